/*
 * oracle/conv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously-correct CPU definition of the operation the CUDA path computes:
 * forward 2-D convolution (cross-correlation) + optional bias + optional ReLU, in double.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library. It shares no code, header or constant with paper_2008_04567_b200/.
 *
 * Definition followed (§2.2 Halide listing
 *     conv(x, y) = sum(filter(r.x, r.y) * in(x + r.x - 1, y + r.y - 1))
 * i.e. an UNFLIPPED window sum with offset -pad; generalised to batch, channels, stride, dilation
 * and groups as written in SURVEY.md §8(c) Part 1; fusion semantics relu(bias_add(conv)) per
 * SPEC.md:136 and PAPER.md:15):
 *
 *   P = floor((H + 2*pad_h - dil_h*(R-1) - 1) / stride_h) + 1        (same for Q with W, S)
 *   Cpg = C/groups, Kpg = K/groups, grp(k) = k / Kpg
 *   pre[n,k,p,q] = sum_{c<Cpg} sum_{r<R} sum_{s<S}
 *                  x[n, grp(k)*Cpg + c, p*stride_h - pad_h + r*dil_h, q*stride_w - pad_w + s*dil_w]
 *                  * w[k, c, r, s]            (x taken as 0 outside [0,H) x [0,W))
 *   y = pre (epilogue 0) | pre + b[k] (1) | max(pre + b[k], 0) (2)
 *     | max(pre + b[k] + z[n,k,p,q], 0) (3: the residual-add fusion of a ResNet block's last
 *       conv, SURVEY.md §8(f) NEXT-1 / PAPER.md:15 operator fusion; z has y's shape)
 *
 * Layout: canonical NCHW for x and y, KCRS for w (the test harness transposes with numpy for
 * NHWC cases). Loop order (n, k, p, q, c, r, s), fixed.
 *
 * shape[] = {N, C, H, W, K, R, S, stride_h, stride_w, pad_h, pad_w, dil_h, dil_w, groups, epilogue}
 */
#include <stdint.h>
#include <stddef.h>

static int out_size(int in, int pad, int dil, int f, int stride)
{
    /* floor division of a possibly negative numerator */
    int num = in + 2 * pad - dil * (f - 1) - 1;
    if (num < 0) return 0;
    return num / stride + 1;
}

int wpk_oracle_out_dims(const int32_t *shape, int32_t *p_out, int32_t *q_out)
{
    *p_out = out_size(shape[2], shape[9], shape[11], shape[5], shape[7]);
    *q_out = out_size(shape[3], shape[10], shape[12], shape[6], shape[8]);
    return (*p_out >= 1 && *q_out >= 1) ? 0 : -1;
}

/* One output element, exactly as the definition above. */
static double one_output(const int32_t *sh, const double *x, const double *w, const double *b,
                         const double *z, int n, int k, int p, int q)
{
    const int C = sh[1], H = sh[2], W = sh[3], K = sh[4], R = sh[5], S = sh[6];
    const int sth = sh[7], stw = sh[8], ph = sh[9], pw = sh[10], dh = sh[11], dw = sh[12];
    const int G = sh[13], epi = sh[14];
    const int Cpg = C / G, Kpg = K / G, grp = k / Kpg;
    double acc = 0.0;
    for (int c = 0; c < Cpg; ++c)
        for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s) {
                int hi = p * sth - ph + r * dh;
                int wi = q * stw - pw + s * dw;
                double xv = 0.0;
                if (hi >= 0 && hi < H && wi >= 0 && wi < W)
                    xv = x[(((size_t)n * C + (size_t)(grp * Cpg + c)) * H + hi) * W + wi];
                acc += xv * w[(((size_t)k * Cpg + c) * R + r) * S + s];
            }
    if (epi >= 1) acc += b[k];
    if (epi == 3) {
        int P, Q;
        wpk_oracle_out_dims(sh, &P, &Q);
        acc += z[(((size_t)n * K + k) * P + p) * Q + q];
    }
    if (epi >= 2 && acc < 0.0) acc = 0.0;
    return acc;
}

/* Full output tensor y[N][K][P][Q].  nthreads > 1 splits the outermost (n,k) loop with OpenMP;
 * the arithmetic per element is unchanged. Returns 0, or -1 on an invalid shape. */
int wpk_oracle_conv2d_res(const int32_t *sh, const double *x, const double *w, const double *b,
                          const double *z, double *y, int nthreads);
int wpk_oracle_conv2d(const int32_t *sh, const double *x, const double *w, const double *b,
                      double *y, int nthreads)
{
    if (sh[14] == 3) return -1;   /* the residual epilogue needs z: wpk_oracle_conv2d_res */
    return wpk_oracle_conv2d_res(sh, x, w, b, NULL, y, nthreads);
}

/* Same, with the residual z[N][K][P][Q] (read only when epilogue == 3). */
int wpk_oracle_conv2d_res(const int32_t *sh, const double *x, const double *w, const double *b,
                          const double *z, double *y, int nthreads)
{
    int P, Q;
    if (sh[0] < 1 || sh[1] < 1 || sh[4] < 1 || sh[13] < 1) return -1;
    if (sh[1] % sh[13] != 0 || sh[4] % sh[13] != 0) return -1;
    if (sh[14] == 3 && z == NULL) return -1;
    if (wpk_oracle_out_dims(sh, &P, &Q) != 0) return -1;
    const int N = sh[0], K = sh[4];
    const long long NK = (long long)N * K;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (long long nk = 0; nk < NK; ++nk) {
        int n = (int)(nk / K), k = (int)(nk % K);
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < Q; ++q)
                y[((size_t)nk * P + p) * Q + q] = one_output(sh, x, w, b, z, n, k, p, q);
    }
    return 0;
}

/* Sampled outputs: pts[i] = (n, k, p, q) as int64; out[i] = y[n,k,p,q]. Each output is an
 * independent dot product, so a sample is exact per element. */
int wpk_oracle_conv2d_points(const int32_t *sh, const double *x, const double *w, const double *b,
                             const int64_t *pts, int64_t npts, double *out, int nthreads)
{
    int P, Q;
    if (wpk_oracle_out_dims(sh, &P, &Q) != 0) return -1;
    if (sh[14] == 3) return -1;   /* sampled outputs: epilogues 0-2 */
    for (int64_t i = 0; i < npts; ++i) {
        const int64_t *t = pts + 4 * i;
        if (t[0] < 0 || t[0] >= sh[0] || t[1] < 0 || t[1] >= sh[4] || t[2] < 0 || t[2] >= P ||
            t[3] < 0 || t[3] >= Q)
            return -1;
    }
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t i = 0; i < npts; ++i) {
        const int64_t *t = pts + 4 * i;
        out[i] = one_output(sh, x, w, b, NULL, (int)t[0], (int)t[1], (int)t[2], (int)t[3]);
    }
    return 0;
}
