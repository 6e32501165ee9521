// KB2b: exact-fp32 implicit-GEMM convolution on CUDA cores (WPK_FAMILY_GEMM32).
//
// y[m, k] = sum_kg A[m, kg] * B[k, kg] with m = (n, p, q), kg = (r, s, c) (c innermost, NHWC
// activations, KRSC weights), every product an fp32 FMA accumulated in increasing kg order (the
// result is a fixed function of the inputs, within the fp32 tolerance of the float64 oracle).
// CTA tile BLOCK_M x BLOCK_N, K step BLOCK_K; each thread owns THREAD x THREAD outputs. Operand
// tiles are gathered into registers (16-byte vectors along c; the launcher pads C to a multiple of
// 4), stored transposed
// into double-buffered shared memory ([k][m] and [k][n]) and consumed as outer products; the next
// K step's loads are in flight while the current one is computed. SPLIT_K > 1 (deep layers with
// few tiles) writes per-split fp32 partials that gemm32_reduce_kernel sums in split order.
//
// This is the strict-comparison path of SURVEY.md 8(a) a8 (north star: "an exact-fp32 CUDA-core
// direct/implicit-GEMM kernel"); WPK_FAMILY_SIMT keeps the paper's own direct-convolution template.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "gemm32.h"

namespace wpk {

// 8x8 thread tiles: at most 128 registers per thread (512 / threads CTAs per SM), except where
// that spills (ptxas -v): the 64-thread BLOCK_K 16 tile and the 128 x 64 tile get 4 / 3 CTAs
constexpr int gemm32_min_blocks(int bm, int bn, int bk, int tt) {
    return tt != 8 ? 1
           : ((bm / tt) * (bn / tt) == 64 && bk == 16) ? 4
           : (bm == 128 && bn == 64) ? 3
                                     : 512 / ((bm / tt) * (bn / tt));
}

template <int BM, int BN, int BK, int TT>
__global__ void __launch_bounds__((BM / TT) * (BN / TT), gemm32_min_blocks(BM, BN, BK, TT))
    gemm32_conv_kernel(const Gemm32Args a) {
    constexpr int TX = BN / TT, TY = BM / TT, NT = TX * TY;
    constexpr int A4 = BM * BK / 4, B4 = BN * BK / 4;                 // float4 slots per tile
    constexpr int AL = (A4 + NT - 1) / NT, BL = (B4 + NT - 1) / NT;   // per-thread vector loads
    __shared__ __align__(16) float As[2][BK][BM];
    __shared__ __align__(16) float Bs[2][BK][BN];
    const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
    const long long m0 = (long long)blockIdx.x * BM;
    const int n0 = blockIdx.y * BN;
    const float *x = a.x, *w = a.w;
    const int Kg = a.R * a.S * a.C;   // a.C % 4 == 0 (the launcher pads C): 16-byte operand vectors

    // rows of the A tile this thread loads: image, top-left input coordinate (or invalid)
    int an[AL], ah[AL], aw[AL];
#pragma unroll
    for (int i = 0; i < AL; ++i) {
        const int idx = tid + i * NT;
        const long long m = m0 + idx / (BK / 4);
        an[i] = -1;
        if (idx < A4 && m < a.M) {
            const int n = (int)(m / a.PQ);
            const int rem = (int)(m - (long long)n * a.PQ);
            const int p = rem / a.Q, q = rem - (rem / a.Q) * a.Q;
            an[i] = n; ah[i] = p * a.sh - a.ph; aw[i] = q * a.sw - a.pw;
        }
    }
    float4 ra[AL], rb[BL];
    auto load_a = [&](int k0) {
#pragma unroll
        for (int i = 0; i < AL; ++i) {
            const int idx = tid + i * NT;
            const int kg = k0 + (idx % (BK / 4)) * 4;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (an[i] >= 0 && kg < Kg) {   // 4 channels of one tap (kg % 4 == 0, C % 4 == 0)
                const int c = kg % a.C, rs = kg / a.C, s = rs % a.S, r = rs / a.S;
                const int h = ah[i] + r * a.dh, ww = aw[i] + s * a.dw;
                if (h >= 0 && h < a.H && ww >= 0 && ww < a.W)
                    v = *reinterpret_cast<const float4 *>(x + (((long long)an[i] * a.H + h) * a.W + ww) * a.C + c);
            }
            ra[i] = v;
        }
    };
    auto load_b = [&](int k0) {
#pragma unroll
        for (int i = 0; i < BL; ++i) {
            const int idx = tid + i * NT;
            const int col = idx / (BK / 4), kg = k0 + (idx % (BK / 4)) * 4;
            const int n = n0 + col;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (idx < B4 && n < a.K && kg < Kg) v = *reinterpret_cast<const float4 *>(w + (long long)n * Kg + kg);
            rb[i] = v;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int i = 0; i < AL; ++i) {
            const int idx = tid + i * NT;
            if (idx < A4) {
                const int row = idx / (BK / 4), kq = (idx % (BK / 4)) * 4;
                As[buf][kq][row] = ra[i].x; As[buf][kq + 1][row] = ra[i].y;
                As[buf][kq + 2][row] = ra[i].z; As[buf][kq + 3][row] = ra[i].w;
            }
        }
#pragma unroll
        for (int i = 0; i < BL; ++i) {
            const int idx = tid + i * NT;
            if (idx < B4) {
                const int col = idx / (BK / 4), kq = (idx % (BK / 4)) * 4;
                Bs[buf][kq][col] = rb[i].x; Bs[buf][kq + 1][col] = rb[i].y;
                Bs[buf][kq + 2][col] = rb[i].z; Bs[buf][kq + 3][col] = rb[i].w;
            }
        }
    };

    float acc[TT][TT];
#pragma unroll
    for (int i = 0; i < TT; ++i)
#pragma unroll
        for (int j = 0; j < TT; ++j) acc[i][j] = 0.f;

    // split-K: this CTA accumulates K steps [kt0, kt1) (blockIdx.z of SPLIT_K)
    const int nk_all = (Kg + BK - 1) / BK;
    const int kt0 = blockIdx.z * a.kper, kt1 = min(nk_all, kt0 + a.kper);
    const int nk = kt1 - kt0;
    const int kbase = kt0 * BK;
    load_a(kbase);
    load_b(kbase);
    store(0);
    __syncthreads();
    for (int t = 0; t < nk; ++t) {
        const int buf = t & 1;
        if (t + 1 < nk) { load_a(kbase + (t + 1) * BK); load_b(kbase + (t + 1) * BK); }
        // operand fragments double-buffered in registers: row kk+1 is read from shared memory
        // while row kk's outer product issues (hides the LDS latency at low occupancy)
        float av[2][TT], bv[2][TT];
        auto frag = [&](int f, int kk) {
#pragma unroll
            for (int i = 0; i < TT; i += 4) {
                const float4 t4 = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * TT + i]);
                av[f][i] = t4.x; av[f][i + 1] = t4.y; av[f][i + 2] = t4.z; av[f][i + 3] = t4.w;
            }
#pragma unroll
            for (int j = 0; j < TT; j += 4) {
                const float4 t4 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * TT + j]);
                bv[f][j] = t4.x; bv[f][j + 1] = t4.y; bv[f][j + 2] = t4.z; bv[f][j + 3] = t4.w;
            }
        };
        frag(0, 0);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            if (kk + 1 < BK) frag((kk + 1) & 1, kk + 1);
#pragma unroll
            for (int i = 0; i < TT; ++i)
#pragma unroll
                for (int j = 0; j < TT; ++j) acc[i][j] = fmaf(av[kk & 1][i], bv[kk & 1][j], acc[i][j]);
        }
        if (t + 1 < nk) {
            store(buf ^ 1);
            __syncthreads();
        }
    }

    if (a.partial) {   // split-K: raw partial sums [split][m][k], reduced in order by gemm32_reduce
        float *pp = a.partial + (long long)blockIdx.z * a.M * a.K;
        const int kb = n0 + tx * TT;
#pragma unroll
        for (int i = 0; i < TT; ++i) {
            const long long m = m0 + ty * TT + i;
            if (m >= a.M) continue;
            float *row = pp + m * a.K;
            if (kb + TT <= a.K && (a.K % 4) == 0) {
#pragma unroll
                for (int j = 0; j < TT; j += 4)
                    *reinterpret_cast<float4 *>(row + kb + j) =
                        make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < TT; ++j)
                    if (kb + j < a.K) row[kb + j] = acc[i][j];
            }
        }
        return;
    }
    // epilogue: + bias, (+ residual), ReLU; layout-strided stores (16-byte vectors for NHWC)
#pragma unroll
    for (int i = 0; i < TT; ++i) {
        const long long m = m0 + ty * TT + i;
        if (m >= a.M) continue;
        const int n = (int)(m / a.PQ);
        const int rem = (int)(m - (long long)n * a.PQ);
        const int p = rem / a.Q, q = rem - (rem / a.Q) * a.Q;
        const long long ybase = (long long)n * a.ys_n + (long long)p * a.ys_p + (long long)q * a.ys_q;
        float v[TT];
#pragma unroll
        for (int j = 0; j < TT; ++j) {
            const int k = n0 + tx * TT + j;
            float o = acc[i][j];
            if (k < a.K) {
                if (a.epilogue >= 1) o += a.b[k];
                if (a.epilogue == 3) o += a.z[ybase + (long long)k * a.ys_k];
                if (a.epilogue >= 2) o = fmaxf(o, 0.f);
            }
            v[j] = o;
        }
        const int kb = n0 + tx * TT;
        if (a.ys_k == 1 && kb + TT <= a.K && (a.K % 4) == 0) {
#pragma unroll
            for (int j = 0; j < TT; j += 4)
                *reinterpret_cast<float4 *>(a.y + ybase + kb + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < TT; ++j)
                if (kb + j < a.K) a.y[ybase + (long long)(kb + j) * a.ys_k] = v[j];
        }
    }
}

// Split-K reduction: y = epilogue(sum over splits 0..S-1 in increasing order); one thread per output.
// All splits' loads are issued before the in-order sum (SPLIT_K <= 8), so one L2/HBM latency is
// paid per output instead of one per split.
__global__ void gemm32_reduce_kernel(const Gemm32Args a, int splits) {
    const long long total = a.M * a.K;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        float v[8];
#pragma unroll
        for (int z = 0; z < 8; ++z) v[z] = z < splits ? __ldcs(a.partial + (long long)z * total + i) : 0.f;
        float o = v[0];
#pragma unroll
        for (int z = 1; z < 8; ++z)
            if (z < splits) o += v[z];
        const long long m = i / a.K;
        const int k = (int)(i - m * a.K);
        const int n = (int)(m / a.PQ);
        const int rem = (int)(m - (long long)n * a.PQ);
        const int p = rem / a.Q, q = rem - (rem / a.Q) * a.Q;
        const long long yi = (long long)n * a.ys_n + (long long)k * a.ys_k + (long long)p * a.ys_p + (long long)q * a.ys_q;
        if (a.epilogue >= 1) o += a.b[k];
        if (a.epilogue == 3) o += a.z[yi];
        if (a.epilogue >= 2) o = fmaxf(o, 0.f);
        a.y[yi] = o;
    }
}

template <int BM, int BN, int BK, int TT>
static cudaError_t launch_t(const Gemm32Args &a, int splits, cudaStream_t st) {
    dim3 grid((unsigned)((a.M + BM - 1) / BM), (unsigned)((a.K + BN - 1) / BN), (unsigned)splits);
    gemm32_conv_kernel<BM, BN, BK, TT><<<grid, (BM / TT) * (BN / TT), 0, st>>>(a);
    return cudaGetLastError();
}

int gemm32_launch(const Gemm32Args &a_in, int bm, int bn, int bk, int tt, int splits, float *partial, int sm_count,
                  void *stream, std::string *err) {
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaErrorInvalidValue;
    Gemm32Args a = a_in;
    const int nk = (a.R * a.S * a.C + bk - 1) / bk;
    a.kper = (nk + splits - 1) / splits;
    splits = (nk + a.kper - 1) / a.kper;   // no empty split
    a.partial = splits > 1 ? partial : nullptr;
#define WPK_G32(BM, BN, BK, TT) \
    if (bm == BM && bn == BN && bk == BK && tt == TT) e = launch_t<BM, BN, BK, TT>(a, splits, st);
    WPK_G32(64, 64, 8, 4) WPK_G32(64, 64, 16, 4) WPK_G32(64, 64, 8, 8) WPK_G32(64, 64, 16, 8)
    WPK_G32(64, 128, 8, 4) WPK_G32(64, 128, 16, 4) WPK_G32(64, 128, 8, 8) WPK_G32(64, 128, 16, 8)
    WPK_G32(128, 64, 8, 4) WPK_G32(128, 64, 16, 4) WPK_G32(128, 64, 8, 8) WPK_G32(128, 64, 16, 8)
    WPK_G32(128, 128, 8, 4) WPK_G32(128, 128, 16, 4) WPK_G32(128, 128, 8, 8) WPK_G32(128, 128, 16, 8)
#undef WPK_G32
    if (e != cudaSuccess) {
        *err = std::string("gemm32_conv_kernel launch: ") + cudaGetErrorString(e);
        return -1;
    }
    if (splits == 1) return 1;
    const long long total = a.M * a.K;
    const long long blocks = std::min<long long>((total + 255) / 256, (long long)sm_count * 8);
    gemm32_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, splits);
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        *err = std::string("gemm32_reduce_kernel launch: ") + cudaGetErrorString(e);
        return -1;
    }
    return 2;
}

}  // namespace wpk
