// Fused depthwise + pointwise convolution, one output tile per CTA (wpk_dwpw_*, A_MODE 1 of a fused
// plan, the MobileNet-V2 block; PAPER.md:15 / :35 operator fusion).
//
//   t[m][c] = RN_T(dw_epi(sum_{r,s} x[n][p*sh - ph + r*dh][q*sw - pw + s*dw][c] * w_dw[r][s][c] + b_dw[c]))
//   y[m][k] = RN_T(pw_epi(sum_c t[m][c] * w_pw[k][c] + b_pw[k]))          (m = (n, p, q), NHWC)
//
// A CTA of 8 warps owns 128 output pixels and ALL K_out channels. The C channels are walked in
// chunks of 64: every thread computes the depthwise result of 4 pixels x 8 channels of the chunk
// (fp32 taps in (r, s) order with FFMA2, bias after the sum, ReLU, one rounding: exactly what the
// unfused depthwise kernel stores) straight into a 128-byte-swizzled K-major smem tile, the chunk's
// pointwise weights are copied next to it, and one elected thread issues the tcgen05 MMAs
// (128 x K_out x 64, fp32 accumulator in TMEM, kind::f16) -- double-buffered, so the depthwise math
// of chunk i+1 overlaps the MMAs of chunk i. t never leaves shared memory. The epilogue reads the
// accumulator with tcgen05.ld (warp w: TMEM lane quarter w % 4, column half w / 4), adds the
// pointwise bias, applies the epilogue and stores bf16 / fp16 rows.
// Unlike the persistent tcgen05 kernel's 4 producer warps (DESIGN.md finding 25) every warp of the
// CTA computes the depthwise part and several CTAs share an SM (41-113 KB of smem, <= 512 TMEM
// columns in total), so its load latency is hidden by occupancy.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "dwpw.h"
#include "ptx.cuh"

namespace wpk {

namespace {

__device__ __forceinline__ float2 up2(uint32_t u, __nv_bfloat16 *) {
    return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
}
__device__ __forceinline__ float2 up2(uint32_t u, __half *) {
    return __half22float2(*reinterpret_cast<const __half2 *>(&u));
}
__device__ __forceinline__ void ffma2(float2 &acc, float2 a, float2 b) {
    unsigned long long c = *reinterpret_cast<unsigned long long *>(&acc);
    asm("fma.rn.f32x2 %0, %1, %2, %0;"
        : "+l"(c)
        : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)));
    acc = *reinterpret_cast<float2 *>(&c);
}
__device__ __forceinline__ uint32_t pack2(float a, float b, __nv_bfloat16 *) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ uint32_t pack2(float a, float b, __half *) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
template <typename T>
__device__ __forceinline__ void mac8(float2 *acc, uint4 x, uint4 w) {
    ffma2(acc[0], up2(x.x, (T *)nullptr), up2(w.x, (T *)nullptr));
    ffma2(acc[1], up2(x.y, (T *)nullptr), up2(w.y, (T *)nullptr));
    ffma2(acc[2], up2(x.z, (T *)nullptr), up2(w.z, (T *)nullptr));
    ffma2(acc[3], up2(x.w, (T *)nullptr), up2(w.w, (T *)nullptr));
}

constexpr int kThreads = 256;
constexpr int kRows = 128;

// depthwise result of the chunk's (row, 16-byte channel vector) pieces. Only the chunk's nvalid
// real vectors are computed (C = 32, 96, 144 leave 4, 4, 2 of a chunk's 8): piece p = (row, j) =
// (p / nvalid, p % nvalid), pieces tid and tid + 256 in flight per iteration (3x3: all 18 loads
// before the math); the padded vectors j >= nvalid are written as zeros (the MMA reads them).
template <typename T, bool R3>
__device__ __forceinline__ void dw_chunk(const DwpwArgs &a, uint32_t sbase, int m0, int cvec0, int tid) {
    const int cv = a.C >> 3;
    const int nvalid = min(8, cv - cvec0);
    const int npieces = kRows * nvalid;
    const uint4 *__restrict__ xv = static_cast<const uint4 *>(a.x);
    const uint4 *__restrict__ wv = static_cast<const uint4 *>(a.w_dw);
    const uint4 *__restrict__ bv = static_cast<const uint4 *>(a.b_dw);
    const int PQ = a.P * a.Q;
#pragma unroll 1
    for (int p0 = tid; p0 < npieces; p0 += 2 * kThreads) {
        float2 acc[2][4];
        bool ok[2];
        int row[2], jj[2];
        uint4 xx[2][R3 ? 9 : 1];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int pc = p0 + u * kThreads;
            const bool inp = pc < npieces;
            row[u] = inp ? pc / nvalid : 0;
            jj[u] = inp ? pc - row[u] * nvalid : 0;
            const int m = m0 + row[u];
            ok[u] = inp && m < a.M;
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[u][e] = make_float2(0.f, 0.f);
            const int mm = ok[u] ? m : 0;
            const int n = mm / PQ;
            const int rem = mm - n * PQ;
            const int p = rem / a.Q, q = rem - p * a.Q;
            const int h0 = p * a.sh - a.ph, w0 = q * a.sw - a.pw;
            const int nh = n * a.H;
            const uint4 *xj = xv + cvec0 + jj[u];
            if constexpr (R3) {
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int s = 0; s < 3; ++s) {
                        const int hi = h0 + r * a.dh, wi = w0 + s * a.dw;
                        xx[u][r * 3 + s] = (ok[u] && hi >= 0 && hi < a.H && wi >= 0 && wi < a.W)
                                               ? __ldg(xj + (size_t)((nh + hi) * a.W + wi) * cv)
                                               : make_uint4(0u, 0u, 0u, 0u);
                    }
            } else if (ok[u]) {
                const uint4 *wj = wv + cvec0 + jj[u];
#pragma unroll 1
                for (int r = 0; r < a.R; ++r) {
                    const int hi = h0 + r * a.dh;
                    if (hi < 0 || hi >= a.H) continue;
#pragma unroll 1
                    for (int s = 0; s < a.S; ++s) {
                        const int wi = w0 + s * a.dw;
                        if (wi < 0 || wi >= a.W) continue;
                        mac8<T>(acc[u], __ldg(xj + (size_t)((nh + hi) * a.W + wi) * cv),
                                __ldg(wj + (size_t)(r * a.S + s) * cv));
                    }
                }
            }
        }
        if constexpr (R3) {
#pragma unroll
            for (int i = 0; i < 9; ++i) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const uint4 wq = __ldg(wv + (size_t)i * cv + cvec0 + jj[u]);
                    mac8<T>(acc[u], xx[u][i], wq);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (p0 + u * kThreads >= npieces) break;
            uint32_t o[4] = {0u, 0u, 0u, 0u};
            if (ok[u]) {
                float2 bf[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
                if (bv) {
                    const uint4 b4 = __ldg(bv + cvec0 + jj[u]);
                    bf[0] = up2(b4.x, (T *)nullptr); bf[1] = up2(b4.y, (T *)nullptr);
                    bf[2] = up2(b4.z, (T *)nullptr); bf[3] = up2(b4.w, (T *)nullptr);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float v0 = acc[u][e].x, v1 = acc[u][e].y;
                    if (a.dw_epi >= 1) { v0 += bf[e].x; v1 += bf[e].y; }
                    if (a.dw_epi == 2) { v0 = fmaxf(v0, 0.f); v1 = fmaxf(v1, 0.f); }
                    o[e] = pack2(v0, v1, (T *)nullptr);
                }
            }
            const int rw = row[u];
            const uint32_t rb = sbase + (uint32_t)(rw >> 3) * 1024u + (uint32_t)(rw & 7) * 128u;
            ptx::st_shared_v4(rb + ((uint32_t)(jj[u] ^ (rw & 7)) << 4), o[0], o[1], o[2], o[3]);
        }
    }
    // the chunk's padded vectors (channels >= C): zeros
    const int npad = 8 - nvalid;
    for (int q = tid; q < kRows * npad; q += kThreads) {
        const int rw = q / npad, jp = nvalid + (q - (q / npad) * npad);
        const uint32_t rb = sbase + (uint32_t)(rw >> 3) * 1024u + (uint32_t)(rw & 7) * 128u;
        ptx::st_shared_v4(rb + ((uint32_t)(jp ^ (rw & 7)) << 4), 0u, 0u, 0u, 0u);
    }
}

}  // namespace

template <typename T>
__global__ void __launch_bounds__(kThreads) dwpw_kernel(const DwpwArgs a) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = ptx::smem_u32(smem_raw);
    uint8_t *sm = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
    const int kp = a.kp;                               // K_out rounded up to 16 (MMA N)
    uint8_t *sA = sm;                                  // [2][128 rows][128 B]
    uint8_t *sB = sm + 2 * 16384;                      // [2][kp rows][128 B]
    uint64_t *bars = reinterpret_cast<uint64_t *>(sB + 2 * (size_t)kp * 128);
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (warp == 0) {
        ptx::tmem_alloc(tmem_holder, a.tmem_cols);
        ptx::tmem_relinquish();
    }
    if (tid == 32) {
        ptx::mbar_init(&bars[0], 1);
        ptx::mbar_init(&bars[1], 1);
        ptx::fence_mbar_init();
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    asm volatile("griddepcontrol.wait;" ::: "memory");   // x may still be written upstream, y read

    const int m0 = blockIdx.x * kRows;
    // split-K over the channel chunks (blockIdx.y = split s of a.splits): chunks [kc0, kc1)
    const int nkc_all = (a.C + 63) / 64;
    const int kc0 = blockIdx.y * a.kc_per_split;
    const int kc1 = min(nkc_all, kc0 + a.kc_per_split);
    const int nkc = kc1 - kc0;
    const int cv = a.C >> 3;
    const uint4 *__restrict__ wpw = static_cast<const uint4 *>(a.w_pw);
    const bool r3 = a.R == 3 && a.S == 3;
    uint32_t ph0 = 0, ph1 = 0;
    for (int kci = 0; kci < nkc; ++kci) {
        const int kc = kc0 + kci;
        const int b = kci & 1;
        if (kci >= 2) {   // the MMAs of chunk kc - 2 have finished reading buffer b
            if (b == 0) { ptx::mbar_wait(&bars[0], ph0); ph0 ^= 1; }
            else { ptx::mbar_wait(&bars[1], ph1); ph1 ^= 1; }
        }
        const uint32_t aB = ptx::smem_u32(sA + b * 16384);
        const uint32_t bB = ptx::smem_u32(sB + (size_t)b * kp * 128);
        if (r3) dw_chunk<T, true>(a, aB, m0, kc * 8, tid);
        else dw_chunk<T, false>(a, aB, m0, kc * 8, tid);
        // the chunk's pointwise weights: kp rows x 8 vectors, zero past K_out / C
        for (int v = tid; v < kp * 8; v += kThreads) {
            const int k = v >> 3, jj = v & 7, c8 = kc * 8 + jj;
            const uint4 val = (k < a.K && c8 < cv) ? __ldg(wpw + (size_t)k * cv + c8) : make_uint4(0u, 0u, 0u, 0u);
            ptx::st_shared_v4(bB + (uint32_t)(k >> 3) * 1024u + (uint32_t)(k & 7) * 128u + ((uint32_t)(jj ^ (k & 7)) << 4),
                              val.x, val.y, val.z, val.w);
        }
        ptx::fence_proxy_async_smem();   // generic-proxy smem writes -> the MMA (async proxy)
        __syncthreads();
        if (warp == 0) {
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
                const uint64_t ad = ptx::sw128_kmajor_desc(aB);
                const uint64_t bd = ptx::sw128_kmajor_desc(bB);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {   // 4 x 16 channels of the 64-channel chunk (+32 B each)
                    ptx::umma<0>(tmem, ad + 2 * kk, bd + 2 * kk, a.idesc0, (kci > 0 || kk > 0) ? 1u : 0u);
                    if (kp > 256)   // columns 256.. of a wide K_out: the next 256 rows of B
                        ptx::umma<0>(tmem + 256, ad + 2 * kk, bd + (uint64_t)((256 * 128) >> 4) + 2 * kk, a.idesc1,
                                     (kci > 0 || kk > 0) ? 1u : 0u);
                }
                ptx::umma_commit(&bars[b]);   // buffer b free (and, for the last chunk, the accumulator ready)
            }
            __syncwarp();
        }
    }
    {   // the last commit tracks every MMA issued before it
        const int b = (nkc - 1) & 1;
        ptx::mbar_wait(&bars[b], b == 0 ? ph0 : ph1);
    }
    ptx::tc_fence_after();

    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 (one output row each), column half w / 4
    const int quarter = warp & 3, half = warp >> 2;
    const int row = quarter * 32 + lane;
    const int m = m0 + row;
    const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16);
    T *__restrict__ y = static_cast<T *>(a.y);
    const T *__restrict__ bpw = static_cast<const T *>(a.b_pw);
    for (int c0 = half * 16; c0 < kp; c0 += 32) {
        uint32_t r[16];
        ptx::tmem_ld16_nowait(tl + (uint32_t)c0, r);
        ptx::tmem_wait_ld();
        if (m < a.M && a.splits > 1) {   // split-K: this split's fp32 partial, no bias / epilogue
            float4 *dst = reinterpret_cast<float4 *>(a.partial + ((size_t)blockIdx.y * a.M + m) * a.K + c0);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (c0 + 4 * q + 4 <= a.K)
                    dst[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                         __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
        } else if (m < a.M) {
            uint32_t o[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                float v0 = __uint_as_float(r[2 * e]), v1 = __uint_as_float(r[2 * e + 1]);
                const int k = c0 + 2 * e;
                if (a.pw_epi >= 1) {
                    v0 += (k < a.K) ? static_cast<float>(bpw[k]) : 0.f;
                    v1 += (k + 1 < a.K) ? static_cast<float>(bpw[k + 1]) : 0.f;
                }
                if (a.pw_epi == 2) { v0 = fmaxf(v0, 0.f); v1 = fmaxf(v1, 0.f); }
                o[e] = pack2(v0, v1, (T *)nullptr);
            }
            uint4 *dst = reinterpret_cast<uint4 *>(y + (size_t)m * a.K + c0);
            if (c0 + 8 <= a.K) dst[0] = make_uint4(o[0], o[1], o[2], o[3]);   // K_out % 8 == 0 (plan)
            if (c0 + 16 <= a.K) dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, a.tmem_cols);
}

// split-K reduction: y = RN(pw_epi(sum_{s = 0..S-1} partial[s] + b_pw)), the partials summed in split
// order (deterministic); one thread per 8 consecutive outputs (K_out % 8 == 0)
template <typename T>
__global__ void dwpw_reduce_kernel(const DwpwArgs a) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const long long n8 = (long long)a.M * a.K / 8;
    const T *__restrict__ bpw = static_cast<const T *>(a.b_pw);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
        const long long e0 = i * 8;
        const int k0 = (int)(e0 % a.K);
        float v[8];
        const float4 *p0 = reinterpret_cast<const float4 *>(a.partial + e0);
        float4 u = p0[0], w = p0[1];
        v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w; v[4] = w.x; v[5] = w.y; v[6] = w.z; v[7] = w.w;
        for (int s = 1; s < a.splits; ++s) {
            const float4 *ps = reinterpret_cast<const float4 *>(a.partial + (size_t)s * a.M * a.K + e0);
            u = ps[0]; w = ps[1];
            v[0] += u.x; v[1] += u.y; v[2] += u.z; v[3] += u.w; v[4] += w.x; v[5] += w.y; v[6] += w.z; v[7] += w.w;
        }
        uint32_t o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float v0 = v[2 * e], v1 = v[2 * e + 1];
            if (a.pw_epi >= 1) { v0 += static_cast<float>(bpw[k0 + 2 * e]); v1 += static_cast<float>(bpw[k0 + 2 * e + 1]); }
            if (a.pw_epi == 2) { v0 = fmaxf(v0, 0.f); v1 = fmaxf(v1, 0.f); }
            o[e] = pack2(v0, v1, (T *)nullptr);
        }
        reinterpret_cast<uint4 *>(static_cast<T *>(a.y))[i] = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

static uint32_t idesc_f16(bool bf16, int n) {   // kind::f16, fp32 accumulate, K-major A and B, M = 128
    uint32_t d = 0;
    d |= 1u << 4;                            // c_format = F32
    d |= (bf16 ? 1u : 0u) << 7;              // a_format
    d |= (bf16 ? 1u : 0u) << 10;             // b_format
    d |= (uint32_t)(n >> 3) << 17;           // n_dim
    d |= (uint32_t)(128 >> 4) << 24;         // m_dim
    return d;
}

size_t dwpw_smem_bytes(int kp) { return 1024 + 2 * 16384 + 2 * (size_t)kp * 128 + 64; }

int dwpw_launch(DwpwArgs a, int dtype, void *stream, std::string *err) {
    a.kp = (a.K + 15) / 16 * 16;
    int cols = 32;
    while (cols < a.kp) cols <<= 1;
    a.tmem_cols = (uint32_t)cols;
    const bool bf16 = dtype == WPK_BF16;
    a.idesc0 = idesc_f16(bf16, std::min(a.kp, 256));
    a.idesc1 = idesc_f16(bf16, a.kp > 256 ? a.kp - 256 : 16);
    const size_t smem = dwpw_smem_bytes(a.kp);
    cudaLaunchConfig_t lc{};
    const int nkc = (a.C + 63) / 64;
    if (a.splits < 1) a.splits = 1;
    a.kc_per_split = (nkc + a.splits - 1) / a.splits;
    lc.gridDim = dim3((unsigned)((a.M + kRows - 1) / kRows), (unsigned)a.splits);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = smem;
    lc.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    cudaError_t ce;
    if (bf16) {
        ce = cudaFuncSetAttribute(dwpw_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ce == cudaSuccess) ce = cudaLaunchKernelEx(&lc, dwpw_kernel<__nv_bfloat16>, a);
    } else {
        ce = cudaFuncSetAttribute(dwpw_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ce == cudaSuccess) ce = cudaLaunchKernelEx(&lc, dwpw_kernel<__half>, a);
    }
    if (ce == cudaSuccess) ce = cudaGetLastError();
    if (ce != cudaSuccess) {
        *err = std::string("dwpw_kernel launch: ") + cudaGetErrorString(ce);
        return -1;
    }
    if (a.splits == 1) return 1;
    cudaLaunchConfig_t rc{};
    const long long n8 = (long long)a.M * a.K / 8;
    rc.gridDim = dim3((unsigned)std::min<long long>((n8 + 255) / 256, 148 * 8));
    rc.blockDim = dim3(256);
    rc.stream = (cudaStream_t)stream;
    rc.attrs = attr;
    rc.numAttrs = 1;
    ce = bf16 ? cudaLaunchKernelEx(&rc, dwpw_reduce_kernel<__nv_bfloat16>, a) : cudaLaunchKernelEx(&rc, dwpw_reduce_kernel<__half>, a);
    if (ce == cudaSuccess) ce = cudaGetLastError();
    if (ce != cudaSuccess) {
        *err = std::string("dwpw_reduce_kernel launch: ") + cudaGetErrorString(ce);
        return -1;
    }
    return 2;
}

}  // namespace wpk
