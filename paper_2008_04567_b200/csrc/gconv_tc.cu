// Grouped convolution on the tensor cores (general groups 1 < g < C; the
// ResNeXt case): the tcgen05 family's A_MODE 1 for a grouped plan.
//
//   y[n][p][q][g*Kpg + k] = epi(b + sum_{r,s,c < Cpg} x[n][p*sh-ph+r*dh][q*sw-pw+s*dw][g*Cpg + c] * w[g*Kpg + k][r][s][c])
//
// Each group is its own small GEMM (M = N*P*Q pixels, N = Kpg, K = R*S*Cpg): a CTA of 8 warps owns
// 128 pixels x GT consecutive groups. For every group of the tile and every 64-wide chunk of that
// group's K, the threads gather the im2col rows (k = (r*S + s)*Cpg + c, zero past R*S*Cpg and out of
// the image) into a 128-byte-swizzled K-major smem tile and copy the group's weight rows
// ([K][R][S][Cpg] = NHWC layout, rows padded to Np = max(16, Kpg rounded to 16) with zeros), and one
// elected thread issues 128 x Np x 64 tcgen05 MMAs into the group's TMEM columns [gl*Np, gl*Np+Np)
// -- double-buffered, the gather of step i+1 overlapping the MMAs of step i. The epilogue reads the
// Kpg valid columns of each group (tcgen05.ld), adds the bias, applies ReLU / the residual and stores.
// Padding waste: N to Np (4x at Kpg = 4) and K to 64 (1.8x at R*S*Cpg = 36); the fp32 accumulate
// order per output is k = 0, 1, ... (exact-integer inputs are bit-exact).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "gconv_tc.h"
#include "ptx.cuh"

namespace wpk {

namespace {

constexpr int kThreads = 256;
constexpr int kRows = 128;

__device__ __forceinline__ uint32_t pk2(float a, float b, __nv_bfloat16 *) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ uint32_t pk2(float a, float b, __half *) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

// im2col rows of one (group, K chunk): thread tid owns the 16-byte pieces (row, j) =
// ((tid >> 3) + 32 i, tid & 7), i < 4. Loaded into registers one step ahead of the smem store
// (software pipeline: the loads of step s+1 are in flight while step s is stored and multiplied).
struct Pieces {
    uint32_t o[4][4];
};
__device__ __forceinline__ void gather_load(const GconvArgs &a, int m0, int g, int k0, int tid, Pieces &P) {
    const unsigned short *__restrict__ x = static_cast<const unsigned short *>(a.x);
    const int KG = a.R * a.S * a.Cpg;
    const int PQ = a.P * a.Q;
    const int j = tid & 7;
    const int kb = k0 + j * 8;                   // first K index of this 16-byte piece
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = (tid >> 3) + 32 * i;
        const int m = m0 + row;
        uint32_t *o = P.o[i];
        o[0] = o[1] = o[2] = o[3] = 0u;
        if (m < a.M && kb < KG) {
            const int n = m / PQ;
            const int rem = m - n * PQ;
            const int p = rem / a.Q, q = rem - p * a.Q;
            const int h0 = p * a.sh - a.ph, w0 = q * a.sw - a.pw;
            const size_t nbase = (size_t)n * a.H;
            if (a.Cpg % 8 == 0) {                // one tap, 8 consecutive channels: one 16-byte load
                const int tap = kb / a.Cpg, c = kb - tap * a.Cpg;
                const int r = tap / a.S, s = tap - r * a.S;
                const int hi = h0 + r * a.dh, wi = w0 + s * a.dw;
                if (hi >= 0 && hi < a.H && wi >= 0 && wi < a.W) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4 *>(
                        x + ((nbase + hi) * a.W + wi) * a.C + (size_t)g * a.Cpg + c));
                    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
                }
            } else if (a.Cpg == 4) {             // two taps of 4 channels: two 8-byte loads
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int tap = kb / 4 + h;
                    if (tap * 4 >= KG) break;
                    const int r = tap / a.S, s = tap - r * a.S;
                    const int hi = h0 + r * a.dh, wi = w0 + s * a.dw;
                    if (hi >= 0 && hi < a.H && wi >= 0 && wi < a.W) {
                        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(
                            x + ((nbase + hi) * a.W + wi) * a.C + (size_t)g * a.Cpg));
                        o[2 * h] = v.x; o[2 * h + 1] = v.y;
                    }
                }
            } else {                             // general Cpg: element by element
                unsigned short e16[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    e16[e] = 0;
                    const int k = kb + e;
                    if (k < KG) {
                        const int tap = k / a.Cpg, c = k - tap * a.Cpg;
                        const int r = tap / a.S, s = tap - r * a.S;
                        const int hi = h0 + r * a.dh, wi = w0 + s * a.dw;
                        if (hi >= 0 && hi < a.H && wi >= 0 && wi < a.W)
                            e16[e] = __ldg(x + ((nbase + hi) * a.W + wi) * a.C + (size_t)g * a.Cpg + c);
                    }
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) o[e] = (uint32_t)e16[2 * e] | ((uint32_t)e16[2 * e + 1] << 16);
            }
        }
    }
}
__device__ __forceinline__ void gather_store(uint32_t sbase, int tid, const Pieces &P) {
    const int j = tid & 7;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = (tid >> 3) + 32 * i;
        ptx::st_shared_v4(sbase + (uint32_t)(row >> 3) * 1024u + (uint32_t)(row & 7) * 128u +
                              ((uint32_t)(j ^ (row & 7)) << 4),
                          P.o[i][0], P.o[i][1], P.o[i][2], P.o[i][3]);
    }
}

// the group's weight rows [Np][64] of the chunk: w [K][R*S*Cpg], zero for k >= Kpg or past KG
__device__ __forceinline__ void weight_chunk(const GconvArgs &a, uint32_t sbase, int g, int k0, int tid) {
    const unsigned short *__restrict__ w = static_cast<const unsigned short *>(a.w);
    const int KG = a.R * a.S * a.Cpg;
    for (int v = tid; v < a.np * 8; v += kThreads) {
        const int kk = v >> 3, jj = v & 7;
        const int kidx = k0 + jj * 8;
        uint32_t o[4] = {0u, 0u, 0u, 0u};
        if (kk < a.Kpg && kidx < KG) {
            const unsigned short *src = w + (size_t)(g * a.Kpg + kk) * KG + kidx;
            if (KG % 8 == 0) {
                const uint4 q = __ldg(reinterpret_cast<const uint4 *>(src));
                o[0] = q.x; o[1] = q.y; o[2] = q.z; o[3] = q.w;
            } else {
                unsigned short e16[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) e16[e] = (kidx + e < KG) ? __ldg(src + e) : (unsigned short)0;
#pragma unroll
                for (int e = 0; e < 4; ++e) o[e] = (uint32_t)e16[2 * e] | ((uint32_t)e16[2 * e + 1] << 16);
            }
        }
        ptx::st_shared_v4(sbase + (uint32_t)(kk >> 3) * 1024u + (uint32_t)(kk & 7) * 128u + ((uint32_t)(jj ^ (kk & 7)) << 4),
                          o[0], o[1], o[2], o[3]);
    }
}

}  // namespace

template <typename T>
__global__ void __launch_bounds__(kThreads) gconv_tc_kernel(const GconvArgs a) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = ptx::smem_u32(smem_raw);
    uint8_t *sm = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
    uint8_t *sA = sm;                                   // [2][128][128 B]
    uint8_t *sB = sm + 2 * 16384;                       // [2][np][128 B]
    uint64_t *bars = reinterpret_cast<uint64_t *>(sB + 2 * (size_t)a.np * 128);
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
    asm volatile("griddepcontrol.wait;" ::: "memory");

    const int m0 = (blockIdx.x % a.m_tiles) * kRows;
    const int g0 = (blockIdx.x / a.m_tiles) * a.gt;
    const int ng = min(a.gt, a.groups - g0);
    const int KG = a.R * a.S * a.Cpg;
    const int nkc = (KG + 63) / 64;
    uint32_t ph0 = 0, ph1 = 0;
    int step = 0;
    Pieces cur;
    gather_load(a, m0, g0, 0, tid, cur);
    for (int gl = 0; gl < ng; ++gl) {
        for (int kc = 0; kc < nkc; ++kc, ++step) {
            const int b = step & 1;
            // next step's loads first: in flight while this step is stored and multiplied
            Pieces nxt;
            const bool more = kc + 1 < nkc || gl + 1 < ng;
            if (more) {
                const int ngl = (kc + 1 < nkc) ? gl : gl + 1, nkc1 = (kc + 1 < nkc) ? kc + 1 : 0;
                gather_load(a, m0, g0 + ngl, nkc1 * 64, tid, nxt);
            }
            if (step >= 2) {
                if (b == 0) { ptx::mbar_wait(&bars[0], ph0); ph0 ^= 1; }
                else { ptx::mbar_wait(&bars[1], ph1); ph1 ^= 1; }
            }
            const uint32_t aB = ptx::smem_u32(sA + b * 16384);
            const uint32_t bB = ptx::smem_u32(sB + (size_t)b * a.np * 128);
            gather_store(aB, tid, cur);
            if (more) cur = nxt;
            weight_chunk(a, bB, g0 + gl, kc * 64, tid);
            ptx::fence_proxy_async_smem();
            __syncthreads();
            if (warp == 0) {
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint64_t ad = ptx::sw128_kmajor_desc(aB), bd = ptx::sw128_kmajor_desc(bB);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        ptx::umma<0>(tmem + (uint32_t)(gl * a.np), ad + 2 * kk, bd + 2 * kk, a.idesc,
                                     (kc > 0 || kk > 0) ? 1u : 0u);
                    ptx::umma_commit(&bars[b]);
                }
                __syncwarp();
            }
        }
    }
    {
        const int b = (step - 1) & 1;
        ptx::mbar_wait(&bars[b], b == 0 ? ph0 : ph1);
    }
    ptx::tc_fence_after();

    // epilogue: warp w -> TMEM lanes 32 (w % 4).., groups gl = w / 4, w / 4 + 2, ...
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int m = m0 + row;
    const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16);
    T *__restrict__ y = static_cast<T *>(a.y);
    const T *__restrict__ bias = static_cast<const T *>(a.b);
    const T *__restrict__ z = static_cast<const T *>(a.z);
    for (int gl = warp >> 2; gl < ng; gl += 2) {
        for (int c0 = 0; c0 < a.Kpg; c0 += 16) {
            uint32_t r[16];
            ptx::tmem_ld16_nowait(tl + (uint32_t)(gl * a.np + c0), r);
            ptx::tmem_wait_ld();
            if (m >= a.M) continue;
            const int kbase = (g0 + gl) * a.Kpg + c0;
            const int nv = min(16, a.Kpg - c0);
            T *dst = y + (size_t)m * a.K + kbase;
#pragma unroll
            for (int e = 0; e < 16; e += 2) {
                if (e >= nv) break;
                float v0 = __uint_as_float(r[e]), v1 = __uint_as_float(r[e + 1]);
                if (a.epilogue >= 1) {
                    v0 += static_cast<float>(bias[kbase + e]);
                    if (e + 1 < nv) v1 += static_cast<float>(bias[kbase + e + 1]);
                }
                if (a.epilogue == 3) {
                    v0 += static_cast<float>(z[(size_t)m * a.K + kbase + e]);
                    if (e + 1 < nv) v1 += static_cast<float>(z[(size_t)m * a.K + kbase + e + 1]);
                }
                if (a.epilogue >= 2) { v0 = fmaxf(v0, 0.f); v1 = fmaxf(v1, 0.f); }
                const uint32_t pr = pk2(v0, v1, (T *)nullptr);
                if (e + 1 < nv && ((kbase + e) & 1) == 0) {
                    *reinterpret_cast<uint32_t *>(dst + e) = pr;   // 4-byte aligned pair
                } else {
                    const unsigned short lo = (unsigned short)(pr & 0xFFFFu), hi = (unsigned short)(pr >> 16);
                    reinterpret_cast<unsigned short *>(dst)[e] = lo;
                    if (e + 1 < nv) reinterpret_cast<unsigned short *>(dst)[e + 1] = hi;
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, a.tmem_cols);
}

size_t gconv_tc_smem_bytes(int np) { return 1024 + 2 * 16384 + 2 * (size_t)np * 128 + 64; }

int gconv_tc_launch(GconvArgs a, int dtype, void *stream, std::string *err) {
    uint32_t d = 0;
    d |= 1u << 4;                                        // c_format = F32
    d |= (dtype == WPK_BF16 ? 1u : 0u) << 7;             // a_format (BF16 = 1, F16 = 0)
    d |= (dtype == WPK_BF16 ? 1u : 0u) << 10;            // b_format
    d |= (uint32_t)(a.np >> 3) << 17;                    // n_dim
    d |= (uint32_t)(128 >> 4) << 24;                     // m_dim
    a.idesc = d;
    int cols = 32;
    while (cols < a.gt * a.np) cols <<= 1;
    a.tmem_cols = (uint32_t)cols;
    a.m_tiles = (a.M + kRows - 1) / kRows;
    const long long grid = (long long)a.m_tiles * ((a.groups + a.gt - 1) / a.gt);
    const size_t smem = gconv_tc_smem_bytes(a.np);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)grid);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = smem;
    lc.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    cudaError_t ce;
    if (dtype == WPK_BF16) {
        ce = cudaFuncSetAttribute(gconv_tc_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ce == cudaSuccess) ce = cudaLaunchKernelEx(&lc, gconv_tc_kernel<__nv_bfloat16>, a);
    } else {
        ce = cudaFuncSetAttribute(gconv_tc_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ce == cudaSuccess) ce = cudaLaunchKernelEx(&lc, gconv_tc_kernel<__half>, a);
    }
    if (ce == cudaSuccess) ce = cudaGetLastError();
    if (ce != cudaSuccess) {
        *err = std::string("gconv_tc_kernel launch: ") + cudaGetErrorString(ce);
        return -1;
    }
    return 1;
}

}  // namespace wpk
