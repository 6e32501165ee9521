// KB1: implicit-GEMM forward convolution on 5th-generation tensor cores (tcgen05 / TMEM / TMA).
//
// GEMM view:  D[m, k] = sum_kg A[m, kg] * B[k, kg]
//   m  = (n, p, q) output pixel (M = N*P*Q),   k = output channel,
//   kg = (r, s, c) reduction index, c innermost (NHWC activations, KRSC weights).
//   A[m, (r,s,c)] = x[n, p*sh - ph + r*dh, q*sw - pw + s*dw, c]  (0 outside) -- never materialised:
//   each K block (one filter tap (r,s) x BK channels) is fetched by ONE TMA im2col load of 128
//   output pixels x BK channels (the hardware walks the pixels, applies stride, zero-fills padding).
//   B[k, (r,s,c)] = w[k, r, s, c]: TMA tiled load of BLOCK_N x BK from the [K][R*S][C] weights.
// Both operands land in shared memory in the canonical K-major 128-byte-swizzle layout (BK =
// 128 bytes of K per stage), consumed by tcgen05.mma (kind::f16 for bf16/fp16, kind::tf32) issued
// by one thread; the fp32 accumulator lives in TMEM (double-buffered: 2 x BLOCK_N columns), so the
// epilogue of tile i overlaps the main loop of tile i+1.
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer,
// warps 2-5 = epilogue (tcgen05.ld -> +bias -> ReLU -> round -> 16-byte vector stores, or fp32
// split-K partials). Persistent grid: CTAs loop over work items (tile, split) with a static
// round-robin schedule; RASTER picks which GEMM dimension varies fastest.
//
// The fused epilogue realises the paper's operator fusion ("write one CUDA kernel
// function for the fused operator"; SPEC.md:136 relu(bias_add(conv))).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ptx.cuh"
#include "umma_conv.h"

namespace wpk {

enum { DT_F16 = 0, DT_BF16 = 1, DT_TF32 = 2 };

template <int DT> struct OutT;
template <> struct OutT<DT_F16> { using T = __half; };
template <> struct OutT<DT_BF16> { using T = __nv_bfloat16; };
template <> struct OutT<DT_TF32> { using T = float; };

__device__ __forceinline__ float ld_bias(const __half *b, int k) { return __half2float(b[k]); }
__device__ __forceinline__ float ld_bias(const __nv_bfloat16 *b, int k) { return __bfloat162float(b[k]); }
__device__ __forceinline__ float ld_bias(const float *b, int k) { return b[k]; }

__device__ __forceinline__ uint32_t pack2(float a, float b, __half *) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ uint32_t pack2(float a, float b, __nv_bfloat16 *) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ uint32_t pack2(float, float, float *) { return 0u; }   // unused (fp32 out)
__device__ __forceinline__ void st_out(__half *p, float v) { *p = __float2half_rn(v); }
__device__ __forceinline__ void st_out(__nv_bfloat16 *p, float v) { *p = __float2bfloat16_rn(v); }
__device__ __forceinline__ void st_out(float *p, float v) { *p = v; }

struct WorkPos {
    int mt, nt, split;
};
__device__ __forceinline__ WorkPos decode_work(long long w, const UmmaArgs &a) {
    WorkPos r;
    r.split = (int)(w % a.splits);
    long long t = w / a.splits;
    if (a.raster == 0) {
        r.mt = (int)(t / a.n_tiles);
        r.nt = (int)(t % a.n_tiles);
    } else {
        r.nt = (int)(t / a.m_tiles);
        r.mt = (int)(t % a.m_tiles);
    }
    return r;
}

// Epilogue for one 32-row x (column chunk) slab: TMEM -> registers -> (+bias, ReLU, round) ->
// swizzled smem staging -> TMA store (epi_tma), or direct global stores.
template <typename T>
struct EpiCtx {
    const UmmaArgs *a;
    const float *sBias;
    uint8_t *sEpi;        // this warp's 2 x 4 KB staging buffers
    uint32_t ebuf;
    int lane;
    int nbufs;
};

template <typename T>
__device__ __forceinline__ void epi_chunk_tma(EpiCtx<T> &E, const CUtensorMap *tmY, uint32_t taddr, int k0, int mrow,
                                              int split, bool final_out) {
    const UmmaArgs &a = *E.a;
    uint32_t pk[32];
    // all TMEM loads of the 128-byte chunk in flight at once, one wait
    uint32_t raw[64];
    const int nsub = (final_out && sizeof(T) == 2) ? 4 : 2;
#pragma unroll
    for (int sub = 0; sub < 4; ++sub)
        if (sub < nsub) ptx::tmem_ld16_nowait(taddr + sub * 16, raw + sub * 16);
    ptx::tmem_wait_ld();
    if (final_out && sizeof(T) == 2) {
#pragma unroll
        for (int sub = 0; sub < 4; ++sub) {
            float v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                v[j] = __uint_as_float(raw[sub * 16 + j]) + E.sBias[min(k0 + sub * 16 + j, a.K - 1)];
                if (a.epilogue == 2) v[j] = fmaxf(v[j], 0.f);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) pk[sub * 8 + j] = pack2(v[2 * j], v[2 * j + 1], (T *)nullptr);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            float v = __uint_as_float(raw[j]);
            if (final_out) {
                v += E.sBias[min(k0 + j, a.K - 1)];
                if (a.epilogue == 2) v = fmaxf(v, 0.f);
            }
            pk[j] = __float_as_uint(v);
        }
    }
    // staging buffer reuse: the TMA store issued two chunks ago must have finished reading it
    if (E.lane == 0) {
        if (E.nbufs == 2) ptx::bulk_wait_read<1>();
        else ptx::bulk_wait_read<0>();
    }
    __syncwarp();
    uint8_t *bufp = E.sEpi + E.ebuf * 4096;
    const uint32_t buf = ptx::smem_u32(bufp) + (uint32_t)E.lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        ptx::st_shared_v4(buf + ((uint32_t)(j ^ (E.lane & 7)) << 4), pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (E.lane == 0) {
        if (final_out) ptx::tma_store_2d(tmY, bufp, k0, mrow);
        else ptx::tma_store_3d(tmY, bufp, k0, mrow, split);
        ptx::bulk_commit();
    }
    if (E.nbufs == 2) E.ebuf ^= 1;
}

template <typename T>
__device__ __forceinline__ void epi_chunk_direct(EpiCtx<T> &E, uint32_t taddr, int k0, long long m, int split,
                                                 bool final_out) {
    const UmmaArgs &a = *E.a;
    float v[16];
    ptx::tmem_ld16(taddr, v);
    if (m >= a.M) return;
    const bool full16 = (k0 + 16 <= a.K);
    if (!final_out) {
        float *dst = a.partial + ((long long)split * a.M + m) * a.K + k0;
        if (full16 && a.vec_ok) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
                *reinterpret_cast<float4 *>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (k0 + j < a.K) dst[j] = v[j];
        }
        return;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        v[j] += E.sBias[min(k0 + j, a.K - 1)];
        if (a.epilogue == 2) v[j] = fmaxf(v[j], 0.f);
    }
    T *y = static_cast<T *>(a.y);
    if (a.out_nchw) {
        const long long nimg = m / a.PQ;
        const long long base = nimg * (long long)a.K * a.PQ + (m - nimg * a.PQ);
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (k0 + j < a.K) st_out(y + base + (long long)(k0 + j) * a.PQ, v[j]);
        return;
    }
    T *dst = y + m * a.K + k0;
    if (full16 && a.vec_ok) {
        if constexpr (sizeof(T) == 2) {
            uint32_t u[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) u[j] = pack2(v[2 * j], v[2 * j + 1], (T *)nullptr);
            reinterpret_cast<uint4 *>(dst)[0] = make_uint4(u[0], u[1], u[2], u[3]);
            reinterpret_cast<uint4 *>(dst)[1] = make_uint4(u[4], u[5], u[6], u[7]);
        } else {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
                *reinterpret_cast<float4 *>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (k0 + j < a.K) st_out(dst + j, v[j]);
    }
}

// In-kernel split-K fixup ("serial reduction by the last arriving split"): every split publishes its
// fp32 partial tile, bumps the tile's counter; the CTA that completes the count sums all partials
// in the fixed split order 0..S-1 (deterministic, independent of arrival order), applies bias+ReLU,
// rounds once and stores the output, then resets the counter for the next launch.
template <typename T>
__device__ __noinline__ void splitk_fixup(const UmmaArgs &a, const float *sBias, volatile int *sFlag, const WorkPos &wp,
                                          int nsub, int warp, int lane) {
    if (a.epi_tma && lane == 0) ptx::bulk_wait_all();   // this warp's partial stores are complete
    __syncwarp();
    __threadfence();
    ptx::named_bar_sync(1, 256);                         // all 8 epilogue warps published
    const int tile = wp.mt * a.n_tiles + wp.nt;
    if (warp == 4 && lane == 0) {
        const int old = atomicAdd(a.counters + tile, 1);
        *sFlag = (old == a.splits - 1) ? 1 : 0;
    }
    ptx::named_bar_sync(1, 256);
    const bool last = (*sFlag != 0);
    if (!last) return;
    __threadfence();
    // Final pass, coalesced: a warp sums 128 consecutive columns (4 per lane) of one output row over
    // the splits (all splits' loads issued before the in-order sum).
    T *y = static_cast<T *>(a.y);
    const int n0 = wp.nt * a.bn;
    const int ncols = min(a.bn, a.K - n0);
    const int cblocks = (ncols + 127) / 128;
    const int items = nsub * 128 * cblocks;
    const long long MK = a.M * (long long)a.K;
    const long long m0 = (long long)wp.mt * a.bm;
    const bool vec = (a.K % 4) == 0;
    // 4 items x 4 splits of 16-byte loads in flight per lane (the fixup is L2-latency bound)
    constexpr int U = 4;
    for (int base = warp - 4; base < items; base += 8 * U) {
        long long mm[U];
        int kk[U];
        bool ok[U];
        float4 acc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int item = base + u * 8;
            const int r = item / cblocks, cb = item - (item / cblocks) * cblocks;
            mm[u] = m0 + r;
            kk[u] = n0 + cb * 128 + lane * 4;
            ok[u] = item < items && mm[u] < a.M && kk[u] < n0 + ncols;
            acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        bool all_v4 = vec;
#pragma unroll
        for (int u = 0; u < U; ++u) all_v4 = all_v4 && (!ok[u] || kk[u] + 3 < a.K);
        if (all_v4) {
            for (int sp0 = 0; sp0 < a.splits; sp0 += 4) {
                float4 q[4][U];
#pragma unroll
                for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        q[s4][u] = (ok[u] && sp0 + s4 < a.splits)
                            ? __ldcg(reinterpret_cast<const float4 *>(a.partial + (sp0 + s4) * MK + mm[u] * a.K + kk[u]))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        acc[u].x += q[s4][u].x; acc[u].y += q[s4][u].y; acc[u].z += q[s4][u].z; acc[u].w += q[s4][u].w;
                    }
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!ok[u]) continue;
                for (int sp = 0; sp < a.splits; ++sp) {
                    const float *s = a.partial + sp * MK + mm[u] * a.K + kk[u];
                    acc[u].x += __ldcg(s);
                    if (kk[u] + 1 < a.K) acc[u].y += __ldcg(s + 1);
                    if (kk[u] + 2 < a.K) acc[u].z += __ldcg(s + 2);
                    if (kk[u] + 3 < a.K) acc[u].w += __ldcg(s + 3);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
            const long long m = mm[u];
            const int k = kk[u];
            float v[4] = {acc[u].x, acc[u].y, acc[u].z, acc[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                v[j] += sBias[min(k + j, a.K - 1)];
                if (a.epilogue == 2) v[j] = fmaxf(v[j], 0.f);
            }
            if (a.out_nchw) {
                const long long nimg = m / a.PQ;
                const long long ob = nimg * (long long)a.K * a.PQ + (m - nimg * a.PQ);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (k + j < a.K) st_out(y + ob + (long long)(k + j) * a.PQ, v[j]);
            } else {
                T *dst = y + m * a.K + k;
                if (vec && k + 3 < a.K) {
                    if constexpr (sizeof(T) == 2) {
                        const uint32_t lo = pack2(v[0], v[1], (T *)nullptr), hi = pack2(v[2], v[3], (T *)nullptr);
                        *reinterpret_cast<uint2 *>(dst) = make_uint2(lo, hi);
                    } else {
                        *reinterpret_cast<float4 *>(dst) = make_float4(v[0], v[1], v[2], v[3]);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (k + j < a.K) st_out(dst + j, v[j]);
                }
            }
        }
    }
    ptx::named_bar_sync(1, 256);
    if (warp == 4 && lane == 0) a.counters[tile] = 0;    // self-resetting for the next launch
}

// 12 warps: 0 = A producer, 1 = TMEM allocator + MMA issuer, 2 = B producer, 3 = spare,
// 4..11 = epilogue (two groups of four; warp w reads TMEM lanes [32*(w%4), +32)).
template <int DT, bool kGather, bool kPair>
__global__ void __launch_bounds__(kGather ? 512 : 384, 1)
    umma_conv_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmY, const __grid_constant__ UmmaArgs a) {
    using T = typename OutT<DT>::T;
    constexpr bool kTF32 = (DT == DT_TF32);

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    uint8_t *smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
    // CTA pair (cta_group::2): each CTA holds 128 rows of A and half of B; the pair computes 256 x BN
    const uint32_t a_bytes = (uint32_t)(kPair ? 128 : a.bm) * 128u;
    const uint32_t b_bytes = (uint32_t)(kPair ? a.bn / 2 : a.bn) * 128u;
    const int nsub = kPair ? 1 : a.bm / 128;                           // 128-row MMAs per tile per CTA
    const uint32_t crank = kPair ? ptx::cluster_ctarank() : 0u;
    const bool leader = (crank == 0);
    const long long wstart = kPair ? (long long)(blockIdx.x >> 1) : (long long)blockIdx.x;
    const long long wstep = kPair ? (long long)(gridDim.x >> 1) : (long long)gridDim.x;
    uint8_t *smA = smem;
    uint8_t *smB = smem + (size_t)a.stages * a_bytes;
    uint8_t *sEpi = smem + a.epi_off;                                  // [8 warps][2][32 rows][128 B]
    float *sBias = reinterpret_cast<float *>(smem + a.bias_off);      // [K]
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + a.bar_off);
    uint64_t *full = bars;            // [8]
    uint64_t *empty = bars + 8;       // [8]
    uint64_t *tfull = bars + 16;      // [2]
    uint64_t *tempty = bars + 18;     // [2]
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 20);
    volatile int *sFlag = reinterpret_cast<volatile int *>(bars + 21);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long *dbg = a.dbg ? a.dbg + blockIdx.x * 16 : nullptr;
    if (dbg && threadIdx.x == 0) dbg[0] = ptx::globaltimer();

    if (warp == 0 && lane == 0) {
        if (!kGather) ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        if (a.epi_tma) ptx::prefetch_tmap(&tmY);
        for (int s = 0; s < a.stages; ++s) {
            ptx::mbar_init(&full[s], kGather ? 5 : 2);   // A (TMA, or 4 gather warps) + B producer
            ptx::mbar_init(&empty[s], 1);      // MMA commit
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&tfull[s], 1);
            ptx::mbar_init(&tempty[s], kPair ? 16 : 8);   // 8 epilogue warps (x2 CTAs for a pair)
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) {
        if (kPair) {
            ptx::tmem_alloc2(tmem_holder, a.tmem_cols);
            ptx::tmem_relinquish2();
        } else {
            ptx::tmem_alloc(tmem_holder, a.tmem_cols);
            ptx::tmem_relinquish();
        }
    }
    // Programmatic dependent launch: this prologue overlaps the previous kernel's tail. Weights and
    // bias are inference constants, so the bias is staged and the first weight tiles of
    // this CTA are prefetched into L2 before waiting; activations (which the previous layer may
    // produce) are only read after griddepcontrol.wait.
    if (warp >= 4) {   // bias -> smem once (fp32); zero when there is no bias or for split-K partials
        const T *bias = static_cast<const T *>(a.bias);
        for (int k = threadIdx.x - 128; k < a.K; k += 256)
            sBias[k] = (a.epilogue >= 1) ? ld_bias(bias, k) : 0.f;
    }
    if (warp == 2 && lane == 0 && wstart < a.work) {
        const WorkPos wp = decode_work(wstart, a);
        const int n0 = wp.nt * a.bn + (int)crank * (kPair ? a.bn / 2 : 0);
        const int kb0 = wp.split * a.kb_per_split;
        const int kb1 = min(a.num_kb, kb0 + min(a.kb_per_split, a.stages));
        for (int kb = kb0; kb < kb1; ++kb)
            ptx::tma_prefetch_3d(&tmB, (kb % a.c_blocks) * a.bk, kb / a.c_blocks, n0);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    if (kPair) ptx::cluster_sync();   // peer barriers initialised before any remote arrive / TMA
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    if (dbg && threadIdx.x == 0) dbg[1] = ptx::globaltimer();

    if (warp == 0 || warp == 2) {
        // ===================== TMA producers: warp 0 -> A (activations), warp 2 -> B (weights) ====
        if (lane == 0 && !(kGather && warp == 0)) {
            const bool isA = (warp == 0);
            uint32_t stage = 0, phase = 0;
            const uint32_t tx = isA ? a_bytes : b_bytes;
            uint8_t *dst0 = isA ? smA : smB;
            for (long long w = wstart; w < a.work; w += wstep) {
                const WorkPos wp = decode_work(w, a);
                const long long m0 = (long long)wp.mt * a.bm + crank * 128;
                const int n0 = wp.nt * a.bn + (int)crank * (a.bn / 2);
                int wc = 0, hc = 0, nimg = 0;
                if (isA && !a.a_tiled) {
                    nimg = (int)(m0 / a.PQ);
                    const int rem = (int)(m0 - (long long)nimg * a.PQ);
                    const int p = rem / a.Q, q = rem - (rem / a.Q) * a.Q;
                    wc = q * a.stride_w - a.pad_w;
                    hc = p * a.stride_h - a.pad_h;
                }
                const int kb0 = wp.split * a.kb_per_split;
                const int kb1 = min(a.num_kb, kb0 + a.kb_per_split);
                // (r, s, c-block) of kb0, then advanced incrementally (no divisions in the k loop)
                int cb = kb0 % a.c_blocks;
                int rs = kb0 / a.c_blocks;
                int r = rs / a.S, s = rs % a.S;
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t *dst = dst0 + stage * tx;
                    if (kPair) {
                        // both CTAs' bytes land on the leader's barrier; only the leader arms it
                        if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * tx);
                        if (!isA)
                            ptx::tma_load_3d_pair(dst, &tmB, &full[stage], cb * a.bk, rs, n0);
                        else if (a.a_tiled)
                            ptx::tma_load_2d_pair(dst, &tmA, &full[stage], cb * a.bk, (int)m0);
                        else
                            ptx::tma_load_im2col_4d_pair(dst, &tmA, &full[stage], cb * a.bk, wc, hc, nimg,
                                                         (uint16_t)(s * a.dil_w), (uint16_t)(r * a.dil_h));
                    } else {
                        ptx::mbar_arrive_expect_tx(&full[stage], tx);
                        if (!isA)
                            ptx::tma_load_3d(dst, &tmB, &full[stage], cb * a.bk, rs, n0);
                        else if (a.a_tiled)
                            ptx::tma_load_2d(dst, &tmA, &full[stage], cb * a.bk, (int)m0);
                        else
                            ptx::tma_load_im2col_4d(dst, &tmA, &full[stage], cb * a.bk, wc, hc, nimg,
                                                    (uint16_t)(s * a.dil_w), (uint16_t)(r * a.dil_h));
                    }
                    if (++cb == a.c_blocks) {
                        cb = 0;
                        ++rs;
                        if (++s == a.S) { s = 0; ++r; }
                    }
                    if (++stage == (uint32_t)a.stages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (kGather && warp >= 12) {
        // ===================== gather producers (A_MODE 2): implicit im2col straight into the
        // 128-byte-swizzled K-major A stage, for layers whose channel count is too small for TMA
        // im2col boxes. kg = (r*S + s)*C + c; one thread owns BM/128 rows of every stage.
        const int t = threadIdx.x - 384;                       // 0..127
        const int RSC = a.R * a.S * a.C;
        uint32_t stage = 0, phase = 0;
        for (long long w = wstart; w < a.work; w += wstep) {
            const WorkPos wp = decode_work(w, a);
            const int kb0 = wp.split * a.kb_per_split;
            const int kb1 = min(a.num_kb, kb0 + a.kb_per_split);
            int rh0[2], rw0[2], rn[2];
            bool rv[2];
            for (int hh = 0; hh < nsub; ++hh) {
                const long long m = (long long)wp.mt * a.bm + hh * 128 + t;
                rv[hh] = m < a.M;
                const long long mm = rv[hh] ? m : 0;
                const int n = (int)(mm / a.PQ);
                const int rem = (int)(mm - (long long)n * a.PQ);
                const int p = rem / a.Q, q = rem - (rem / a.Q) * a.Q;
                rn[hh] = n;
                rh0[hh] = p * a.stride_h - a.pad_h;
                rw0[hh] = q * a.stride_w - a.pad_w;
            }
            for (int kb = kb0; kb < kb1; ++kb) {
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                for (int hh = 0; hh < nsub; ++hh) {
                    const int row = hh * 128 + t;
                    const uint32_t rbase = ptx::smem_u32(smA + stage * a_bytes) + (uint32_t)(row >> 3) * 1024u +
                                           (uint32_t)(row & 7) * 128u;
                    constexpr int PC = kTF32 ? 4 : 8;          // elements per 16-byte chunk
                    int kg = kb * PC * 8;                      // first element of this 128-byte K block
                    int c = kg % a.C, rs_ = kg / a.C;
                    int s = rs_ % a.S, r = rs_ / a.S;
                    // two chunks (16 independent loads) in flight at a time; 32-bit offsets
#pragma unroll 1
                    for (int j = 0; j < 8; j += 2) {
                        int off[2 * PC];
                        bool okv[2 * PC];
#pragma unroll
                        for (int e = 0; e < 2 * PC; ++e, ++kg) {
                            const int hi = rh0[hh] + r * a.dil_h, wi = rw0[hh] + s * a.dil_w;
                            okv[e] = rv[hh] && kg < RSC && hi >= 0 && hi < a.H && wi >= 0 && wi < a.W;
                            off[e] = a.x_nchw ? ((rn[hh] * a.C + c) * a.H + hi) * a.W + wi
                                              : ((rn[hh] * a.H + hi) * a.W + wi) * a.C + c;
                            if (++c == a.C) { c = 0; if (++s == a.S) { s = 0; ++r; } }
                        }
                        uint32_t bits[2 * PC];
#pragma unroll
                        for (int e = 0; e < 2 * PC; ++e)
                            bits[e] = !okv[e] ? 0u
                                      : kTF32 ? __ldg(reinterpret_cast<const unsigned *>(a.x) + off[e])
                                              : (uint32_t)__ldg(reinterpret_cast<const unsigned short *>(a.x) + off[e]);
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            uint32_t wv[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                wv[q] = kTF32 ? bits[jj * 4 + q]
                                              : (bits[jj * 8 + 2 * q] | (bits[jj * 8 + 2 * q + 1] << 16));
                            ptx::st_shared_v4(rbase + ((uint32_t)((j + jj) ^ (row & 7)) << 4), wv[0], wv[1], wv[2], wv[3]);
                        }
                    }
                }
                ptx::fence_proxy_async_smem();                 // generic-proxy writes -> async-proxy (MMA) reads
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&full[stage]);
                if (++stage == (uint32_t)a.stages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (single thread; the leader CTA of a pair) =====================
        if (lane == 0 && leader) {
            uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
            const uint64_t a_desc0 = ptx::sw128_kmajor_desc(ptx::smem_u32(smA));
            const uint64_t b_desc0 = ptx::sw128_kmajor_desc(ptx::smem_u32(smB));
            const uint32_t acc_cols = (uint32_t)(nsub * a.bn);
            for (long long w = wstart; w < a.work; w += wstep) {
                const WorkPos wp = decode_work(w, a);
                const int kb0 = wp.split * a.kb_per_split;
                const int kb1 = min(a.num_kb, kb0 + a.kb_per_split);
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * acc_cols;
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    if (dbg && w == blockIdx.x && kb == kb0) dbg[2] = ptx::globaltimer();
                    const uint64_t ad = a_desc0 + (uint64_t)((stage * a_bytes) >> 4);
                    const uint64_t bd = b_desc0 + (uint64_t)((stage * b_bytes) >> 4);
                    if (kPair) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            ptx::umma2<kTF32>(d_tmem, ad + 2 * kk, bd + 2 * kk, a.idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
                        ptx::umma_commit2_multicast(&empty[stage]);   // frees the stage in both CTAs
                    } else {
                        for (int h = 0; h < nsub; ++h) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)   // 4 x 32 bytes of K per 128-byte stage (+2 desc units)
                                ptx::umma<kTF32>(d_tmem + h * a.bn, ad + h * (16384 >> 4) + 2 * kk, bd + 2 * kk, a.idesc,
                                                 (kb > kb0 || kk > 0) ? 1u : 0u);
                        }
                        ptx::umma_commit(&empty[stage]);   // frees this smem stage when the MMAs finish
                    }
                    if (++stage == (uint32_t)a.stages) { stage = 0; phase ^= 1; }
                }
                if (kPair) ptx::umma_commit2_multicast(&tfull[acc]);   // both CTAs' accumulator halves ready
                else ptx::umma_commit(&tfull[acc]);                     // accumulator ready for the epilogue
                if (dbg && w == blockIdx.x) dbg[3] = ptx::globaltimer();
                if (++acc == (uint32_t)a.acc_stages) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else if (warp >= 4 && warp < 12) {
        // ===================== epilogue warps 4..11 =====================
        const int quarter = warp & 3;          // TMEM lane quarter this warp may access
        const int grp = (warp - 4) >> 2;       // 0 or 1
        uint32_t acc = 0, acc_phase = 0;
        const bool final_out = (a.splits == 1);
        EpiCtx<T> E{&a, sBias, sEpi + (size_t)(warp - 4) * a.epi_bufs * 4096, 0u, lane, a.epi_bufs};
        const uint32_t acc_cols = (uint32_t)(nsub * a.bn);
        const int cw = a.epi_tma ? (final_out ? (int)(128 / sizeof(T)) : 32) : 16;
        const int nchunks = (a.bn + cw - 1) / cw;
        for (long long w = wstart; w < a.work; w += wstep) {
            const WorkPos wp = decode_work(w, a);
            const int n0 = wp.nt * a.bn;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            // slabs = (h, chunk) pairs; group g takes h == g when nsub == 2, else every other chunk
            for (int h = 0; h < nsub; ++h) {
                if (nsub == 2 && h != grp) continue;
                const int mrow = wp.mt * a.bm + (int)crank * 128 + h * 128 + quarter * 32;
                const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * acc_cols + h * a.bn;
                for (int ci = (nsub == 2 ? 0 : grp); ci < nchunks; ci += (nsub == 2 ? 1 : 2)) {
                    const int c0 = ci * cw;
                    const int k0 = n0 + c0;
                    if (k0 >= a.K) break;   // warp-uniform
                    if (a.epi_tma) {
                        epi_chunk_tma<T>(E, &tmY, tbase + c0, k0, mrow, wp.split, final_out);
                    } else {
                        epi_chunk_direct<T>(E, tbase + c0, k0, (long long)mrow + lane, wp.split, final_out);
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (dbg && warp == 4 && lane == 0 && w == blockIdx.x) dbg[4] = ptx::globaltimer();
            if (dbg && warp == 4 && lane == 0) {   // per-tile epilogue completion times (first 8 tiles)
                const long long it = (w - wstart) / wstep;
                if (it < 8) dbg[8 + it] = ptx::globaltimer();
            }
            if (lane == 0) {                                  // TMEM free: the MMA may start the next tile
                if (kPair) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
                else ptx::mbar_arrive(&tempty[acc]);
            }
            if (++acc == (uint32_t)a.acc_stages) { acc = 0; acc_phase ^= 1; }
            if (!final_out) splitk_fixup<T>(a, sBias, sFlag, wp, nsub, warp, lane);
        }
        if (a.epi_tma && lane == 0) ptx::bulk_wait_all();
        if (dbg && warp == 4 && lane == 0) dbg[5] = ptx::globaltimer();
    }

    __syncthreads();
    if (kPair) ptx::cluster_sync();   // the peer no longer touches our barriers / TMEM
    if (dbg && threadIdx.x == 0) dbg[6] = ptx::globaltimer();
    if (warp == 1) {
        ptx::tc_fence_after();
        if (kPair) ptx::tmem_dealloc2(tmem_base, a.tmem_cols);
        else ptx::tmem_dealloc(tmem_base, a.tmem_cols);
    }
}

// ---------------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*EncodeIm2colFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const int *, const int *, cuuint32_t, cuuint32_t,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void *driver_sym(const char *name) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
    return fn;
}

static EncodeTiledFn encode_tiled() {
    static EncodeTiledFn f = (EncodeTiledFn)driver_sym("cuTensorMapEncodeTiled");
    return f;
}
static EncodeIm2colFn encode_im2col() {
    static EncodeIm2colFn f = (EncodeIm2colFn)driver_sym("cuTensorMapEncodeIm2col");
    return f;
}

static uint32_t make_idesc(int dt, int bm, int bn) {
    uint32_t fmt = (dt == DT_F16) ? 0u : (dt == DT_BF16) ? 1u : 2u;
    uint32_t d = 0;
    d |= 1u << 4;                          // c_format = F32
    d |= fmt << 7;                         // a_format
    d |= fmt << 10;                        // b_format
    // a_major = b_major = 0 (K-major), no negate, dense
    d |= (uint32_t)(bn >> 3) << 17;        // n_dim
    d |= (uint32_t)(bm >> 4) << 24;        // m_dim
    return d;
}

template <int DT, bool G, bool PAIR>
static bool set_smem_attr() {
    static bool done = false;
    if (!done) {
        if (cudaFuncSetAttribute(umma_conv_kernel<DT, G, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) !=
            cudaSuccess)
            return false;
        done = true;
    }
    return true;
}

int umma_launch(const UmmaLaunch &L, std::string *err) {
    const int dt = L.dtype == WPK_F16 ? DT_F16 : L.dtype == WPK_BF16 ? DT_BF16 : DT_TF32;
    const int e = (dt == DT_TF32) ? 4 : 2;
    const CUtensorMapDataType tdt = (dt == DT_F16)    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                    : (dt == DT_BF16) ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                      : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    if (!encode_tiled() || !encode_im2col()) {
        *err = "cuTensorMapEncode* driver entry points unavailable";
        return -1;
    }
    const UmmaGeom &g = L.g;
    CUtensorMap tmA, tmB, tmY;
    UmmaMapCache *mc = L.cache;
    const bool hit = mc && mc->valid && mc->x == L.x && mc->w == L.w && mc->y == L.y && mc->partial == L.partial &&
                     mc->cfg == L.cfg;
    if (hit) {
        tmA = mc->a;
        tmB = mc->b;
        tmY = mc->yy;
        goto launch;
    }
    // ---- A: im2col view of x[N][H][W][Cp] (or a plain [N*H*W][Cp] matrix for 1x1/s1/p0) --------
    std::memset(&tmY, 0, sizeof tmY);
    std::memset(&tmA, 0, sizeof tmA);
    if (g.a_mode == 2) {
        // gather producer: no A tensor map
    } else if (g.a_tiled) {
        cuuint64_t dims[2] = {(cuuint64_t)g.cpad, (cuuint64_t)L.a_rows};
        cuuint64_t strides[1] = {(cuuint64_t)g.cpad * e};
        cuuint32_t box[2] = {(cuuint32_t)g.bk, (cuuint32_t)(g.pair ? 128 : g.bm)};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = encode_tiled()(&tmA, tdt, 2, const_cast<void *>(L.x), dims, strides, box, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            *err = "cuTensorMapEncodeTiled(A) failed (" + std::to_string((int)r) + ")";
            return -1;
        }
    } else {
        cuuint64_t dims[4] = {(cuuint64_t)g.cpad, (cuuint64_t)L.W, (cuuint64_t)L.H, (cuuint64_t)L.N};
        cuuint64_t strides[3] = {(cuuint64_t)g.cpad * e, (cuuint64_t)g.cpad * e * L.W,
                                 (cuuint64_t)g.cpad * e * L.W * L.H};
        int lower[2] = {-L.pad_w, -L.pad_h};
        int upper[2] = {L.pad_w - (L.S - 1) * L.dil_w, L.pad_h - (L.R - 1) * L.dil_h};
        cuuint32_t estr[4] = {1, (cuuint32_t)L.stride_w, (cuuint32_t)L.stride_h, 1};
        CUresult r = encode_im2col()(&tmA, tdt, 4, const_cast<void *>(L.x), dims, strides, lower, upper,
                                     (cuuint32_t)g.bk, (cuuint32_t)(g.pair ? 128 : g.bm), estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            *err = "cuTensorMapEncodeIm2col failed (" + std::to_string((int)r) + ")";
            return -1;
        }
    }
    // ---- Y: TMA-store view of the NHWC output [M][K] (or the fp32 split-K partials [S][M][K]) ---
    if (g.epi_tma) {
        const long long M = (long long)L.N * L.P * L.Q;
        CUresult r;
        if (g.splits == 1) {
            cuuint64_t dims[2] = {(cuuint64_t)L.K, (cuuint64_t)M};
            cuuint64_t strides[1] = {(cuuint64_t)L.K * e};
            cuuint32_t box[2] = {(cuuint32_t)(128 / e), 32};
            cuuint32_t estr[2] = {1, 1};
            r = encode_tiled()(&tmY, tdt, 2, L.y, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t dims[3] = {(cuuint64_t)L.K, (cuuint64_t)M, (cuuint64_t)g.splits};
            cuuint64_t strides[2] = {(cuuint64_t)L.K * 4, (cuuint64_t)L.K * 4 * M};
            cuuint32_t box[3] = {32, 32, 1};
            cuuint32_t estr[3] = {1, 1, 1};
            r = encode_tiled()(&tmY, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, L.partial, dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) {
            *err = "cuTensorMapEncodeTiled(Y) failed (" + std::to_string((int)r) + ")";
            return -1;
        }
    }
    // ---- B: tiled view of w[K][R*S][Cp] ---------------------------------------------------------
    {
        cuuint64_t dims[3] = {(cuuint64_t)g.cpad, (cuuint64_t)L.b_rs, (cuuint64_t)L.K};
        cuuint64_t strides[2] = {(cuuint64_t)g.cpad * e, (cuuint64_t)g.cpad * e * L.b_rs};
        cuuint32_t box[3] = {(cuuint32_t)g.bk, 1, (cuuint32_t)(g.pair ? g.bn / 2 : g.bn)};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode_tiled()(&tmB, tdt, 3, const_cast<void *>(L.w), dims, strides, box, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            *err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
            return -1;
        }
    }
    if (mc) {
        mc->x = L.x; mc->w = L.w; mc->y = L.y; mc->partial = L.partial; mc->cfg = L.cfg;
        mc->a = tmA; mc->b = tmB; mc->yy = tmY; mc->valid = true;
    }
launch:
    UmmaArgs a{};
    a.bias = L.b;
    a.y = L.y;
    a.partial = L.partial;
    a.M = (long long)L.N * L.P * L.Q;
    a.K = L.K;
    a.P = L.P;
    a.Q = L.Q;
    a.PQ = (long long)L.P * L.Q;
    a.stride_h = L.stride_h; a.stride_w = L.stride_w; a.pad_h = L.pad_h; a.pad_w = L.pad_w;
    a.dil_h = L.dil_h; a.dil_w = L.dil_w; a.S = L.S;
    a.c_blocks = g.c_blocks; a.num_kb = g.num_kb; a.kb_per_split = g.kb_per_split; a.splits = g.splits;
    a.m_tiles = g.m_tiles; a.n_tiles = g.n_tiles; a.raster = g.raster; a.work = g.work;
    a.bm = g.bm; a.bn = g.bn; a.bk = g.bk; a.stages = g.stages; a.acc_stages = g.acc_stages;
    a.idesc = make_idesc(dt, g.pair ? 256 : 128, g.bn);   // 1-CTA: 128 x BN (BLOCK_M 256 = two); pair: 256 x BN
    a.tmem_cols = (uint32_t)g.tmem_cols;
    a.epilogue = L.epilogue;
    a.out_nchw = L.out_nchw;
    a.vec_ok = (L.K % 16 == 0) ? 1 : 0;   // 16-element chunks start 32/64-byte aligned
    a.a_tiled = g.a_tiled;
    a.epi_tma = g.epi_tma;
    a.epi_off = (uint32_t)g.epi_off;
    a.epi_bufs = g.epi_bufs;
    a.bias_off = (uint32_t)g.bias_off;
    a.bar_off = (uint32_t)g.bar_off;
    a.dbg = L.dbg;
    a.counters = L.counters;
    a.x = L.x;
    a.x_nchw = L.x_nchw;
    a.C = L.C; a.H = L.H; a.W = L.W; a.R = L.R;
    cudaStream_t st = (cudaStream_t)L.stream;
    long long grid = (long long)L.sm_count * g.ctas_per_sm;
    if (grid > g.work) grid = g.work;
    if (g.pair) grid = 2 * std::min<long long>(g.work, L.sm_count / 2);
    int launches = 0;
    cudaError_t ce = cudaSuccess;
#define WPK_LAUNCH_UMMA(DTV)                                                                          \
    do {                                                                                              \
        if (g.a_mode == 2) {                                                                          \
            if (!set_smem_attr<DTV, true, false>()) { *err = "cudaFuncSetAttribute failed"; return -1; } \
            ce = cudaLaunchKernelEx(&lc, umma_conv_kernel<DTV, true, false>, tmA, tmB, tmY, a);      \
        } else if (g.pair) {                                                                          \
            if (!set_smem_attr<DTV, false, true>()) { *err = "cudaFuncSetAttribute failed"; return -1; } \
            ce = cudaLaunchKernelEx(&lc, umma_conv_kernel<DTV, false, true>, tmA, tmB, tmY, a);      \
        } else {                                                                                      \
            if (!set_smem_attr<DTV, false, false>()) { *err = "cudaFuncSetAttribute failed"; return -1; } \
            ce = cudaLaunchKernelEx(&lc, umma_conv_kernel<DTV, false, false>, tmA, tmB, tmY, a);     \
        }                                                                                             \
    } while (0)
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)grid);
    lc.blockDim = dim3(g.a_mode == 2 ? 512 : 384);
    lc.dynamicSmemBytes = g.smem_bytes;
    lc.stream = st;
    cudaLaunchAttribute attr[2];
    int nattr = 0;
    if (!getenv("WPK_NO_PDL")) {
        attr[nattr].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[nattr].val.programmaticStreamSerializationAllowed = 1;
        ++nattr;
    }
    if (g.pair) {   // the two CTAs of a tcgen05 CTA pair form a cluster
        attr[nattr].id = cudaLaunchAttributeClusterDimension;
        attr[nattr].val.clusterDim.x = 2;
        attr[nattr].val.clusterDim.y = 1;
        attr[nattr].val.clusterDim.z = 1;
        ++nattr;
    }
    lc.attrs = attr;
    lc.numAttrs = nattr;
    if (dt == DT_F16) WPK_LAUNCH_UMMA(DT_F16);
    else if (dt == DT_BF16) WPK_LAUNCH_UMMA(DT_BF16);
    else WPK_LAUNCH_UMMA(DT_TF32);
#undef WPK_LAUNCH_UMMA
    if (ce == cudaSuccess) ce = cudaGetLastError();
    if (ce != cudaSuccess) {
        *err = std::string("umma_conv_kernel launch: ") + cudaGetErrorString(ce);
        return -1;
    }
    ++launches;
    return launches;
}

}  // namespace wpk
