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
// by one thread; the fp32 accumulator lives in TMEM (1, 2 or 4 accumulator stages), so the
// epilogue of tile i overlaps the main loop of tiles i+1...
//
// The kernel is a template over (dtype, A producer kind, epilogue kind) so that each launched
// variant carries only the code it runs: the warps of one SM sub-partition execute different
// roles at once, and a kernel image larger than the instruction caches stalls them all
// ("no instruction" stalls measured with ncu on the first, single-variant version).
//
// Warp roles (384 threads, 512 with gather producers): warp 0 = A TMA producer, warp 1 = TMEM
// allocator + MMA issuer, warp 2 = B TMA producer, warp 3 spare, warps 4-11 = epilogue
// (tcgen05.ld -> +bias -> ReLU -> round -> swizzled smem -> TMA store), warps 12-15 = gather
// producers (A_MODE 2/3). Persistent grid: CTAs loop over work items (tile, split) with a static
// round-robin schedule; RASTER picks which GEMM dimension varies fastest.
//
// The fused epilogue realises the paper's operator fusion ("write one CUDA kernel
// function for the fused operator"; SPEC.md:136 relu(bias_add(conv))).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <atomic>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "umma_conv.h"

#ifdef WPK_TIMELINE
#define WPK_DBG_FLAGS(a) ((a).dbg_flags)   // experiment switches (tools only)
#else
#define WPK_DBG_FLAGS(a) 0
#endif

namespace wpk {

template <int DT> struct OutT;
template <> struct OutT<DT_F16> { using T = __half; };
template <> struct OutT<DT_BF16> { using T = __nv_bfloat16; };
template <> struct OutT<DT_TF32> { using T = float; };
template <> struct OutT<DT_FP8> { using T = __nv_bfloat16; };   // e4m3 operands, bf16 output

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
    const int wi = (int)w;   // work counts are < 2^31 (plan validation)
    r.split = wi % a.splits;
    const int t = wi / a.splits;
    if (a.raster == 0) {
        r.mt = t / a.n_tiles;
        r.nt = t - r.mt * a.n_tiles;
    } else {
        r.nt = t / a.m_tiles;
        r.mt = t - r.nt * a.m_tiles;
    }
    return r;
}

// element e (0/1) of a packed pair of 16-bit values, as float
__device__ __forceinline__ float to_f2(uint32_t u, int e, __half *) {
    return __half2float(__ushort_as_half((unsigned short)(e ? (u >> 16) : (u & 0xFFFFu))));
}
__device__ __forceinline__ float to_f2(uint32_t u, int e, __nv_bfloat16 *) {
    return __bfloat162float(__ushort_as_bfloat16((unsigned short)(e ? (u >> 16) : (u & 0xFFFFu))));
}
__device__ __forceinline__ float to_f2(uint32_t, int, float *) { return 0.f; }
__device__ __forceinline__ float ld_elem(const __half *p) { return __half2float(*p); }
__device__ __forceinline__ float ld_elem(const __nv_bfloat16 *p) { return __bfloat162float(*p); }
__device__ __forceinline__ float ld_elem(const float *p) { return *p; }

// bias + ReLU for 4 consecutive columns (bias staged in smem as fp32, zero-padded past K)
__device__ __forceinline__ void bias_relu4(float *v, const float *sBias, int k, bool relu) {
    const float4 b = *reinterpret_cast<const float4 *>(sBias + k);
    v[0] += b.x; v[1] += b.y; v[2] += b.z; v[3] += b.w;
    if (relu) {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = fmaxf(v[j], 0.f);
    }
}

// Epilogue state of one warp: its staging buffers (2 x 4 KB = 32 rows x 128 B, or 1).
struct EpiCtx {
    const float *sBias;
    uint8_t *sEpi;
    uint32_t ebuf;
    int lane;
    int nbufs;
};

// 32 rows x 128 bytes (packed in pk, one row per lane) -> 128-byte-swizzled smem staging buffer ->
// TMA store: FINAL into the output [M][K], else into the fp32 partials [split][M][K].
template <bool FINAL>
__device__ __forceinline__ void stage_and_store(EpiCtx &E, const UmmaArgs &a, const CUtensorMap *tmY, const uint32_t *pk,
                                                int k0, int mrow, int split) {
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
    if (E.lane == 0 && !(WPK_DBG_FLAGS(a) & 2)) {
        if constexpr (FINAL) ptx::tma_store_2d(tmY, bufp, k0, mrow);
        else ptx::tma_store_3d(tmY, bufp, k0, mrow, split);
        ptx::bulk_commit();
    }
    if (E.nbufs == 2) E.ebuf ^= 1;
}

// Final-output chunk of a dual-accumulator tile (MODE bit 2): 32 columns at a time, the two
// accumulators (even K steps at taddr, odd at taddr + BN) summed in fp32, then bias, residual, ReLU and
// one rounding as in epi_chunk_tma.
template <typename T, bool RES>
__device__ __forceinline__ void epi_chunk_tma_dual(EpiCtx &E, const UmmaArgs &a, const CUtensorMap *tmY, uint32_t taddr,
                                                int k0, int mrow) {
    constexpr int CW = 128 / sizeof(T);   // 64 (16-bit) or 32 (fp32) columns per chunk
    uint32_t pk[32];
#pragma unroll
    for (int half = 0; half < CW / 32; ++half) {
        uint32_t ra[32], rb[32];
        ptx::tmem_ld32_nowait(taddr + half * 32, ra);
        ptx::tmem_ld32_nowait(taddr + (uint32_t)a.bn + half * 32, rb);
        uint4 zr[RES ? 4 : 1];   // this lane's row: 32 columns of the residual
        if constexpr (RES) {
            const long long m = (long long)mrow + E.lane;
            const int kz = k0 + half * 32;
            constexpr int EPV = 16 / sizeof(T);   // elements per 16-byte vector
            const uint4 *zp = reinterpret_cast<const uint4 *>(static_cast<const T *>(a.z) + m * a.K + kz);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                zr[j] = (m < a.M && kz + (j + 1) * EPV <= a.K && (sizeof(T) == 2 || j < 32 / EPV)) ? __ldg(zp + j)
                                                                                                : make_uint4(0u, 0u, 0u, 0u);
        }
        ptx::tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            float v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = __uint_as_float(ra[4 * q + j]) + __uint_as_float(rb[4 * q + j]);
            bias_relu4(v, E.sBias, k0 + half * 32 + 4 * q, false);
            if constexpr (RES) {
                if constexpr (sizeof(T) == 2) {   // 4 16-bit residual values = half of zr[q / 2]
                    const uint32_t lo = (q & 1) ? zr[q >> 1].z : zr[q >> 1].x, hi = (q & 1) ? zr[q >> 1].w : zr[q >> 1].y;
                    v[0] += to_f2(lo, 0, (T *)nullptr); v[1] += to_f2(lo, 1, (T *)nullptr);
                    v[2] += to_f2(hi, 0, (T *)nullptr); v[3] += to_f2(hi, 1, (T *)nullptr);
                } else {
                    // fp32: 32 columns = 8 vectors, but zr holds 4 (the first 16 columns); reload the rest
                    const long long m = (long long)mrow + E.lane;
                    const int kk = k0 + half * 32 + 4 * q;
                    const uint4 z4 = (q < 4) ? zr[q]
                                             : ((m < a.M && kk + 4 <= a.K)
                                                    ? __ldg(reinterpret_cast<const uint4 *>(static_cast<const T *>(a.z) + m * a.K + kk))
                                                    : make_uint4(0u, 0u, 0u, 0u));
                    v[0] += __uint_as_float(z4.x); v[1] += __uint_as_float(z4.y);
                    v[2] += __uint_as_float(z4.z); v[3] += __uint_as_float(z4.w);
                }
            }
            if (a.epilogue >= 2) {
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = fmaxf(v[j], 0.f);
            }
            if constexpr (sizeof(T) == 2) {
                pk[half * 16 + 2 * q] = pack2(v[0], v[1], (T *)nullptr);
                pk[half * 16 + 2 * q + 1] = pack2(v[2], v[3], (T *)nullptr);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) pk[4 * q + j] = __float_as_uint(v[j]);
            }
        }
    }
    stage_and_store<true>(E, a, tmY, pk, k0, mrow, 0);
}

// One 32-row x 128-byte chunk through smem + TMA store. FINAL: +bias, ReLU, RN-round to T (64
// columns for 16-bit T, 32 for fp32); else fp32 split-K partials (32 columns) into [split][M][K].
template <typename T, bool FINAL, bool RES = false, bool DUAL = false>
__device__ __forceinline__ void epi_chunk_tma(EpiCtx &E, const UmmaArgs &a, const CUtensorMap *tmY, uint32_t taddr,
                                              int k0, int mrow, int split) {
    constexpr bool k16 = FINAL && sizeof(T) == 2;
    if constexpr (FINAL && DUAL) {   // dual accumulators: (even K steps at taddr) + (odd at taddr + BN)
        epi_chunk_tma_dual<T, RES>(E, a, tmY, taddr, k0, mrow);
        return;
    }
    uint32_t raw[k16 ? 64 : 32];
    ptx::tmem_ld32_nowait(taddr, raw);
    if constexpr (k16) ptx::tmem_ld32_nowait(taddr + 32, raw + 32);
    // residual (epilogue 3): this lane's row, the chunk's 128 bytes, loaded while TMEM drains
    // (a compile-time switch: the residual variant is its own kernel instantiation, so the plain
    // epilogue does not carry the residual's 32 registers)
    uint4 zr[RES ? 8 : 1];
    constexpr bool res = FINAL && RES;
    if constexpr (res) {
        const long long m = (long long)mrow + E.lane;
        const uint4 *zp = reinterpret_cast<const uint4 *>(static_cast<const T *>(a.z) + m * a.K + k0);
#pragma unroll
        for (int j = 0; j < 8; ++j)
            zr[j] = (m < a.M && k0 + (j + 1) * (int)(16 / sizeof(T)) <= a.K) ? __ldg(zp + j) : make_uint4(0u, 0u, 0u, 0u);
    }
    ptx::tmem_wait_ld();
    uint32_t pk[32];
    if constexpr (k16) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            float v[4] = {__uint_as_float(raw[4 * q]), __uint_as_float(raw[4 * q + 1]), __uint_as_float(raw[4 * q + 2]),
                          __uint_as_float(raw[4 * q + 3])};
            bias_relu4(v, E.sBias, k0 + 4 * q, false);
            if constexpr (res) {   // 4 16-bit residual values = half of zr[q / 2]
                const uint32_t lo = (q & 1) ? zr[q >> 1].z : zr[q >> 1].x, hi = (q & 1) ? zr[q >> 1].w : zr[q >> 1].y;
                v[0] += to_f2(lo, 0, (T *)nullptr); v[1] += to_f2(lo, 1, (T *)nullptr);
                v[2] += to_f2(hi, 0, (T *)nullptr); v[3] += to_f2(hi, 1, (T *)nullptr);
            }
            if (a.epilogue >= 2) {
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = fmaxf(v[j], 0.f);
            }
            pk[2 * q] = pack2(v[0], v[1], (T *)nullptr);
            pk[2 * q + 1] = pack2(v[2], v[3], (T *)nullptr);
        }
    } else if constexpr (FINAL) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            float v[4] = {__uint_as_float(raw[4 * q]), __uint_as_float(raw[4 * q + 1]), __uint_as_float(raw[4 * q + 2]),
                          __uint_as_float(raw[4 * q + 3])};
            bias_relu4(v, E.sBias, k0 + 4 * q, false);
            if constexpr (res) {
                v[0] += __uint_as_float(zr[q].x); v[1] += __uint_as_float(zr[q].y);
                v[2] += __uint_as_float(zr[q].z); v[3] += __uint_as_float(zr[q].w);
            }
            if (a.epilogue >= 2) {
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = fmaxf(v[j], 0.f);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) pk[4 * q + j] = __float_as_uint(v[j]);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) pk[j] = raw[j];
    }
    stage_and_store<FINAL>(E, a, tmY, pk, k0, mrow, split);
}

// The split-K owner's whole slab (its chunks ci0, ci0 + cstep, ... of one 32-row group), software
// pipelined: the previous splits' fp32 partials of the next 32 columns are loaded from L2 while the
// current 32 columns are reduced, so an L2 round trip (~1-2 us under load) is paid once per slab
// instead of once per 32 columns (measured: pair split-2 owners finished up to 11 us after the
// last MMA, tools/timeline.py). Same arithmetic and order as before: partials of splits 0..S-2 in
// split order, then the owner's own TMEM accumulator, bias, ReLU, one rounding. Each 32-column
// half goes straight into the swizzled staging row (no packed copy of the whole chunk is held).
template <typename T>
__device__ __forceinline__ void epi_owner_run(EpiCtx &E, const UmmaArgs &a, const CUtensorMap *tmY, uint32_t tbase,
                                              int n0, int mrow, int ci0, int cstep, int nchunks) {
    constexpr int CW = 128 / sizeof(T);          // columns per 128-byte output chunk (64 or 32)
    constexpr int HPC = CW / 32;                 // 32-column halves per chunk
    constexpr int JPH = 8 / HPC;                 // 16-byte row pieces per half
    const long long m = (long long)mrow + E.lane;
    const bool mok = m < a.M;
    const long long MK = a.M * (long long)a.K;
    const float *prow = a.partial + m * a.K;
    const int nprev = a.splits - 1;
    auto chunk_of = [&](int j) { return ci0 + (j / HPC) * cstep; };
    auto valid = [&](int j) { const int ci = chunk_of(j); return ci < nchunks && n0 + ci * CW < a.K; };
    auto col_of = [&](int j) { return n0 + chunk_of(j) * CW + (j % HPC) * 32; };
    auto ld8 = [&](float4 *v, const float *src, int kh) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            v[q] = (mok && kh + 4 * q < a.K) ? __ldcg(reinterpret_cast<const float4 *>(src + kh + 4 * q))
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    // reduce 32 columns (partials in cur) and write them into the staging row
    auto step = [&](int j, float4 *cur, uint32_t row_addr) {
        const int half = j % HPC, kh = col_of(j);
        uint32_t raw[32];
        ptx::tmem_ld32_nowait(tbase + (uint32_t)(chunk_of(j) * CW + half * 32), raw);
        for (int sp = 1; sp < nprev; ++sp) {                  // splits 1 .. S-2 (S > 2), in order
            float4 v[8];
            ld8(v, prow + sp * MK, kh);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                cur[q].x += v[q].x; cur[q].y += v[q].y; cur[q].z += v[q].z; cur[q].w += v[q].w;
            }
        }
        ptx::tmem_wait_ld();
#pragma unroll
        for (int jj = 0; jj < JPH; ++jj) {
            uint32_t w4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {   // 16 bytes: 8 (16-bit) or 4 (fp32) columns
                if constexpr (sizeof(T) == 2) {
                    const int q = jj * 2 + e / 2;
                    float v2[4] = {cur[q].x + __uint_as_float(raw[4 * q]), cur[q].y + __uint_as_float(raw[4 * q + 1]),
                                   cur[q].z + __uint_as_float(raw[4 * q + 2]), cur[q].w + __uint_as_float(raw[4 * q + 3])};
                    bias_relu4(v2, E.sBias, kh + 4 * q, a.epilogue == 2);
                    w4[e] = (e & 1) ? pack2(v2[2], v2[3], (T *)nullptr) : pack2(v2[0], v2[1], (T *)nullptr);
                } else {
                    const int q = jj;
                    float v2[4] = {cur[q].x + __uint_as_float(raw[4 * q]), cur[q].y + __uint_as_float(raw[4 * q + 1]),
                                   cur[q].z + __uint_as_float(raw[4 * q + 2]), cur[q].w + __uint_as_float(raw[4 * q + 3])};
                    bias_relu4(v2, E.sBias, kh + 4 * q, a.epilogue == 2);
                    w4[e] = __float_as_uint(v2[e]);
                }
            }
            const int piece = half * JPH + jj;
            ptx::st_shared_v4(row_addr + ((uint32_t)(piece ^ (E.lane & 7)) << 4), w4[0], w4[1], w4[2], w4[3]);
        }
    };
    float4 bA[8], bB[8];
    if (valid(0)) ld8(bA, prow, col_of(0));
    uint32_t row_addr = 0;
    for (int j = 0; valid(j); j += 2) {
        // (j even: bA holds its partials; j + 1 uses bB)
        if (j % HPC == 0) {   // a new output chunk: its staging buffer must be free
            if (E.nbufs == 2) ptx::bulk_wait_read<1>();
            else ptx::bulk_wait_read<0>();
            __syncwarp();
            row_addr = ptx::smem_u32(E.sEpi + E.ebuf * 4096) + (uint32_t)E.lane * 128;
        }
        const bool v1 = valid(j + 1);
        if (v1) ld8(bB, prow, col_of(j + 1));
        step(j, bA, row_addr);
        if ((j + 1) % HPC == 0 || !v1) {   // chunk complete
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (E.lane == 0 && !(WPK_DBG_FLAGS(a) & 2)) {
                ptx::tma_store_2d(tmY, E.sEpi + E.ebuf * 4096, n0 + chunk_of(j) * CW, mrow);
                ptx::bulk_commit();
            }
            if (E.nbufs == 2) E.ebuf ^= 1;
        }
        if (!v1) break;
        if ((j + 1) % HPC == 0) {
            if (E.nbufs == 2) ptx::bulk_wait_read<1>();
            else ptx::bulk_wait_read<0>();
            __syncwarp();
            row_addr = ptx::smem_u32(E.sEpi + E.ebuf * 4096) + (uint32_t)E.lane * 128;
        }
        if (valid(j + 2)) ld8(bA, prow, col_of(j + 2));
        step(j + 1, bB, row_addr);
        if ((j + 2) % HPC == 0 || !valid(j + 2)) {
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (E.lane == 0 && !(WPK_DBG_FLAGS(a) & 2)) {
                ptx::tma_store_2d(tmY, E.sEpi + E.ebuf * 4096, n0 + chunk_of(j + 1) * CW, mrow);
                ptx::bulk_commit();
            }
            if (E.nbufs == 2) E.ebuf ^= 1;
        }
    }
}

// Split-K owner, bulk variant (the CTA's last work item, so its pipeline stages are idle): every
// epilogue warp TMA-loads the previous splits' fp32 partials of ITS rows and chunks into the stage
// area (32 x 32 boxes through the partials' tensor map), all 8 warps wait on one barrier, then each
// lane reads its row back from the 128-byte-swizzled boxes. One L2 round trip per tile instead of
// one per 32 columns of per-lane row loads (measured: ~10 us of owner reduction).
// Sum order as everywhere: splits 0..S-2, then the owner's own TMEM accumulator; bias, ReLU, one
// rounding. Slab layout: box (sp, rq = 32-row group, c = 32-column block) at
// ((sp * nrq + rq) * ncb + c) * 4 KB.
template <typename T>
__device__ __forceinline__ void epi_owner_bulk(EpiCtx &E, const UmmaArgs &a, const CUtensorMap *tmY,
                                               const CUtensorMap *tmP, uint8_t *slab, uint64_t *pbar,
                                               uint32_t tbase, int n0, int mrow, int rq, int nrq, int ci0,
                                               int cstep, int nchunks) {
    constexpr int CW = 128 / sizeof(T);
    constexpr int HPC = CW / 32;
    const int ncb = a.bn / 32;
    const int nprev = a.splits - 1;
    // (1) this warp's loads: every previous split x its chunks' 32-column blocks, its 32 rows
    uint32_t bytes = 0;
    for (int ci = ci0; ci < nchunks && n0 + ci * CW < a.K; ci += cstep) bytes += (uint32_t)(nprev * HPC) * 4096u;
    if (E.lane == 0) {
        ptx::mbar_arrive_expect_tx(pbar, bytes);
        for (int ci = ci0; ci < nchunks && n0 + ci * CW < a.K; ci += cstep)
            for (int sp = 0; sp < nprev; ++sp)
                for (int hf = 0; hf < HPC; ++hf) {
                    const int c = ci * HPC + hf;
                    ptx::tma_load_3d(slab + (size_t)((sp * nrq + rq) * ncb + c) * 4096u, tmP, pbar, n0 + c * 32, mrow, sp);
                }
    }
    __syncwarp();
    ptx::mbar_wait(pbar, 0);   // (2) all 8 warps' boxes landed (one phase per launch: the CTA's last item)
    const uint32_t slab_u = ptx::smem_u32(slab);
    const uint32_t swz = (uint32_t)(E.lane & 7);
    // (3) reduce chunk by chunk into the staging buffers, TMA store
    for (int ci = ci0; ci < nchunks; ci += cstep) {
        const int k0 = n0 + ci * CW;
        if (k0 >= a.K) break;
        if (E.nbufs == 2) ptx::bulk_wait_read<1>();
        else ptx::bulk_wait_read<0>();
        __syncwarp();
        const uint32_t row_addr = ptx::smem_u32(E.sEpi + E.ebuf * 4096) + (uint32_t)E.lane * 128;
#pragma unroll
        for (int hf = 0; hf < HPC; ++hf) {
            const int c = ci * HPC + hf;
#pragma unroll
            for (int sb = 0; sb < 2; ++sb) {   // 16 columns at a time (register pressure)
                const int kh = k0 + hf * 32 + sb * 16;
                uint32_t raw[16];
                ptx::tmem_ld16_nowait(tbase + (uint32_t)(ci * CW + hf * 32 + sb * 16), raw);
                float acc[16];
                for (int sp = 0; sp < nprev; ++sp) {
                    const uint32_t rb = slab_u + (uint32_t)((sp * nrq + rq) * ncb + c) * 4096u + (uint32_t)E.lane * 128u;
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        uint32_t x0, x1, x2, x3;
                        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                                     : "r"(rb + (((uint32_t)(sb * 4 + p) ^ swz) << 4)));
                        const float f[4] = {__uint_as_float(x0), __uint_as_float(x1), __uint_as_float(x2), __uint_as_float(x3)};
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc[4 * p + e] = (sp == 0) ? f[e] : acc[4 * p + e] + f[e];
                    }
                }
                ptx::tmem_wait_ld();
#pragma unroll
                for (int q = 0; q < 4; ++q) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[4 * q + e] += __uint_as_float(raw[4 * q + e]);
                    bias_relu4(acc + 4 * q, E.sBias, kh + 4 * q, a.epilogue == 2);
                }
                if constexpr (sizeof(T) == 2) {   // 16 columns = two 16-byte pieces
#pragma unroll
                    for (int pc = 0; pc < 2; ++pc) {
                        const float *v = acc + 8 * pc;
                        const int piece = hf * 4 + sb * 2 + pc;
                        ptx::st_shared_v4(row_addr + (((uint32_t)piece ^ swz) << 4), pack2(v[0], v[1], (T *)nullptr),
                                          pack2(v[2], v[3], (T *)nullptr), pack2(v[4], v[5], (T *)nullptr),
                                          pack2(v[6], v[7], (T *)nullptr));
                    }
                } else {                          // fp32: four pieces
#pragma unroll
                    for (int pc = 0; pc < 4; ++pc) {
                        const float *v = acc + 4 * pc;
                        const int piece = sb * 4 + pc;
                        ptx::st_shared_v4(row_addr + (((uint32_t)piece ^ swz) << 4), __float_as_uint(v[0]),
                                          __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3]));
                    }
                }
            }
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (E.lane == 0 && !(WPK_DBG_FLAGS(a) & 2)) {
            ptx::tma_store_2d(tmY, E.sEpi + E.ebuf * 4096, k0, mrow);
            ptx::bulk_commit();
        }
        __syncwarp();
        if (E.nbufs == 2) E.ebuf ^= 1;
    }
}

// Cluster split-K owner chunk: columns [k0, k0 + 128 B) of this CTA's output slice; the other
// splits' fp32 partials of them were delivered into this CTA's shared memory (recv_row = this
// lane's row in source slot 0 at the chunk's first column, slot_bytes apart). Summed in split
// order 0..S-1 (this CTA's own TMEM accumulator at position q) -> deterministic; then bias, ReLU,
// one rounding, TMA store.
template <typename T>
__device__ __forceinline__ void epi_chunk_csplit(EpiCtx &E, const UmmaArgs &a, const CUtensorMap *tmY, uint32_t taddr,
                                                 int k0, int mrow, uint32_t recv_row, uint32_t slot_bytes, int q,
                                                 int S) {
    constexpr int CW = 128 / sizeof(T);
    uint32_t pk[32];
#pragma unroll
    for (int half = 0; half < CW / 32; ++half) {
        uint32_t raw[32];
        ptx::tmem_ld32_nowait(taddr + half * 32, raw);
        ptx::tmem_wait_ld();
        float acc[32];
        for (int rk = 0; rk < S; ++rk) {
            float v[32];
            if (rk == q) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(raw[j]);
            } else {
                const uint32_t src = recv_row + (uint32_t)(rk < q ? rk : rk - 1) * slot_bytes + half * 128;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    uint32_t x0, x1, x2, x3;
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                                 : "r"(src + j * 16));
                    v[4 * j] = __uint_as_float(x0); v[4 * j + 1] = __uint_as_float(x1);
                    v[4 * j + 2] = __uint_as_float(x2); v[4 * j + 3] = __uint_as_float(x3);
                }
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] = (rk == 0) ? v[j] : acc[j] + v[j];
        }
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) {
            float v[4] = {acc[4 * qq], acc[4 * qq + 1], acc[4 * qq + 2], acc[4 * qq + 3]};
            bias_relu4(v, E.sBias, k0 + half * 32 + 4 * qq, a.epilogue == 2);
            if constexpr (sizeof(T) == 2) {
                pk[half * 16 + 2 * qq] = pack2(v[0], v[1], (T *)nullptr);
                pk[half * 16 + 2 * qq + 1] = pack2(v[2], v[3], (T *)nullptr);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) pk[4 * qq + j] = __float_as_uint(v[j]);
            }
        }
    }
    stage_and_store<true>(E, a, tmY, pk, k0, mrow, 0);
}

// Direct-store epilogue for one 32-row x 16-column chunk (NCHW output, unaligned K, partials).
template <typename T, bool DUAL = false>
__device__ __noinline__ void epi_chunk_direct(const UmmaArgs &a, const float *sBias, uint32_t taddr, int k0,
                                              long long m, int split, bool final_out) {
    float v[16];
    ptx::tmem_ld16(taddr, v);
    if constexpr (DUAL) {   // dual accumulators: + the odd K steps' accumulator, BN columns further
        float v2[16];
        ptx::tmem_ld16(taddr + (uint32_t)a.bn, v2);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += v2[j];
    }
    if (m >= a.M) return;
    const bool full16 = (k0 + 16 <= a.K);
    if (!final_out) {
        float *dst = a.partial + ((long long)split * a.M + m) * a.K + k0;
        if (full16 && a.vec_ok) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
                *reinterpret_cast<float4 *>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
            for (int j = 0; j < 16; ++j)
                if (k0 + j < a.K) dst[j] = v[j];
        }
        return;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) bias_relu4(v + 4 * q, sBias, k0 + 4 * q, false);
    T *y = static_cast<T *>(a.y);
    const T *z = static_cast<const T *>(a.z);
    if (a.out_nchw) {
        const long long nimg = m / a.PQ;
        const long long base = nimg * (long long)a.K * a.PQ + (m - nimg * a.PQ);
        for (int j = 0; j < 16; ++j)
            if (k0 + j < a.K) {
                const long long yi = base + (long long)(k0 + j) * a.PQ;
                float o = v[j];
                if (a.epilogue == 3) o += ld_elem(z + yi);
                if (a.epilogue >= 2) o = fmaxf(o, 0.f);
                st_out(y + yi, o);
            }
        return;
    }
    for (int j = 0; j < 16; ++j) {
        if (a.epilogue == 3 && k0 + j < a.K) v[j] += ld_elem(z + m * a.K + k0 + j);
        if (a.epilogue >= 2) v[j] = fmaxf(v[j], 0.f);
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
        for (int j = 0; j < 16; ++j)
            if (k0 + j < a.K) st_out(dst + j, v[j]);
    }
}

// In-kernel split-K fixup ("serial reduction by the last arriving split"): every split publishes its
// fp32 partial tile, bumps the tile's counter; the CTA that completes the count sums all partials
// in the fixed split order 0..S-1 (deterministic, independent of arrival order), applies bias+ReLU,
// rounds once and stores the output, then resets the counter for the next launch. For a CTA pair
// each CTA owns its 128 rows of the 256-row tile and has its own counter.
template <typename T>
__device__ __noinline__ void splitk_fixup(const UmmaArgs &a, const float *sBias, volatile int *sFlag, const WorkPos &wp,
                                          int nsub, int warp, int lane, uint32_t crank, int pair) {
    if (a.epi_tma && lane == 0) ptx::bulk_wait_all();   // this warp's partial stores are complete
    __syncwarp();
    __threadfence();
    ptx::named_bar_sync(1, 256);                         // all 8 epilogue warps published
    const int tile = (wp.mt * a.n_tiles + wp.nt) * (pair ? 2 : 1) + (int)crank;
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
    const long long m0 = (long long)wp.mt * a.bm + crank * 128;
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
        for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
            const long long m = mm[u];
            const int k = kk[u];
            float v[4] = {acc[u].x, acc[u].y, acc[u].z, acc[u].w};
            bias_relu4(v, sBias, k, a.epilogue == 2);
            if (a.out_nchw) {
                const long long nimg = m / a.PQ;
                const long long ob = nimg * (long long)a.K * a.PQ + (m - nimg * a.PQ);
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
                    for (int j = 0; j < 4; ++j)
                        if (k + j < a.K) st_out(dst + j, v[j]);
                }
            }
        }
    }
    ptx::named_bar_sync(1, 256);
    if (warp == 4 && lane == 0) a.counters[tile] = 0;    // self-resetting for the next launch
}

// A_MODE 2 producer: element gather (small C, NHWC or NCHW x) straight into the 128-byte-swizzled
// K-major A stage; kg = (r*S + s)*C + c; thread t owns rows t and 128 + t of every stage.
template <bool kTF32>
__device__ __forceinline__ void element_gather(const UmmaArgs &a, uint8_t *smA, uint32_t a_bytes, uint64_t *full,
                                               uint64_t *empty, int nsub, long long wstart, long long wstep, int t,
                                               int lane) {
    const int RSC = a.R * a.S * a.C;
    uint32_t stage = 0, phase = 0;
    for (long long w = wstart; w < a.work; w += wstep) {
        const WorkPos wp = decode_work(w, a);
        const int kb0 = wp.split * a.kb_per_split;
        const int kb1 = min(a.num_kb, kb0 + a.kb_per_split);
        int rh0[2], rw0[2], rn[2];
        bool rv[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const long long m = (long long)wp.mt * a.bm + hh * 128 + t;
            rv[hh] = hh < nsub && m < a.M;
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
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                if (hh >= nsub) break;
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
                            wv[q] = kTF32 ? bits[jj * 4 + q] : (bits[jj * 8 + 2 * q] | (bits[jj * 8 + 2 * q + 1] << 16));
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
}

// Fused depthwise producer (wpk_dwpw_*, NEXT-4: the MobileNet-V2 block's depthwise 3x3 feeding its
// 1x1 projection in ONE kernel): the A operand of the pointwise GEMM -- row m = output pixel of the
// depthwise conv, K = its C channels -- is computed here, never stored to global memory:
//   a[m][c] = RN_T(dw_epilogue(sum_{r,s} x[n][p*sh - ph + r*dh][q*sw - pw + s*dw][c] * w_dw[r][s][c] + b_dw[c]))
// (fp32 products and sum in (r, s) order, the bias added after the sum, one rounding to the I/O
// dtype: what the unfused depthwise conv stores). NHWC x, C % 8 == 0, 16-bit T.
// Work split: a K block is rows x 8 channel vectors (16 B = 8 channels each); thread t of the 4
// producer warps owns vector j = t & 7 of rows (t >> 3) + 16 i, so the 8 threads of a row read
// its 128 contiguous bytes per tap (one L1 line: a warp touches 4 lines per load instead of 32).
// The tap's weight vector is the same for all rows of the thread: loaded once per K block (3x3:
// kept in registers). Two rows are in flight per iteration; rows >= M and channels >= C are
// written as zeros.
// 16-bit pair -> two fp32 (exact): bf16 is the high half of an fp32; fp16 via the converter
__device__ __forceinline__ float2 up2(uint32_t u, __nv_bfloat16 *) {
    return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
}
__device__ __forceinline__ float2 up2(uint32_t u, __half *) {
    return __half22float2(*reinterpret_cast<const __half2 *>(&u));
}
// acc.{x,y} = fma(a.{x,y}, b.{x,y}, acc.{x,y}) in one FFMA2 (each lane rounds once, as fmaf)
__device__ __forceinline__ void ffma2(float2 &acc, float2 a, float2 b) {
    unsigned long long c = *reinterpret_cast<unsigned long long *>(&acc);
    asm("fma.rn.f32x2 %0, %1, %2, %0;"
        : "+l"(c)
        : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)));
    acc = *reinterpret_cast<float2 *>(&c);
}
// acc[0..3] += x[8 channels] * w[8 channels] (16-byte vectors of 16-bit values)
template <typename T>
__device__ __forceinline__ void mac8(float2 *acc, uint4 x, uint4 w) {
    ffma2(acc[0], up2(x.x, (T *)nullptr), up2(w.x, (T *)nullptr));
    ffma2(acc[1], up2(x.y, (T *)nullptr), up2(w.y, (T *)nullptr));
    ffma2(acc[2], up2(x.z, (T *)nullptr), up2(w.z, (T *)nullptr));
    ffma2(acc[3], up2(x.w, (T *)nullptr), up2(w.w, (T *)nullptr));
}

template <typename T, int R3>
__device__ __forceinline__ void dw_rows(const UmmaArgs &a, uint32_t sbase, int mbase, int nrows, int t, int c0,
                                       const uint4 *__restrict__ xv, const uint4 *__restrict__ wv,
                                       const uint4 *__restrict__ bv) {
    const int cv = a.C >> 3;
    const int j = t & 7;
    const int cvec = c0 + j;
    const bool cok = cvec < cv;
    const uint4 *wj = wv + cvec;   // tap i's weight vector: wj[i * cv] (an L1 hit shared by the row's threads)
    const uint4 *xj = xv + cvec;
    const int M = (int)a.M, PQ = (int)a.PQ;   // < 2^31 (plan validation)
    uint32_t bb[4] = {0u, 0u, 0u, 0u};
    if (bv && cok) {
        const uint4 b4 = __ldg(bv + cvec);
        bb[0] = b4.x; bb[1] = b4.y; bb[2] = b4.z; bb[3] = b4.w;
    }
#pragma unroll 1
    for (int row0 = (t >> 3); row0 < nrows; row0 += 32) {
        float2 acc[2][4];
        bool ok[2];
        uint4 xx[2][R3 ? 9 : 1];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int row = row0 + 16 * u;
            const int m = mbase + row;
            ok[u] = row < nrows && m < M && cok;
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[u][e] = make_float2(0.f, 0.f);
            const int mm = ok[u] ? m : 0;
            const int n = mm / PQ;
            const int rem = mm - n * PQ;
            const int p = rem / a.Q, q = rem - p * a.Q;
            const int h0 = p * a.stride_h - a.pad_h, w0 = q * a.stride_w - a.pad_w;
            const int nh = n * a.H;
            if constexpr (R3 != 0) {   // all 9 taps' loads issued before any math
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int s = 0; s < 3; ++s) {
                        const int hi = h0 + r * a.dil_h, wi = w0 + s * a.dil_w;
                        xx[u][r * 3 + s] = (ok[u] && hi >= 0 && hi < a.H && wi >= 0 && wi < a.W)
                                               ? __ldg(xj + (size_t)((nh + hi) * a.W + wi) * cv)
                                               : make_uint4(0u, 0u, 0u, 0u);
                    }
            } else if (ok[u]) {
#pragma unroll 1
                for (int r = 0; r < a.R; ++r) {
                    const int hi = h0 + r * a.dil_h;
                    if (hi < 0 || hi >= a.H) continue;
#pragma unroll 1
                    for (int s = 0; s < a.S; ++s) {
                        const int wi = w0 + s * a.dil_w;
                        if (wi < 0 || wi >= a.W) continue;
                        mac8<T>(acc[u], __ldg(xj + (size_t)((nh + hi) * a.W + wi) * cv),
                                __ldg(wj + (size_t)(r * a.S + s) * cv));
                    }
                }
            }
        }
        if constexpr (R3 != 0) {
#pragma unroll
            for (int i = 0; i < 9; ++i) {
                const uint4 wq = cok ? __ldg(wj + (size_t)i * cv) : make_uint4(0u, 0u, 0u, 0u);
                mac8<T>(acc[0], xx[0][i], wq);
                mac8<T>(acc[1], xx[1][i], wq);
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int row = row0 + 16 * u;
            if (row >= nrows) break;
            uint32_t o[4] = {0u, 0u, 0u, 0u};
            if (ok[u]) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 bf = up2(bb[e], (T *)nullptr);
                    float v0 = acc[u][e].x + bf.x, v1 = acc[u][e].y + bf.y;
                    if (a.dw_relu) { v0 = fmaxf(v0, 0.f); v1 = fmaxf(v1, 0.f); }
                    o[e] = pack2(v0, v1, (T *)nullptr);
                }
            }
            const uint32_t rbase = sbase + (uint32_t)(row >> 3) * 1024u + (uint32_t)(row & 7) * 128u;
            ptx::st_shared_v4(rbase + ((uint32_t)(j ^ (row & 7)) << 4), o[0], o[1], o[2], o[3]);
        }
    }
}

template <typename T>
__device__ __forceinline__ void dw_producer(const UmmaArgs &a, uint8_t *smA, uint32_t a_bytes, uint64_t *full,
                                           uint64_t *empty, int nsub, long long wstart, long long wstep, int t,
                                           int lane) {
    const uint4 *xv = reinterpret_cast<const uint4 *>(a.x);
    const uint4 *wv = reinterpret_cast<const uint4 *>(a.dw_w);
    const uint4 *bv = reinterpret_cast<const uint4 *>(a.dw_b);
    const bool r3 = a.R == 3 && a.S == 3;
    uint32_t stage = 0, phase = 0;
    for (long long w = wstart; w < a.work; w += wstep) {
        const WorkPos wp = decode_work(w, a);
        const int kb0 = wp.split * a.kb_per_split;
        const int kb1 = min(a.num_kb, kb0 + a.kb_per_split);
        const int mbase = wp.mt * a.bm;
        for (int kb = kb0; kb < kb1; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t sbase = ptx::smem_u32(smA + stage * a_bytes);
            if (r3) dw_rows<T, 3>(a, sbase, mbase, nsub * 128, t, kb * 8, xv, wv, bv);
            else dw_rows<T, 0>(a, sbase, mbase, nsub * 128, t, kb * 8, xv, wv, bv);
            ptx::fence_proxy_async_smem();                 // generic-proxy writes -> async-proxy (MMA) reads
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&full[stage]);
            if (++stage == (uint32_t)a.stages) { stage = 0; phase ^= 1; }
        }
    }
}

// A_MODE 3 producer: pixel-segment gather (C <= 4). x is re-laid as a zero-padded NHWC image
// with 4 channels per pixel (a.H x a.W = padded size), so every tap is in bounds. K row =
// (r, s', c), s' < Sp; a 16-byte smem chunk holds PPC whole pixels of one filter row. FAST: the
// chunk is one aligned 16-byte cp.async (tf32; 16-bit with dil_w 1, rows of odd q*stride_w reading
// a copy of the image shifted by one pixel); else two 8-byte copies. The copies of a stage
// are asynchronous: a thread keeps up to LAG stages in flight and signals a stage full only after
// cp.async.wait_group + a proxy fence, so the load latency overlaps across stages with no
// registers held. Thread t owns rows t and 128 + t of every stage.
template <bool kTF32, bool FAST, int LAG>
__device__ __forceinline__ void segment_gather(const UmmaArgs &a, uint8_t *smA, uint32_t a_bytes, uint64_t *full,
                                               uint64_t *empty, int nsub, long long wstart, long long wstep, int t,
                                               int lane) {
    constexpr int PPC = kTF32 ? 1 : 2;                 // pixels per 16-byte chunk
    constexpr int PB = 16 / PPC;                       // bytes per stored pixel
    const int chunks_per_r = a.seg_sp / PPC;
    const int rstep = a.dil_h * a.W * PB;              // bytes between filter rows
    const int sstep = a.dil_w * PB;                    // bytes between filter columns
    const long long img_bytes = (long long)a.M / a.PQ * a.H * a.W * PB;   // N * Hp * Wp pixels
    const char *xb = static_cast<const char *>(a.x);
    const uint32_t swz = (uint32_t)(t & 7) << 4;       // rows t and 128 + t share the swizzle phase
    uint32_t stage = 0, phase = 0;
    // stages issued but not yet signalled: the npend stages before `stage` (in issue order, so no
    // FIFO array -- a runtime-indexed array would live in local memory on this hot loop)
    int npend = 0;
    for (long long w = wstart; w < a.work; w += wstep) {
        const WorkPos wp = decode_work(w, a);
        // per row: pointer to tap (0,0) in the padded image (nullptr: row past M, zero-filled)
        const char *rptr[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            rptr[hh] = nullptr;
            const long long m = (long long)wp.mt * a.bm + hh * 128 + t;
            if (hh < nsub && m < a.M && !(WPK_DBG_FLAGS(a) & 1)) {
                const int n = (int)(m / a.PQ);
                const int rem = (int)(m - (long long)n * a.PQ);
                const int p = rem / a.Q, q = rem - (rem / a.Q) * a.Q;
                const int col = q * a.stride_w;
                const int sh = (a.seg_two && (col & 1)) ? 1 : 0;   // shifted copy keeps chunks aligned
                rptr[hh] = xb + sh * img_bytes + (((long long)n * a.H + p * a.stride_h) * a.W + col + sh) * PB;
            }
        }
        const int kb0 = wp.split * a.kb_per_split;
        const int kb1 = min(a.num_kb, kb0 + a.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
            // chunk offsets of this K block (uniform over rows); bit j of vmask: chunk j is a real tap
            int off[8];
            uint32_t vmask = 0;
            {
                const int cj = kb * 8;
                int r = cj / chunks_per_r, s0 = (cj - r * chunks_per_r) * PPC;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    off[j] = r * rstep + s0 * sstep;
                    if (r < a.R) vmask |= 1u << j;
                    s0 += PPC;
                    if (s0 == a.seg_sp) { s0 = 0; ++r; }
                }
            }
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t sbase = ptx::smem_u32(smA + stage * a_bytes) + (uint32_t)(t >> 3) * 1024u +
                                   (uint32_t)(t & 7) * 128u;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                if (hh >= nsub) break;
                const uint32_t rbase = sbase + (uint32_t)hh * 16384u;     // row 128 + t: 16 atoms further
                const char *rp = rptr[hh];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const bool ok = rp != nullptr && ((vmask >> j) & 1u);
                    const char *src = ok ? rp + off[j] : xb;
                    const uint32_t dst = rbase + (((uint32_t)j << 4) ^ swz);
                    if constexpr (FAST) {
                        ptx::cp_async_16(dst, src, ok ? 16u : 0u);
                    } else {
                        ptx::cp_async_8(dst, src, ok ? 8u : 0u);
                        ptx::cp_async_8(dst + 8, ok ? src + sstep : xb, ok ? 8u : 0u);
                    }
                }
            }
            ptx::cp_async_commit();
            if (npend == LAG) {                          // oldest stage's copies done -> signal it
                ptx::cp_async_wait<LAG>();
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    uint32_t oldest = stage + (uint32_t)a.stages - LAG;
                    if (oldest >= (uint32_t)a.stages) oldest -= (uint32_t)a.stages;
                    ptx::mbar_arrive(&full[oldest]);
                }
                --npend;
            }
            ++npend;
            if (++stage == (uint32_t)a.stages) { stage = 0; phase ^= 1; }
        }
    }
    ptx::cp_async_wait<0>();
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0)
        for (int i = 0; i < npend; ++i) {
            uint32_t st = stage + (uint32_t)a.stages - (uint32_t)npend + (uint32_t)i;
            if (st >= (uint32_t)a.stages) st -= (uint32_t)a.stages;
            ptx::mbar_arrive(&full[st]);
        }
}

// L2 prefetch of the activation rows one work item's A loads will read: NHWC rows [h_lo, h_hi]
// of the images its output pixels m0 .. m0 + rows - 1 belong to (whole rows: contiguous bytes);
// for the plain 2-D A view (1x1/s1/p0) the pixel rows themselves.
__device__ __forceinline__ void prefetch_a_rows(const UmmaArgs &a, long long m0, int rows) {
    if (m0 >= a.M) return;
    const long long m1 = min(a.M, m0 + rows) - 1;
    const long long rowb = (long long)a.C * a.e_size;             // bytes per input pixel
    const char *x = static_cast<const char *>(a.x);
    if (a.a_tiled) {
        ptx::bulk_prefetch_l2(x + m0 * rowb, (unsigned long long)((m1 - m0 + 1) * rowb));
        return;
    }
    const long long n0 = m0 / a.PQ, n1 = m1 / a.PQ;
    const int p0 = (int)((m0 - n0 * a.PQ) / a.Q), p1 = (int)((m1 - n1 * a.PQ) / a.Q);
    const int hlo = max(0, p0 * a.stride_h - a.pad_h);
    const int hhi = min(a.H - 1, p1 * a.stride_h - a.pad_h + (a.R - 1) * a.dil_h);
    const long long b0 = ((n0 * a.H + hlo) * a.W) * rowb;
    const long long b1 = ((n1 * a.H + hhi + 1) * a.W) * rowb;
    if (b1 > b0) ptx::bulk_prefetch_l2(x + b0, (unsigned long long)(b1 - b0));
}

// 12 warps (16 with gather producers): 0 = A producer, 1 = TMEM allocator + MMA issuer,
// 2 = B producer, 3 = spare, 4..11 = epilogue (two groups of four; warp w reads TMEM lanes
// [32*(w%4), +32)), 12..15 = gather producers.
template <int DT, int AK, int EK, bool RES = false, bool DUAL = false>
__global__ void __launch_bounds__((AK >= AK_GATHER && AK <= AK_DW) ? 512 : 384, 1)
    umma_conv_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmP,
                     const __grid_constant__ UmmaArgs a) {
    using T = typename OutT<DT>::T;
    constexpr bool kTF32 = (DT == DT_TF32);
    constexpr int kKind = (DT == DT_TF32) ? 1 : (DT == DT_FP8) ? 2 : 0;   // tcgen05.mma kind
    constexpr bool kPair = (AK == AK_PAIR || AK == AK_PAIR_KG2);
    constexpr bool kGather = (AK >= AK_GATHER && AK <= AK_DW);
    // K blocks per full / empty barrier group: a compile-time constant, so the one-block variants
    // keep the plain loops (a runtime group size cost ~5% of the step in instruction footprint)
    constexpr int KG = (AK == AK_TMA_KG2 || AK == AK_PAIR_KG2) ? 2 : 1;

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
    float *sBias = reinterpret_cast<float *>(smem + a.bias_off);      // [Kpad]
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + a.bar_off);
    uint64_t *full = bars;            // [8]
    uint64_t *empty = bars + 8;       // [8]
    uint64_t *tfull = bars + 16;      // [4]
    uint64_t *tempty = bars + 20;     // [4]
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 24);
    volatile int *sFlag = reinterpret_cast<volatile int *>(bars + 25);
    uint64_t *freeb = bars + 26;      // EK_CSPLIT: every peer's stages are idle (S - 1 remote arrives)
    uint64_t *datab = bars + 27;      // EK_CSPLIT: every peer delivered its partials (8 (S - 1) arrives)
    uint64_t *pbar = bars + 28;       // EK_SPLIT owner: the other splits' partial slab landed (8 warps)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef WPK_TIMELINE   // per-CTA globaltimer stamps for tools/timeline.py (libwpk_timeline.so only)
    unsigned long long *dbg = a.dbg ? a.dbg + blockIdx.x * 64 : nullptr;
#else                 // production build: every stamp and experiment switch folds away
    unsigned long long *const dbg = nullptr;
#endif
    if (dbg && threadIdx.x == 0) dbg[0] = ptx::globaltimer();

    if (warp == 0 && lane == 0) {
        if (!kGather) ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        if (EK != EK_DIRECT) ptx::prefetch_tmap(&tmY);
        if (EK == EK_SPLIT) ptx::prefetch_tmap(&tmP);
        for (int s = 0; s < a.stages; ++s) {
            // A (TMA: 1 or 2 issuing threads; or 4 gather warps) + B producer
            ptx::mbar_init(&full[s], kGather ? 5 : a.prod_rr ? 1 : (a.a_split ? 3 : 2));
            ptx::mbar_init(&empty[s], 1);      // MMA commit
        }
        for (int s = 0; s < a.acc_stages; ++s) {
            ptx::mbar_init(&tfull[s], 1);
            ptx::mbar_init(&tempty[s], kPair ? 16 : 8);   // 8 epilogue warps (x2 CTAs for a pair)
        }
        if (EK == EK_CSPLIT) {
            ptx::mbar_init(freeb, a.splits - 1);
            ptx::mbar_init(datab, 8 * (a.splits - 1));
        }
        if (EK == EK_SPLIT) ptx::mbar_init(pbar, 8);
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
    // Programmatic dependent launch: this prologue overlaps the previous kernel's tail. Weights are
    // inference constants, so the B producer starts streaming weight tiles into shared
    // memory before the previous grid has finished; only the threads that read activations (A
    // producers) or write the output (epilogue) execute griddepcontrol.wait.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    if (kPair || EK == EK_CSPLIT) ptx::cluster_sync();   // peer barriers initialised before remote arrives / TMA
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    if (dbg && threadIdx.x == 0) dbg[1] = ptx::globaltimer();

    if (!kGather && a.prod_rr && (warp == 0 || warp == 2 || warp == 3)) {
        // ===================== TMA producers, round robin (a.prod_rr) =====================
        // K block g of this CTA's schedule (ring stage g % STAGES) is loaded by producer warp
        // g % NPROD (warps 0, 2, 3; lane 0): its A box and B box under one expect_tx (full barrier
        // count 1). One issuing thread sustains ~1 box per 200-450 ns while the SM ingests far more
        // (tools/kloop_feed.cu: 3 producers 279 ns per 128x128 K block vs 548-575 ns for the A/B split).
        // A producer may run ahead of the others; before loading block g it waits on the parity of
        // the stage's empty barrier for block g - STAGES, unambiguous only if block g - 2 STAGES has
        // been consumed: its own previous wait (block g - NPROD) saw g - NPROD - STAGES consumed, so
        // NPROD <= STAGES suffices.
        // K groups (a.kgroup = G in {1, 2}): G consecutive K blocks of a work item share one full /
        // empty barrier pair (the first slot's), so one expect_tx / wait / commit serves G blocks;
        // a producer loads whole groups: group gi (ring group gi % NG) belongs to producer gi % NPROD.
        constexpr int G = KG;
        const int NG = a.stages / G;                   // barrier groups in the ring
        const int NPROD = min(3, NG);
        const int pid = (warp == 0) ? 0 : warp - 1;
        if (lane == 0 && pid < NPROD) {
            const uint32_t a_rows = kPair ? 128u : (uint32_t)a.bm;
            const uint32_t tx = (a_rows * 128u + b_bytes) * (kPair ? 2u : 1u);   // a pair's loads land on the leader's barrier
            struct ItemPos {
                int m0, nimg, wc, hc, n0;
            };
            auto walk = [&](auto &&fn) {
                long long gi = 0;   // group index in this CTA's schedule
                for (long long w = wstart; w < a.work; w += wstep) {
                    const WorkPos wp = decode_work(w, a);
                    const int kb0 = wp.split * a.kb_per_split;
                    const int kb1 = min(a.num_kb, kb0 + a.kb_per_split);
                    const int ngi = (kb1 - kb0 + G - 1) / G;
                    int i = (int)((pid - gi % NPROD + NPROD) % NPROD);
                    if (i < ngi) {
                        ItemPos ip;
                        ip.m0 = wp.mt * a.bm + (int)crank * 128;   // M < 2^31 (plan validation)
                        ip.nimg = ip.m0 / (int)a.PQ;
                        const int rem = ip.m0 - ip.nimg * (int)a.PQ;
                        const int p = rem / a.Q, q = rem - p * a.Q;
                        ip.wc = q * a.stride_w - a.pad_w;
                        ip.hc = p * a.stride_h - a.pad_h;
                        ip.n0 = wp.nt * a.bn + (int)crank * (a.bn / 2);
                        for (; i < ngi; i += NPROD) {
                            const int kb = kb0 + i * G;
                            if (!fn(gi + i, ip, kb, min(G, kb1 - kb))) return;
                        }
                    }
                    gi += ngi;
                }
            };
            auto load_b = [&](long long gi, const ItemPos &ip, int kb, int nblk) {
                const uint32_t grp = (uint32_t)(gi % NG);
                if (leader) ptx::mbar_arrive_expect_tx(&full[grp * G], tx * (uint32_t)nblk);
#pragma unroll 1
                for (int j = 0; j < nblk; ++j) {
                    const uint32_t slot = grp * G + j;
                    const int rs = (kb + j) / a.c_blocks, cb = (kb + j) - rs * a.c_blocks;
                    if constexpr (kPair) ptx::tma_load_3d_pair(smB + slot * b_bytes, &tmB, &full[grp * G], cb * a.bk, rs, ip.n0);
                    else ptx::tma_load_3d(smB + slot * b_bytes, &tmB, &full[grp * G], cb * a.bk, rs, ip.n0);
                }
            };
            auto load_a = [&](long long gi, const ItemPos &ip, int kb, int nblk) {
                const uint32_t grp = (uint32_t)(gi % NG);
#pragma unroll 1
                for (int j = 0; j < nblk; ++j) {
                    const uint32_t slot = grp * G + j;
                    uint8_t *dst = smA + slot * a_bytes;
                    const int rs = (kb + j) / a.c_blocks, cb = (kb + j) - rs * a.c_blocks;
                    if (a.a_tiled) {
                        if constexpr (kPair) ptx::tma_load_2d_pair(dst, &tmA, &full[grp * G], cb * a.bk, ip.m0);
                        else ptx::tma_load_2d(dst, &tmA, &full[grp * G], cb * a.bk, ip.m0);
                    } else {
                        const int r = rs / a.S, s = rs - r * a.S;
                        if constexpr (kPair)
                            ptx::tma_load_im2col_4d_pair(dst, &tmA, &full[grp * G], cb * a.bk, ip.wc, ip.hc, ip.nimg,
                                                         (uint16_t)(s * a.dil_w), (uint16_t)(r * a.dil_h));
                        else
                            ptx::tma_load_im2col_4d(dst, &tmA, &full[grp * G], cb * a.bk, ip.wc, ip.hc, ip.nimg,
                                                    (uint16_t)(s * a.dil_w), (uint16_t)(r * a.dil_h));
                    }
                }
            };
            // PDL: the ring starts empty, so this producer's first-pass weight boxes go out before
            // griddepcontrol.wait (the previous grid may still write this conv's input, never its weights)
            walk([&](long long gi, const ItemPos &ip, int kb, int nblk) {
                if (gi >= NG) return false;
                load_b(gi, ip, kb, nblk);
                return true;
            });
            asm volatile("griddepcontrol.wait;" ::: "memory");
            if (dbg && pid == 0) dbg[7] = ptx::globaltimer();
            walk([&](long long gi, const ItemPos &ip, int kb, int nblk) {
                if (gi >= NG) {
                    ptx::mbar_wait(&empty[(uint32_t)(gi % NG) * G], (uint32_t)((gi / NG) & 1) ^ 1u);
                    load_b(gi, ip, kb, nblk);
                }
                load_a(gi, ip, kb, nblk);
                return true;
            });
        }
    } else if (warp == 0 || warp == 2 || (warp == 3 && !kGather && a.a_split)) {
        // ===================== TMA producers: warp 0 -> A (activations), warp 2 -> B (weights) ====
        // With a_split, warp 3 loads the second half of each A stage: one thread issues one TMA
        // instruction per ~430 cycles whatever the box size (tools/tma_bench.cu), so two issuing
        // threads double the A feed rate up to the SM's ~76 B/clk ingest.
        if (lane == 0 && !(kGather && warp == 0)) {
            const bool isA = (warp != 2);
            const int half = (warp == 3) ? 1 : 0;
            // weights are inference constants: this CTA's 1/grid slice of them goes to L2 while the
            // previous grid (PDL) is still running, so no K block waits on DRAM for its B tile
            if (!isA && (a.l2pf & 1)) {
                const long long chunk = ((a.w_bytes + gridDim.x - 1) / gridDim.x + 255) / 256 * 256;
                const long long off = (long long)blockIdx.x * chunk;
                if (off < a.w_bytes)
                    ptx::bulk_prefetch_l2(static_cast<const char *>(a.wgt) + off,
                                          (unsigned long long)min(chunk, a.w_bytes - off));
            }
            if (isA) asm volatile("griddepcontrol.wait;" ::: "memory");
            const int pf_rows = (int)((kPair ? 128u : (uint32_t)a.bm) >> (a.a_split ? 1 : 0));
            if (isA && half == 0 && (a.l2pf & 2) && wstart < a.work) {   // the first work item's input rows
                const WorkPos wp0 = decode_work(wstart, a);
                prefetch_a_rows(a, (long long)wp0.mt * a.bm + crank * 128, pf_rows << (a.a_split ? 1 : 0));
            }
            if (dbg && isA && half == 0) dbg[7] = ptx::globaltimer();   // previous grid complete
            uint32_t stage = 0, phase = 0;
            const uint32_t a_rows = (kPair ? 128u : (uint32_t)a.bm) >> (a.a_split ? 1 : 0);   // rows per A load
            const uint32_t tx = isA ? a_rows * 128u : b_bytes;
            const uint32_t sstride = isA ? a_bytes : b_bytes;
            uint8_t *dst0 = isA ? smA + (size_t)half * a_rows * 128u : smB;
            for (long long w = wstart; w < a.work; w += wstep) {
                const WorkPos wp = decode_work(w, a);
                const long long m0 = (long long)wp.mt * a.bm + crank * 128 + (long long)half * a_rows;
                if (isA && half == 0 && (a.l2pf & 2) && w + wstep < a.work) {   // one work item ahead
                    const WorkPos wn = decode_work(w + wstep, a);
                    if (wn.mt != wp.mt) prefetch_a_rows(a, (long long)wn.mt * a.bm + crank * 128, pf_rows << (a.a_split ? 1 : 0));
                }
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
                constexpr int G = KG;   // K blocks per barrier group (slot stage .. stage + G - 1)
                for (int kb = kb0; kb < kb1; kb += G) {
                    const int nblk = min(G, kb1 - kb);
                    uint64_t *fb = &full[stage];
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    // experiment (dbg_flags & 8): issue times of the first tile's A (B) loads
                    if (dbg && (WPK_DBG_FLAGS(a) & 8) && w == wstart && kb - kb0 < 16 && half == 0)
                        dbg[(isA ? 16 : 32) + (kb - kb0)] = ptx::globaltimer();
                    if constexpr (kPair) {   // both CTAs' bytes land on the leader's barrier; only the leader arms it
                        if (leader) ptx::mbar_arrive_expect_tx(fb, 2 * tx * (uint32_t)nblk);
                    } else {
                        ptx::mbar_arrive_expect_tx(fb, tx * (uint32_t)nblk);
                    }
#pragma unroll 1
                    for (int j = 0; j < nblk; ++j) {
                        uint8_t *dst = dst0 + (stage + j) * sstride;
                        if constexpr (kPair) {
                            if (!isA)
                                ptx::tma_load_3d_pair(dst, &tmB, fb, cb * a.bk, rs, n0);
                            else if (a.a_tiled)
                                ptx::tma_load_2d_pair(dst, &tmA, fb, cb * a.bk, (int)m0);
                            else
                                ptx::tma_load_im2col_4d_pair(dst, &tmA, fb, cb * a.bk, wc, hc, nimg,
                                                             (uint16_t)(s * a.dil_w), (uint16_t)(r * a.dil_h));
                        } else {
                            if (!isA)
                                ptx::tma_load_3d(dst, &tmB, fb, cb * a.bk, rs, n0);
                            else if (a.a_tiled)
                                ptx::tma_load_2d(dst, &tmA, fb, cb * a.bk, (int)m0);
                            else
                                ptx::tma_load_im2col_4d(dst, &tmA, fb, cb * a.bk, wc, hc, nimg,
                                                        (uint16_t)(s * a.dil_w), (uint16_t)(r * a.dil_h));
                        }
                        if (++cb == a.c_blocks) {
                            cb = 0;
                            ++rs;
                            if (++s == a.S) { s = 0; ++r; }
                        }
                    }
                    stage += G;
                    if (stage == (uint32_t)a.stages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (kGather && warp >= 12) {
        // ===================== gather producers (A_MODE 2 / 3) =====================
        const int t = threadIdx.x - 384;                       // 0..127
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if constexpr (AK == AK_SEG) {
            // LAG = STAGES - 1 stages of copies in flight per thread
#define WPK_SEG(L)                                                                                          \
    do {                                                                                                  \
        if (a.seg_fast) segment_gather<kTF32, true, L>(a, smA, a_bytes, full, empty, nsub, wstart, wstep, t, lane); \
        else segment_gather<kTF32, false, L>(a, smA, a_bytes, full, empty, nsub, wstart, wstep, t, lane);        \
    } while (0)
            switch (a.stages) {
                case 3: WPK_SEG(2); break;
                case 4: WPK_SEG(3); break;
                case 5: WPK_SEG(4); break;
                case 6: WPK_SEG(5); break;
                case 7: WPK_SEG(6); break;
                default: WPK_SEG(7); break;
            }
#undef WPK_SEG
        } else if constexpr (AK == AK_GATHER) {
            element_gather<kTF32>(a, smA, a_bytes, full, empty, nsub, wstart, wstep, t, lane);
        } else if constexpr (AK == AK_DW) {
            dw_producer<T>(a, smA, a_bytes, full, empty, nsub, wstart, wstep, t, lane);
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (single thread; the leader CTA of a pair) =====================
#ifdef WPK_MMA_LANE0
        constexpr bool kConv = false;   // A/B experiment: the old single-lane issue loop
#else
        constexpr bool kConv = true;    // the whole warp runs the loop; elect_one() issues
#endif
        if (leader && (kConv || lane == 0)) {
            uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
            const uint64_t a_desc0 = ptx::sw128_kmajor_desc(ptx::smem_u32(smA));
            const uint64_t b_desc0 = ptx::sw128_kmajor_desc(ptx::smem_u32(smB));
            const uint32_t acc_cols = (uint32_t)(nsub * a.bn * (DUAL ? 2 : 1));
            for (long long w = wstart; w < a.work; w += wstep) {
                const WorkPos wp = decode_work(w, a);
                const int kb0 = wp.split * a.kb_per_split;
                const int kb1 = min(a.num_kb, kb0 + a.kb_per_split);
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const long long dit = (w - wstart) / wstep;     // debug: per-tile events of the first 8 tiles
                if (dbg && dit < 8 && !(WPK_DBG_FLAGS(a) & 8)) dbg[16 + dit * 6 + 0] = ptx::globaltimer();
                const uint32_t d_tmem = tmem_base + acc * acc_cols;
                const bool cyc = dbg && (WPK_DBG_FLAGS(a) & 128) && w == wstart;   // cycle accounting, first tile
                long long c_wait = 0, c_issue = 0, c_t0 = cyc ? clock64() : 0, c1 = 0;
                constexpr int G = KG;   // K blocks per barrier group (slots stage .. stage + G - 1)
                for (int kb = kb0; kb < kb1; kb += G) {
                    const int nblk = min(G, kb1 - kb);
                    const long long c0 = cyc ? clock64() : 0;
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    if (cyc) {
                        c1 = clock64();
                        c_wait += c1 - c0;
                    }
                    if (dbg && w == wstart && kb == kb0) dbg[2] = ptx::globaltimer();
                    if (dbg && dit < 8 && kb == kb0 && !(WPK_DBG_FLAGS(a) & 8)) dbg[16 + dit * 6 + 1] = ptx::globaltimer();
                    if (dbg && (WPK_DBG_FLAGS(a) & 8) && w == wstart && kb - kb0 < 16) dbg[48 + (kb - kb0)] = ptx::globaltimer();
                    if (!kConv || ptx::elect_one()) {
#pragma unroll 1
                    for (int j = 0; j < nblk; ++j) {
                    const uint64_t ad = a_desc0 + (uint64_t)(((stage + j) * a_bytes) >> 4);
                    const uint64_t bd = b_desc0 + (uint64_t)(((stage + j) * b_bytes) >> 4);
                    const bool first = (kb == kb0 && j == 0);   // the work item's first K block
                    if constexpr (kPair) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            if constexpr (DUAL)   // even K steps -> accumulator 0, odd -> accumulator 1
                                ptx::umma2<kKind>(d_tmem + (kk & 1) * a.bn, ad + 2 * kk, bd + 2 * kk, a.idesc,
                                                  (!first || kk > 1) ? 1u : 0u);
                            else
                                ptx::umma2<kKind>(d_tmem, ad + 2 * kk, bd + 2 * kk, a.idesc, (!first || kk > 0) ? 1u : 0u);
                        }
                    } else {
                        if constexpr (DUAL) {   // even K steps -> accumulator 0, odd -> accumulator 1 (BN columns on)
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                ptx::umma<kKind>(d_tmem + (kk & 1) * a.bn, ad + 2 * kk, bd + 2 * kk, a.idesc,
                                                 (!first || kk > 1) ? 1u : 0u);
                        } else {
                            for (int h = 0; h < nsub; ++h) {
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk)   // 4 x 32 bytes of K per 128-byte stage (+2 desc units)
                                    ptx::umma<kKind>(d_tmem + h * a.bn, ad + h * (16384 >> 4) + 2 * kk, bd + 2 * kk, a.idesc,
                                                     (!first || kk > 0) ? 1u : 0u);
                            }
                        }
                    }
                    }
                    if constexpr (kPair) ptx::umma_commit2_multicast(&empty[stage]);   // frees the group's slots in both CTAs
                    else ptx::umma_commit(&empty[stage]);                               // frees the group's slots when the MMAs finish
                    }
                    if (kConv) __syncwarp();
                    if (cyc) c_issue += clock64() - c1;
                    stage += G;
                    if (stage == (uint32_t)a.stages) { stage = 0; phase ^= 1; }
                }
                if (cyc && lane == 0) {
                    dbg[60] = (unsigned long long)c_wait;
                    dbg[61] = (unsigned long long)c_issue;
                    dbg[62] = (unsigned long long)(clock64() - c_t0);
                    dbg[63] = (unsigned long long)(kb1 - kb0);
                }
                if (!kConv || ptx::elect_one()) {
                    if constexpr (kPair) ptx::umma_commit2_multicast(&tfull[acc]);   // both CTAs' halves ready
                    else ptx::umma_commit(&tfull[acc]);                               // accumulator ready
                }
                if (kConv) __syncwarp();
                if (dbg && w == wstart) dbg[3] = ptx::globaltimer();
                if (dbg && dit < 8 && !(WPK_DBG_FLAGS(a) & 8)) dbg[16 + dit * 6 + 2] = ptx::globaltimer();
                if (dbg && dit < 8 && (WPK_DBG_FLAGS(a) & 4) && !(WPK_DBG_FLAGS(a) & 8)) {   // experiment: MMA completion seen by a spinning thread
                    while (!ptx::mbar_test_wait(&tfull[acc], acc_phase)) {}
                    dbg[16 + dit * 6 + 5] = ptx::globaltimer();
                }
                if (++acc == (uint32_t)a.acc_stages) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else if (warp >= 4 && warp < 12) {
        // ===================== epilogue warps 4..11 =====================
        // bias -> smem once (fp32, zero past K; zero without bias), off the prologue's critical
        // path: the epilogue needs it only after the first tile's K loop
        {
            const T *bias = static_cast<const T *>(a.bias);
            for (int k = threadIdx.x - 128; k < a.kpad_bias; k += 256)
                sBias[k] = (a.epilogue >= 1 && k < a.K) ? ld_bias(bias, k) : 0.f;
            ptx::named_bar_sync(1, 256);
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");   // y may still be in use upstream
        const int quarter = warp & 3;          // TMEM lane quarter this warp may access
        const int grp = (warp - 4) >> 2;       // 0 or 1
        uint32_t acc = 0, acc_phase = 0;
        EpiCtx E{sBias, sEpi + (size_t)(warp - 4) * a.epi_bufs * 4096, 0u, lane, a.epi_bufs};
        const uint32_t acc_cols = (uint32_t)(nsub * a.bn * (DUAL ? 2 : 1));
        constexpr int cwf = (EK == EK_DIRECT) ? 16 : (int)(128 / sizeof(T));   // final-output chunk width
        constexpr int cwp = (EK == EK_DIRECT) ? 16 : 32;                        // fp32-partial chunk width
        for (long long w = wstart; w < a.work; w += wstep) {
            const WorkPos wp = decode_work(w, a);
            const int n0 = wp.nt * a.bn;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            const long long dit = (w - wstart) / wstep;
            if (dbg && warp == 4 && lane == 0 && dit < 8 && !(WPK_DBG_FLAGS(a) & 8)) dbg[16 + dit * 6 + 3] = ptx::globaltimer();
            // split-K (EK_SPLIT): the tile's last split owns the output; it waits until the other
            // splits have published their partials (they precede it in the static schedule, so they
            // are resident or done: no deadlock), then reduces them in split order.
            const bool owner = (EK != EK_SPLIT) || wp.split == a.splits - 1;
            const int ctile = (wp.mt * a.n_tiles + wp.nt) * (kPair ? 2 : 1) + (int)crank;
            if (EK == EK_SPLIT && owner) {
                if (warp == 4 && lane == 0) {
                    if (dbg && w == wstart) dbg[59] = ptx::globaltimer();   // owner starts waiting
                    while (ptx::ld_acquire_gpu(a.counters + ctile) < a.splits - 1) __nanosleep(32);
                    if (dbg && w == wstart) dbg[57] = ptx::globaltimer();   // owner saw every split published
                }
                ptx::named_bar_sync(1, 256);
            }
            const int cw = owner ? cwf : cwp;
            const int nchunks = (a.bn + cw - 1) / cw;
            if constexpr (EK == EK_CSPLIT) {
                // ---- split-K over the cluster: the S splits of this tile are the S CTAs; CTA q owns
                // output columns [q*BN/S, (q+1)*BN/S) and receives the others' partials of them into
                // its own (idle after the last MMA) pipeline stages.
                const int S = a.splits;
                const int q = (int)ptx::cluster_ctarank();
                const int slice = a.bn / S;
                const uint32_t slot_bytes = (uint32_t)a.bm * (uint32_t)a.recv_stride;
                const uint32_t recv0 = ptx::smem_u32(smem);
                if (warp == 4 && lane == 0)                     // (1) our stages are free
                    for (int j = 0; j < S; ++j)
                        if (j != q) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(freeb), (uint32_t)j));
                ptx::mbar_wait_cluster(freeb, 0);               // (2) every peer's stages are free
                // (3) send: our accumulator columns of the other slices, 32 at a time, into slot
                // (q < j ? q : q - 1) of destination j
                const int sends = (S - 1) * (slice / 32);
                for (int h = 0; h < nsub; ++h) {
                    if (nsub == 2 && h != grp) continue;
                    const int row = h * 128 + quarter * 32 + lane;
                    const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * acc_cols + h * a.bn;
                    for (int ci = (nsub == 2 ? 0 : grp); ci < sends; ci += (nsub == 2 ? 1 : 2)) {
                        const int jd = ci / (slice / 32);
                        const int j = jd < q ? jd : jd + 1;                   // destination rank
                        const int cl = (ci - jd * (slice / 32)) * 32;         // column within its slice
                        uint32_t raw[32];
                        ptx::tmem_ld32_nowait(tbase + j * slice + cl, raw);
                        ptx::tmem_wait_ld();
                        const uint32_t dst = ptx::mapa(recv0 + (uint32_t)(q < j ? q : q - 1) * slot_bytes +
                                                           (uint32_t)row * a.recv_stride + (uint32_t)cl * 4u,
                                                       (uint32_t)j);
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            ptx::st_cluster_v4(dst + x * 16, raw[4 * x], raw[4 * x + 1], raw[4 * x + 2], raw[4 * x + 3]);
                    }
                }
                ptx::fence_acq_rel_cluster();
                __syncwarp();
                if (lane == 0)
                    for (int j = 0; j < S; ++j)
                        if (j != q) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(datab), (uint32_t)j));
                ptx::mbar_wait_cluster(datab, 0);               // (4) all partials of our slice arrived
                // (5) reduce our slice in 128-byte output chunks
                const int own_chunks = slice / cwf;
                for (int h = 0; h < nsub; ++h) {
                    if (nsub == 2 && h != grp) continue;
                    const int row = h * 128 + quarter * 32 + lane;
                    const int mrow = wp.mt * a.bm + h * 128 + quarter * 32;
                    const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * acc_cols + h * a.bn;
                    for (int ci = (nsub == 2 ? 0 : grp); ci < own_chunks; ci += (nsub == 2 ? 1 : 2)) {
                        const int cl = ci * cwf;
                        const int k0 = n0 + q * slice + cl;
                        if (k0 >= a.K) break;
                        epi_chunk_csplit<T>(E, a, &tmY, tbase + q * slice + cl, k0, mrow,
                                            recv0 + (uint32_t)row * a.recv_stride + (uint32_t)cl * 4u, slot_bytes, q, S);
                    }
                }
            } else
            // slabs = (h, chunk) pairs; group g takes h == g when nsub == 2, else every other chunk
            for (int h = 0; h < nsub; ++h) {
                if (nsub == 2 && h != grp) continue;
                const int mrow = wp.mt * a.bm + (int)crank * 128 + h * 128 + quarter * 32;
                const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * acc_cols + h * a.bn;
                if (EK == EK_SPLIT && owner) {
                    if (a.owner_bulk && w + wstep >= a.work)   // the CTA's last item: its stages are idle
                        epi_owner_bulk<T>(E, a, &tmY, &tmP, smem, pbar, tbase, n0, mrow, h * 4 + quarter, nsub * 4,
                                          nsub == 2 ? 0 : grp, nsub == 2 ? 1 : 2, nchunks);
                    else
                        epi_owner_run<T>(E, a, &tmY, tbase, n0, mrow, nsub == 2 ? 0 : grp, nsub == 2 ? 1 : 2, nchunks);
                    continue;
                }
                for (int ci = (nsub == 2 ? 0 : grp); ci < nchunks; ci += (nsub == 2 ? 1 : 2)) {
                    const int c0 = ci * cw;
                    const int k0 = n0 + c0;
                    if (k0 >= a.K) break;   // warp-uniform
                    if constexpr (EK == EK_TMA) {
                        epi_chunk_tma<T, true, RES, DUAL>(E, a, &tmY, tbase + c0, k0, mrow, 0);
                    } else if constexpr (EK == EK_SPLIT) {
                        epi_chunk_tma<T, false>(E, a, &tmP, tbase + c0, k0, mrow, wp.split);   // (owner: above)
                    } else {
                        epi_chunk_direct<T, DUAL>(a, sBias, tbase + c0, k0, (long long)mrow + lane, wp.split, a.splits == 1);
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (dbg && warp == 4 && lane == 0 && w == wstart) dbg[4] = ptx::globaltimer();
            if (dbg && warp == 4 && lane == 0 && dit < 8) {
                dbg[8 + dit] = ptx::globaltimer();
                if (!(WPK_DBG_FLAGS(a) & 8)) dbg[16 + dit * 6 + 4] = ptx::globaltimer();
            }
            if (lane == 0) {                                  // TMEM free: the MMA may start the next tile
                if constexpr (kPair) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
                else ptx::mbar_arrive(&tempty[acc]);
            }
            if (++acc == (uint32_t)a.acc_stages) { acc = 0; acc_phase ^= 1; }
            if constexpr (EK == EK_SPLIT) {
                if (!owner) {   // publish: partial stores complete and visible, then count this split in
                    if (lane == 0) ptx::bulk_wait_all();
                    __syncwarp();
                    __threadfence();
                    ptx::named_bar_sync(1, 256);
                    if (warp == 4 && lane == 0) atomicAdd(a.counters + ctile, 1);
                    if (dbg && warp == 4 && lane == 0 && w == wstart) dbg[56] = ptx::globaltimer();   // published
                } else {        // all 8 warps have consumed the partials: reset for the next launch
                    ptx::named_bar_sync(1, 256);
                    if (warp == 4 && lane == 0) a.counters[ctile] = 0;
                    if (dbg && warp == 4 && lane == 0 && w == wstart) dbg[58] = ptx::globaltimer();   // owner done
                }
            }
            if (EK == EK_DIRECT && a.splits > 1) splitk_fixup<T>(a, sBias, sFlag, wp, nsub, warp, lane, crank, kPair ? 1 : 0);
        }
        // the staging buffers must not be released while TMA stores still read them; the global
        // writes themselves complete with the grid (a dependent grid's griddepcontrol.wait sees them)
        if (EK != EK_DIRECT && lane == 0) ptx::bulk_wait_read<0>();
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

// ---- launch of one (dtype) instantiation family -----------------------------------------------
template <int DT, int AK, int EK, bool RES = false, bool DUAL = false>
static cudaError_t launch_variant(cudaLaunchConfig_t &lc, const CUtensorMap &tmA, const CUtensorMap &tmB,
                                  const CUtensorMap &tmY, const CUtensorMap &tmP, const UmmaArgs &a) {
    // the shared-memory opt-in is per device context: remember it per device (bit d), so a plan
    // on a second device of the same process sets it again; racing host threads at worst set it twice
    static std::atomic<unsigned long long> attr_done{0ull};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cudaGetLastError();
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load(std::memory_order_acquire) & bit)) {
        cudaError_t e = cudaFuncSetAttribute(umma_conv_kernel<DT, AK, EK, RES, DUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e != cudaSuccess) return e;
        // one shared-memory carveout for every variant and config: consecutive convs whose dynamic
        // smem differs would otherwise get different L1/smem splits, and an SM can only switch
        // carveout once drained -- no overlap of one conv's tail with the next conv's CTAs
        if (!getenv("WPK_NO_CARVEOUT")) {
            e = cudaFuncSetAttribute(umma_conv_kernel<DT, AK, EK, RES, DUAL>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)cudaSharedmemCarveoutMaxShared);
            if (e != cudaSuccess) return e;
        }
        attr_done.fetch_or(bit, std::memory_order_acq_rel);
    }
    return cudaLaunchKernelEx(&lc, umma_conv_kernel<DT, AK, EK, RES, DUAL>, tmA, tmB, tmY, tmP, a);
}

template <int DT, int AK>
static cudaError_t launch_ak(int ek, cudaLaunchConfig_t &lc, const CUtensorMap &tmA, const CUtensorMap &tmB,
                             const CUtensorMap &tmY, const CUtensorMap &tmP, const UmmaArgs &a) {
    if constexpr (AK == AK_TMA || AK == AK_PAIR || AK == AK_TMA_KG2 || AK == AK_PAIR_KG2) {   // dual accumulators (MODE bit 2): TMA A producers only (plan validation)
        if (a.kdual) {
            if (ek == EK_TMA)
                return a.epilogue == 3 ? launch_variant<DT, AK, EK_TMA, true, true>(lc, tmA, tmB, tmY, tmP, a)
                                       : launch_variant<DT, AK, EK_TMA, false, true>(lc, tmA, tmB, tmY, tmP, a);
            if (ek == EK_DIRECT) return launch_variant<DT, AK, EK_DIRECT, false, true>(lc, tmA, tmB, tmY, tmP, a);
            return cudaErrorInvalidConfiguration;
        }
    }
    if (ek == EK_TMA)
        return a.epilogue == 3 ? launch_variant<DT, AK, EK_TMA, true>(lc, tmA, tmB, tmY, tmP, a)
                               : launch_variant<DT, AK, EK_TMA, false>(lc, tmA, tmB, tmY, tmP, a);
    if (ek == EK_SPLIT) return launch_variant<DT, AK, EK_SPLIT>(lc, tmA, tmB, tmY, tmP, a);
    if (ek == EK_CSPLIT) {
        if constexpr (AK == AK_TMA || AK == AK_TMA_KG2) return launch_variant<DT, AK, EK_CSPLIT>(lc, tmA, tmB, tmY, tmP, a);
        else return cudaErrorInvalidConfiguration;   // plan validation never pairs these
    }
    return launch_variant<DT, AK, EK_DIRECT>(lc, tmA, tmB, tmY, tmP, a);
}

template <int DT>
cudaError_t umma_launch_dt(int ak, int ek, cudaLaunchConfig_t &lc, const CUtensorMap &tmA, const CUtensorMap &tmB,
                           const CUtensorMap &tmY, const CUtensorMap &tmP, const UmmaArgs &a) {
    if (ak == AK_PAIR) return a.kgroup == 2 ? launch_ak<DT, AK_PAIR_KG2>(ek, lc, tmA, tmB, tmY, tmP, a)
                                            : launch_ak<DT, AK_PAIR>(ek, lc, tmA, tmB, tmY, tmP, a);
    if constexpr (DT == DT_FP8) {   // e4m3: TMA A producers only (plan validation)
        if (ak != AK_TMA) return cudaErrorInvalidConfiguration;
    } else {
        if (ak == AK_GATHER) return launch_ak<DT, AK_GATHER>(ek, lc, tmA, tmB, tmY, tmP, a);
        if (ak == AK_SEG) return launch_ak<DT, AK_SEG>(ek, lc, tmA, tmB, tmY, tmP, a);
        if constexpr (DT == DT_BF16 || DT == DT_F16) {   // fused depthwise producer: 16-bit data
            if (ak == AK_DW) return launch_ak<DT, AK_DW>(ek, lc, tmA, tmB, tmY, tmP, a);
        }
    }
    return a.kgroup == 2 ? launch_ak<DT, AK_TMA_KG2>(ek, lc, tmA, tmB, tmY, tmP, a)
                         : launch_ak<DT, AK_TMA>(ek, lc, tmA, tmB, tmY, tmP, a);
}

}  // namespace wpk
