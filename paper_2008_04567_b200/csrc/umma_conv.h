// Host/device interface of the tcgen05 implicit-GEMM convolution (umma_conv.cu).
#pragma once
#include <cstdint>
#include <string>

#include <cuda.h>
#include <cuda_runtime.h>

#include "wpk_internal.h"

namespace wpk {

enum { DT_F16 = 0, DT_BF16 = 1, DT_TF32 = 2, DT_FP8 = 3 };   // DT_FP8: e4m3 x / w, bf16 b / z / y
// A producer kinds: TMA (im2col / tiled), TMA for a CTA pair, element gather (A_MODE 2),
// pixel-segment gather (A_MODE 3)
// AK_DW: fused depthwise producer (wpk_dwpw_*); AK_TMA_KG2 / AK_PAIR_KG2: the TMA producers with K groups
// of two blocks per barrier pair (A_MODE 5 / 6; the group size is a template constant)
enum { AK_TMA = 0, AK_PAIR = 1, AK_GATHER = 2, AK_SEG = 3, AK_DW = 4, AK_TMA_KG2 = 5, AK_PAIR_KG2 = 6 };
// epilogue kinds: final output via TMA store, split-K partials via TMA store (+ in-kernel fixup),
// direct global stores (NCHW output or K not a multiple of the 128-byte chunk; final or partial)
enum { EK_TMA = 0, EK_SPLIT = 1, EK_DIRECT = 2, EK_CSPLIT = 3 };   // EK_CSPLIT: split-K over a cluster (DSMEM)

struct UmmaArgs {
    const void *bias;
    void *y;
    float *partial;
    long long M, PQ, work;
    int K, P, Q;
    int stride_h, stride_w, pad_h, pad_w, dil_h, dil_w, S;
    int c_blocks, num_kb, kb_per_split, splits;
    int m_tiles, n_tiles, raster;
    int bm, bn, bk, stages, acc_stages;
    uint32_t idesc, tmem_cols;
    int epilogue, out_nchw, vec_ok;
    int a_tiled, epi_tma, epi_bufs;
    uint32_t epi_off, bias_off, bar_off;
    unsigned long long *dbg;        // optional per-CTA timeline (globaltimer ns), debug only
    int *counters;                  // split-K arrival counters, one per output tile (self-resetting)
    const void *x;                  // A_MODE 2 gather source (the caller's activations)
    int x_nchw, C, H, W, R;
    int a_mode, seg_sp, seg_fast;   // A_MODE 3: pixel-segment gather, filter columns padded to seg_sp
    int seg_two;                    // A_MODE 3: shifted second image copy for odd stride_w
    int kpad_bias;                  // staged bias length (K rounded up to 256, zero-padded)
    int owner_bulk;                 // EK_SPLIT: the other splits' partial slab fits in the stage area
    int kdual;                      // two accumulators per 128-row tile (even / odd K steps)
    int prod_rr;                    // TMA producers: K blocks dealt round robin over warps 0, 2, 3
    int kgroup;                     // K blocks per full / empty barrier group (1, or 2 for TMA producers)
    int recv_stride;                // EK_CSPLIT: bytes per received partial row
    int a_split;                    // A stage loaded by two threads (two half-height boxes)
    const void *z;                  // residual (epilogue 3), laid out as y
    int dbg_flags;                  // experiments only (WPK_DBG_FLAGS): 1 = gather zero-fills, 2 = no y stores
    // L2 prefetch (bit 0: weights, this CTA's 1/grid slice of the packed tensor, before the PDL wait;
    // bit 1: activations, the input rows of this CTA's next work item, TMA producers only)
    int l2pf;
    const void *wgt;                // packed weights [K][R*S][C] as the B tensor map sees them
    long long w_bytes;
    int e_size;                     // bytes per element of x / w
    const void *dw_w;               // AK_DW: depthwise weights packed [R][S][C] (I/O dtype)
    const void *dw_b;               // AK_DW: depthwise bias [C] or NULL
    int dw_relu;                    // AK_DW: ReLU after the depthwise bias
};

// Tensor maps of the last launch, reused while pointers and config are unchanged (host-side
// encode is a few microseconds per map).
struct UmmaMapCache {
    bool valid = false;
    const void *x = nullptr, *w = nullptr;
    void *y = nullptr, *partial = nullptr;
    Config cfg;
    int a_split = 0;
    CUtensorMap a, b, yy, pp;
};

struct UmmaLaunch {
    int dtype;                       // wpk_dtype (F16 / BF16 / TF32)
    const void *x;                   // NHWC activations, channels padded to g.cpad
    const void *w;                   // [K][R][S][g.cpad]
    const void *b;
    void *y;
    const void *z = nullptr;         // residual (epilogue 3), laid out as y
    const void *dw_w = nullptr;      // fused depthwise (A_MODE 5): weights [R][S][C], bias [C] or NULL
    const void *dw_b = nullptr;
    int dw_relu = 0;
    float *partial;                  // split-K workspace (splits x M x K fp32) or nullptr
    int *counters = nullptr;         // split-K tile counters (zeroed once per workspace)
    int N, H, W, K, R, S, P, Q;
    int stride_h, stride_w, pad_h, pad_w, dil_h, dil_w;
    int epilogue, out_nchw;
    long long a_rows;                // rows of the 2-D A view when g.a_tiled (N*H*W, or M for explicit im2col)
    int b_rs;                        // taps folded in B's middle dim (R*S, or 1 for explicit im2col)
    int sm_count;
    void *stream;
    unsigned long long *dbg = nullptr;
    int C = 0, x_nchw = 0;
    UmmaMapCache *cache = nullptr;
    Config cfg;
    UmmaGeom g;
};

// Returns the number of kernel launches issued (1 or 2), or -1 with *err set.
int umma_launch(const UmmaLaunch &L, std::string *err);

// Per-dtype kernel instantiations (umma_conv_{f16,bf16,tf32}.cu): launch variant (ak, ek).
cudaError_t umma_launch_f16(int ak, int ek, cudaLaunchConfig_t &lc, const CUtensorMap &tmA, const CUtensorMap &tmB,
                            const CUtensorMap &tmY, const CUtensorMap &tmP, const UmmaArgs &a);
cudaError_t umma_launch_bf16(int ak, int ek, cudaLaunchConfig_t &lc, const CUtensorMap &tmA, const CUtensorMap &tmB,
                             const CUtensorMap &tmY, const CUtensorMap &tmP, const UmmaArgs &a);
cudaError_t umma_launch_tf32(int ak, int ek, cudaLaunchConfig_t &lc, const CUtensorMap &tmA, const CUtensorMap &tmB,
                             const CUtensorMap &tmY, const CUtensorMap &tmP, const UmmaArgs &a);
cudaError_t umma_launch_fp8(int ak, int ek, cudaLaunchConfig_t &lc, const CUtensorMap &tmA, const CUtensorMap &tmB,
                             const CUtensorMap &tmY, const CUtensorMap &tmP, const UmmaArgs &a);

}  // namespace wpk
