// Host/device interface of the tcgen05 implicit-GEMM convolution (umma_conv.cu).
#pragma once
#include <cstdint>
#include <string>

#include <cuda.h>

#include "wpk_internal.h"

namespace wpk {

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
};

// Tensor maps of the last launch, reused while pointers and config are unchanged (host-side
// encode is a few microseconds per map).
struct UmmaMapCache {
    bool valid = false;
    const void *x = nullptr, *w = nullptr;
    void *y = nullptr, *partial = nullptr;
    Config cfg;
    CUtensorMap a, b, yy;
};

struct UmmaLaunch {
    int dtype;                       // wpk_dtype (F16 / BF16 / TF32)
    const void *x;                   // NHWC activations, channels padded to g.cpad
    const void *w;                   // [K][R][S][g.cpad]
    const void *b;
    void *y;
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

}  // namespace wpk
