// Host/device interface of the tcgen05 implicit-GEMM convolution (umma_conv.cu).
#pragma once
#include <cstdint>
#include <string>

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
    int bn, bk, stages, acc_stages;
    uint32_t idesc, tmem_cols;
    int epilogue, out_nchw, vec_ok;
};

struct UmmaLaunch {
    int dtype;                       // wpk_dtype (F16 / BF16 / TF32)
    const void *x;                   // NHWC activations, channels padded to g.cpad
    const void *w;                   // [K][R][S][g.cpad]
    const void *b;
    void *y;
    float *partial;                  // split-K workspace (splits x M x K fp32) or nullptr
    int N, H, W, K, R, S, P, Q;
    int stride_h, stride_w, pad_h, pad_w, dil_h, dil_w;
    int epilogue, out_nchw;
    int sm_count;
    void *stream;
    UmmaGeom g;
};

// Returns the number of kernel launches issued (1 or 2), or -1 with *err set.
int umma_launch(const UmmaLaunch &L, std::string *err);

}  // namespace wpk
