// Grouped convolution on the tensor cores (gconv_tc.cu; tcgen05 family, A_MODE 1 of a grouped plan).
#pragma once
#include <cstdint>
#include <string>

#include "wpk_internal.h"

namespace wpk {

struct GconvArgs {
    const void *x;          // NHWC [N][H][W][C]
    const void *w;          // NHWC grouped weights [K][R][S][Cpg]
    const void *b;          // [K] or NULL
    const void *z;          // residual (epilogue 3), NHWC like y
    void *y;                // NHWC [N][P][Q][K]
    int N, C, H, W, P, Q, R, S, K, M;
    int sh, sw, ph, pw, dh, dw;
    int groups, Cpg, Kpg;
    int np;                 // MMA N per group: max(16, Kpg rounded up to 16)
    int gt;                 // groups per CTA tile
    int epilogue;
    int m_tiles;            // set by gconv_tc_launch
    uint32_t tmem_cols, idesc;
};

size_t gconv_tc_smem_bytes(int np);
int gconv_tc_launch(GconvArgs a, int dtype, void *stream, std::string *err);

}  // namespace wpk
