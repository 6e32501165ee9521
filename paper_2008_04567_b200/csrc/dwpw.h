// Fused depthwise + pointwise kernel, one output tile per CTA (dwpw.cu; A_MODE 1 of a fused plan).
#pragma once
#include <cstdint>
#include <string>

#include "wpk_internal.h"

namespace wpk {

struct DwpwArgs {
    const void *x;          // NHWC [N][H][W][C]
    const void *w_dw;       // depthwise weights packed [R][S][C]
    const void *b_dw;       // [C] or NULL (dw epilogue NONE)
    const void *w_pw;       // pointwise weights [K][C]
    const void *b_pw;       // [K] or NULL (pw epilogue NONE)
    void *y;                // NHWC [N][P][Q][K]
    int N, C, H, W, P, Q, R, S, K, M;
    int sh, sw, ph, pw, dh, dw;
    int dw_epi, pw_epi;     // 0 none, 1 bias, 2 bias + ReLU
    int kp;                 // K rounded up to 16 (set by dwpw_launch)
    int splits;             // split-K over the 64-channel chunks (>= 1); > 1: fp32 partials + a reduction
    int kc_per_split;       // chunks per split (set by dwpw_launch)
    float *partial;         // [splits][M][K] fp32 (workspace) when splits > 1
    uint32_t tmem_cols, idesc0, idesc1;
};

size_t dwpw_smem_bytes(int kp);
// returns the number of launches (1) or -1 with *err set
int dwpw_launch(DwpwArgs a, int dtype, void *stream, std::string *err);

}  // namespace wpk
