// Depthwise convolution (KB3) host interface.
#pragma once
#include <string>

#include "wpk_internal.h"

namespace wpk {

struct DwArgs {
    const void *x, *w, *b;   // w packed [R][S][C] (depthwise) or [R][S][C/g][K] (grouped)
    void *y;
    const void *z;           // residual (epilogue 3), laid out as y
    int N, C, H, W, R, S, P, Q;
    int K, Cpg, Kpg;         // grouped: output channels, channels per group (in, out); 0 = depthwise
    int sh, sw, ph, pw, dh, dw;
    long long xs_n, xs_c, xs_h, xs_w;
    long long ys_n, ys_c, ys_p, ys_q;   // ys_c: output-channel stride
    int epilogue;
};

int dw_launch(const DwArgs &a, int dtype, int vec, int pix, int threads, int sm_count, void *stream,
              std::string *err);

}  // namespace wpk
