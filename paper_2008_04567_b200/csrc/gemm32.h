// Exact-fp32 implicit-GEMM convolution on CUDA cores (KB2b, WPK_FAMILY_GEMM32) host interface.
#pragma once
#include <string>

namespace wpk {

struct Gemm32Args {
    const float *x;   // NHWC [N][H][W][C], C % 4 == 0 (zero-padded by the launcher otherwise)
    const float *w;   // KRSC [K][R][S][C]
    const float *b;   // [K] (epilogue >= 1)
    float *y;         // output, element (n, k, p, q) at n*ys_n + k*ys_k + p*ys_p + q*ys_q
    const float *z;   // residual (epilogue 3), laid out as y
    long long M;      // N * P * Q
    int PQ, Q, K, C, H, W, R, S;
    int sh, sw, ph, pw, dh, dw;
    long long ys_n, ys_k, ys_p, ys_q;
    int epilogue;
    int kper;          // K steps per split (set by gemm32_launch)
    float *partial;    // [splits][M][K] fp32 partials when SPLIT_K > 1 (set by gemm32_launch)
};

// genes (BLOCK_M, BLOCK_N, BLOCK_K, THREAD_TILE, SPLIT_K); partial = workspace of
// gemm32_partial_bytes(); returns launches (1, or 2 with the split-K reduction) or -1 with *err set
int gemm32_launch(const Gemm32Args &a, int bm, int bn, int bk, int tt, int splits, float *partial, int sm_count,
                  void *stream, std::string *err);

}  // namespace wpk
