// KB2: direct convolution on CUDA cores with fp32 FMA -- the exact-fp32 strict-comparison path and
// the universal fallback (any layout, dtype, stride, padding, dilation, groups).
//
// Schedule template = the paper's own genes (O_conv entries T_x..Tile_rz):
//   T_x, T_y, T_z   threads of a block along output column q, output row p, output channel k
//   Tile_x, Tile_y, Tile_z   outputs per thread along q, p, k (strided by the block extent so that
//                            adjacent threads touch adjacent q -> coalesced NCHW accesses)
//   Tile_rz         unroll of the reduction over input channels ("split and unroll size in a
//                   reduce domain")
// Every output is summed in the same order (c ascending, then r, then s) with fp32 FMA.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace wpk {

struct SimtArgs {
    const void *x, *w, *b;
    void *y;
    const void *z;          // residual (epilogue 3), laid out as y
    int N, C, H, W, K, R, S, P, Q;
    int sh, sw, ph, pw, dh, dw, Cpg, Kpg, groups;
    long long xs_n, xs_c, xs_h, xs_w;
    long long ws_k, ws_c, ws_r, ws_s;
    long long ys_n, ys_k, ys_p, ys_q;
    int epilogue;
    int kblocks;
};

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <> __device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ __half from_f<__half>(float v) { return __float2half_rn(v); }

template <typename T, int TX, int TY, int TZ, int TRZ>
__global__ void simt_conv_kernel(const SimtArgs a) {
    const T *__restrict__ x = static_cast<const T *>(a.x);
    const T *__restrict__ w = static_cast<const T *>(a.w);
    const int bx = blockDim.x, by = blockDim.y, bz = blockDim.z;
    const int q0 = blockIdx.x * bx * TX + threadIdx.x;
    const int p0 = blockIdx.y * by * TY + threadIdx.y;
    const int n = blockIdx.z / a.kblocks;
    const int k0 = (blockIdx.z % a.kblocks) * bz * TZ + threadIdx.z;

    float acc[TZ][TY][TX];
#pragma unroll
    for (int j = 0; j < TZ; ++j)
#pragma unroll
        for (int i = 0; i < TY; ++i)
#pragma unroll
            for (int l = 0; l < TX; ++l) acc[j][i][l] = 0.f;

    int cbase[TZ];
    bool kval[TZ];
#pragma unroll
    for (int j = 0; j < TZ; ++j) {
        const int k = k0 + j * bz;
        kval[j] = k < a.K;
        cbase[j] = kval[j] ? (k / a.Kpg) * a.Cpg : 0;
    }
    const T *xn = x + (long long)n * a.xs_n;

    for (int c = 0; c < a.Cpg; c += TRZ) {
#pragma unroll
        for (int cc = 0; cc < TRZ; ++cc) {
            const int ci = c + cc;
            if (ci < a.Cpg) {
                for (int r = 0; r < a.R; ++r) {
                    for (int s = 0; s < a.S; ++s) {
                        float wv[TZ];
#pragma unroll
                        for (int j = 0; j < TZ; ++j) {
                            const int k = k0 + j * bz;
                            wv[j] = kval[j] ? to_f<T>(w[k * a.ws_k + ci * a.ws_c + r * a.ws_r + s * a.ws_s]) : 0.f;
                        }
#pragma unroll
                        for (int i = 0; i < TY; ++i) {
                            const int hi = (p0 + i * by) * a.sh - a.ph + r * a.dh;
                            const bool hok = (p0 + i * by) < a.P && hi >= 0 && hi < a.H;
#pragma unroll
                            for (int l = 0; l < TX; ++l) {
                                const int wi = (q0 + l * bx) * a.sw - a.pw + s * a.dw;
                                const bool ok = hok && (q0 + l * bx) < a.Q && wi >= 0 && wi < a.W;
                                if (a.groups == 1) {
                                    const float xv = ok ? to_f<T>(xn[ci * a.xs_c + hi * a.xs_h + wi * a.xs_w]) : 0.f;
#pragma unroll
                                    for (int j = 0; j < TZ; ++j) acc[j][i][l] = fmaf(xv, wv[j], acc[j][i][l]);
                                } else {
#pragma unroll
                                    for (int j = 0; j < TZ; ++j) {
                                        const float xv = (ok && kval[j])
                                            ? to_f<T>(xn[(cbase[j] + ci) * a.xs_c + hi * a.xs_h + wi * a.xs_w]) : 0.f;
                                        acc[j][i][l] = fmaf(xv, wv[j], acc[j][i][l]);
                                    }
                                }
                            }
                        }
                    }
                }
            }
        }
    }
    T *y = static_cast<T *>(a.y);
    const T *b = static_cast<const T *>(a.b);
#pragma unroll
    for (int j = 0; j < TZ; ++j) {
        const int k = k0 + j * bz;
        if (!kval[j]) continue;
        const float bias = (a.epilogue >= 1) ? to_f<T>(b[k]) : 0.f;
#pragma unroll
        for (int i = 0; i < TY; ++i) {
            const int p = p0 + i * by;
            if (p >= a.P) continue;
#pragma unroll
            for (int l = 0; l < TX; ++l) {
                const int q = q0 + l * bx;
                if (q >= a.Q) continue;
                float v = acc[j][i][l] + bias;
                const long long yi = n * a.ys_n + k * a.ys_k + p * a.ys_p + q * a.ys_q;
                if (a.epilogue == 3) v += to_f<T>(static_cast<const T *>(a.z)[yi]);
                if (a.epilogue >= 2) v = fmaxf(v, 0.f);
                y[yi] = from_f<T>(v);
            }
        }
    }
}

using SimtKernelFn = void (*)(const SimtArgs);

// Tables of all (Tile_x, Tile_y, Tile_z, Tile_rz) instantiations, one per element type
// (defined in simt_conv_{f32,bf16,f16}.cu).
SimtKernelFn simt_get_f32(int tx, int ty, int tz, int trz);
SimtKernelFn simt_get_bf16(int tx, int ty, int tz, int trz);
SimtKernelFn simt_get_f16(int tx, int ty, int tz, int trz);

}  // namespace wpk

#define WPK_SIMT_TABLE_IMPL(T, NAME, FULL)                                                                        \
    namespace wpk {                                                                                     \
    template <int TX, int TY, int TZ>                                                                   \
    static SimtKernelFn simt_pick_rz(int trz) {                                                         \
        switch (trz) {                                                                                  \
        case 1: return simt_conv_kernel<T, TX, TY, TZ, 1>;                                              \
        case 2: return FULL ? simt_conv_kernel<T, TX, TY, TZ, FULL ? 2 : 1> : nullptr;                   \
        case 4: return FULL ? simt_conv_kernel<T, TX, TY, TZ, FULL ? 4 : 1> : nullptr;                   \
        case 8: return FULL ? simt_conv_kernel<T, TX, TY, TZ, FULL ? 8 : 1> : nullptr;                   \
        }                                                                                               \
        return nullptr;                                                                                 \
    }                                                                                                   \
    template <int TX, int TY>                                                                           \
    static SimtKernelFn simt_pick_z(int tz, int trz) {                                                  \
        switch (tz) {                                                                                   \
        case 1: return simt_pick_rz<TX, TY, 1>(trz);                                                    \
        case 2: return simt_pick_rz<TX, TY, 2>(trz);                                                    \
        case 4: return simt_pick_rz<TX, TY, 4>(trz);                                                    \
        }                                                                                               \
        return nullptr;                                                                                 \
    }                                                                                                   \
    template <int TX>                                                                                   \
    static SimtKernelFn simt_pick_y(int ty, int tz, int trz) {                                          \
        switch (ty) {                                                                                   \
        case 1: return simt_pick_z<TX, 1>(tz, trz);                                                     \
        case 2: return simt_pick_z<TX, 2>(tz, trz);                                                     \
        case 4: return simt_pick_z<TX, 4>(tz, trz);                                                     \
        }                                                                                               \
        return nullptr;                                                                                 \
    }                                                                                                   \
    SimtKernelFn NAME(int tx, int ty, int tz, int trz) {                                                \
        switch (tx) {                                                                                   \
        case 1: return simt_pick_y<1>(ty, tz, trz);                                                     \
        case 2: return simt_pick_y<2>(ty, tz, trz);                                                     \
        case 4: return simt_pick_y<4>(ty, tz, trz);                                                     \
        }                                                                                               \
        return nullptr;                                                                                 \
    }                                                                                                   \
    }
