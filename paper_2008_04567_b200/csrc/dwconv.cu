// KB3: depthwise convolution (groups == C == K), the bandwidth-bound path of MobileNet-V2
// (BASELINE.json configs[3]). Not in the paper; same definition as KB1/KB2 with C/g = 1:
//   y[n,c,p,q] = act(b[c] + sum_{r,s} x[n,c,p*sh-ph+r*dh,q*sw-pw+s*dw] * w[c,r,s]).
// NHWC: each thread owns VEC_C consecutive channels (one 4..16-byte vector) x PIX consecutive
// output columns; weights are pre-packed to [R][S][C] so they load as vectors too.
// Per output the taps are summed in (r, s) order with fp32 FMA. grouped_conv_kernel below covers
// the other groups (1 < g < C).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <string>

#include "dwconv.h"
#include "simt_conv.cuh"   // to_f / from_f

namespace wpk {

template <typename T, int VEC, int PIX>
__global__ void dw_conv_kernel(const DwArgs a) {
    const T *__restrict__ x = static_cast<const T *>(a.x);
    const T *__restrict__ wp = static_cast<const T *>(a.w);   // [R][S][C]
    const T *__restrict__ b = static_cast<const T *>(a.b);
    T *__restrict__ y = static_cast<T *>(a.y);
    const int cvecs = a.C / VEC;
    const int qblocks = (a.Q + PIX - 1) / PIX;
    const long long total = (long long)a.N * a.P * qblocks * cvecs;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int cv = (int)(idx % cvecs);
        long long t = idx / cvecs;
        const int qb = (int)(t % qblocks);
        t /= qblocks;
        const int p = (int)(t % a.P);
        const int n = (int)(t / a.P);
        const int c0 = cv * VEC;
        float acc[PIX][VEC];
#pragma unroll
        for (int i = 0; i < PIX; ++i)
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[i][v] = 0.f;
        for (int r = 0; r < a.R; ++r) {
            const int hi = p * a.sh - a.ph + r * a.dh;
            if (hi < 0 || hi >= a.H) continue;
            for (int s = 0; s < a.S; ++s) {
                T wv[VEC];
                const T *wsrc = wp + ((long long)r * a.S + s) * a.C + c0;
                if constexpr (VEC * sizeof(T) >= 4) {
                    constexpr int NB = VEC * sizeof(T);
                    if constexpr (NB == 16) *reinterpret_cast<uint4 *>(wv) = *reinterpret_cast<const uint4 *>(wsrc);
                    else if constexpr (NB == 8) *reinterpret_cast<uint2 *>(wv) = *reinterpret_cast<const uint2 *>(wsrc);
                    else *reinterpret_cast<uint32_t *>(wv) = *reinterpret_cast<const uint32_t *>(wsrc);
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) wv[v] = wsrc[v];
                }
#pragma unroll
                for (int i = 0; i < PIX; ++i) {
                    const int q = qb * PIX + i;
                    const int wi = q * a.sw - a.pw + s * a.dw;
                    if (q >= a.Q || wi < 0 || wi >= a.W) continue;
                    const T *xs = x + (long long)n * a.xs_n + (long long)hi * a.xs_h + (long long)wi * a.xs_w;
                    T xv[VEC];
                    if (a.xs_c == 1 && VEC * sizeof(T) >= 4) {
                        constexpr int NB = VEC * sizeof(T);
                        if constexpr (NB == 16) *reinterpret_cast<uint4 *>(xv) = *reinterpret_cast<const uint4 *>(xs + c0);
                        else if constexpr (NB == 8) *reinterpret_cast<uint2 *>(xv) = *reinterpret_cast<const uint2 *>(xs + c0);
                        else if constexpr (NB == 4) *reinterpret_cast<uint32_t *>(xv) = *reinterpret_cast<const uint32_t *>(xs + c0);
                        else {
#pragma unroll
                            for (int v = 0; v < VEC; ++v) xv[v] = xs[(c0 + v) * a.xs_c];
                        }
                    } else {
#pragma unroll
                        for (int v = 0; v < VEC; ++v) xv[v] = xs[(long long)(c0 + v) * a.xs_c];
                    }
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[i][v] = fmaf(to_f<T>(xv[v]), to_f<T>(wv[v]), acc[i][v]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < PIX; ++i) {
            const int q = qb * PIX + i;
            if (q >= a.Q) continue;
            T out[VEC];
            const long long yo = (long long)n * a.ys_n + (long long)p * a.ys_p + (long long)q * a.ys_q;
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                float o = acc[i][v];
                if (a.epilogue >= 1) o += to_f<T>(b[c0 + v]);
                if (a.epilogue == 3) o += to_f<T>(static_cast<const T *>(a.z)[yo + (long long)(c0 + v) * a.ys_c]);
                if (a.epilogue >= 2) o = fmaxf(o, 0.f);
                out[v] = from_f<T>(o);
            }
            T *yd = y + yo;
            if (a.ys_c == 1 && VEC * sizeof(T) >= 4) {
                constexpr int NB = VEC * sizeof(T);
                if constexpr (NB == 16) *reinterpret_cast<uint4 *>(yd + c0) = *reinterpret_cast<uint4 *>(out);
                else if constexpr (NB == 8) *reinterpret_cast<uint2 *>(yd + c0) = *reinterpret_cast<uint2 *>(out);
                else if constexpr (NB == 4) *reinterpret_cast<uint32_t *>(yd + c0) = *reinterpret_cast<uint32_t *>(out);
                else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) yd[c0 + v] = out[v];
                }
            } else {
#pragma unroll
                for (int v = 0; v < VEC; ++v) yd[(long long)(c0 + v) * a.ys_c] = out[v];
            }
        }
    }
}

// General groups (1 < g, C/g or K/g > 1), the same thread layout with the
// vector over VEC consecutive OUTPUT channels of one group (K/g % VEC == 0): every output of the
// thread reads the same C/g input channels of its group, so each activation is loaded once per
// (tap, channel) and multiplied into VEC accumulators; weights are pre-packed to fp32 [R][S][C/g][K]
// so the VEC weights of one (r, s, c) are one or two vector loads with no conversion. Per output: taps in (r, s, c) order, fp32 FMA.
// VEC consecutive fp32 weights (16-byte vectors where they fit; K/g % VEC == 0 keeps them aligned)
template <int VEC>
__device__ __forceinline__ void load_wvec(float *wv, const float *src) {
    if constexpr (VEC % 4 == 0) {
#pragma unroll
        for (int v = 0; v < VEC; v += 4) *reinterpret_cast<float4 *>(wv + v) = *reinterpret_cast<const float4 *>(src + v);
    } else if constexpr (VEC == 2) {
        *reinterpret_cast<float2 *>(wv) = *reinterpret_cast<const float2 *>(src);
    } else {
        wv[0] = src[0];
    }
}

template <typename T, int VEC, int PIX>
__global__ void grouped_conv_kernel(const DwArgs a) {
    const T *__restrict__ x = static_cast<const T *>(a.x);
    const float *__restrict__ wp = static_cast<const float *>(a.w);   // fp32 [R][S][Cpg][K]
    const T *__restrict__ b = static_cast<const T *>(a.b);
    T *__restrict__ y = static_cast<T *>(a.y);
    const int kvecs = a.K / VEC;
    const int qblocks = (a.Q + PIX - 1) / PIX;
    const long long total = (long long)a.N * a.P * qblocks * kvecs;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int kv = (int)(idx % kvecs);
        long long t = idx / kvecs;
        const int qb = (int)(t % qblocks);
        t /= qblocks;
        const int p = (int)(t % a.P);
        const int n = (int)(t / a.P);
        const int k0 = kv * VEC;
        const int cbase = (k0 / a.Kpg) * a.Cpg;
        float acc[PIX][VEC];
#pragma unroll
        for (int i = 0; i < PIX; ++i)
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[i][v] = 0.f;
        for (int r = 0; r < a.R; ++r) {
            const int hi = p * a.sh - a.ph + r * a.dh;
            if (hi < 0 || hi >= a.H) continue;
            for (int s = 0; s < a.S; ++s) {
                const T *xs[PIX];
#pragma unroll
                for (int i = 0; i < PIX; ++i) {
                    const int q = qb * PIX + i;
                    const int wi = q * a.sw - a.pw + s * a.dw;
                    xs[i] = (q < a.Q && wi >= 0 && wi < a.W)
                                ? x + (long long)n * a.xs_n + (long long)hi * a.xs_h + (long long)wi * a.xs_w +
                                      (long long)cbase * a.xs_c
                                : nullptr;
                }
                const float *wrs = wp + ((long long)(r * a.S + s) * a.Cpg) * a.K + k0;
                int c = 0;
                if (a.xs_c == 1 && (a.Cpg & 3) == 0) {   // NHWC, C/g % 4 == 0: 4 channels per load
                    for (; c < a.Cpg; c += 4) {
                        float xv[PIX][4];
#pragma unroll
                        for (int i = 0; i < PIX; ++i) {
                            if (!xs[i]) continue;
                            T t4[4];
                            if constexpr (sizeof(T) == 2) *reinterpret_cast<uint2 *>(t4) = *reinterpret_cast<const uint2 *>(xs[i] + c);
                            else *reinterpret_cast<uint4 *>(t4) = *reinterpret_cast<const uint4 *>(xs[i] + c);
#pragma unroll
                            for (int j = 0; j < 4; ++j) xv[i][j] = to_f<T>(t4[j]);
                        }
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            float wv[VEC];
                            load_wvec<VEC>(wv, wrs + (long long)(c + j) * a.K);
#pragma unroll
                            for (int i = 0; i < PIX; ++i) {
                                if (!xs[i]) continue;
#pragma unroll
                                for (int v = 0; v < VEC; ++v) acc[i][v] = fmaf(xv[i][j], wv[v], acc[i][v]);
                            }
                        }
                    }
                }
                for (; c < a.Cpg; ++c) {
                    float wv[VEC];
                    load_wvec<VEC>(wv, wrs + (long long)c * a.K);
#pragma unroll
                    for (int i = 0; i < PIX; ++i) {
                        if (!xs[i]) continue;
                        const float xv = to_f<T>(xs[i][(long long)c * a.xs_c]);
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[i][v] = fmaf(xv, wv[v], acc[i][v]);
                    }
                }
            }
        }
#pragma unroll
        for (int i = 0; i < PIX; ++i) {
            const int q = qb * PIX + i;
            if (q >= a.Q) continue;
            T out[VEC];
            const long long yo = (long long)n * a.ys_n + (long long)p * a.ys_p + (long long)q * a.ys_q;
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                float o = acc[i][v];
                if (a.epilogue >= 1) o += to_f<T>(b[k0 + v]);
                if (a.epilogue == 3) o += to_f<T>(static_cast<const T *>(a.z)[yo + (long long)(k0 + v) * a.ys_c]);
                if (a.epilogue >= 2) o = fmaxf(o, 0.f);
                out[v] = from_f<T>(o);
            }
            T *yd = y + yo;
            if (a.ys_c == 1 && VEC * sizeof(T) == 16) *reinterpret_cast<uint4 *>(yd + k0) = *reinterpret_cast<uint4 *>(out);
            else if (a.ys_c == 1 && VEC * sizeof(T) == 8) *reinterpret_cast<uint2 *>(yd + k0) = *reinterpret_cast<uint2 *>(out);
            else {
#pragma unroll
                for (int v = 0; v < VEC; ++v) yd[(long long)(k0 + v) * a.ys_c] = out[v];
            }
        }
    }
}

template <typename T, int VEC>
static int dw_launch_pix(const DwArgs &a, int pix, int threads, long long blocks, cudaStream_t st) {
    const bool grouped = a.Cpg > 0;
#define WPK_DWL(P)                                                                                   \
    if (grouped) grouped_conv_kernel<T, VEC, P><<<(unsigned)blocks, threads, 0, st>>>(a);          \
    else dw_conv_kernel<T, VEC, P><<<(unsigned)blocks, threads, 0, st>>>(a);                        \
    return 0;
    switch (pix) {
    case 1: WPK_DWL(1)
    case 2: WPK_DWL(2)
    case 4: WPK_DWL(4)
    }
#undef WPK_DWL
    return -1;
}

template <typename T>
static int dw_launch_t(const DwArgs &a, int vec, int pix, int threads, long long blocks, cudaStream_t st) {
    switch (vec) {
    case 1: return dw_launch_pix<T, 1>(a, pix, threads, blocks, st);
    case 2: return dw_launch_pix<T, 2>(a, pix, threads, blocks, st);
    case 4: return dw_launch_pix<T, 4>(a, pix, threads, blocks, st);
    case 8: return (sizeof(T) == 2) ? dw_launch_pix<T, (sizeof(T) == 2 ? 8 : 4)>(a, pix, threads, blocks, st) : -1;
    }
    return -1;
}

int dw_launch(const DwArgs &a, int dtype, int vec, int pix, int threads, int sm_count, void *stream,
              std::string *err) {
    const int qblocks = (a.Q + pix - 1) / pix;
    const long long total = (long long)a.N * a.P * qblocks * ((a.Cpg > 0 ? a.K : a.C) / vec);
    long long blocks = (total + threads - 1) / threads;
    const long long cap = (long long)sm_count * (2048 / threads) * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    cudaStream_t st = (cudaStream_t)stream;
    int rc;
    if (dtype == WPK_BF16) rc = dw_launch_t<__nv_bfloat16>(a, vec, pix, threads, blocks, st);
    else if (dtype == WPK_F16) rc = dw_launch_t<__half>(a, vec, pix, threads, blocks, st);
    else rc = dw_launch_t<float>(a, vec, pix, threads, blocks, st);
    if (rc != 0) {
        *err = "no depthwise/grouped instantiation for this (VEC_C, PIX) pair";
        return -1;
    }
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) {
        *err = std::string("dw_conv_kernel launch: ") + cudaGetErrorString(ce);
        return -1;
    }
    return 1;
}

}  // namespace wpk
