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

// Depthwise 3x3, NHWC, 16-bit data, 16-byte channel vectors (the VEC_C = 8 instantiations of the
// common MobileNet case: dilation 1, stride SW in {1, 2}, C % 8 == 0, < 2^31 work items). The same
// definition and per-output order as dw_conv_kernel -- taps in (r, s) order, one fp32 FMA each, the
// bias after the sum -- with the memory traffic of a sliding window: a thread's PIX consecutive
// outputs of one row need (PIX-1)*SW + 3 input columns per filter row, each loaded once (16 B) and
// reused by every tap that reads it; two channels per FFMA2 (bit-identical to two FFMAs); 32-bit
// index arithmetic. Consecutive threads take consecutive channel vectors of one pixel (coalesced).
__device__ __forceinline__ float2 dw_up2(uint32_t u, __nv_bfloat16 *) {
    return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
}
__device__ __forceinline__ float2 dw_up2(uint32_t u, __half *) {
    return __half22float2(*reinterpret_cast<const __half2 *>(&u));
}
__device__ __forceinline__ void dw_ffma2(float2 &acc, float2 a, float2 b) {
    unsigned long long c = *reinterpret_cast<unsigned long long *>(&acc);
    asm("fma.rn.f32x2 %0, %1, %2, %0;"
        : "+l"(c)
        : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)));
    acc = *reinterpret_cast<float2 *>(&c);
}
__device__ __forceinline__ uint32_t dw_pack2(float a, float b, __nv_bfloat16 *) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ uint32_t dw_pack2(float a, float b, __half *) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

template <typename T, int PIX, int SW>
__global__ void dw3_nhwc_kernel(const DwArgs a) {
    constexpr int NCOL = (PIX - 1) * SW + 3;
    const uint4 *__restrict__ x = static_cast<const uint4 *>(a.x);
    const uint4 *__restrict__ wp = static_cast<const uint4 *>(a.w);   // [3][3][C] in 16-byte vectors
    const uint4 *__restrict__ b = static_cast<const uint4 *>(a.b);
    const uint4 *__restrict__ z = static_cast<const uint4 *>(a.z);
    uint4 *__restrict__ y = static_cast<uint4 *>(a.y);
    const int cvecs = a.C >> 3;
    const int qblocks = (a.Q + PIX - 1) / PIX;
    const int total = a.N * a.P * qblocks * cvecs;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int cv = idx % cvecs;
        int t = idx / cvecs;
        const int qb = t % qblocks;
        t /= qblocks;
        const int p = t % a.P;
        const int n = t / a.P;
        const int q0 = qb * PIX;
        const int w0 = q0 * SW - a.pw;
        float2 acc[PIX][4];
#pragma unroll
        for (int i = 0; i < PIX; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[i][e] = make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const int hi = p * a.sh - a.ph + r;
            if (hi < 0 || hi >= a.H) continue;
            const uint4 *xr = x + (size_t)((n * a.H + hi) * a.W) * cvecs + cv;
            uint4 col[NCOL];
#pragma unroll
            for (int c = 0; c < NCOL; ++c) {
                const int wi = w0 + c;
                col[c] = (wi >= 0 && wi < a.W) ? __ldg(xr + (size_t)wi * cvecs) : make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                const uint4 wv = __ldg(wp + (size_t)(r * 3 + s) * cvecs + cv);
                const float2 w0f = dw_up2(wv.x, (T *)nullptr), w1f = dw_up2(wv.y, (T *)nullptr);
                const float2 w2f = dw_up2(wv.z, (T *)nullptr), w3f = dw_up2(wv.w, (T *)nullptr);
#pragma unroll
                for (int i = 0; i < PIX; ++i) {
                    const uint4 xv = col[i * SW + s];
                    dw_ffma2(acc[i][0], dw_up2(xv.x, (T *)nullptr), w0f);
                    dw_ffma2(acc[i][1], dw_up2(xv.y, (T *)nullptr), w1f);
                    dw_ffma2(acc[i][2], dw_up2(xv.z, (T *)nullptr), w2f);
                    dw_ffma2(acc[i][3], dw_up2(xv.w, (T *)nullptr), w3f);
                }
            }
        }
        float2 bf[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        if (a.epilogue >= 1) {
            const uint4 bv = __ldg(b + cv);
            bf[0] = dw_up2(bv.x, (T *)nullptr); bf[1] = dw_up2(bv.y, (T *)nullptr);
            bf[2] = dw_up2(bv.z, (T *)nullptr); bf[3] = dw_up2(bv.w, (T *)nullptr);
        }
#pragma unroll
        for (int i = 0; i < PIX; ++i) {
            const int q = q0 + i;
            if (q >= a.Q) break;
            const size_t yo = (size_t)((n * a.P + p) * a.Q + q) * cvecs + cv;
            float2 zf[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            if (a.epilogue == 3) {
                const uint4 zv = __ldg(z + yo);
                zf[0] = dw_up2(zv.x, (T *)nullptr); zf[1] = dw_up2(zv.y, (T *)nullptr);
                zf[2] = dw_up2(zv.z, (T *)nullptr); zf[3] = dw_up2(zv.w, (T *)nullptr);
            }
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float v0 = acc[i][e].x, v1 = acc[i][e].y;
                if (a.epilogue >= 1) { v0 += bf[e].x; v1 += bf[e].y; }
                if (a.epilogue == 3) { v0 += zf[e].x; v1 += zf[e].y; }
                if (a.epilogue >= 2) { v0 = fmaxf(v0, 0.f); v1 = fmaxf(v1, 0.f); }
                o[e] = dw_pack2(v0, v1, (T *)nullptr);
            }
            y[yo] = make_uint4(o[0], o[1], o[2], o[3]);
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

// the sliding-window 3x3 NHWC kernel applies (else the generic dw_conv_kernel)
static bool dw3_fast_ok(const DwArgs &a, int elem, int vec) {
    if (elem != 2 || vec != 8 || a.Cpg > 0 || a.C % 8 || a.xs_c != 1 || a.ys_c != 1) return false;
    if (a.R != 3 || a.S != 3 || a.dh != 1 || a.dw != 1 || (a.sw != 1 && a.sw != 2)) return false;
    if (a.xs_w != a.C || a.ys_q != a.C) return false;   // dense NHWC
    return (double)a.N * a.P * a.Q * (a.C / 8) < 2.0e9 && (double)a.N * a.H * a.W * a.C < 2.0e9;
}

template <typename T, int VEC>
static int dw_launch_pix(const DwArgs &a, int pix, int threads, long long blocks, cudaStream_t st) {
    const bool grouped = a.Cpg > 0;
    if constexpr (VEC == 8 && sizeof(T) == 2) {
        if (dw3_fast_ok(a, 2, VEC)) {
#define WPK_DW3(P)                                                                                   \
    if (a.sw == 1) dw3_nhwc_kernel<T, P, 1><<<(unsigned)blocks, threads, 0, st>>>(a);                 \
    else dw3_nhwc_kernel<T, P, 2><<<(unsigned)blocks, threads, 0, st>>>(a);                         \
    return 0;
            switch (pix) {
            case 1: WPK_DW3(1)
            case 2: WPK_DW3(2)
            case 4: WPK_DW3(4)
            }
#undef WPK_DW3
            return -1;
        }
    }
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
