// Does TMA multicast of the weight tile raise the per-SM K-loop feed? (DESIGN.md finding 22)
// Clusters of 2 CTAs stream K blocks = A box (im2col, 128 pixels x 64 ch, own) + B tile (128 weight
// rows x 64 ch). Unicast: each CTA loads its whole B tile. Multicast: each CTA loads one 64-row half
// with .multicast::cluster to both CTAs (the pair of M tiles shares the weight tile). A consumer
// thread holds each full stage 130 ns (the MMA time of a 128x128x64 block) and frees it in both
// CTAs (the peer writes into our B half). Reports ns per K block.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2008_04567_b200/csrc kloop_mc.cu -lcuda -o kloop_mc
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace wpk;

__device__ __forceinline__ void tma_2d_mc(void *smem, const CUtensorMap *m, uint64_t *bar, int c0, int c1, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(ptx::smem_u32(smem)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}

struct P {
    int stages, iters, hold_ns, mc, img, nimg;
    long long mrows;
};

__global__ void __launch_bounds__(128, 1) kloop(const __grid_constant__ CUtensorMap tmAi,
                                               const __grid_constant__ CUtensorMap tmB,
                                               const __grid_constant__ CUtensorMap tmBh, P p, unsigned long long *out) {
    extern __shared__ uint8_t smraw[];
    uint8_t *sm = smraw + ((1024 - (ptx::smem_u32(smraw) & 1023)) & 1023);
    const uint32_t box = 128 * 128;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)p.stages * 2 * box);
    uint64_t *empty = full + 16;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = ptx::cluster_ctarank();
    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmAi);
        ptx::prefetch_tmap(&tmB);
        ptx::prefetch_tmap(&tmBh);
        for (int s = 0; s < p.stages; ++s) {
            ptx::mbar_init(&full[s], 2);                 // A producer + B producer of this CTA
            ptx::mbar_init(&empty[s], p.mc ? 2 : 1);    // multicast: our consumer and the peer's
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    ptx::cluster_sync();
    const unsigned long long t0 = ptx::globaltimer();
    const int pq = p.img * p.img;
    if ((warp == 0 || warp == 2) && lane == 0) {
        const bool isA = warp == 0;
        uint32_t st = 0, ph = 0;
        long long m = ((long long)blockIdx.x * 128) % (p.mrows - 128);
        for (int i = 0; i < p.iters; ++i) {
            ptx::mbar_wait(&empty[st], ph ^ 1);
            const int kb = i % 36;
            uint8_t *dst = sm + (size_t)st * 2 * box;
            if (isA) {
                ptx::mbar_arrive_expect_tx(&full[st], box);
                const int n = (int)(m / pq), rem = (int)(m % pq), pp = rem / p.img, q = rem % p.img;
                const int tap = kb % 9;
                ptx::tma_load_im2col_4d(dst, &tmAi, &full[st], 64 * ((kb / 9) % 4), q - 1, pp - 1, n,
                                        (uint16_t)(tap % 3), (uint16_t)(tap / 3));
                if (kb == 35) {
                    m += 128 * gridDim.x;
                    if (m + 128 > p.mrows) m = ((long long)blockIdx.x * 128) % (p.mrows - 128);
                }
            } else {
                ptx::mbar_arrive_expect_tx(&full[st], box);   // the whole B tile lands here either way
                if (p.mc) tma_2d_mc(dst + box + rank * box / 2, &tmBh, &full[st], 64 * kb, (int)rank * 64, 0x3);
                else ptx::tma_load_2d(dst + box, &tmB, &full[st], 64 * kb, 0);
            }
            if (++st == (uint32_t)p.stages) { st = 0; ph ^= 1; }
        }
    } else if (warp == 1 && lane == 0) {
        uint32_t st = 0, ph = 0;
        const uint32_t peer = rank ^ 1u;
        for (int i = 0; i < p.iters; ++i) {
            ptx::mbar_wait(&full[st], ph);
            const unsigned long long h0 = ptx::globaltimer();
            while (ptx::globaltimer() - h0 < (unsigned long long)p.hold_ns) {
            }
            ptx::mbar_arrive(&empty[st]);
            if (p.mc) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&empty[st]), peer));
            if (++st == (uint32_t)p.stages) { st = 0; ph ^= 1; }
        }
    }
    __syncthreads();
    ptx::cluster_sync();
    if (threadIdx.x == 0) out[blockIdx.x] = ptx::globaltimer() - t0;
}

typedef CUresult (*EncT)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                         const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                         CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*EncI)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                         const int *, const int *, cuuint32_t, cuuint32_t, const cuuint32_t *, CUtensorMapInterleave,
                         CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    void *f1 = nullptr, *f2 = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f1, cudaEnableDefault, &q) != cudaSuccess || !f1 ||
        cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f2, cudaEnableDefault, &q) != cudaSuccess || !f2) {
        printf("no tensor-map encoders (no GPU?)\n");
        return 1;
    }
    EncT enc = (EncT)f1;
    EncI enci = (EncI)f2;
    cudaFuncSetAttribute(kloop, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    unsigned long long *out;
    cudaMalloc(&out, 1024 * 8);
    const int img = 14, C = 256, nimg = 32;
    void *xa, *wb;
    cudaMalloc(&xa, (size_t)nimg * img * img * C * 2);
    cudaMemset(xa, 1, (size_t)nimg * img * img * C * 2);
    const long long brows = 256, bk = 2304;
    cudaMalloc(&wb, (size_t)brows * bk * 2);
    cudaMemset(wb, 1, (size_t)brows * bk * 2);
    CUtensorMap tAi, tB, tBh;
    const cuuint32_t e4[4] = {1, 1, 1, 1};
    {
        cuuint64_t d[4] = {(cuuint64_t)C, (cuuint64_t)img, (cuuint64_t)img, (cuuint64_t)nimg};
        cuuint64_t s[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * img, (cuuint64_t)C * 2 * img * img};
        int lo[2] = {-1, -1}, hi[2] = {-1, -1};
        enci(&tAi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, xa, d, s, lo, hi, 64, 128, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    for (int half = 0; half < 2; ++half) {
        cuuint64_t d[2] = {(cuuint64_t)bk, (cuuint64_t)brows};
        cuuint64_t s[1] = {(cuuint64_t)bk * 2};
        cuuint32_t b[2] = {64, half ? 64u : 128u};
        enc(half ? &tBh : &tB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, wb, d, s, b, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    printf("%-6s %-6s %-5s %-5s %9s\n", "mc", "stages", "hold", "grid", "ns/kblk");
    for (int mc : {0, 1})
        for (int stages : {4, 6})
            for (int hold : {0, 130}) {
                P p{stages, 36 * 20, hold, mc, img, nimg, (long long)nimg * img * img};
                const size_t smem = (size_t)stages * 2 * 16384 + 1024 + 512;
                cudaLaunchConfig_t lc{};
                lc.gridDim = dim3(148);
                lc.blockDim = dim3(128);
                lc.dynamicSmemBytes = smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = 2;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                lc.attrs = at;
                lc.numAttrs = 1;
                cudaLaunchKernelEx(&lc, kloop, tAi, tB, tBh, p, out);
                cudaDeviceSynchronize();
                cudaLaunchKernelEx(&lc, kloop, tAi, tB, tBh, p, out);
                cudaError_t err = cudaDeviceSynchronize();
                std::vector<unsigned long long> o(148);
                cudaMemcpy(o.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
                double avg = 0;
                for (auto v : o) avg += v;
                avg /= 148;
                printf("%-6d %-6d %-5d %-5d %9.1f %s\n", mc, stages, hold, 148, avg / p.iters,
                       err == cudaSuccess ? "" : cudaGetErrorString(err));
            }
    return 0;
}
