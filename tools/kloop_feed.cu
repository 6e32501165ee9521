// The conv kernel's K loop without the MMAs (DESIGN.md finding 17): every CTA streams K blocks
// = one A box (im2col of 128 output pixels x 64 channels, 3x3 taps cycling, or a tiled 128-row box)
// + one B box (128 weight rows x 64 channels) into a ring of STAGES shared-memory stages; a consumer
// thread holds each full stage HOLD ns (the MMA time of a 128x128x64 block is ~130 ns) before
// freeing it. Variants: B rows shared by all CTAs at the same K block (the conv: every M tile reads
// the same weight tile) or distinct per CTA; A and B issued by one thread or by two.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2008_04567_b200/csrc kloop_feed.cu -lcuda -o kloop_feed
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace wpk;

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\t@P1 mov.s32 %0, 1;\n\t}"
        : "+r"(pred));
    return pred != 0;
}

struct P {
    int stages, iters, hold_ns, a_im2col, b_shared, two_threads, img, nimg, kblocks, nprod;
    long long mrows, brows;
};

__global__ void __launch_bounds__(256, 1) kloop(const __grid_constant__ CUtensorMap tmA2,
                                               const __grid_constant__ CUtensorMap tmAi,
                                               const __grid_constant__ CUtensorMap tmB, P p,
                                               unsigned long long *out) {
    extern __shared__ uint8_t smraw[];
    uint8_t *sm = smraw + ((1024 - (ptx::smem_u32(smraw) & 1023)) & 1023);
    const uint32_t box = 128 * 128;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)p.stages * 2 * box);
    uint64_t *empty = full + 16;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmA2);
        ptx::prefetch_tmap(&tmAi);
        ptx::prefetch_tmap(&tmB);
        for (int s = 0; s < p.stages; ++s) {
            ptx::mbar_init(&full[s], p.two_threads ? 2 : 1);   // producers of one stage
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const unsigned long long t0 = ptx::globaltimer();
    // producers: two_threads -> warp 0 issues A, warp 2 issues B (every stage); else nprod warps
    // 0, 2, 3, 4 (skipping the consumer warp 1), warp j-th producer loads stages i % nprod == j
    const int pw = warp == 0 ? 0 : warp - 1;
    const bool prod = p.two_threads ? (warp == 0 || warp == 2) : (warp != 1 && pw < p.nprod);
    const bool isA = p.two_threads ? warp == 0 : true, isB = p.two_threads ? warp == 2 : true;
    const int step = p.two_threads ? 1 : p.nprod, first = p.two_threads ? 0 : pw;
    if (prod) {   // the whole warp runs the loop (warp-uniform operands: no per-thread waterfall around UTMALDG)
        long long m = ((long long)blockIdx.x * 128) % (p.mrows - 128);
        const int pq = p.img * p.img;
        for (int i = first; i < p.iters; i += step) {
            const uint32_t st = (uint32_t)(i % p.stages), ph = (uint32_t)((i / p.stages) & 1);
            if (i >= p.stages) ptx::mbar_wait(&empty[st], ph ^ 1);
            const int kb = i % p.kblocks;
            const uint32_t tx = (p.two_threads ? 1u : 2u) * box;
            uint8_t *dst = sm + (size_t)st * 2 * box;
            if (elect_one()) {
            ptx::mbar_arrive_expect_tx(&full[st], tx);
            if (isA) {
                if (p.a_im2col) {
                    const int n = (int)(m / pq), rem = (int)(m % pq), pp = rem / p.img, q = rem % p.img;
                    const int tap = kb % 9;
                    ptx::tma_load_im2col_4d(dst, &tmAi, &full[st], 64 * ((kb / 9) % 4), q - 1, pp - 1, n,
                                            (uint16_t)(tap % 3), (uint16_t)(tap / 3));
                } else {
                    ptx::tma_load_2d(dst, &tmA2, &full[st], 64 * (kb % 4), (int)m);
                }
            }
            if (isB) {
                const long long brow = p.b_shared ? 0 : ((long long)blockIdx.x * 128) % (p.brows - 128);
                ptx::tma_load_2d(dst + box, &tmB, &full[st], 64 * (kb % 36), (int)brow);
            }
            }
            __syncwarp();
            if (kb + step > p.kblocks - 1 && i / p.kblocks != (i + step) / p.kblocks) {   // next M tile
                m += 128 * gridDim.x;
                if (m + 128 > p.mrows) m = ((long long)blockIdx.x * 128) % (p.mrows - 128);
            }
        }
    } else if (warp == 1 && lane == 0) {
        uint32_t st = 0, ph = 0;
        for (int i = 0; i < p.iters; ++i) {
            ptx::mbar_wait(&full[st], ph);
            const unsigned long long h0 = ptx::globaltimer();
            while (ptx::globaltimer() - h0 < (unsigned long long)p.hold_ns) {
            }
            ptx::mbar_arrive(&empty[st]);
            if (++st == (uint32_t)p.stages) { st = 0; ph ^= 1; }
        }
    }
    __syncthreads();
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
    // activations: s4-like 14x14x256 x 32 images (3.2 MB, L2-resident); weights [256 rows][2304]
    const int img = 14, C = 256, nimg = 32;
    void *xa, *wb;
    cudaMalloc(&xa, (size_t)nimg * img * img * C * 2);
    cudaMemset(xa, 1, (size_t)nimg * img * img * C * 2);
    const long long brows = 512, bk = 2304;
    cudaMalloc(&wb, (size_t)brows * bk * 2);
    cudaMemset(wb, 1, (size_t)brows * bk * 2);
    CUtensorMap tA2, tAi, tB;
    const cuuint32_t e4[4] = {1, 1, 1, 1};
    {
        cuuint64_t d[2] = {(cuuint64_t)C, (cuuint64_t)nimg * img * img};
        cuuint64_t s[1] = {(cuuint64_t)C * 2};
        cuuint32_t b[2] = {64, 128};
        enc(&tA2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xa, d, s, b, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    {
        cuuint64_t d[4] = {(cuuint64_t)C, (cuuint64_t)img, (cuuint64_t)img, (cuuint64_t)nimg};
        cuuint64_t s[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * img, (cuuint64_t)C * 2 * img * img};
        int lo[2] = {-1, -1}, hi[2] = {-1, -1};
        enci(&tAi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, xa, d, s, lo, hi, 64, 128, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    {
        cuuint64_t d[2] = {(cuuint64_t)bk, (cuuint64_t)brows};
        cuuint64_t s[1] = {(cuuint64_t)bk * 2};
        cuuint32_t b[2] = {64, 128};
        enc(&tB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, wb, d, s, b, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    printf("%-7s %-6s %-4s %-5s %-5s %-5s %9s %9s\n", "A", "Bshare", "prod", "stg", "hold", "grid", "ns/kblk", "B/clk/SM");
    for (int a_im2col : {1, 0})
        for (int b_shared : {1})
            for (int nprod : {0, 1, 2, 3, 4})
                for (int stages : {4, 6})
                    for (int hold : {130})
                        for (int grid : {98, 148}) {
                            if (stages < nprod) continue;
                            P p{stages, 36 * 20, hold, a_im2col, b_shared, nprod == 0, img, nimg, 36,
                                nprod == 0 ? 1 : nprod, (long long)nimg * img * img, brows};
                            const size_t smem = (size_t)stages * 2 * 16384 + 1024 + 512;
                            kloop<<<grid, 256, smem>>>(tA2, tAi, tB, p, out);
                            cudaDeviceSynchronize();
                            kloop<<<grid, 256, smem>>>(tA2, tAi, tB, p, out);
                            cudaError_t err = cudaDeviceSynchronize();
                            std::vector<unsigned long long> o(grid);
                            cudaMemcpy(o.data(), out, grid * 8, cudaMemcpyDeviceToHost);
                            double avg = 0;
                            for (auto v : o) avg += v;
                            avg /= grid;
                            const double ns = avg / p.iters;
                            printf("%-7s %-6d %-4d %-5d %-5d %-5d %9.1f %9.1f %s\n", a_im2col ? "im2col" : "tiled",
                                   b_shared, nprod, stages, hold, grid, ns, 32768.0 / (ns * 1.965),
                                   err == cudaSuccess ? "" : cudaGetErrorString(err));
                        }
    return 0;
}
