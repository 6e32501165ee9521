// Micro-benchmark of the per-SM TMA operand feed that bounds the implicit-GEMM K loop (DESIGN.md
// finding 1/6). Every CTA streams "K blocks" into a ring of shared-memory stages: an A box (tiled
// 2-D rows, or an im2col box of output pixels x 64 channels cycling over the 9 taps of a 3x3
// conv, as the conv kernel's A producer issues them) plus a B box (tiled rows), 128 bytes per row.
// Reported: bytes landing in each SM's shared memory per SM clock, versus
//   box rows (64 / 128), stages in flight, A kind, one or two issuing threads, active SMs,
//   L2-resident (8 MB) or DRAM-streamed (3 GB) source.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2008_04567_b200/csrc tma_feed.cu -lcuda -o tma_feed
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace wpk;

struct Geo {
    long long rows_total;   // rows of the 2-D view (pixels)
    int img;                // 4-D view: H = W = img
    long long nimg;
};

// warp 0 lane 0: A (+ B unless split), warp 2 lane 0: B (split), warp 1 lane 0: consumer
__global__ void __launch_bounds__(96, 1) feed(const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmAi,
                                             const __grid_constant__ CUtensorMap tmB, int iters, Geo geo, int stages,
                                             int rows, int a_im2col, int split, unsigned long long *cycles) {
    extern __shared__ uint8_t smraw[];
    uint8_t *sm = smraw + ((1024 - (ptx::smem_u32(smraw) & 1023)) & 1023);
    const uint32_t box = (uint32_t)rows * 128;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)stages * 2 * box);
    uint64_t *empty = full + 16;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            ptx::mbar_init(&full[s], split ? 2 : 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    if (lane == 0 && (warp == 0 || (warp == 2 && split))) {
        const bool doA = (warp == 0), doB = (warp == 2) || !split;
        long long m = ((long long)blockIdx.x * 7919 * rows) % (geo.rows_total - rows);
        long long mb = ((long long)blockIdx.x * 104729 * rows) % (geo.rows_total - rows);
        int tap = 0;
        uint32_t st = 0, ph = 0;
        const int pq = geo.img * geo.img;
        for (int i = 0; i < iters; ++i) {
            ptx::mbar_wait(&empty[st], ph ^ 1);
            ptx::mbar_arrive_expect_tx(&full[st], (doA ? box : 0) + (doB ? box : 0));
            uint8_t *dst = sm + (size_t)st * 2 * box;
            if (doA) {
                if (a_im2col) {
                    const int n = (int)(m / pq), rem = (int)(m % pq);
                    const int p = rem / geo.img, q = rem % geo.img;
                    ptx::tma_load_im2col_4d(dst, &tmAi, &full[st], 0, q - 1, p - 1, n, (uint16_t)(tap % 3),
                                            (uint16_t)(tap / 3));
                } else {
                    ptx::tma_load_2d(dst, &tmA2, &full[st], 0, (int)m);
                }
            }
            if (doB) ptx::tma_load_2d(dst + box, &tmB, &full[st], 0, (int)mb);
            if (++tap == 9) {           // next M tile after the 9 taps
                tap = 0;
                m += rows;
                if (m + rows > geo.rows_total) m = 0;
            }
            mb += rows;
            if (mb + rows > geo.rows_total) mb = 0;
            if (++st == (uint32_t)stages) { st = 0; ph ^= 1; }
        }
    } else if (warp == 1 && lane == 0) {
        uint32_t st = 0, ph = 0;
        for (int i = 0; i < iters; ++i) {
            ptx::mbar_wait(&full[st], ph);
            ptx::mbar_arrive(&empty[st]);
            if (++st == (uint32_t)stages) { st = 0; ph ^= 1; }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
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
    cudaFuncSetAttribute(feed, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    unsigned long long *cyc;
    cudaMalloc(&cyc, 1024 * 8);
    const int img = 14;
    void *buf;
    const long long big = 3LL << 30;
    cudaMalloc(&buf, big);
    cudaMemset(buf, 1, big);
    printf("%-5s %-6s %-5s %-6s %-5s %-5s %8s %9s %9s\n", "data", "A", "rows", "stages", "split", "grid", "GB/s",
           "B/clk/SM", "ns/kblk");
    for (int dram = 0; dram < 2; ++dram) {
        const long long bytes = dram ? big : (8LL << 20);
        Geo geo;
        geo.img = img;
        geo.nimg = bytes / (128LL * img * img);
        geo.rows_total = geo.nimg * img * img;
        for (int rows : {64, 128}) {
            CUtensorMap tA2, tAi, tB;
            cuuint64_t d2[2] = {64, (cuuint64_t)geo.rows_total};
            cuuint64_t s2[1] = {128};
            cuuint32_t b2[2] = {64, (cuuint32_t)rows};
            cuuint32_t e2[2] = {1, 1};
            enc(&tA2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            enc(&tB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            cuuint64_t d4[4] = {64, (cuuint64_t)img, (cuuint64_t)img, (cuuint64_t)geo.nimg};
            cuuint64_t s4[3] = {128, 128ull * img, 128ull * img * img};
            int lo[2] = {-1, -1}, hi[2] = {-1, -1};
            cuuint32_t e4[4] = {1, 1, 1, 1};
            CUresult r = enci(&tAi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, d4, s4, lo, hi, 64, (cuuint32_t)rows, e4,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) printf("im2col encode failed %d\n", (int)r);
            for (int a_im2col : {0, 1})
                for (int stages : {4, 6, 8, 12})
                    for (int split : {0, 1})
                        for (int grid : {74, 148}) {
                            const size_t smem = (size_t)stages * 2 * rows * 128 + 2048;
                            if (smem > 227 * 1024) continue;
                            if (!(grid == 148 || (stages == 6 && split == 1))) continue;
                            const int iters = dram ? 600 : 3000;
                            feed<<<grid, 96, smem>>>(tA2, tAi, tB, 20, geo, stages, rows, a_im2col, split, cyc);
                            cudaEvent_t e0, e1;
                            cudaEventCreate(&e0);
                            cudaEventCreate(&e1);
                            cudaEventRecord(e0);
                            feed<<<grid, 96, smem>>>(tA2, tAi, tB, iters, geo, stages, rows, a_im2col, split, cyc);
                            cudaEventRecord(e1);
                            cudaError_t err = cudaEventSynchronize(e1);
                            float ms = 0;
                            cudaEventElapsedTime(&ms, e0, e1);
                            std::vector<unsigned long long> c(grid);
                            cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
                            double avg = 0;
                            for (auto v : c) avg += v;
                            avg /= grid;
                            const double per_cta = (double)iters * 2 * rows * 128;
                            printf("%-5s %-6s %-5d %-6d %-5d %-5d %8.0f %9.1f %9.1f %s\n", dram ? "dram" : "l2",
                                   a_im2col ? "im2col" : "tiled", rows, stages, split, grid,
                                   per_cta * grid / (ms * 1e-3) / 1e9, per_cta / avg, ms * 1e6 / iters,
                                   err == cudaSuccess ? "" : cudaGetErrorString(err));
                        }
        }
    }
    return 0;
}
