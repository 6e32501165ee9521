// Micro-benchmark: TMA tile-load throughput into shared memory per SM (no MMA), to size the
// implicit-GEMM pipeline. One CTA per SM; thread 0 streams boxes of ROWS x 128 B into a ring of
// STAGES buffers, thread 32 consumes (waits full, re-arms empty). Reports GB/s and B/clk/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2008_04567_b200/csrc tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "ptx.cuh"

using namespace wpk;
__device__ __forceinline__ bool test_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(ptx::smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void wait_any(uint64_t *bar, uint32_t parity, int mode) {
    if (mode == 0) ptx::mbar_wait(bar, parity);
    else while (!test_wait(bar, parity)) {}
}

__global__ void __launch_bounds__(256, 1) tma_stream(const __grid_constant__ CUtensorMap tm, int stages, int rows,
                                                     int iters, int total_rows, unsigned long long *cycles, int nb, int warpmode) {
    extern __shared__ uint8_t smraw[];
    uint32_t base = ptx::smem_u32(smraw);
    uint8_t *sm = smraw + ((1024 - (base & 1023)) & 1023);
    const uint32_t box = rows * 128 * nb;
    const int P = blockDim.x / 64;              // independent producer/consumer pairs
    const int pid = (threadIdx.x / 32) % P;
    const bool is_prod = threadIdx.x / 32 < P;
    uint64_t *full0 = (uint64_t *)(sm + P * stages * box);
    uint64_t *full = full0 + pid * 16;
    uint64_t *empty = full + 8;
    sm += pid * stages * box;
    if (threadIdx.x % 32 == 0 && is_prod) {
        for (int s = 0; s < stages; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    long long t0 = clock64();
    if (is_prod && threadIdx.x % 32 == 0) {
        uint32_t st = 0, ph = 0;
        int row = (blockIdx.x * 977 + pid * 131) * rows % (total_rows - rows * nb);
        for (int i = 0; i < iters; ++i) {
            wait_any(&empty[st], ph ^ 1, warpmode);
            
            if (threadIdx.x % 32 == 0) {
            ptx::mbar_arrive_expect_tx(&full[st], box);
            row += rows * nb;
            if (row + rows * nb > total_rows) row = 0;
            for (int j = 0; j < nb; ++j)
                ptx::tma_load_2d(sm + st * box + j * rows * 128, &tm, &full[st], 0, row + j * rows);
            }
            
            if (++st == (uint32_t)stages) { st = 0; ph ^= 1; }
        }
    } else if (!is_prod && threadIdx.x % 32 == 0) {
        uint32_t st = 0, ph = 0;
        for (int i = 0; i < iters; ++i) {
            wait_any(&full[st], ph, warpmode);
            
            if (threadIdx.x % 32 == 0) ptx::mbar_arrive(&empty[st]);
            if (++st == (uint32_t)stages) { st = 0; ph ^= 1; }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

int main(int argc, char **argv) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long long total_rows = 1 << 16;            // 8 MB of 128-byte rows (L2 resident)
    void *buf;
    cudaMalloc(&buf, total_rows * 128);
    cudaMemset(buf, 1, total_rows * 128);
    unsigned long long *cyc;
    cudaMalloc(&cyc, sms * 8);
    void *fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (CUresult(*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fn;
    cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    printf("rows stages grid  GB/s   B/clk/SM(at %s)\n", "clock64");
    for (int wm : {0})
    for (int P : {1, 2, 4})
    for (int nb : {1})
    for (int rows : {64, 128, 256}) {
        for (int stages : {2, 4, 6}) {
            if ((size_t)P * stages * rows * 128 * nb + 4096 > 227 * 1024) continue;
            for (int grid : {sms}) {
                CUtensorMap tm;
                cuuint64_t dims[2] = {64, (cuuint64_t)total_rows};
                cuuint64_t str[1] = {128};
                cuuint32_t boxd[2] = {64, (cuuint32_t)rows};
                cuuint32_t es[2] = {1, 1};
                enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                int iters = 4000;
                size_t smem = 1024 + P * stages * rows * 128 * nb + 1024;
                tma_stream<<<grid, 64 * P, smem>>>(tm, stages, rows, 200, total_rows, cyc, nb, wm);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                tma_stream<<<grid, 64 * P, smem>>>(tm, stages, rows, iters, total_rows, cyc, nb, wm);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                std::vector<unsigned long long> c(grid);
                cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
                double avgc = 0;
                for (auto v : c) avgc += v;
                avgc /= grid;
                double bytes = (double)grid * iters * rows * 128 * nb * P;
                printf("wm=%d P=%d nb=%d %4d %6d %4d %7.0f %8.1f   err=%s\n", wm, P, nb, rows, stages, grid, bytes / ms / 1e6,
                       (double)iters * rows * 128 * nb * P / avgc, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
