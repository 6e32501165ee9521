// Issue N TMA loads back-to-back from one thread (each to its own mbarrier), record when each lands.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "ptx.cuh"
using namespace wpk;
__global__ void k(const __grid_constant__ CUtensorMap tm, int n, int rows, long long *out) {
    extern __shared__ uint8_t smraw[];
    uint32_t base = ptx::smem_u32(smraw);
    uint8_t *sm = smraw + ((1024 - (base & 1023)) & 1023);
    uint64_t *bar = (uint64_t *)(sm + n * rows * 128);
    if (threadIdx.x == 0) {
        for (int i = 0; i < n; ++i) ptx::mbar_init(&bar[i], 1);
        ptx::fence_mbar_init();
        long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
            ptx::mbar_arrive_expect_tx(&bar[i], rows * 128);
            ptx::tma_load_2d(sm + i * rows * 128, &tm, &bar[i], 0, (blockIdx.x * n + i) * rows);
        }
        long long t1 = clock64();
        for (int i = 0; i < n; ++i) {
            while (!ptx::mbar_try_wait(&bar[i], 0)) {}
            out[blockIdx.x * 40 + i] = clock64() - t0;
        }
        out[blockIdx.x * 40 + 39] = t1 - t0;
    }
}
int main() {
    void *buf; cudaMalloc(&buf, 64 << 20); cudaMemset(buf, 1, 64 << 20);
    long long *out; cudaMalloc(&out, 148 * 40 * 8);
    void *fn; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (CUresult(*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fn;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (int rows : {64, 128}) for (int grid : {1, 148}) {
        CUtensorMap tm; cuuint64_t dims[2] = {64, (64 << 20) / 128}; cuuint64_t str[1] = {128};
        cuuint32_t box[2] = {64, (cuuint32_t)rows}; cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        int n = 8;
        for (int rep = 0; rep < 3; ++rep) k<<<grid, 32, n * rows * 128 + 2048>>>(tm, n, rows, out);
        cudaDeviceSynchronize();
        long long h[40]; cudaMemcpy(h, out, 40 * 8, cudaMemcpyDeviceToHost);
        printf("rows=%d grid=%d issue=%lld land:", rows, grid, h[39]);
        for (int i = 0; i < n; ++i) printf(" %lld", h[i]);
        printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
    }
}
