// tcgen05.mma issue rate from shared-memory operands (DESIGN.md finding 17): one thread per CTA
// issues K blocks of 4 x (128 x N x 16) bf16 MMAs (nsub = 2: two 128-row MMAs sharing B, as
// BLOCK_M 256) from a 2-stage operand ring, with or without concurrent TMA writes into other
// shared memory (3 threads streaming 16 KB tiled boxes from an L2-resident buffer). Reports
// clocks per K block vs the 8192 FLOP/clk/SM dense peak.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2008_04567_b200/csrc mma_rate.cu -lcuda -o mma_rate
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

__global__ void __launch_bounds__(192, 1) mma_rate(const __grid_constant__ CUtensorMap tm, int n, int nsub, int iters,
                                                  int tma_threads, int mode, long long rows, unsigned long long *out,
                                                  unsigned long long *tma_bytes) {
    extern __shared__ uint8_t smraw[];
    uint8_t *sm = smraw + ((1024 - (ptx::smem_u32(smraw) & 1023)) & 1023);
    const uint32_t a_bytes = (uint32_t)nsub * 16384u, b_bytes = (uint32_t)n * 128u;
    const uint32_t stage = a_bytes + b_bytes;
    uint8_t *tbuf = sm + 2 * stage;                                // TMA region: 3 threads x 2 x 16 KB
    uint64_t *bars = reinterpret_cast<uint64_t *>(tbuf + 6 * 16384);
    uint64_t *done = bars;                                         // MMA completion
    uint64_t *tfull = bars + 1;                                    // [6]
    uint32_t *holder = reinterpret_cast<uint32_t *>(bars + 8);
    volatile int *stop = reinterpret_cast<volatile int *>(bars + 9);
    uint64_t *ring = bars + 10;                                    // [2] per-K-block commit targets
    uint64_t *ready = bars + 12;                                   // completed barrier (mode 2)
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tm);
        ptx::mbar_init(done, 1);
        for (int i = 0; i < 6; ++i) ptx::mbar_init(&tfull[i], 1);
        ptx::mbar_init(&ring[0], 1);
        ptx::mbar_init(&ring[1], 1);
        ptx::mbar_init(ready, 1);
        *stop = 0;
        ptx::fence_mbar_init();
        ptx::mbar_arrive(ready);   // phase 0 complete
    }
    if (warp == 1) {
        ptx::tmem_alloc(holder, 512);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *holder;
    if (warp == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t a0 = ptx::sw128_kmajor_desc(ptx::smem_u32(sm));
        const uint64_t b0 = ptx::sw128_kmajor_desc(ptx::smem_u32(sm + a_bytes));
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (mode >= 2) {   // the kernel's per-K-block wait on a (complete) full barrier
                ptx::mbar_wait(ready, 0);
                ptx::tc_fence_after();
            }
            const uint32_t st = (uint32_t)(i & 1) * stage;
            const uint64_t ad = a0 + (st >> 4), bd = b0 + (st >> 4);
            if (elect_one()) {
                for (int h = 0; h < nsub; ++h)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        ptx::umma<false>(tmem + h * n, ad + h * (16384 >> 4) + 2 * kk, bd + 2 * kk, idesc, (i | kk) ? 1u : 0u);
                if (mode >= 1) ptx::umma_commit(&ring[i & 1]);   // the kernel frees each stage by a commit
            }
            __syncwarp();
        }
        if (elect_one()) ptx::umma_commit(done);
        __syncwarp();
        ptx::mbar_wait(done, 0);
        if (lane == 0) {
            out[blockIdx.x] = clock64() - t0;
            *stop = 1;
        }
    } else if (warp >= 2 && warp < 2 + tma_threads && lane == 0) {
        const int t = warp - 2;
        unsigned long long bytes = 0;
        long long m = ((long long)blockIdx.x * 997 * 128 + t * 40000) % (rows - 128);
        uint32_t ph[2] = {0, 0};
        int i = 0;
        for (; !*stop; ++i) {
            const int s = i & 1;
            if (i >= 2) {
                ptx::mbar_wait(&tfull[2 * t + s], ph[s]);
                ph[s] ^= 1;
                bytes += 16384;
            }
            ptx::mbar_arrive_expect_tx(&tfull[2 * t + s], 16384);
            ptx::tma_load_2d(tbuf + (size_t)(2 * t + s) * 16384, &tm, &tfull[2 * t + s], 0, (int)m);
            m += 128;
            if (m + 128 > rows) m = 0;
        }
        for (int k = 0; k < 2 && k < i; ++k) {   // drain
            const int s = (i - 1 - k) & 1;
            ptx::mbar_wait(&tfull[2 * t + s], ph[s]);
            ph[s] ^= 1;
        }
        atomicAdd(tma_bytes + blockIdx.x, bytes);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

typedef CUresult (*EncT)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                         const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                         CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    void *f1 = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f1, cudaEnableDefault, &q) != cudaSuccess || !f1) {
        printf("no tensor-map encoder (no GPU?)\n");
        return 1;
    }
    EncT enc = (EncT)f1;
    cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    unsigned long long *out, *tb;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&tb, 1024 * 8);
    const long long rows = (16 << 20) / 128;   // 16 MB of 128-byte rows, L2-resident
    void *buf;
    cudaMalloc(&buf, rows * 128);
    cudaMemset(buf, 0, rows * 128);
    CUtensorMap tm;
    cuuint64_t d[2] = {64, (cuuint64_t)rows};
    cuuint64_t s[1] = {128};
    cuuint32_t b[2] = {64, 128};
    cuuint32_t e[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("%-5s %-5s %-4s %-5s %-6s %10s %10s %10s\n", "N", "nsub", "tma", "mode", "grid", "clk/kblk", "%peak", "tmaB/clk");
    for (int n : {64, 128, 256})
        for (int nsub : {1, 2})
            for (int tt : {0, 3})
              for (int mode : {0, 1, 2})
                for (int grid : {148}) {
                    const int iters = 2000;
                    const size_t smem = 2 * ((size_t)nsub * 16384 + n * 128) + 6 * 16384 + 256 + 1024;
                    if (smem > 227 * 1024) continue;
                    cudaMemset(tb, 0, 1024 * 8);
                    mma_rate<<<grid, 192, smem>>>(tm, n, nsub, iters, tt, mode, rows, out, tb);
                    cudaError_t err = cudaDeviceSynchronize();
                    std::vector<unsigned long long> o(grid), t(grid);
                    cudaMemcpy(o.data(), out, grid * 8, cudaMemcpyDeviceToHost);
                    cudaMemcpy(t.data(), tb, grid * 8, cudaMemcpyDeviceToHost);
                    double avg = 0, tbytes = 0;
                    for (int i = 0; i < grid; ++i) {
                        avg += o[i];
                        tbytes += t[i];
                    }
                    avg /= grid;
                    tbytes /= grid;
                    const double clk = avg / iters;
                    const double ideal = (double)nsub * 128 * n * 64 * 2 / 8192.0;
                    printf("%-5d %-5d %-4d %-5d %-6d %10.1f %10.1f %10.1f %s\n", n, nsub, tt, mode, grid, clk, 100.0 * ideal / clk,
                           tbytes / avg, err == cudaSuccess ? "" : cudaGetErrorString(err));
                }
    return 0;
}
