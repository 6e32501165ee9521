// The conv kernel's stage ring without data (DESIGN.md finding 17): a producer warp (elected lane)
// waits for a stage to be freed and arrives on its "full" barrier (no TMA); the MMA warp waits
// "full", issues 4 x (128 x N x 16) (nsub x) bf16 MMAs and frees the stage with tcgen05.commit.
// Measures clocks per K block for STAGES and wait flavours (suspending try_wait / spinning
// test_wait), i.e. what the synchronisation alone costs next to the MMAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2008_04567_b200/csrc mma_ring.cu -o mma_ring
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace wpk;

__device__ __forceinline__ void wait_flavour(uint64_t *bar, uint32_t ph, int spin) {
    if (spin) {
        while (!ptx::mbar_test_wait(bar, ph)) {
        }
    } else {
        ptx::mbar_wait(bar, ph);
    }
}

__global__ void __launch_bounds__(384, 1) ring(int n, int nsub, int stages, int iters, int spin, int no_wait_mma,
                                              int waiters, unsigned long long *out) {
    extern __shared__ uint8_t smraw[];
    uint8_t *sm = smraw + ((1024 - (ptx::smem_u32(smraw) & 1023)) & 1023);
    const uint32_t a_bytes = (uint32_t)nsub * 16384u, b_bytes = (uint32_t)n * 128u;
    const uint32_t stage_bytes = a_bytes + b_bytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + 2 * stage_bytes);
    uint64_t *full = bars, *empty = bars + 16, *done = bars + 32;
    uint32_t *holder = reinterpret_cast<uint32_t *>(bars + 33);
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(done, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) {
        ptx::tmem_alloc(holder, 512);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *holder;
    const long long t0 = clock64();
    if (warp == 0 && no_wait_mma != 2) {
        for (int g = 0; g < iters; ++g) {
            const uint32_t st = (uint32_t)(g % stages), ph = (uint32_t)((g / stages) & 1);
            if (g >= stages) wait_flavour(&empty[st], ph ^ 1u, spin);
            if (ptx::elect_one()) ptx::mbar_arrive(&full[st]);
            __syncwarp();
        }
    } else if (warp == 1) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t a0 = ptx::sw128_kmajor_desc(ptx::smem_u32(sm));
        const uint64_t b0 = ptx::sw128_kmajor_desc(ptx::smem_u32(sm + a_bytes));
        long long t_issue = 0, t_wait = 0;
        if (no_wait_mma == 2) {   // constant operands: the loop body is 4 (8) UTCHMMA, nothing else
            const long long ti0 = clock64();
            if (ptx::elect_one()) {
                for (int g = 0; g < iters; ++g) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        ptx::umma<false>(tmem, a0 + 2 * kk, b0 + 2 * kk, idesc, 1u);
                        if (nsub == 2) ptx::umma<false>(tmem + n, a0 + 1024 + 2 * kk, b0 + 2 * kk, idesc, 1u);
                    }
                }
            }
            __syncwarp();
            t_issue = clock64() - ti0;
        } else
        for (int g = 0; g < iters; ++g) {
            const uint32_t st = (uint32_t)(g % stages), ph = (uint32_t)((g / stages) & 1);
            const long long tw0 = clock64();
            if (!no_wait_mma) {
                wait_flavour(&full[st], ph, spin);
                ptx::tc_fence_after();
            }
            const uint32_t so = (uint32_t)(g & 1) * stage_bytes;   // operands: 2 buffers (data irrelevant)
            const uint64_t ad = a0 + (so >> 4), bd = b0 + (so >> 4);
            const long long ti0 = clock64();
            t_wait += ti0 - tw0;
            if (ptx::elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    for (int h = 0; h < nsub; ++h)
                        ptx::umma<false>(tmem + h * n, ad + h * (16384 >> 4) + 2 * kk, bd + 2 * kk, idesc, (g | kk) ? 1u : 0u);
                ptx::umma_commit(&empty[st]);
            }
            __syncwarp();
            t_issue += clock64() - ti0;
        }
        if (ptx::elect_one()) ptx::umma_commit(done);
        __syncwarp();
        ptx::mbar_wait(done, 0);
        if (threadIdx.x == 32) {
            out[blockIdx.x] = clock64() - t0;
            out[256 + blockIdx.x] = t_issue;
            out[512 + blockIdx.x] = t_wait;
        }
    }
    else if (warp >= 4 && warp < 4 + waiters) {
        // the kernel's 8 epilogue warps wait on the first accumulator meanwhile (mbar_wait: try_wait +
        // globaltimer watchdog); waiters < 0 selects a plain try_wait loop
        ptx::mbar_wait(done, 0);
    } else if (warp >= 4 && warp < 4 - waiters) {
        while (!ptx::mbar_try_wait(done, 0)) {
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    unsigned long long *out;
    cudaMalloc(&out, 1024 * 8);
    printf("%-5s %-5s %-6s %-8s %10s %8s %8s %8s\n", "N", "nsub", "stages", "waiters", "clk/kblk", "%peak", "issue", "wait");
    for (int n : {128, 256})
        for (int nsub : {1, 2})
            for (int waiters : {0, 8, -8}) {
                const int stages = 4, iters = 36 * 30;
                const size_t smem = 2 * ((size_t)nsub * 16384 + n * 128) + 1024 + 512;
                ring<<<148, 384, smem>>>(n, nsub, stages, iters, 0, 0, waiters, out);
                cudaError_t err = cudaDeviceSynchronize();
                std::vector<unsigned long long> o(768);
                cudaMemcpy(o.data(), out, 768 * 8, cudaMemcpyDeviceToHost);
                double avg = 0, ti = 0, tw = 0;
                for (int i = 0; i < 148; ++i) {
                    avg += o[i];
                    ti += o[256 + i];
                    tw += o[512 + i];
                }
                avg /= 148;
                ti /= 148.0 * iters;
                tw /= 148.0 * iters;
                const double clk = avg / iters, ideal = (double)nsub * 128 * n * 64 * 2 / 8192.0;
                printf("%-5d %-5d %-6d %-8d %10.1f %8.1f %8.1f %8.1f %s\n", n, nsub, stages, waiters, clk,
                       100.0 * ideal / clk, ti, tw, err == cudaSuccess ? "" : cudaGetErrorString(err));
            }
    return 0;
}
