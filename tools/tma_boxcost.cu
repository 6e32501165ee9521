// Per-box cost of the TMA engine (DESIGN.md finding 17): one thread per CTA streams boxes of one
// kind into a ring of shared-memory stages (a consumer thread frees them), L2-resident source.
// Kinds: tiled 2-D {64 bf16, rows}; tiled 3-D {64, rows, kb} over a [K/64][M][64] view of an M x K
// matrix (kb K-blocks per instruction); im2col 4-D (pixels x 64 channels, 3x3 taps cycling); tiled
// 4-D {64, bw, bh, 1} over NHWC with tap offsets (zero fill at the borders).
// Reported: ns per box, bytes per SM clock, for 148 and 32 active CTAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2008_04567_b200/csrc tma_boxcost.cu -lcuda -o tma_boxcost
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace wpk;

__device__ __forceinline__ void tma_load_4d(void *smem, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(ptx::smem_u32(smem)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

struct P {
    int kind;        // 0 tiled2d, 1 tiled3d, 2 im2col, 3 tiled4d
    int rows;        // rows / pixels per box (kind 0-2); bw (kind 3)
    int kb;          // K blocks per box (kind 1); bh (kind 3)
    int box_bytes;
    int stages;
    int iters;
    int img, nimg;   // NHWC geometry for kinds 2, 3 (C = 64)
    int mrows;       // rows of the 2-D / 3-D views
    int bps;         // boxes per stage (one mbarrier)
    int npairs;      // independent producer/consumer pairs (rings) per CTA
    int spin;        // consumer/producer spin on test_wait instead of the suspending try_wait
};

__device__ __forceinline__ void wait_bar(uint64_t *bar, uint32_t ph, int spin) {
    if (spin) {
        while (!ptx::mbar_test_wait(bar, ph)) {
        }
    } else {
        while (!ptx::mbar_try_wait(bar, ph)) {
        }
    }
}

__global__ void __launch_bounds__(256, 1) feed(const __grid_constant__ CUtensorMap tm, P p,
                                             unsigned long long *cycles) {
    extern __shared__ uint8_t smraw[];
    uint8_t *sm = smraw + ((1024 - (ptx::smem_u32(smraw) & 1023)) & 1023);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int pair = warp / 2;
    const size_t ring = (size_t)p.stages * p.box_bytes * p.bps;
    uint64_t *full0 = reinterpret_cast<uint64_t *>(sm + ring * p.npairs);
    uint64_t *full = full0 + pair * 32;
    uint64_t *empty = full + 16;
    sm += ring * pair;
    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tm);
        for (int s = 0; s < 32 * p.npairs; ++s) ptx::mbar_init(&full0[s], 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    if (pair < p.npairs && warp % 2 == 0 && lane == 0) {
        uint32_t st = 0, ph = 0;
        int m = (int)(((long long)blockIdx.x * 7919 * 128) % (p.mrows - 256));
        int tap = 0, kblk = 0;
        const int pq = p.img * p.img;
        for (int i = 0; i < p.iters; ++i) {
            wait_bar(&empty[st], ph ^ 1, p.spin);
            ptx::mbar_arrive_expect_tx(&full[st], p.box_bytes * p.bps);
            for (int bx = 0; bx < p.bps; ++bx) {
            uint8_t *dst = sm + ((size_t)st * p.bps + bx) * p.box_bytes;
            if (p.kind == 0) {
                ptx::tma_load_2d(dst, &tm, &full[st], kblk * 64, m);
            } else if (p.kind == 1) {
                ptx::tma_load_3d(dst, &tm, &full[st], 0, m, kblk);
            } else if (p.kind == 2) {
                const int n = m / pq, rem = m % pq, pp = rem / p.img, q = rem % p.img;
                ptx::tma_load_im2col_4d(dst, &tm, &full[st], 0, q - 1, pp - 1, n, (uint16_t)(tap % 3),
                                        (uint16_t)(tap / 3));
            } else {
                const int n = (m / pq) % p.nimg;
                const int y0 = ((m % pq) / p.img / p.kb) * p.kb, x0 = 0;
                tma_load_4d(dst, &tm, &full[st], 0, x0 + tap % 3 - 1, y0 + tap / 3 - 1, n);
            }
            if (p.kind == 2 || p.kind == 3) {
                if (++tap == 9) {
                    tap = 0;
                    m += p.kind == 2 ? p.rows : p.rows * p.kb;
                }
            } else {
                kblk += (p.kind == 1 ? p.kb : 1);
                if (kblk >= 8) {
                    kblk = 0;
                    m += p.rows;
                }
            }
            if (m + 1024 > p.mrows) m = 0;
            }
            if (++st == (uint32_t)p.stages) { st = 0; ph ^= 1; }
        }
    } else if (pair < p.npairs && warp % 2 == 1 && lane == 0) {
        uint32_t st = 0, ph = 0;
        for (int i = 0; i < p.iters; ++i) {
            wait_bar(&full[st], ph, p.spin);
            ptx::mbar_arrive(&empty[st]);
            if (++st == (uint32_t)p.stages) { st = 0; ph ^= 1; }
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
    const size_t bytes = 16u << 20;   // L2-resident
    void *buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    const int K = 512;                 // 2-D / 3-D views: M x 512 bf16 (1 KB rows)
    const int mrows = (int)(bytes / (K * 2));
    printf("%-8s %-5s %-4s %-7s %-6s %-5s %8s %9s %9s\n", "kind", "rows", "kb", "bytes", "stages", "grid", "GB/s",
           "B/clk/SM", "ns/box");
    struct V { int kind, rows, kb, bps, npairs, spin, stages, grid; };
    std::vector<V> vs;
    for (int kind : {0, 2})
        for (int spin : {0, 1}) {
            vs.push_back({kind, 128, 1, 1, 1, spin, 8, 148});
            vs.push_back({kind, 128, 1, 2, 1, spin, 4, 148});
            vs.push_back({kind, 128, 1, 4, 1, spin, 2, 148});
            vs.push_back({kind, 64, 1, 4, 1, spin, 4, 148});
            vs.push_back({kind, 128, 1, 1, 2, spin, 4, 148});
            vs.push_back({kind, 128, 1, 1, 4, spin, 2, 148});
            vs.push_back({kind, 64, 1, 1, 4, spin, 4, 148});
            vs.push_back({kind, 128, 1, 1, 1, spin, 4, 296});
        }
    const int img = 28, nimg = (int)(bytes / (128ull * img * img));
    printf("%-8s %-5s %-4s %-4s %-6s %-4s %-6s %-5s %8s %9s %9s\n", "kind", "rows", "bps", "pairs", "spin", "stg",
           "bytes", "grid", "GB/s", "B/clk/SM", "ns/box");
    for (auto v : vs) {
        CUtensorMap tm;
        CUresult r;
        P p{};
        p.kind = v.kind;
        p.rows = v.rows;
        p.kb = v.kb;
        p.img = img;
        p.nimg = nimg;
        p.bps = v.bps;
        p.npairs = v.npairs;
        p.spin = v.spin;
        p.stages = v.stages;
        p.mrows = v.kind >= 2 ? nimg * img * img : mrows;
        cuuint32_t e4[4] = {1, 1, 1, 1};
        if (v.kind == 0) {
            cuuint64_t d[2] = {(cuuint64_t)K, (cuuint64_t)mrows};
            cuuint64_t s[1] = {(cuuint64_t)K * 2};
            cuuint32_t b[2] = {64, (cuuint32_t)v.rows};
            r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d, s, b, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t d[4] = {64, (cuuint64_t)img, (cuuint64_t)img, (cuuint64_t)nimg};
            cuuint64_t s[3] = {128, 128ull * img, 128ull * img * img};
            int lo[2] = {-1, -1}, hi[2] = {-1, -1};
            r = enci(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, d, s, lo, hi, 64, (cuuint32_t)v.rows, e4,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        p.box_bytes = v.rows * 128;
        if (r != CUDA_SUCCESS) {
            printf("encode failed %d\n", (int)r);
            continue;
        }
        const size_t smem = (size_t)v.stages * p.box_bytes * v.bps * v.npairs + 32 * 8 * v.npairs + 2048;
        if (smem > (v.grid > 148 ? 113 : 227) * 1024) {
            printf("skip (smem %zu)\n", smem);
            continue;
        }
        p.iters = 20;
        feed<<<v.grid, 256, smem>>>(tm, p, cyc);
        p.iters = 3000 / v.bps;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        feed<<<v.grid, 256, smem>>>(tm, p, cyc);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double boxes = (double)p.iters * v.bps * v.npairs * v.grid;
        const double sms = v.grid > 148 ? 148 : v.grid;
        printf("%-8s %-5d %-4d %-4d %-6d %-4d %-6d %-5d %8.0f %9.1f %9.1f %s\n", v.kind ? "im2col" : "tiled2d", v.rows,
               v.bps, v.npairs, v.spin, v.stages, p.box_bytes, v.grid, boxes * p.box_bytes / (ms * 1e-3) / 1e9,
               boxes * p.box_bytes / sms / (ms * 1e-3 * 1.965e9), ms * 1e6 / (boxes / sms),
               err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
    return 0;
}
