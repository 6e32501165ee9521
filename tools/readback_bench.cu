// How fast can ONE CTA (256 threads) read back a 512 KB fp32 region (4 splits x 128 rows x 256 cols
// of a [S][M][K] buffer) right after other SMs wrote it, vs. when it was written long ago?
#include <cuda_runtime.h>
#include <cstdio>
__global__ void writer(float *p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 1.0f;
}
__global__ void reader(const float *p, long long MK, int K, int S, int U, float *out, long long *cyc) {
    long long t0 = clock64();
    float acc = 0.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int items = 128 * 2;   // 128 rows x 2 blocks of 128 columns
    for (int base = warp; base < items; base += 8 * U) {
        float4 a[8];
        for (int u = 0; u < U; ++u) a[u] = make_float4(0, 0, 0, 0);
        for (int sp = 0; sp < S; ++sp) {
#pragma unroll 8
            for (int u = 0; u < U; ++u) {
                const int item = base + u * 8;
                if (item >= items) continue;
                const int r = item / 2, cb = item % 2;
                const float4 q = __ldcg(reinterpret_cast<const float4 *>(p + sp * MK + (long long)r * K + cb * 128 + lane * 4));
                a[u].x += q.x; a[u].y += q.y; a[u].z += q.z; a[u].w += q.w;
            }
        }
        for (int u = 0; u < U; ++u) acc += a[u].x + a[u].y + a[u].z + a[u].w;
    }
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) *cyc = clock64() - t0;
}
int main() {
    const int S = 4, M = 6272, K = 256;
    const long long MK = (long long)M * K;
    float *p, *out; long long *cyc;
    cudaMalloc(&p, S * MK * 4); cudaMalloc(&out, 1024 * 4); cudaMalloc(&cyc, 8);
    for (int U : {1, 4, 8}) {
        for (int fresh : {1, 0}) {
            writer<<<1184, 256>>>(p, S * MK);
            cudaDeviceSynchronize();
            if (!fresh) { float *q; cudaMalloc(&q, 512 << 20); writer<<<1184, 256>>>(q, (512 << 20) / 4); cudaDeviceSynchronize(); cudaFree(q); }
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            reader<<<1, 256>>>(p, MK, K, S, U, out, cyc);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("U=%d fresh=%d: %.1f us (%lld cycles) %s\n", U, fresh, ms * 1e3, c, cudaGetErrorString(cudaGetLastError()));
        }
    }
}
