// Latency micro-benchmarks for the small dense algebra in K2 (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float warp_sum(float v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ void warp_vecmat(const float *v, const float *S, int n, int ld, float *y) {
    const int lane = threadIdx.x & 31;
    for (int j = lane; j < n; j += 32) {
        float acc0 = 0.f, acc1 = 0.f;
        int i = 0;
        for (; i + 1 < n; i += 2) {
            acc0 = fmaf(v[i], S[i * ld + j], acc0);
            acc1 = fmaf(v[i + 1], S[(i + 1) * ld + j], acc1);
        }
        y[j] = acc0 + acc1;
    }
    __syncwarp();
}
__global__ void k(float *out, long long *cyc, int n, const float *g) {
    __shared__ float S[32 * 36], v[32], y[32];
    __shared__ float b0[32 * 36], b1[32 * 36];
    for (int e = threadIdx.x; e < 32 * 36; e += blockDim.x) { S[e] = (e % 37) * 0.01f; b0[e] = (e % 37 == 0) ? 2.f : 0.01f; }
    if (threadIdx.x < 32) v[threadIdx.x] = threadIdx.x * 0.1f;
    __syncthreads();
    long long t0 = clock64();
    float acc = 0;
    if (threadIdx.x < 32) {
        for (int it = 0; it < 100; ++it) { warp_vecmat(v, S, n, 36, y); v[threadIdx.x] = y[threadIdx.x] * 0.5f; __syncwarp(); }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x < 32) for (int it = 0; it < 100; ++it) acc = warp_sum(acc + 1.f);
    __syncthreads();
    long long t2 = clock64();
    for (int it = 0; it < 100; ++it) __syncthreads();
    long long t3 = clock64();
    // dependent L2 loads
    float x = 0; int idx = 0;
    if (threadIdx.x == 0) for (int it = 0; it < 100; ++it) { x += __ldcg(g + idx); idx = ((int)x) & 1023; }
    __syncthreads();
    long long t4 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / 100; cyc[1] = (t2 - t1) / 100; cyc[2] = (t3 - t2) / 100; cyc[3] = (t4 - t3) / 100;
        out[0] = acc + x + y[0];
    }
}
int main() {
    float *out, *g; long long *cyc, h[4];
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 64); cudaMalloc(&g, 4096 * 4); cudaMemset(g, 0, 4096 * 4);
    for (int rep = 0; rep < 3; ++rep) k<<<1, 256>>>(out, cyc, 32, g);
    cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    printf("vecmat32 %lld cyc, warp_sum %lld cyc, syncthreads %lld cyc, L2 dep load %lld cyc\n", h[0], h[1], h[2], h[3]);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock %d kHz\n", clk);
    return 0;
}
