// Calibration: %globaltimer vs clock64, dependent L2 / DRAM load latency,
// and a 512-thread block's dependent-load phase, from inside a kernel (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(const unsigned *g, size_t n, unsigned long long *o) {
    __shared__ unsigned s;
    unsigned long long t0 = gt(); long long c0 = clock64();
    unsigned idx = threadIdx.x;
    // 64 dependent loads, stride that walks a large buffer (DRAM)
    for (int i = 0; i < 64; ++i) idx = __ldcg(g + ((size_t)idx * 2654435761u) % n) + threadIdx.x;
    __syncthreads();
    unsigned long long t1 = gt(); long long c1 = clock64();
    // 64 dependent loads in a small buffer (L2 hits after first touch)
    unsigned j = threadIdx.x;
    for (int i = 0; i < 64; ++i) j = __ldcg(g + (j & 4095)) + threadIdx.x;
    __syncthreads();
    unsigned long long t2 = gt(); long long c2 = clock64();
    for (int i = 0; i < 1000; ++i) __syncthreads();
    unsigned long long t3 = gt(); long long c3 = clock64();
    if (threadIdx.x == 0) { s = idx + j; o[0] = t1 - t0; o[1] = c1 - c0; o[2] = t2 - t1; o[3] = c2 - c1; o[4] = t3 - t2; o[5] = c3 - c2; o[6] = s; }
}
int main1() {
    size_t n = (size_t)1 << 28;  // 1 GiB of uint32
    unsigned *g; unsigned long long *o, h[8];
    cudaMalloc(&g, n * 4); cudaMemset(g, 0, n * 4); cudaMalloc(&o, 64);
    for (int blocks : {1, 148, 296}) {
        for (int rep = 0; rep < 3; ++rep) k<<<blocks, 512>>>(g, n, o);
        cudaDeviceSynchronize();
        cudaMemcpy(h, o, 56, cudaMemcpyDeviceToHost);
        printf("blocks=%d: 64 dep DRAM loads %.2f us (%lld cyc) | 64 dep L2 loads %.2f us (%lld cyc) | 1000 syncthreads(512) %.2f us (%lld cyc)\n",
               blocks, h[0] / 1e3, h[1], h[2] / 1e3, h[3], h[4] / 1e3, h[5]);
    }
    return 0;
}
// globaltimer read cost
__global__ void kg(unsigned long long *o) {
    long long c0 = clock64();
    unsigned long long s = 0;
    for (int i = 0; i < 100; ++i) s += gt();
    long long c1 = clock64();
    if (threadIdx.x == 0) { o[0] = (c1 - c0) / 100; o[1] = s; }
}
int main2() {
    unsigned long long *o, h[2];
    cudaMalloc(&o, 16);
    for (int r = 0; r < 3; ++r) kg<<<1, 32>>>(o);
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("globaltimer read: %llu cycles\n", h[0]);
    return 0;
}
int main() { main1(); return main2(); }
