// %globaltimer update granularity (dev tool): one thread spins reading it and
// records the first 16 distinct values' deltas and the clock64 cycles between.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long *o) {
    unsigned long long prev, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
    long long c0 = clock64();
    int n = 0;
    while (n < 16) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t != prev) { long long c = clock64(); o[2 * n] = t - prev; o[2 * n + 1] = c - c0; c0 = c; prev = t; ++n; }
    }
}
int main() {
    unsigned long long *o, h[32];
    cudaMalloc(&o, 256);
    for (int r = 0; r < 2; ++r) k<<<1, 1>>>(o);
    cudaMemcpy(h, o, 256, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 16; ++i) printf("delta %llu ns, %llu cycles\n", h[2 * i], h[2 * i + 1]);
    return 0;
}
