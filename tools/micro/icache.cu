// Instruction-fetch cost of cold straight-line code (dev tool): a kernel whose
// body is N unrolled dependent-free FMA chains, run once by 32 blocks.
#include <cstdio>
#include <cuda_runtime.h>
template <int NI>
__global__ void straight(float *out, long long *cyc) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        a0 = fmaf(a0, 1.0001f, 0.5f); a1 = fmaf(a1, 0.9999f, 0.25f);
        a2 = fmaf(a2, 1.0002f, 0.125f); a3 = fmaf(a3, 0.9998f, 0.0625f);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
template <int NI>
void run(float *out, long long *cyc) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        straight<NI><<<32, 256>>>(out, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("NI=%d (%d FMA instrs, %d KB code) rep %d: %.2f us\n", NI, 4 * NI, 4 * NI * 16 / 1024, rep, ms * 1e3);
    }
}
int main() {
    float *out; long long *cyc;
    cudaMalloc(&out, 32 * 256 * 4); cudaMalloc(&cyc, 32 * 8);
    run<256>(out, cyc);
    run<1024>(out, cyc);
    run<4096>(out, cyc);
    return 0;
}
