// Micro-benchmark of the block-wide Gauss-Jordan used by K2 (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kCompressThreads = 256;
template <int E>
__device__ bool block_gj_t(float *M, int R, int ld, float *s_rc) {
    const int tid = threadIdx.x;
    const int e0 = tid * E;
    const bool act = e0 < R * R;
    const int i = act ? e0 / R : 0, c0 = act ? e0 - (e0 / R) * R : 0;
    float own[E];
#pragma unroll
    for (int e = 0; e < E; ++e) own[e] = act ? M[i * ld + c0 + e] : 0.f;
    __syncthreads();
    for (int k = 0; k < R; ++k) {
        float *rowb = s_rc + (k & 1) * 128;
        float *colb = rowb + 64;
        if (act) {
            if (i == k) {
#pragma unroll
                for (int e = 0; e < E; ++e) rowb[c0 + e] = own[e];
            }
#pragma unroll
            for (int e = 0; e < E; ++e)
                if (c0 + e == k) colb[i] = own[e];
        }
        __syncthreads();
        const float p = rowb[k];
        if (!(p > 0.f) || !isfinite(p)) return false;
        if (act) {
            const float ip = __frcp_rn(p);
            const float f = colb[i] * ip;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int j = c0 + e;
                const float piv = rowb[j];
                if (i == k) own[e] = (j == k) ? ip : own[e] * ip;
                else own[e] = (j == k) ? -f : fmaf(-f, piv, own[e]);
            }
        }
    }
    if (act) for (int e = 0; e < E; ++e) M[i * ld + c0 + e] = own[e];
    __syncthreads();
    return true;
}
__global__ void k(float *out, long long *cyc, int R) {
    __shared__ float M[64 * 68], s_rc[256];
    const int ld = R + 4;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) M[(e / R) * ld + e % R] = (e / R == e % R) ? 4.f : 0.01f;
    __syncthreads();
    long long t0 = clock64();
    bool ok = block_gj_t<4>(M, R, ld, s_rc);
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = M[0] + ok; }
}
int main() {
    float *out; long long *cyc, h[2];
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 64);
    for (int rep = 0; rep < 3; ++rep) k<<<1, 256>>>(out, cyc, 32);
    cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
    printf("block_gj R=32: %lld cycles\n", h[0]);
    return 0;
}
