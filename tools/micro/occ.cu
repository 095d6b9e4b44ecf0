// Occupancy probe: blocks/SM for 288-thread (9-warp) blocks vs register cap.
#include <cstdio>
template <int NR>
__global__ void __maxnreg__(NR) k(float *o, int n) {
    float a[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) a[i] = o[i * n + threadIdx.x];
    for (int it = 0; it < n; ++it)
#pragma unroll
        for (int i = 0; i < 64; ++i) a[i] = a[i] * a[(i + 1) & 63] + 1.f;
    float s = 0;
#pragma unroll
    for (int i = 0; i < 64; ++i) s += a[i];
    o[threadIdx.x] = s;
}
template <int NR> void probe() {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k<NR>);
    for (int thr : {256, 288, 320, 384}) {
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k<NR>, thr, 0);
        printf("maxnreg %3d (uses %3d): %d threads -> %d blocks/SM\n", NR, fa.numRegs, thr, o);
    }
}
template <int NR> void probe_smem(int maxdyn, int carve) {
    cudaFuncSetAttribute(k<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxdyn);
    if (carve >= 0) cudaFuncSetAttribute(k<NR>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    for (int dyn : {0, 65536, 90240}) {
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k<NR>, 288, dyn);
        printf("maxnreg %3d maxdyn %d carve %d: 288 threads, dyn %d -> %d blocks/SM\n", NR, maxdyn, carve, dyn, o);
    }
}
int main() {
    probe_smem<104>(90240, -1);
    probe_smem<104>(90240, 100);
    probe<64>(); probe<72>(); probe<80>(); probe<88>(); probe<96>(); probe<104>(); probe<112>();
    return 0;
}
