// Microbenchmark of the gathered-row attention phase alone (development
// tool): 32 heads x P parts, each block attends ~S/P random ascending rows of
// its part from a 128K-row bf16 K/V/A store (C4 shapes), through
// attend_reduce_list (cp.async stages + online softmax + tensor-core Y|G) or
// straight register loads (attend_list).  Reports the kernel time and the
// per-block phase clock (first chunk in, end).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include "../../paper_2510_23649_b200/csrc/attend_common.cuh"

namespace lrqk {
__device__ int g_lrqk_trace_on = 0;
__device__ unsigned long long g_lrqk_trace[kTraceCap][2];
}
using namespace lrqk;
using T = __nv_bfloat16;

constexpr int kThr = 288;

template <int CR, int NS, int MODE, bool AROW = false, int YGM = 2, int PPH = 9>
__global__ void __maxnreg__(96) bench_kernel(lrqk_layer_t L, const int *rows_all, const int *nrows, int cap,
                                                    const T *q, float *parts, long long *clk) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ float s_m[9], s_l[9];
    int *s_rows = reinterpret_cast<int *>(smem + (PPH == 9 ? 90 : 42) * 1024);
    const int blk = blockIdx.x, h = blk / PPH, g = h / 4;
    const int n = nrows[blk];
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_rows[i] = rows_all[blk * cap + i];
    __syncthreads();
    long long t0 = clock64();
    const int lane = threadIdx.x & 31, sl = lane % 16;
    const T *kb = reinterpret_cast<const T *>(L.slow_k) + (size_t)g * L.t_max * 128;
    const T *vb = reinterpret_cast<const T *>(L.slow_v) + (size_t)g * L.t_max * 128;
    const T *proxy = reinterpret_cast<const T *>(L.proxy) + (size_t)h * L.t_max * 32;
    float qv[1][8];
    Pack<T>::load(q + (size_t)h * 128 + sl * 8, qv[0]);
    float m = -INFINITY, l = 0.f, acc[1][8] = {};
    float yacc[YGM > 0 ? YGM : 1][2][4] = {}, gacc[4][4] = {};
    const float c = 1.4426950408889634f * rsqrtf(128.f);
    if constexpr (MODE == 0)
        attend_reduce_list<T, 16, 1, YGM, CR, NS>(L, kb, vb, proxy, AROW ? proxy : nullptr, s_rows, n, qv, c, m, l, acc,
                                                  smem, yacc, gacc);
    else
        attend_list<T, 16, 1, 8>(kb, vb, s_rows, n, qv, c, 128, m, l, acc);
    long long t1 = clock64();
    float *s_acc = reinterpret_cast<float *>(smem);
    block_partial<T, 16, 1>(m, l, acc, 128, s_m, s_l, s_acc, parts + (size_t)blk * 130);
    if (MODE == 0) {
        float s = 0;
        for (int j = 0; j < 2; ++j) for (int k = 0; k < 4; ++k) s += yacc[0][j][k];
        if (s == 12345.f) parts[0] = s;  // keep the reduction alive
    }
    if (threadIdx.x == 0) { clk[blk * 2] = t0; clk[blk * 2 + 1] = t1; }
}

// pure gather: every warp streams 16-byte pieces of its rows' K and V (U rows
// per 16-lane group in flight), summing them -- the random-row HBM ceiling
template <int U>
__global__ void __launch_bounds__(kThr) gather_kernel(lrqk_layer_t L, const int *rows_all, const int *nrows, int cap,
                                                      float *parts) {
    const int blk = blockIdx.x, h = blk / 9, g = h / 4;
    const int n = nrows[blk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = lane >> 4, sl = lane & 15;
    const uint4 *kb = reinterpret_cast<const uint4 *>(reinterpret_cast<const T *>(L.slow_k) + (size_t)g * L.t_max * 128);
    const uint4 *vb = reinterpret_cast<const uint4 *>(reinterpret_cast<const T *>(L.slow_v) + (size_t)g * L.t_max * 128);
    const int *rows = rows_all + blk * cap;
    const int step = (blockDim.x >> 5) * 2;
    uint32_t acc = 0;
    for (int b0 = warp * 2 + sub; b0 < n; b0 += step * U) {
        uint4 x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = b0 + u * step;
            const int r = j < n ? __ldg(rows + j) : 0;
            x[u] = kb[(size_t)r * 16 + sl];
            y[u] = vb[(size_t)r * 16 + sl];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += x[u].x ^ y[u].y ^ x[u].z ^ y[u].w;
    }
    if (acc == 0x12345u) parts[blk] = acc;
}

// K|V interleaved rows (512 contiguous bytes per token): 32 lanes per row
template <int U>
__global__ void __launch_bounds__(kThr) gather_kv_kernel(const T *kv, int t_max, const int *rows_all, const int *nrows,
                                                         int cap, float *parts) {
    const int blk = blockIdx.x, h = blk / 9, g = h / 4;
    const int n = nrows[blk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint4 *b = reinterpret_cast<const uint4 *>(kv + (size_t)g * t_max * 256);
    const int *rows = rows_all + blk * cap;
    const int step = blockDim.x >> 5;
    uint32_t acc = 0;
    for (int b0 = warp; b0 < n; b0 += step * U) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = b0 + u * step;
            const int r = j < n ? __ldg(rows + j) : 0;
            x[u] = b[(size_t)r * 32 + lane];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += x[u].x ^ x[u].w;
    }
    if (acc == 0x12345u) parts[blk] = acc;
}

// TMA bulk gather: warp 8 issues one 256-byte bulk copy per K row and per V
// row into a ring of NS stages of CR rows (mbarrier completion); warps 0-7
// wait and release each stage
template <int CR, int NS>
__global__ void __launch_bounds__(kThr) gather_tma_kernel(lrqk_layer_t L, const int *rows_all, const int *nrows, int cap,
                                                          float *parts) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[NS], empty[NS];
    const int blk = blockIdx.x, h = blk / 9, g = h / 4;
    const int n = nrows[blk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const T *kb = reinterpret_cast<const T *>(L.slow_k) + (size_t)g * L.t_max * 128;
    const T *vb = reinterpret_cast<const T *>(L.slow_v) + (size_t)g * L.t_max * 128;
    const int *rows = rows_all + blk * cap;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nch = (n + CR - 1) / CR;
    constexpr int SB = CR * 512;
    if (warp == 8) {
        for (int ch = 0; ch < nch; ++ch) {
            const int s2 = ch % NS;
            if (ch >= NS) mbar_wait(empty + s2, ((ch / NS) - 1) & 1);
            const int r0 = ch * CR, nr = min(CR, n - r0);
            if (lane == 0) mbar_expect_tx(full + s2, (uint32_t)nr * 512);
            __syncwarp();
            for (int j = lane; j < nr; j += 32) {
                const int r = rows[r0 + j];
                bulk_g2s(smem + s2 * SB + j * 256, kb + (size_t)r * 128, 256, full + s2);
                bulk_g2s(smem + s2 * SB + CR * 256 + j * 256, vb + (size_t)r * 128, 256, full + s2);
            }
        }
    } else {
        uint32_t acc = 0;
        for (int ch = 0; ch < nch; ++ch) {
            const int s2 = ch % NS;
            mbar_wait(full + s2, (ch / NS) & 1);
            acc += reinterpret_cast<const uint32_t *>(smem + s2 * SB)[threadIdx.x];
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s2);
        }
        if (acc == 0x12345u) parts[blk] = acc;
    }
}

void *g_flush;
template <int CR, int NS>
void run_gather_tma(lrqk_layer_t L, const int *rows, const int *nrows, int cap, float *parts, int nblk) {
    auto fn = gather_tma_kernel<CR, NS>;
    const int sm = NS * CR * 512;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms = 0.f;
    const int reps = 20;
    for (int w = 0; w < reps + 2; ++w) {
        cudaMemsetAsync(g_flush, w, (size_t)256 << 20);
        cudaEventRecord(a);
        fn<<<nblk, kThr, sm>>>(L, rows, nrows, cap, parts);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float x; cudaEventElapsedTime(&x, a, b);
        if (w >= 2) ms += x;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThr, sm);
    const double bytes = (double)nblk * 229 * 512;
    printf("gather TMA bulk CR=%d NS=%d (%d blocks/SM): %7.2f us  %6.0f GB/s  %s\n", CR, NS, occ, ms * 1e3 / reps,
           bytes / (ms * 1e-3 / reps) / 1e9, cudaGetErrorString(cudaGetLastError()));
}
template <int U>
void run_gather_kv(const T *kv, int t_max, const int *rows, const int *nrows, int cap, float *parts, int nblk) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms = 0.f;
    const int reps = 20;
    for (int w = 0; w < reps + 2; ++w) {
        cudaMemsetAsync(g_flush, w, (size_t)256 << 20);
        cudaEventRecord(a);
        gather_kv_kernel<U><<<nblk, kThr>>>(kv, t_max, rows, nrows, cap, parts);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float x; cudaEventElapsedTime(&x, a, b);
        if (w >= 2) ms += x;
    }
    const double bytes = (double)nblk * 229 * 512;
    printf("gather K|V interleaved U=%2d: %7.2f us  %6.0f GB/s\n", U, ms * 1e3 / reps, bytes / (ms * 1e-3 / reps) / 1e9);
}
template <int U>
void run_gather(lrqk_layer_t L, const int *rows, const int *nrows, int cap, float *parts, int nblk, int per_sm_bytes) {
    auto fn = gather_kernel<U>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, per_sm_bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms = 0.f;
    const int reps = 20;
    for (int w = 0; w < reps + 2; ++w) {
        cudaMemsetAsync(g_flush, w, (size_t)256 << 20);
        cudaEventRecord(a);
        fn<<<nblk, kThr, per_sm_bytes>>>(L, rows, nrows, cap, parts);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float x; cudaEventElapsedTime(&x, a, b);
        if (w >= 2) ms += x;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThr, per_sm_bytes);
    const double bytes = (double)nblk * 229 * 512;
    printf("gather U=%2d smem %6d (%d blocks/SM): %7.2f us  %6.0f GB/s\n", U, per_sm_bytes, occ, ms * 1e3 / reps,
           bytes / (ms * 1e-3 / reps) / 1e9);
}
template <int CR, int NS, int MODE, bool AROW = false, int YGM = 2, int PPH = 9>
void run(const char *name, lrqk_layer_t L, const int *rows, const int *nrows, int cap, const T *q, float *parts,
         long long *clk, int nblk) {
    auto fn = bench_kernel<CR, NS, MODE, AROW, YGM, PPH>;
    const int smem = (PPH == 9 ? 90 : 42) * 1024 + cap * 4;
    const int thr = PPH == 9 ? kThr : 160;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) fn<<<nblk, thr, smem>>>(L, rows, nrows, cap, q, parts, clk);
    const int reps = 20;
    float ms = 0.f;
    for (int w = 0; w < reps; ++w) {
        cudaMemsetAsync(g_flush, w, (size_t)256 << 20);  // evict the gathered rows from L2
        cudaEventRecord(a);
        fn<<<nblk, thr, smem>>>(L, rows, nrows, cap, q, parts, clk);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float x; cudaEventElapsedTime(&x, a, b);
        ms += x;
    }
    std::vector<long long> c(nblk * 2);
    cudaMemcpy(c.data(), clk, nblk * 16, cudaMemcpyDeviceToHost);
    std::vector<double> d;
    for (int i = 0; i < nblk; ++i) d.push_back((c[2 * i + 1] - c[2 * i]) / 1965.0);
    std::sort(d.begin(), d.end());
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, thr, smem);
    printf("%-28s kernel %7.2f us  attend phase med %6.2f max %6.2f us  (%d blocks/SM) %s\n", name, ms * 1e3 / reps,
           d[nblk / 2], d.back(), occ, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char **argv) {
    const int T_ = 131072 + 64, Hq = 32, P = 9, S = 2064;
    const int nblk = Hq * P, cap = 1024;
    const int mode_rows = argc < 2 ? 1 : atoi(argv[1]);  // 1 ascending random, 0 shuffled, 2 consecutive
    const bool sorted_rows = mode_rows != 0;
    T *K, *V, *A, *q;
    cudaMalloc(&K, (size_t)8 * T_ * 128 * 2);
    cudaMalloc(&V, (size_t)8 * T_ * 128 * 2);
    cudaMalloc(&A, (size_t)Hq * T_ * 32 * 2);
    cudaMalloc(&q, Hq * 128 * 2);
    cudaMemset(K, 0, (size_t)8 * T_ * 128 * 2);
    cudaMemset(V, 0, (size_t)8 * T_ * 128 * 2);
    cudaMemset(A, 0, (size_t)Hq * T_ * 32 * 2);
    cudaMemset(q, 0, Hq * 128 * 2);
    std::vector<int> rows(nblk * cap), nr(nblk), rows18(2 * nblk * cap), nr18(2 * nblk);
    std::mt19937 rng(1);
    const int part = 131072 / P, part18 = 131072 / 18;
    for (int h = 0; h < Hq; ++h) {
        std::vector<int> pick;
        std::uniform_int_distribution<int> U(0, 131071);
        while ((int)pick.size() < S) pick.push_back(U(rng));
        std::sort(pick.begin(), pick.end());
        pick.erase(std::unique(pick.begin(), pick.end()), pick.end());
        for (int p = 0; p < P; ++p) nr[h * P + p] = 0;
        for (int p = 0; p < 18; ++p) nr18[h * 18 + p] = 0;
        for (int x : pick) {
            const int p = std::min(P - 1, x / part);
            rows[(h * P + p) * cap + nr[h * P + p]++] = x;
            const int p2 = std::min(17, x / part18);
            rows18[(h * 18 + p2) * cap + nr18[h * 18 + p2]++] = x;
        }
    }
    int *drows, *dnr, *drows18, *dnr18; float *parts; long long *clk;
    cudaMalloc(&drows, rows.size() * 4); cudaMalloc(&dnr, nblk * 4);
    cudaMalloc(&drows18, rows18.size() * 4); cudaMalloc(&dnr18, 2 * nblk * 4);
    cudaMemcpy(drows18, rows18.data(), rows18.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dnr18, nr18.data(), 2 * nblk * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&parts, 2 * nblk * 130 * 4); cudaMalloc(&clk, 2 * nblk * 16);
    cudaMemcpy(drows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dnr, nr.data(), nblk * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&g_flush, (size_t)256 << 20);
    lrqk_layer_t L = {};
    L.t_max = T_; L.dim_stride = 128; L.rank_stride = 32; L.head_dim = 128;
    L.slow_k = K; L.slow_v = V; L.proxy = A;
    printf("rows per block ~%d, %s\n", S / P, sorted_rows ? "ascending" : "shuffled");
    setvbuf(stdout, nullptr, _IONBF, 0);
    T *KV = nullptr;
    if (cudaMalloc(&KV, (size_t)8 * T_ * 256 * 2) != cudaSuccess) { printf("alloc KV failed\n"); return 1; }
    cudaMemset(KV, 0, (size_t)8 * T_ * 256 * 2);
    run<64, 2, 0, true, 0>("P=9  288thr CR=64 NS=2 no YG", L, drows, dnr, cap, q, parts, clk, nblk);
    run<32, 2, 0, true, 0, 18>("P=18 160thr CR=32 NS=2 no YG", L, drows18, dnr18, cap, q, parts, clk, 2 * nblk);
    run<0, 0, 1>("P=9  288thr registers U=8", L, drows, dnr, cap, q, parts, clk, nblk);
    run<0, 0, 1, false, 0, 18>("P=18 160thr registers U=8", L, drows18, dnr18, cap, q, parts, clk, 2 * nblk);
    return 0;
}
