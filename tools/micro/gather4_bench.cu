// Microbenchmark (development tool): the random-row gather of the attend
// phase (C4 shapes: 32 heads x 9 parts, ~229 ascending random rows of 128
// bf16 per part, K and V of 8 KV heads x 128K rows) through
//   (a) plain 16-byte register loads (U rows in flight per 16-lane group),
//   (b) one TMA bulk copy per row (cp.async.bulk, 256 B),
//   (c) TMA tile::gather4 (cp.async.bulk.tensor.2d ... tile::gather4: four
//       rows of a 2-D tensor map per instruction),
// each with L2 flushed between launches.  Checks that (c) lands the right
// rows.  Usage: gather4_bench [rows per head] [1: consecutive rows]
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

using T = __nv_bfloat16;
constexpr int kThr = 288;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
    } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void gather4(void *dst, const CUtensorMap *m, int c0, int r0, int r1, int r2, int r3,
                                        uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"(smem_u32(bar))
        : "memory");
}

// (a) plain loads
template <int U>
__global__ void __launch_bounds__(kThr) plain_kernel(const T *K, const T *V, int t_max, const int *rows_all,
                                                     const int *nrows, int cap, unsigned *sink) {
    const int blk = blockIdx.x, g = blk / 9 / 4;
    const int n = nrows[blk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = lane >> 4, sl = lane & 15;
    const uint4 *kb = reinterpret_cast<const uint4 *>(K + (size_t)g * t_max * 128);
    const uint4 *vb = reinterpret_cast<const uint4 *>(V + (size_t)g * t_max * 128);
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
    if (acc == 0x12345u) sink[blk] = acc;
}

// (a') plain loads after an L2 prefetch of every row of the block: PF 1 =
// prefetch.global.L2 per 128-byte line, PF 2 = cp.async.bulk.prefetch.L2 per row
template <int U, int PF>
__global__ void __launch_bounds__(kThr) plain_pf_kernel(const T *K, const T *V, int t_max, const int *rows_all,
                                                        const int *nrows, int cap, unsigned *sink) {
    const int blk = blockIdx.x, g = blk / 9 / 4;
    const int n = nrows[blk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = lane >> 4, sl = lane & 15;
    const T *kr = K + (size_t)g * t_max * 128, *vr = V + (size_t)g * t_max * 128;
    const int *rows = rows_all + blk * cap;
    if (PF == 1) {
        for (int e = threadIdx.x; e < n * 4; e += blockDim.x) {
            const int j = e >> 2, part = e & 3;
            const T *base = (part & 2) ? vr : kr;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (size_t)rows[j] * 128 + (part & 1) * 64));
        }
    } else if (PF == 2) {
        for (int e = threadIdx.x; e < n * 2; e += blockDim.x) {
            const int j = e >> 1;
            const T *base = (e & 1) ? vr : kr;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], 256;" ::"l"(base + (size_t)rows[j] * 128) : "memory");
        }
    }
    const uint4 *kb = reinterpret_cast<const uint4 *>(kr);
    const uint4 *vb = reinterpret_cast<const uint4 *>(vr);
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
    if (acc == 0x12345u) sink[blk] = acc;
}

// (b) / (c): producer warp 8 fills a ring of NS stages of CR rows (K then V);
// warps 0-7 check each stage's rows and release it
template <int CR, int NS, bool G4>
__global__ void __launch_bounds__(kThr) tma_kernel(const __grid_constant__ CUtensorMap mk,
                                                   const __grid_constant__ CUtensorMap mv, const T *K, const T *V,
                                                   int t_max, const int *rows_all, const int *nrows, int cap,
                                                   unsigned *sink, unsigned *bad) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[NS], empty[NS];
    const int blk = blockIdx.x, g = blk / 9 / 4;
    const int n = nrows[blk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int *rows = rows_all + blk * cap;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nch = (n + CR - 1) / CR;
    constexpr int SB = CR * 512;
    const int gbase = g * t_max;  // first row of this KV head in the 2-D maps
    if (warp == 8) {
        for (int ch = 0; ch < nch; ++ch) {
            const int s2 = ch % NS;
            if (ch >= NS) mbar_wait(empty + s2, ((ch / NS) - 1) & 1);
            const int r0 = ch * CR, nr = min(CR, n - r0);
            if (G4) {
                const int ng = (nr + 3) / 4;
                if (lane == 0) mbar_expect_tx(full + s2, (uint32_t)ng * 4 * 512);
                __syncwarp();
                for (int q = lane; q < ng; q += 32) {
                    int r[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) r[u] = gbase + rows[r0 + min(4 * q + u, nr - 1)];
                    gather4(smem + s2 * SB + q * 4 * 256, &mk, 0, r[0], r[1], r[2], r[3], full + s2);
                    gather4(smem + s2 * SB + CR * 256 + q * 4 * 256, &mv, 0, r[0], r[1], r[2], r[3], full + s2);
                }
            } else {
                if (lane == 0) mbar_expect_tx(full + s2, (uint32_t)nr * 512);
                __syncwarp();
                for (int j = lane; j < nr; j += 32) {
                    const int r = rows[r0 + j];
                    bulk_g2s(smem + s2 * SB + j * 256, K + ((size_t)gbase + r) * 128, 256, full + s2);
                    bulk_g2s(smem + s2 * SB + CR * 256 + j * 256, V + ((size_t)gbase + r) * 128, 256, full + s2);
                }
            }
        }
    } else {
        uint32_t acc = 0, nbad = 0;
        for (int ch = 0; ch < nch; ++ch) {
            const int s2 = ch % NS;
            mbar_wait(full + s2, (ch / NS) & 1);
            const int r0 = ch * CR, nr = min(CR, n - r0);
            for (int j = threadIdx.x; j < nr; j += 256) {  // K and V rows carry their row index in element 0
                const uint16_t kx = reinterpret_cast<const uint16_t *>(smem + s2 * SB + j * 256)[0];
                const uint16_t vx = reinterpret_cast<const uint16_t *>(smem + s2 * SB + CR * 256 + j * 256)[0];
                const uint16_t want = (uint16_t)((gbase + rows[r0 + j]) & 0x7FFF);
                nbad += (kx != want) + (vx != want);
                acc += kx;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s2);
        }
        if (acc == 0x12345u) sink[blk] = acc;
        if (nbad) atomicAdd(bad, nbad);
    }
}

__global__ void fill_kernel(T *X, long long rows) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x)
        reinterpret_cast<uint16_t *>(X)[r * 128] = (uint16_t)(r & 0x7FFF);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
        return nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

int main(int argc, char **argv) {
    // argv[1]: rows per head (default 2064 = C4's S); argv[2]: 1 = consecutive rows
    const int T_ = 131072 + 64, Hq = 32, P = 9, Hkv = 8;
    const int S = argc > 1 ? atoi(argv[1]) : 2064;
    const bool consecutive = argc > 2 && atoi(argv[2]) == 1;
    const int nblk = Hq * P, cap = std::max(1024, 2 * S / P + 64);
    const long long nrows_all = (long long)Hkv * T_;
    T *K, *V;
    cudaMalloc(&K, nrows_all * 256);
    cudaMalloc(&V, nrows_all * 256);
    cudaMemset(K, 0, nrows_all * 256);
    cudaMemset(V, 0, nrows_all * 256);
    fill_kernel<<<1184, 256>>>(K, nrows_all);
    fill_kernel<<<1184, 256>>>(V, nrows_all);
    std::vector<int> rows(nblk * cap), nr(nblk);
    std::mt19937 rng(1);
    const int part = 131072 / P;
    for (int h = 0; h < Hq; ++h) {
        std::vector<int> pick;
        std::uniform_int_distribution<int> U(0, 131071);
        if (consecutive) {
            const int start = U(rng) % (131072 - S);
            for (int i = 0; i < S; ++i) pick.push_back(start + i);
        }
        while ((int)pick.size() < S) pick.push_back(U(rng));
        std::sort(pick.begin(), pick.end());
        pick.erase(std::unique(pick.begin(), pick.end()), pick.end());
        for (int p = 0; p < P; ++p) nr[h * P + p] = 0;
        for (int x : pick) {
            const int p = std::min(P - 1, x / part);
            rows[(h * P + p) * cap + nr[h * P + p]++] = x;
        }
    }
    long long total_rows = 0;
    for (int b = 0; b < nblk; ++b) total_rows += nr[b];
    int *drows, *dnr;
    unsigned *sink, *bad;
    cudaMalloc(&drows, rows.size() * 4);
    cudaMalloc(&dnr, nblk * 4);
    cudaMalloc(&sink, nblk * 4);
    cudaMalloc(&bad, 4);
    cudaMemcpy(drows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dnr, nr.data(), nblk * 4, cudaMemcpyHostToDevice);
    void *flush;
    cudaMalloc(&flush, (size_t)256 << 20);
    setvbuf(stdout, nullptr, _IONBF, 0);

    CUtensorMap mk, mv;
    auto fn = encode_fn();
    if (!fn) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
    const cuuint64_t dims[2] = {128, (cuuint64_t)nrows_all};
    const cuuint64_t strides[1] = {256};
    const cuuint32_t box[2] = {128, 1};
    const cuuint32_t es[2] = {1, 1};
    CUresult rk = fn(&mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult rv = fn(&mv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, V, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("tensor maps: %d %d; rows per block ~%lld\n", (int)rk, (int)rv, total_rows / nblk);
    const double bytes = (double)total_rows * 512;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto time = [&](const char *name, auto launch) {
        float ms = 0.f;
        const int reps = 20;
        cudaMemset(bad, 0, 4);
        for (int w = 0; w < reps + 2; ++w) {
            cudaMemsetAsync(flush, w, (size_t)256 << 20);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float x;
            cudaEventElapsedTime(&x, a, b);
            if (w >= 2) ms += x;
        }
        unsigned hb = 0;
        cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
        printf("%-36s %7.2f us  %6.0f GB/s  bad rows %u  %s\n", name, ms * 1e3 / reps, bytes / (ms * 1e-3 / reps) / 1e9,
               hb, cudaGetErrorString(cudaGetLastError()));
    };
    time("plain loads U=8", [&] { plain_kernel<8><<<nblk, kThr>>>(K, V, T_, drows, dnr, cap, sink); });
    time("plain loads U=2", [&] { plain_kernel<2><<<nblk, kThr>>>(K, V, T_, drows, dnr, cap, sink); });
    time("L2 prefetch (lines) + loads U=8", [&] { plain_pf_kernel<8, 1><<<nblk, kThr>>>(K, V, T_, drows, dnr, cap, sink); });
    time("L2 prefetch (bulk rows) + loads U=8", [&] { plain_pf_kernel<8, 2><<<nblk, kThr>>>(K, V, T_, drows, dnr, cap, sink); });
    time("L2 prefetch (lines) + loads U=2", [&] { plain_pf_kernel<2, 1><<<nblk, kThr>>>(K, V, T_, drows, dnr, cap, sink); });
#define TMA_RUN(CR, NS, G4, NAME)                                                                          \
    {                                                                                                      \
        auto kf = tma_kernel<CR, NS, G4>;                                                                  \
        const int sm = NS * CR * 512;                                                                      \
        cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);                         \
        time(NAME, [&] { kf<<<nblk, kThr, sm>>>(mk, mv, K, V, T_, drows, dnr, cap, sink, bad); });         \
    }
    TMA_RUN(64, 2, false, "bulk per row CR=64 NS=2");
    TMA_RUN(64, 2, true, "gather4 CR=64 NS=2");
    TMA_RUN(32, 4, true, "gather4 CR=32 NS=4");
    TMA_RUN(64, 3, true, "gather4 CR=64 NS=3");
    TMA_RUN(128, 2, true, "gather4 CR=128 NS=2");
    TMA_RUN(256, 1, true, "gather4 CR=256 NS=1 (all rows at once)");
    return 0;
}
