// Warp-level bf16 tensor-core helpers (mma.sync m16n8k16, ldmatrix, cp.async)
// shared by compress.cu (K2p) and select_attend.cu (K4+K6).
#pragma once
#include "common.cuh"

namespace lrqk {

// L2 prefetches (no destination, no completion tracking)
LRQK_DEV void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
LRQK_DEV void bulk_prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
LRQK_DEV void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src) : "memory");
}
LRQK_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> LRQK_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
LRQK_DEV void ldsm_x4_trans(uint32_t (&r)[4], const void *p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
LRQK_DEV void ldsm_x2_trans(uint32_t (&r)[2], const void *p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
                 : "=r"(r[0]), "=r"(r[1]) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
LRQK_DEV void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

constexpr int kMmaRows = 64;  // rows per sub-chunk

// smem bytes of the two gather buffers (row strides padded by 16 bytes)
__host__ __device__ inline int mma_stage_bytes(int R, int d) { return kMmaRows * ((d * 2 + 16) + (R * 2 + 16)); }

// Y += A^T K and G += A^T A over one staged tile of kMmaRows rows (rows
// beyond the valid ones must be zero in A).  A tile: [kMmaRows][lda bytes]
// bf16 rows of rank_stride R; K tile: [kMmaRows][ldk bytes] bf16 rows of d.
// Eight warps: warp w owns Y columns [w*8*NTW, (w+1)*8*NTW) and G tiles
// w, w+8, ...  MT = R/16 m tiles, NTW = d/64 n tiles per warp.
template <int MT, int NTW, int KR = kMmaRows>
LRQK_DEV void mma_reduce_tile(const uint8_t *kb_s, int ldk, const uint8_t *ab_s, int lda, int R,
                              float (&yacc)[MT][NTW][4], float (&gacc)[4][4]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane >> 3, i8 = lane & 7;
    constexpr int RR = MT * 16;  // rank_stride (== R)
    constexpr int GT = (RR / 16) * (RR / 8);
    (void)R;
#pragma unroll 1  // one k-step of code: the gather loop around it must stay in the instruction cache
    for (int ks = 0; ks < KR; ks += 16) {
        uint32_t af[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int m0 = mt * 16 + ((q & 1) ? 8 : 0), k0 = ks + ((q & 2) ? 8 : 0);
            ldsm_x4_trans(af[mt], ab_s + (k0 + i8) * lda + m0 * 2);
        }
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) {
            const int n0 = (warp * NTW + nt) * 8;
            uint32_t bfr[2];
            const int k0 = ks + ((lane >> 3) & 1) * 8;
            ldsm_x2_trans(bfr, kb_s + (k0 + i8) * ldk + n0 * 2);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) mma_bf16_16816(yacc[mt][nt], af[mt], bfr);
        }
#pragma unroll
        for (int w2 = 0; w2 < 4; ++w2) {
            const int gtile = warp + 8 * w2;
            if (gtile >= GT) break;
            const int mt = gtile / (RR / 8), n0 = (gtile % (RR / 8)) * 8;
            uint32_t bfr[2];
            const int k0 = ks + ((lane >> 3) & 1) * 8;
            ldsm_x2_trans(bfr, ab_s + (k0 + i8) * lda + n0 * 2);
#pragma unroll
            for (int m2 = 0; m2 < MT; ++m2)
                if (m2 == mt) mma_bf16_16816(gacc[w2], af[m2], bfr);
        }
    }
}

// Accumulator fragments -> partial [Y (R x d, row-major) | G (R x R)].
template <int MT, int NTW>
LRQK_DEV void mma_write_partial(const float (&yacc)[MT][NTW][4], const float (&gacc)[4][4], int R, int d,
                                float *part) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane >> 2, fc = (lane & 3) * 2;
    const int GT = (R / 16) * (R / 8);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) {
            const int n0 = (warp * NTW + nt) * 8;
            float *y = part + (mt * 16 + fr) * d + n0 + fc;
            *reinterpret_cast<float2 *>(y) = make_float2(yacc[mt][nt][0], yacc[mt][nt][1]);
            *reinterpret_cast<float2 *>(y + 8 * d) = make_float2(yacc[mt][nt][2], yacc[mt][nt][3]);
        }
#pragma unroll
    for (int w2 = 0; w2 < 4; ++w2) {
        const int gtile = warp + 8 * w2;
        if (gtile >= GT) break;
        const int mt = gtile / (R / 8), n0 = (gtile % (R / 8)) * 8;
        float *gp = part + R * d + (mt * 16 + fr) * R + n0 + fc;
        *reinterpret_cast<float2 *>(gp) = make_float2(gacc[w2][0], gacc[w2][1]);
        *reinterpret_cast<float2 *>(gp + 8 * R) = make_float2(gacc[w2][2], gacc[w2][3]);
    }
}

// Y = A^T K and G = A^T A over n <= kMmaRows listed rows (bf16 storage), on
// the CUDA cores, ADDED to dst[R*d | R*R]: the rows are staged as fp32 in
// shared memory (stage >= kMmaRows * (d + R) floats), then each thread owns
// (R*d + R*R) / blockDim.x outputs.
template <typename T>
__device__ void yg_rows_small(const lrqk_layer_t &L, const T *kb, const T *proxy, const int *rows, int n,
                              float *stage, float *dst) {
    const int d = L.dim_stride, R = L.rank_stride, ap = R * (int)sizeof(T) / 16;
    constexpr int N = Pack<T>::N;
    float *sK = stage, *sA = stage + (size_t)kMmaRows * d;
    for (int e = threadIdx.x; e < n * (d / N + ap); e += blockDim.x) {
        float f[N];
        if (e < n * (d / N)) {
            const int j = e / (d / N), pk = e - j * (d / N);
            unpack16<T>(*reinterpret_cast<const uint4 *>(kb + (size_t)rows[j] * d + pk * N), f);
#pragma unroll
            for (int u = 0; u < N; ++u) sK[j * d + pk * N + u] = f[u];
        } else {
            const int e2 = e - n * (d / N), j = e2 / ap, pk = e2 - j * ap;
            unpack16<T>(*reinterpret_cast<const uint4 *>(proxy + proxy_pack_offset(rows[j], pk, ap) * N), f);
#pragma unroll
            for (int u = 0; u < N; ++u) sA[j * R + pk * N + u] = f[u];
        }
    }
    __syncthreads();
    for (int o = threadIdx.x; o < R * d + R * R; o += blockDim.x) {
        float acc = 0.f;
        if (o < R * d) {
            const int p = o / d, i = o - p * d;
            for (int j = 0; j < n; ++j) acc = fmaf(sA[j * R + p], sK[j * d + i], acc);
        } else {
            const int o2 = o - R * d, p = o2 / R, q = o2 - p * R;
            for (int j = 0; j < n; ++j) acc = fmaf(sA[j * R + p], sA[j * R + q], acc);
        }
        dst[o] += acc;
    }
    __syncthreads();
}

}  // namespace lrqk
