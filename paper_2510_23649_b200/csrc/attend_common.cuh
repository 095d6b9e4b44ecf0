// Gathered-row attention helpers shared by select_attend.cu (K4+K6) and
// score_attend.cu (K3+K4+K6 fused): online softmax over listed K/V rows,
// the staged gather with the tensor-core Y|G reduction, and the block /
// multi-part (max, sum, acc) merges.  ref: attention.py:23-34.
#pragma once
#include "common.cuh"
#include "mma_common.cuh"

namespace lrqk {

// Online softmax over the K/V rows listed in rows[0, n) (shared memory),
// continuing (m, l, acc) of this lane group.  LPR lanes per row, PPL 16-byte
// packs per lane; all lanes of a warp run the same trip count.
template <typename T, int LPR, int PPL, int U = 8>
__device__ void attend_list(const T *kb, const T *vb, const int *rows, int n, const float (&qv)[PPL][Pack<T>::N],
                            float c, int d, float &m, float &l, float (&acc)[PPL][Pack<T>::N]) {
    constexpr int N = Pack<T>::N;
    constexpr int RPW = 32 / LPR;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int sub = lane / LPR, sl = lane - sub * LPR;
    const int step = nw * RPW;
    for (int b0 = warp * RPW; b0 < n; b0 += step * U) {
        uint4 kx[U][PPL], vx[U][PPL];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = b0 + sub + u * step;
            if (j < n) {
                const size_t row = (size_t)rows[j] * d;
#pragma unroll
                for (int pp = 0; pp < PPL; ++pp) {
                    kx[u][pp] = *reinterpret_cast<const uint4 *>(kb + row + (sl + pp * LPR) * N);
                    vx[u][pp] = *reinterpret_cast<const uint4 *>(vb + row + (sl + pp * LPR) * N);
                }
            } else {
#pragma unroll
                for (int pp = 0; pp < PPL; ++pp) { kx[u][pp] = make_uint4(0, 0, 0, 0); vx[u][pp] = make_uint4(0, 0, 0, 0); }
            }
        }
        float x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float s = 0.f;
#pragma unroll
            for (int pp = 0; pp < PPL; ++pp) {
                float f[N];
                unpack16<T>(kx[u][pp], f);
#pragma unroll
                for (int e = 0; e < N; ++e) s = fmaf(f[e], qv[pp][e], s);
            }
            x[u] = s;
        }
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < U; ++u) x[u] += __shfl_xor_sync(0xffffffffu, x[u], o);
        float mx = m;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            x[u] = (b0 + sub + u * step < n) ? x[u] * c : -INFINITY;
            mx = fmaxf(mx, x[u]);
        }
        if (mx == -INFINITY) continue;
        const float scale = exp2f(m - mx);
        l *= scale;
#pragma unroll
        for (int pp = 0; pp < PPL; ++pp)
#pragma unroll
            for (int e = 0; e < N; ++e) acc[pp][e] *= scale;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float p = exp2f(x[u] - mx);
            l += p;
#pragma unroll
            for (int pp = 0; pp < PPL; ++pp) {
                float f[N];
                unpack16<T>(vx[u][pp], f);
#pragma unroll
                for (int e = 0; e < N; ++e) acc[pp][e] = fmaf(p, f[e], acc[pp][e]);
            }
        }
        m = mx;
    }
}

// Staged variant: the listed rows' K and V (and, with YG, their proxy rows
// A) are gathered CR at a time into shared memory with cp.async (NS
// buffers); each chunk feeds the online softmax of this block and, with YG,
// the tensor-core reduction Y += A^T K, G += A^T A that the next step's
// compression needs over Omega_t (compress.cu K2p), so compress_prepare
// does not gather these rows again.
template <typename T, int LPR, int PPL, int YGM, int CR = kMmaRows, int NS = 2>
__device__ void attend_reduce_list(const lrqk_layer_t &L, const T *kb, const T *vb, const T *proxy, const T *arows,
                                   const int *rows,
                                   int n, const float (&qv)[PPL][Pack<T>::N], float c, float &m, float &l,
                                   float (&acc)[PPL][Pack<T>::N], uint8_t *stage,
                                   float (&yacc)[YGM > 0 ? YGM : 1][2][4],
                                   float (&gacc)[4][4]) {
    constexpr int N = Pack<T>::N;
    constexpr int RPW = 32 / LPR;
    const int d = L.dim_stride, R = L.rank_stride;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int sub = lane / LPR, sl = lane - sub * LPR;
    const int ng = nw * RPW, gidx = warp * RPW + sub;
    const int ldk = d * (int)sizeof(T) + 16, lda = R * 2 + 16;  // bytes (padded rows)
    const int kp = d * (int)sizeof(T) / 16;
    constexpr bool YG = YGM > 0;
    constexpr int PA = 2 * YGM;  // 16-byte packs per proxy row (R = 16 * YGM, bf16)
    const int tile_kv = CR * ldk, buf = 2 * tile_kv + (YG ? CR * lda : 0);
    const int nch = (n + CR - 1) / CR;
    auto issue = [&](int ch) {
        uint8_t *kS = stage + (ch % NS) * buf, *vS = kS + tile_kv, *aS = vS + tile_kv;
        const int r0 = ch * CR, nr = min(CR, n - r0);
        if constexpr (YG) {
            // bf16, d = 128, R = 16 * YGM: 16 packs per K/V row, PA per proxy row (shifts only)
            for (int e = tid; e < CR * 16; e += blockDim.x) {
                const int j = e >> 4, pk = e & 15;
                uint8_t *dk = kS + j * ldk + pk * 16, *dv = vS + j * ldk + pk * 16;
                if (j < nr) {
                    const size_t row = (size_t)rows[r0 + j] * 128 + pk * 8;
                    cp_async16(dk, kb + row);
                    cp_async16(dv, vb + row);
                } else {
                    *reinterpret_cast<uint4 *>(dk) = make_uint4(0, 0, 0, 0);
                    *reinterpret_cast<uint4 *>(dv) = make_uint4(0, 0, 0, 0);
                }
            }
            for (int e = tid; e < CR * PA; e += blockDim.x) {
                const int j = e / PA, pk = e % PA;
                uint8_t *da = aS + j * lda + pk * 16;
                if (j < nr)  // the row-major copy when the layer keeps one: one contiguous run per row
                    cp_async16(da, arows ? arows + (size_t)rows[r0 + j] * (PA * 8) + pk * 8
                                         : proxy + proxy_pack_offset(rows[r0 + j], pk, PA) * 8);
                else *reinterpret_cast<uint4 *>(da) = make_uint4(0, 0, 0, 0);
            }
        } else {
            for (int e = tid; e < CR * kp; e += blockDim.x) {
                const int j = e / kp, pk = e - j * kp;
                uint8_t *dk = kS + j * ldk + pk * 16, *dv = vS + j * ldk + pk * 16;
                if (j < nr) {
                    const size_t row = (size_t)rows[r0 + j] * d + pk * (16 / sizeof(T));
                    cp_async16(dk, kb + row);
                    cp_async16(dv, vb + row);
                } else {
                    *reinterpret_cast<uint4 *>(dk) = make_uint4(0, 0, 0, 0);
                    *reinterpret_cast<uint4 *>(dv) = make_uint4(0, 0, 0, 0);
                }
            }
        }
        cp_async_commit();
    };
    // NS-stage pipeline: NS - 1 chunks in flight while one is consumed (a
    // commit group per chunk slot, empty past the end, so wait_group counts).
    // One loop issues the prologue too (ch < 0), so the gather code exists
    // once and the loop stays in the instruction cache.
#pragma unroll 1
    for (int ch = -(NS - 1); ch < nch; ++ch) {
        if (ch + NS - 1 < nch) issue(ch + NS - 1);
        else cp_async_commit();
        if (ch < 0) continue;
        cp_async_wait<NS - 1>();
        __syncthreads();
        const uint8_t *kS = stage + (ch % NS) * buf, *vS = kS + tile_kv, *aS = vS + tile_kv;
        const int nr = min(CR, n - ch * CR);
        // online softmax over this chunk: group gidx takes rows gidx, gidx + ng, ...
        for (int j0 = 0; j0 < CR; j0 += ng * 4) {
            float x[4];
            uint4 vx[4][PPL];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = j0 + gidx + u * ng;
                float sdot = 0.f;
#pragma unroll
                for (int pp = 0; pp < PPL; ++pp) {
                    const uint4 kx = j < CR ? *reinterpret_cast<const uint4 *>(kS + j * ldk + (sl + pp * LPR) * 16)
                                                  : make_uint4(0, 0, 0, 0);
                    vx[u][pp] = j < CR ? *reinterpret_cast<const uint4 *>(vS + j * ldk + (sl + pp * LPR) * 16)
                                             : make_uint4(0, 0, 0, 0);
                    float f[N];
                    unpack16<T>(kx, f);
#pragma unroll
                    for (int e = 0; e < N; ++e) sdot = fmaf(f[e], qv[pp][e], sdot);
                }
                x[u] = sdot;
            }
#pragma unroll
            for (int o = LPR / 2; o > 0; o >>= 1)
#pragma unroll
                for (int u = 0; u < 4; ++u) x[u] += __shfl_xor_sync(0xffffffffu, x[u], o);
            float mx = m;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                x[u] = (j0 + gidx + u * ng < nr) ? x[u] * c : -INFINITY;
                mx = fmaxf(mx, x[u]);
            }
            if (mx != -INFINITY) {
                const float scale = exp2f(m - mx);
                l *= scale;
#pragma unroll
                for (int pp = 0; pp < PPL; ++pp)
#pragma unroll
                    for (int e = 0; e < N; ++e) acc[pp][e] *= scale;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float pr = exp2f(x[u] - mx);
                    l += pr;
#pragma unroll
                    for (int pp = 0; pp < PPL; ++pp) {
                        float f[N];
                        unpack16<T>(vx[u][pp], f);
#pragma unroll
                        for (int e = 0; e < N; ++e) acc[pp][e] = fmaf(pr, f[e], acc[pp][e]);
                    }
                }
                m = mx;
            }
        }
        if constexpr (YG) {
            if (warp < 8) mma_reduce_tile<YGM, 2, CR>(kS, ldk, aS, lda, R, yacc, gacc);  // 8 MMA warps own Y|G
        }
        __syncthreads();
    }
}

// Merge the lane groups' (m, l, acc) into one block partial: dst[0] = max,
// dst[1] = sum, dst[2 + i] = acc (log2 domain, as the attention kernel).
// Groups of a warp merge through shuffles, warps through shared memory with
// precomputed weights.
LRQK_DEV void merge_pair(float &m, float &l, float m2, float l2, float &w1, float &w2) {
    const float M = fmaxf(m, m2);
    w1 = m == -INFINITY ? 0.f : exp2f(m - M);
    w2 = m2 == -INFINITY ? 0.f : exp2f(m2 - M);
    l = l * w1 + l2 * w2;
    m = M;
}
template <typename T, int LPR, int PPL>
__device__ void block_partial(float m, float l, float (&acc)[PPL][Pack<T>::N], int d, float *s_m, float *s_l,
                              float *s_acc, float *dst) {
    constexpr int N = Pack<T>::N;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int sl = lane % LPR;
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o), l2 = __shfl_xor_sync(0xffffffffu, l, o);
        float w1, w2;
        merge_pair(m, l, m2, l2, w1, w2);
#pragma unroll
        for (int pp = 0; pp < PPL; ++pp)
#pragma unroll
            for (int e = 0; e < N; ++e) {
                const float a2 = __shfl_xor_sync(0xffffffffu, acc[pp][e], o);
                acc[pp][e] = acc[pp][e] * w1 + a2 * w2;
            }
    }
    if (lane < LPR) {
        if (lane == 0) { s_m[warp] = m; s_l[warp] = l; }
#pragma unroll
        for (int pp = 0; pp < PPL; ++pp)
#pragma unroll
            for (int e = 0; e < N; ++e) s_acc[warp * d + (sl + pp * LPR) * N + e] = acc[pp][e];
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // warp weights
        const float mw = lane < nw ? s_m[lane] : -INFINITY;
        float M = mw;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float w = (lane < nw && mw != -INFINITY) ? exp2f(mw - M) : 0.f;
        float lw = lane < nw ? s_l[lane] * w : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lw += __shfl_xor_sync(0xffffffffu, lw, o);
        if (lane < nw) s_l[lane] = w;  // now the warp weight
        if (lane == 0) { dst[0] = M; dst[1] = lw; }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        float a = 0.f;
        for (int w = 0; w < nw; ++w) a = fmaf(s_acc[w * d + i], s_l[w], a);
        dst[2 + i] = a;
    }
    __syncthreads();
}

// Merge np softmax partials of one head (each max, sum, acc[d]; log2
// domain, written by block_partial) into out[0, d), summed in partial order.
// s_w: 64 floats of shared memory, s_red: 2.  Whole block.
static __device__ __noinline__ void merge_partials(const float *parts, int np, int d, float *out, float *s_w, float *s_red) {
    if (threadIdx.x < 32) {
        float mx = -INFINITY;
        for (int p = threadIdx.x; p < np; p += 32) mx = fmaxf(mx, __ldcg(parts + (size_t)p * (d + 2)));
        mx = warp_max(mx);
        float den = 0.f;
        for (int p = threadIdx.x; p < np; p += 32) {
            const float pm = __ldcg(parts + (size_t)p * (d + 2));
            const float w = pm == -INFINITY ? 0.f : exp2f(pm - mx);
            if (p < 64) s_w[p] = w;
            den = fmaf(__ldcg(parts + (size_t)p * (d + 2) + 1), w, den);
        }
        den = warp_sum(den);
        if (threadIdx.x == 0) { s_red[0] = den; s_red[1] = mx; }
    }
    __syncthreads();
    const float inv = 1.f / s_red[0];
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        float o = 0.f;
        for (int p0 = 0; p0 < np; p0 += 8) {  // 8 partials' loads in flight, summed in order
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (p0 + u < np) v[u] = __ldcg(parts + (size_t)(p0 + u) * (d + 2) + 2 + i);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int p = p0 + u;
                if (p >= np) break;
                float w;
                if (p < 64) {
                    w = s_w[p];
                } else {
                    const float pm = __ldcg(parts + (size_t)p * (d + 2));
                    w = pm == -INFINITY ? 0.f : exp2f(pm - s_red[1]);
                }
                o = fmaf(v[u], w, o);
            }
        }
        out[i] = o * inv;
    }
    __syncthreads();
}

}  // namespace lrqk
