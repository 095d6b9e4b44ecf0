#include <cstdlib>
// K1: prefill joint rank-r factorisation, batched over heads.
//
// ref: prefill.py:142-230 (lagrangian_value, update_B, update_AK, update_AQ,
//      _factor_delta, prefill_run).
//
// The reference sweep (B_Q, B_K, A_K, A_Q) is re-associated so that every
// sweep streams each of K and Q exactly once:
//
//   pass P1 (over K):  A_K' = K W_K,   W_K = (C_Q + lk B_K^T)(G_AQ + lk B_K B_K^T)^-1
//                      and, fused,  G_AK' = A_K'^T A_K',  C_K' = K^T A_K'
//   pass P2 (over Q):  A_Q' = Q W_Q,   W_Q = (C_K' + lq B_Q^T)(G_AK' + lq B_Q B_Q^T)^-1
//                      and, fused,  G_AQ' = A_Q'^T A_Q',  C_Q' = Q^T A_Q'
//
// where C_X = X^T A_X (d x r) and G_AX = A_X^T A_X (r x r).  update_B is then
// B_X = G_AX^-1 C_X^T, computed from the fused reductions of the previous
// pass without touching X again (prefill.py:161-163).  The objective uses the
// same Gram-trace expansion as the reference (prefill.py:142-158) plus
// ||X - A B||^2 = ||X||^2 - 2<B, C^T> + <G_A, B B^T>.
//
// Each pass kernel block owns a slab of rows of one head, keeps its C/G
// partial sums in registers across 128-row chunks staged in shared memory,
// and writes one partial; a per-head solve kernel reduces the partials and
// does the r x r algebra (Gauss-Jordan inverse with the reference jitter
// retry, linalg.py:80-91).
#include "common.cuh"
#include "mma_common.cuh"

namespace lrqk {

constexpr int kPfThreads = 256;
constexpr int kPfRows = 128;

struct PfDims {
    int H, group, l, d, ds, r, rs, NB;
    size_t psz;        // floats per partial
    size_t head_sz;    // floats of scratch per head
};

LRQK_DEV size_t pf_part_off(const PfDims &D, int h, int nb) {
    return (size_t)h * D.head_sz + (size_t)nb * D.psz;
}
// state block offsets (floats) inside one head's scratch
struct PfState {
    size_t CQ, CK, GQ, GK, W, BQp, BKp, misc;
};
__host__ __device__ inline PfState pf_state(const PfDims &D) {
    PfState s;
    size_t o = (size_t)D.NB * D.psz;
    const size_t dr = (size_t)D.ds * D.rs, rr = (size_t)D.rs * D.rs;
    s.CQ = o; o += dr;
    s.CK = o; o += dr;
    s.GQ = o; o += rr;
    s.GK = o; o += rr;
    s.W = o; o += dr;
    s.BQp = o; o += dr;
    s.BKp = o; o += dr;
    s.misc = o;
    return s;
}
enum PfMisc { PF_ACTIVE = 0, PF_XQ2 = 1, PF_XK2 = 2, PF_QK2 = 3, PF_DAK = 4, PF_DAQ = 5, PF_SWEEP = 6 };
constexpr int kPfMisc = 16;

// ---------------------------------------------------------------------------
// pass kernel: optional A update (A_out = X W), then fused C, G reductions
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kPfThreads)
pf_pass_kernel(const PfDims D, const T *X, int is_k, const float *A_in, float *A_out, int update,
               int want_x2, float *scratch) {
    extern __shared__ __align__(16) float sm[];
    const int h = blockIdx.y, nb = blockIdx.x, tid = threadIdx.x;
    const PfState st = pf_state(D);
    float *hs = scratch + (size_t)h * D.head_sz;
    if (hs[st.misc + PF_ACTIVE] == 0.f) return;
    const int ds = D.ds, rs = D.rs;
    const int ldx = ds + 4, lda = rs + 4;
    float *sX = sm;                        // [kPfRows][ldx]
    float *sA = sX + kPfRows * ldx;        // [kPfRows][lda]
    float *sW = sA + kPfRows * lda;        // [ds][rs]
    float *sRed = sW + ds * rs;            // reduction scratch
    const int xh = is_k ? h / D.group : h;
    const T *Xh = X + (size_t)xh * D.l * ds;
    const float *Ain = A_in + (size_t)h * D.l * rs;
    float *Aout = A_out + (size_t)h * D.l * rs;
    if (update) {
        const float *W = hs + st.W;
        for (int e = tid; e < ds * rs; e += blockDim.x) sW[e] = W[e];
    }
    // slab of rows for this block
    const int nchunks = (D.l + kPfRows - 1) / kPfRows;
    const int c0 = (int)((long long)nchunks * nb / D.NB), c1 = (int)((long long)nchunks * (nb + 1) / D.NB);

    // C tiles (4 k x 4 p) owned by this thread, up to 4
    const int nCt = (ds / 4) * (rs / 4);
    float cacc[4][16];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int e = 0; e < 16; ++e) cacc[a][e] = 0.f;
    // G tiles (4 p x 4 q), row groups
    const int nGt = (rs / 4) * (rs / 4);
    const int ngr = max(1, (int)blockDim.x / nGt);
    float gacc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) gacc[e] = 0.f;
    float diff = 0.f, x2 = 0.f;

    for (int c = c0; c < c1; ++c) {
        const int row0 = c * kPfRows;
        const int nrow = min(kPfRows, D.l - row0);
        __syncthreads();
        // stage X chunk (fp32), zero rows beyond nrow
        for (int e = tid; e < kPfRows * ds; e += blockDim.x) {
            const int i = e / ds, k = e - i * ds;
            float v = i < nrow ? to_float<T>(Xh[(size_t)(row0 + i) * ds + k]) : 0.f;
            sX[i * ldx + k] = v;
            x2 = fmaf(v, v, x2);
        }
        if (!update) {
            for (int e = tid; e < kPfRows * rs; e += blockDim.x) {
                const int i = e / rs, p = e - i * rs;
                sA[i * lda + p] = i < nrow ? Ain[(size_t)(row0 + i) * rs + p] : 0.f;
            }
        }
        __syncthreads();
        if (update) {
            // A_new = X W, 4 rows x 4 cols per tile
            const int nAt = (kPfRows / 4) * (rs / 4);
            for (int tI = tid; tI < nAt; tI += blockDim.x) {
                const int i0 = (tI / (rs / 4)) * 4, p0 = (tI % (rs / 4)) * 4;
                float acc[4][4] = {};
                for (int k = 0; k < ds; k += 4) {
                    float4 xr[4], wr[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) xr[u] = *reinterpret_cast<const float4 *>(sX + (i0 + u) * ldx + k);
#pragma unroll
                    for (int u = 0; u < 4; ++u) wr[u] = *reinterpret_cast<const float4 *>(sW + (k + u) * rs + p0);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float xs[4] = {xr[u].x, xr[u].y, xr[u].z, xr[u].w};
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            acc[u][0] = fmaf(xs[kk], wr[kk].x, acc[u][0]);
                            acc[u][1] = fmaf(xs[kk], wr[kk].y, acc[u][1]);
                            acc[u][2] = fmaf(xs[kk], wr[kk].z, acc[u][2]);
                            acc[u][3] = fmaf(xs[kk], wr[kk].w, acc[u][3]);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u;
                    if (i < nrow) {
                        const float4 old = *reinterpret_cast<const float4 *>(Ain + (size_t)(row0 + i) * rs + p0);
                        const float o4[4] = {old.x, old.y, old.z, old.w};
                        float n4[4];
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            // padded rank columns stay exactly zero
                            n4[v] = (p0 + v < D.r) ? acc[u][v] : 0.f;
                            const float df = n4[v] - o4[v];
                            diff = fmaf(df, df, diff);
                        }
                        *reinterpret_cast<float4 *>(Aout + (size_t)(row0 + i) * rs + p0) = make_float4(n4[0], n4[1], n4[2], n4[3]);
#pragma unroll
                        for (int v = 0; v < 4; ++v) sA[i * lda + p0 + v] = n4[v];
                    } else {
#pragma unroll
                        for (int v = 0; v < 4; ++v) sA[i * lda + p0 + v] = 0.f;
                    }
                }
            }
            __syncthreads();
        }
        // C += X^T A  (4 k x 4 p tiles)
        for (int a = 0; a < 4; ++a) {
            const int tI = tid + a * blockDim.x;
            if (tI >= nCt) break;
            const int k0 = (tI / (rs / 4)) * 4, p0 = (tI % (rs / 4)) * 4;
            for (int i = 0; i < nrow; ++i) {
                const float4 xv = *reinterpret_cast<const float4 *>(sX + i * ldx + k0);
                const float4 av = *reinterpret_cast<const float4 *>(sA + i * lda + p0);
                const float xs[4] = {xv.x, xv.y, xv.z, xv.w}, as[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) cacc[a][u * 4 + v] = fmaf(xs[u], as[v], cacc[a][u * 4 + v]);
            }
        }
        // G += A^T A
        if (tid < nGt * ngr) {
            const int tI = tid % nGt, grp = tid / nGt;
            const int p0 = (tI / (rs / 4)) * 4, q0 = (tI % (rs / 4)) * 4;
            for (int i = grp; i < nrow; i += ngr) {
                const float4 ap = *reinterpret_cast<const float4 *>(sA + i * lda + p0);
                const float4 aq = *reinterpret_cast<const float4 *>(sA + i * lda + q0);
                const float ps[4] = {ap.x, ap.y, ap.z, ap.w}, qs[4] = {aq.x, aq.y, aq.z, aq.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) gacc[u * 4 + v] = fmaf(ps[u], qs[v], gacc[u * 4 + v]);
            }
        }
    }
    // ---- write this block's partial ------------------------------------------
    float *part = scratch + pf_part_off(D, h, nb);
    for (int a = 0; a < 4; ++a) {
        const int tI = tid + a * blockDim.x;
        if (tI >= nCt) break;
        const int k0 = (tI / (rs / 4)) * 4, p0 = (tI % (rs / 4)) * 4;
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) part[(k0 + u) * rs + p0 + v] = cacc[a][u * 4 + v];
    }
    __syncthreads();
    if (tid < nGt * ngr) {
#pragma unroll
        for (int e = 0; e < 16; ++e) sRed[tid * 16 + e] = gacc[e];
    }
    __syncthreads();
    for (int e = tid; e < nGt * 16; e += blockDim.x) {
        const int tI = e / 16, uv = e - tI * 16;
        float s = 0.f;
        for (int gI = 0; gI < ngr; ++gI) s += sRed[(gI * nGt + tI) * 16 + uv];
        const int p0 = (tI / (rs / 4)) * 4, q0 = (tI % (rs / 4)) * 4;
        part[ds * rs + (p0 + uv / 4) * rs + q0 + (uv & 3)] = s;
    }
    __syncthreads();
    float v2[2] = {diff, x2};
    for (int j = 0; j < 2; ++j) {
        float s = warp_sum(v2[j]);
        if ((tid & 31) == 0) sRed[j * 32 + (tid >> 5)] = s;
    }
    __syncthreads();
    if (tid == 0) {
        float sd = 0.f, sx = 0.f;
        for (int w = 0; w < (int)blockDim.x / 32; ++w) { sd += sRed[w]; sx += sRed[32 + w]; }
        part[ds * rs + rs * rs] = sd;
        part[ds * rs + rs * rs + 1] = want_x2 ? sx : 0.f;
    }
}

// ---------------------------------------------------------------------------
// Tensor-core pass (bf16 X, d = 128, rank_stride RS in {16, 32, 64}): the
// same three products as pf_pass_kernel on mma.sync m16n8k16 with fp32
// accumulation.  X is exact in bf16; the fp32 operands W and A are split
// into bf16 hi + lo parts (3xBF16: hi*hi + hi*lo + lo*hi), which keeps the
// products to ~2^-16 relative, the accuracy class of the fp32 CUDA-core
// pass.  Per 128-row tile, 8 warps:
//   A_new = X W      warp w: rows [16w, 16w+16) x all RS columns
//   C    += X^T A    warp w: d rows [16w, 16w+16) x all RS columns
//   G    += A^T A    RS/16 x RS/8 tiles spread over the warps
// The pass is memory-bound (X streamed once, A read/written once), so
// mma.sync already reaches the HBM roofline.
// ---------------------------------------------------------------------------
constexpr int kPfD = 128;

LRQK_DEV void ldsm_x4(uint32_t (&r)[4], const void *p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
LRQK_DEV void ldsm_x2(uint32_t (&r)[2], const void *p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                 : "=r"(r[0]), "=r"(r[1]) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
LRQK_DEV void split_bf16(float v, __nv_bfloat16 &hi, __nv_bfloat16 &lo) {
    hi = __float2bfloat16_rn(v);
    lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

template <int RS>
__global__ void __launch_bounds__(kPfThreads)
pf_pass_mma_kernel(const PfDims D, const __nv_bfloat16 *X, int is_k, const float *A_in, float *A_out, int update,
                   int want_x2, float *scratch) {
    constexpr int NT = RS / 8;                        // n tiles over the rank
    constexpr int GT = (RS / 16) * (RS / 8);          // G tiles
    constexpr int GPW = (GT + 7) / 8;                 // G tiles per warp
    constexpr int LDX = kPfD * 2 + 16, LDA = RS * 2 + 16, LDW = kPfD * 2 + 16;  // bytes
    extern __shared__ __align__(16) uint8_t pm[];
    uint8_t *sXb = pm;                                // 2 x [128][LDX]  X tiles (bf16), double buffered
    uint8_t *sAh = sXb + 2 * kPfRows * LDX;           // [128][LDA]  A tile hi
    uint8_t *sAl = sAh + kPfRows * LDA;               // [128][LDA]  A tile lo
    uint8_t *sWh = sAl + kPfRows * LDA;               // [RS][LDW]   W^T hi
    uint8_t *sWl = sWh + RS * LDW;                    // [RS][LDW]   W^T lo
    float *sRed = reinterpret_cast<float *>(sWl + RS * LDW);
    const int h = blockIdx.y, nb = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const PfState st = pf_state(D);
    float *hs = scratch + (size_t)h * D.head_sz;
    if (hs[st.misc + PF_ACTIVE] == 0.f) return;
    const int xh = is_k ? h / D.group : h;
    const __nv_bfloat16 *Xh = X + (size_t)xh * D.l * kPfD;
    const float *Ain = A_in + (size_t)h * D.l * RS;
    float *Aout = A_out + (size_t)h * D.l * RS;
    if (update) {  // W^T (RS x d), split
        const float *W = hs + st.W;  // [d][RS]
        for (int e = tid; e < kPfD * RS; e += blockDim.x) {
            const int k = e / RS, p = e - k * RS;
            __nv_bfloat16 hi, lo;
            split_bf16(W[e], hi, lo);
            reinterpret_cast<__nv_bfloat16 *>(sWh + p * LDW)[k] = hi;
            reinterpret_cast<__nv_bfloat16 *>(sWl + p * LDW)[k] = lo;
        }
    }
    const int nchunks = (D.l + kPfRows - 1) / kPfRows;
    const int c0 = (int)((long long)nchunks * nb / D.NB), c1 = (int)((long long)nchunks * (nb + 1) / D.NB);
    const int q = lane >> 3, i8 = lane & 7, fr = lane >> 2, fc = (lane & 3) * 2;
    float cacc[NT][4], gacc[GPW][4];
    static_assert(kPfD / 8 == 16, "X rows are 16 packs");
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) cacc[n][e] = 0.f;
#pragma unroll
    for (int g = 0; g < GPW; ++g)
#pragma unroll
        for (int e = 0; e < 4; ++e) gacc[g][e] = 0.f;
    float diff = 0.f, x2 = 0.f;
    // X tiles stream through shared memory with cp.async, one tile ahead
    auto issue_x = [&](int c) {
        uint8_t *dst = sXb + (c & 1) * kPfRows * LDX;
        const int row0 = c * kPfRows, nrow = min(kPfRows, D.l - row0);
        for (int e = tid; e < kPfRows * (kPfD / 8); e += blockDim.x) {
            const int i = e >> 4, pk = e & 15;
            if (i < nrow) cp_async16(dst + i * LDX + pk * 16, Xh + (size_t)(row0 + i) * kPfD + pk * 8);
            else *reinterpret_cast<uint4 *>(dst + i * LDX + pk * 16) = make_uint4(0, 0, 0, 0);
        }
        cp_async_commit();
    };
    if (c0 < c1) issue_x(c0);
    for (int c = c0; c < c1; ++c) {
        const int row0 = c * kPfRows;
        const int nrow = min(kPfRows, D.l - row0);
        uint8_t *sX = sXb + (c & 1) * kPfRows * LDX;
        __syncthreads();  // the other buffer is free again
        if (c + 1 < c1) { issue_x(c + 1); cp_async_wait<1>(); }
        else cp_async_wait<0>();
        // old A of this warp's rows (update: the convergence measure), early
        float2 aold[NT][2];
        if (update) {
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    const int i = warp * 16 + fr + hf * 8;
                    aold[n][hf] = i < nrow ? __ldcs(reinterpret_cast<const float2 *>(Ain + (size_t)(row0 + i) * RS + n * 8 + fc))
                                           : make_float2(0.f, 0.f);
                }
        }
        __syncthreads();
        if (want_x2) {
            for (int e = tid; e < kPfRows * (kPfD / 8); e += blockDim.x) {
                float f[8];
                unpack16<__nv_bfloat16>(*reinterpret_cast<const uint4 *>(sX + (e >> 4) * LDX + (e & 15) * 16), f);
#pragma unroll
                for (int u = 0; u < 8; ++u) x2 = fmaf(f[u], f[u], x2);
            }
        }
        if (!update) {  // A tile from A_in, split
            for (int e = tid; e < kPfRows * RS; e += blockDim.x) {
                const int i = e / RS, p2 = e - i * RS;
                const float v = i < nrow ? Ain[(size_t)(row0 + i) * RS + p2] : 0.f;
                __nv_bfloat16 hi, lo;
                split_bf16(v, hi, lo);
                reinterpret_cast<__nv_bfloat16 *>(sAh + i * LDA)[p2] = hi;
                reinterpret_cast<__nv_bfloat16 *>(sAl + i * LDA)[p2] = lo;
            }
        }
        __syncthreads();
        if (update) {
            // ---- A_new = X W: warp rows [16w, 16w+16) -------------------------
            float aacc[NT][4];
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int e = 0; e < 4; ++e) aacc[n][e] = 0.f;
#pragma unroll
            for (int ks = 0; ks < kPfD; ks += 16) {
                uint32_t af[4];
                ldsm_x4(af, sX + (warp * 16 + (lane & 15)) * LDX + (ks + (lane >> 4) * 8) * 2);
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    uint32_t bh[2], bl[2];
                    const uint8_t *wrow = (lane & 7) * LDW + (ks + ((lane >> 3) & 1) * 8) * 2 + (size_t)n * 8 * LDW + sWh;
                    ldsm_x2(bh, wrow);
                    ldsm_x2(bl, wrow + (sWl - sWh));
                    mma_bf16_16816(aacc[n], af, bh);
                    mma_bf16_16816(aacc[n], af, bl);
                }
            }
            // fragment rows fr, fr + 8 of this warp's 16, columns n*8 + fc, +1
#pragma unroll
            for (int n = 0; n < NT; ++n) {
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    const int i = warp * 16 + fr + hf * 8, p2 = n * 8 + fc;
                    float v0 = p2 < D.r ? aacc[n][hf * 2] : 0.f, v1 = p2 + 1 < D.r ? aacc[n][hf * 2 + 1] : 0.f;
                    if (i >= nrow) { v0 = 0.f; v1 = 0.f; }
                    if (i < nrow) {
                        const float2 old = aold[n][hf];
                        diff = fmaf(v0 - old.x, v0 - old.x, diff);
                        diff = fmaf(v1 - old.y, v1 - old.y, diff);
                        *reinterpret_cast<float2 *>(Aout + (size_t)(row0 + i) * RS + p2) = make_float2(v0, v1);
                    }
                    __nv_bfloat16 h0, l0, h1, l1;
                    split_bf16(v0, h0, l0);
                    split_bf16(v1, h1, l1);
                    __nv_bfloat162 hh, ll;
                    hh.x = h0; hh.y = h1; ll.x = l0; ll.y = l1;
                    *reinterpret_cast<__nv_bfloat162 *>(sAh + i * LDA + p2 * 2) = hh;
                    *reinterpret_cast<__nv_bfloat162 *>(sAl + i * LDA + p2 * 2) = ll;
                }
            }
            __syncthreads();
        }
        // ---- C += X^T A: warp d rows [16w, 16w+16) ---------------------------
#pragma unroll
        for (int ks = 0; ks < kPfRows; ks += 16) {
            uint32_t af[4];
            ldsm_x4_trans(af, sX + (ks + ((q & 2) ? 8 : 0) + i8) * LDX + (warp * 16 + ((q & 1) ? 8 : 0)) * 2);
            const int k0 = ks + ((lane >> 3) & 1) * 8;
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                uint32_t bh[2], bl[2];
                ldsm_x2_trans(bh, sAh + (k0 + i8) * LDA + n * 16);
                ldsm_x2_trans(bl, sAl + (k0 + i8) * LDA + n * 16);
                mma_bf16_16816(cacc[n], af, bh);
                mma_bf16_16816(cacc[n], af, bl);
            }
        }
        // ---- G += A^T A (hi hi + hi lo + lo hi) -------------------------------
#pragma unroll
        for (int g = 0; g < GPW; ++g) {
            const int gt = warp + 8 * g;
            if (gt >= GT) break;
            const int mt = gt / NT, n0 = (gt % NT) * 8;
#pragma unroll
            for (int ks = 0; ks < kPfRows; ks += 16) {
                uint32_t ah[4], al[4];
                const int m0 = mt * 16 + ((q & 1) ? 8 : 0), kk = ks + ((q & 2) ? 8 : 0);
                ldsm_x4_trans(ah, sAh + (kk + i8) * LDA + m0 * 2);
                ldsm_x4_trans(al, sAl + (kk + i8) * LDA + m0 * 2);
                uint32_t bh[2], bl[2];
                const int k0 = ks + ((lane >> 3) & 1) * 8;
                ldsm_x2_trans(bh, sAh + (k0 + i8) * LDA + n0 * 2);
                ldsm_x2_trans(bl, sAl + (k0 + i8) * LDA + n0 * 2);
                mma_bf16_16816(gacc[g], ah, bh);
                mma_bf16_16816(gacc[g], ah, bl);
                mma_bf16_16816(gacc[g], al, bh);
            }
        }
    }
    // ---- this block's partial: C (d x RS) | G (RS x RS) | diff | x2 ---------
    float *part = scratch + pf_part_off(D, h, nb);
#pragma unroll
    for (int n = 0; n < NT; ++n) {
        const int k = warp * 16 + fr, p2 = n * 8 + fc;
        *reinterpret_cast<float2 *>(part + k * RS + p2) = make_float2(cacc[n][0], cacc[n][1]);
        *reinterpret_cast<float2 *>(part + (k + 8) * RS + p2) = make_float2(cacc[n][2], cacc[n][3]);
    }
#pragma unroll
    for (int g = 0; g < GPW; ++g) {
        const int gt = warp + 8 * g;
        if (gt >= GT) break;
        const int mt = gt / NT, n0 = (gt % NT) * 8;
        float *gp = part + kPfD * RS + (mt * 16 + fr) * RS + n0 + fc;
        *reinterpret_cast<float2 *>(gp) = make_float2(gacc[g][0], gacc[g][1]);
        *reinterpret_cast<float2 *>(gp + 8 * RS) = make_float2(gacc[g][2], gacc[g][3]);
    }
    float v2[2] = {diff, x2};
    for (int j = 0; j < 2; ++j) {
        const float sj = warp_sum(v2[j]);
        if (lane == 0) sRed[j * 32 + warp] = sj;
    }
    __syncthreads();
    if (tid == 0) {
        float sd = 0.f, sx = 0.f;
        for (int w = 0; w < (int)blockDim.x / 32; ++w) { sd += sRed[w]; sx += sRed[32 + w]; }
        part[kPfD * RS + RS * RS] = sd;
        part[kPfD * RS + RS * RS + 1] = want_x2 ? sx : 0.f;
    }
}

template <int RS>
static size_t pf_mma_smem() {
    return 2 * (size_t)kPfRows * (kPfD * 2 + 16) + 2 * (size_t)kPfRows * (RS * 2 + 16) +
           2 * (size_t)RS * (kPfD * 2 + 16) + 64 * sizeof(float);
}

// d x d Gram of X (objective only): GX[i][j] = sum_l X[l][i] X[l][j]
template <typename T>
__global__ void pf_gram_dd_kernel(const PfDims D, const T *X, int n_x, float *out /* [n_x][ds][ds] */) {
    const int xh = blockIdx.y;
    const int i = blockIdx.x;  // row of the Gram
    const T *Xh = X + (size_t)xh * D.l * D.ds;
    for (int j = threadIdx.x; j < D.ds; j += blockDim.x) {
        double acc = 0.0;
        for (int l = 0; l < D.l; ++l)
            acc += (double)to_float<T>(Xh[(size_t)l * D.ds + i]) * (double)to_float<T>(Xh[(size_t)l * D.ds + j]);
        out[((size_t)xh * D.ds + i) * D.ds + j] = (float)acc;
    }
    (void)n_x;
}

// sum of GQ o GK over the d x d Grams, per query head
__global__ void pf_qk2_kernel(const PfDims D, const float *gq, const float *gk, float *scratch) {
    const int h = blockIdx.x;
    const float *a = gq + (size_t)h * D.ds * D.ds;
    const float *b = gk + (size_t)(h / D.group) * D.ds * D.ds;
    __shared__ double s[32];
    double acc = 0.0;
    for (int e = threadIdx.x; e < D.ds * D.ds; e += blockDim.x) acc += (double)a[e] * (double)b[e];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)blockDim.x / 32; ++w) t += s[w];
        const PfState st = pf_state(D);
        scratch[(size_t)h * D.head_sz + st.misc + PF_QK2] = (float)t;
    }
}

// ---------------------------------------------------------------------------
// per-head r x r algebra
// ---------------------------------------------------------------------------
// Invert an SPD n x n (row stride ld) into Minv (stride ld) with the
// reference's single jitter retry.  Returns 0 ok, 1 jittered, 2 failed.
__device__ int spd_inverse(const float *M, int n, int ld, float *Minv) {
    const int tid = threadIdx.x, nt = blockDim.x;
    __shared__ int s_fail;
    for (int attempt = 0; attempt < 2; ++attempt) {
        float jit = 0.f;
        if (attempt) {
            float tr = 0.f, dmax = 0.f;
            for (int i = 0; i < n; ++i) { tr += M[i * ld + i]; dmax = fmaxf(dmax, fabsf(M[i * ld + i])); }
            jit = fmaxf(1e-10f * (tr / n + 1.f), dmax * 1.2e-7f);
        }
        __syncthreads();
        for (int e = tid; e < n * n; e += nt) {
            const int i = e / n, j = e - i * n;
            Minv[i * ld + j] = M[i * ld + j] + (i == j ? jit : 0.f);
        }
        if (tid == 0) s_fail = 0;
        for (int k = 0; k < n; ++k) {
            __syncthreads();
            const float p = Minv[k * ld + k];
            if (!(p > 0.f) || !isfinite(p)) { if (tid == 0) s_fail = 1; break; }
            const float ip = 1.f / p;
            float nv[24];
            int cnt = 0;
            for (int e = tid; e < n * n; e += nt) {
                const int i = e / n, j = e - i * n;
                const float a = Minv[i * ld + j];
                float rr;
                if (i == k && j == k) rr = ip;
                else if (i == k) rr = a * ip;
                else if (j == k) rr = -a * ip;
                else rr = a - Minv[i * ld + k] * Minv[k * ld + j] * ip;
                nv[cnt++] = rr;
            }
            __syncthreads();
            cnt = 0;
            for (int e = tid; e < n * n; e += nt) {
                const int i = e / n, j = e - i * n;
                Minv[i * ld + j] = nv[cnt++];
            }
        }
        __syncthreads();
        if (!s_fail) return attempt;
    }
    return 2;
}

// stage: 0 = after the init passes, 1 = after the K pass, 2 = after the Q pass
__global__ void __launch_bounds__(kPfThreads)
pf_solve_kernel(const PfDims D, lrqk_prefill_t P, int stage, int sweep) {
    extern __shared__ __align__(16) float sm[];
    const int h = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    const PfState st = pf_state(D);
    float *hs = P.scratch + (size_t)h * D.head_sz;
    float *misc = hs + st.misc;
    const int ds = D.ds, rs = D.rs, r = D.r, d = D.d;
    const float lq = P.lambda_q, lk = P.lambda_k;
    if (misc[PF_ACTIVE] == 0.f) return;
    const int ldm = rs + 1;
    float *sM = sm;                 // [rs][ldm]
    float *sMi = sM + rs * ldm;     // [rs][ldm]
    float *sB = sMi + rs * ldm;     // [rs][ds]  current B (side being solved)
    float *sRed = sB + rs * ds;     // 64
    float *BQ = P.B_Q + (size_t)h * rs * ds;
    float *BK = P.B_K + (size_t)h * rs * ds;

    // reduce the pass partials into C (ds x rs), G (rs x rs), diff, x2
    auto reduce_into = [&](float *C, float *G, float *diff, float *x2) {
        for (int e = tid; e < ds * rs + rs * rs + 2; e += nt) {
            float s = 0.f;
            for (int nb = 0; nb < D.NB; ++nb) s += hs[(size_t)nb * D.psz + e];
            if (e < ds * rs) C[e] = s;
            else if (e < ds * rs + rs * rs) {
                const int f = e - ds * rs;
                const int p = f / rs, q = f - p * rs;
                if (p <= q) { G[p * rs + q] = s; }
            } else if (e == ds * rs + rs * rs) *diff = s;
            else if (x2) *x2 = s;
        }
        __syncthreads();
        for (int e = tid; e < rs * rs; e += nt) {  // mirror upper -> lower (linalg.py:53-54)
            const int p = e / rs, q = e - p * rs;
            if (p > q) G[p * rs + q] = G[q * rs + p];
        }
        __syncthreads();
    };
    // B = G^-1 C^T  (update_B, prefill.py:161-163) into dst (rs x ds)
    auto solve_B = [&](const float *G, const float *C, float *dst) -> bool {
        for (int e = tid; e < r * r; e += nt) sM[(e / r) * ldm + e % r] = G[(e / r) * rs + e % r];
        const int rc = spd_inverse(sM, r, ldm, sMi);
        if (rc == 2) return false;
        if (rc == 1 && tid == 0) set_status(P.status, LRQK_ST_JITTERED);
        for (int e = tid; e < rs * ds; e += nt) {
            const int p = e / ds, i = e - p * ds;
            float acc = 0.f;
            if (p < r && i < d)
                for (int q = 0; q < r; ++q) acc = fmaf(sMi[p * ldm + q], C[i * rs + q], acc);
            dst[e] = acc;
        }
        __syncthreads();
        return true;
    };
    // W = (C + lam B^T) (G + lam B B^T)^-1  (update_AK / update_AQ)
    auto solve_W = [&](const float *G, const float *C, const float *B, float lam, float *W) -> bool {
        for (int e = tid; e < r * r; e += nt) {
            const int p = e / r, q = e - p * r;
            float bb = 0.f;
            for (int i = 0; i < d; ++i) bb = fmaf(B[p * ds + i], B[q * ds + i], bb);
            sM[p * ldm + q] = G[p * rs + q] + lam * bb;
        }
        __syncthreads();
        for (int e = tid; e < r * r; e += nt) {  // exact symmetry
            const int p = e / r, q = e - p * r;
            if (p > q) sM[p * ldm + q] = sM[q * ldm + p];
        }
        const int rc = spd_inverse(sM, r, ldm, sMi);
        if (rc == 2) return false;
        if (rc == 1 && tid == 0) set_status(P.status, LRQK_ST_JITTERED);
        for (int e = tid; e < ds * rs; e += nt) {
            const int i = e / rs, p = e - i * rs;
            float acc = 0.f;
            if (p < r && i < d)
                for (int q = 0; q < r; ++q) acc = fmaf(C[i * rs + q] + lam * B[q * ds + i], sMi[q * ldm + p], acc);
            W[e] = acc;
        }
        __syncthreads();
        return true;
    };
    // objective (prefill.py:142-158) from the reduced quantities
    auto objective = [&]() -> float {
        const float *CQ = hs + st.CQ, *CK = hs + st.CK, *GQ = hs + st.GQ, *GK = hs + st.GK;
        double acc[4] = {0, 0, 0, 0};  // cross, approx, q-resid-part, k-resid-part
        for (int e = tid; e < ds * rs; e += nt) {
            acc[0] += (double)CQ[e] * CK[e];
            const int i = e / rs, p = e - i * rs;
            acc[2] += -2.0 * (double)BQ[p * ds + i] * CQ[e];
            acc[3] += -2.0 * (double)BK[p * ds + i] * CK[e];
        }
        for (int e = tid; e < rs * rs; e += nt) {
            const int p = e / rs, q = e - p * rs;
            acc[1] += (double)GQ[e] * GK[e];
            double bbq = 0, bbk = 0;
            for (int i = 0; i < ds; ++i) {
                bbq += (double)BQ[p * ds + i] * BQ[q * ds + i];
                bbk += (double)BK[p * ds + i] * BK[q * ds + i];
            }
            acc[2] += (double)GQ[e] * bbq;
            acc[3] += (double)GK[e] * bbk;
        }
        __shared__ double sacc[4][32];
        for (int j = 0; j < 4; ++j) {
            double v = acc[j];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if ((tid & 31) == 0) sacc[j][tid >> 5] = v;
        }
        __syncthreads();
        double tot[4] = {0, 0, 0, 0};
        for (int j = 0; j < 4; ++j)
            for (int w = 0; w < nt / 32; ++w) tot[j] += sacc[j][w];
        __syncthreads();
        const double fit = fmax((double)misc[PF_QK2] - 2.0 * tot[0] + tot[1], 0.0);
        const double rq = fmax((double)misc[PF_XQ2] + tot[2], 0.0);
        const double rk = fmax((double)misc[PF_XK2] + tot[3], 0.0);
        return (float)(0.5 * fit + 0.5 * lq * rq + 0.5 * lk * rk);
    };
    auto fail = [&]() {
        if (tid == 0) { set_status(P.status, LRQK_ST_SOLVE_FAILED); misc[PF_ACTIVE] = 0.f; }
    };

    if (stage == 0) {
        // partials of the two init passes were written to the Q slot (CQ/GQ)
        // and K slot by the host sequencing: Q pass -> reduce now into CQ/GQ
        // is done by the caller splitting stage 0 into 0a/0b (see below).
        return;
    }
    if (stage == 3 || stage == 4) {  // 3: reduce init Q pass, 4: reduce init K pass + first B/W
        float dummy;
        if (stage == 3) {
            reduce_into(hs + st.CQ, hs + st.GQ, &dummy, misc + PF_XQ2);
            return;
        }
        reduce_into(hs + st.CK, hs + st.GK, &dummy, misc + PF_XK2);
        if (P.want_objective && tid == 0) misc[PF_SWEEP] = 0.f;
        // B factors start at zero (prefill.py:137-139) for the initial objective
        for (int e = tid; e < rs * ds; e += nt) { BQ[e] = 0.f; BK[e] = 0.f; }
        __syncthreads();
        if (P.want_objective) {
            const float obj = objective();
            if (tid == 0) P.objective[(size_t)h * (P.max_iter + 1)] = obj;
        }
        // first sweep: B_Q, B_K from the init factors, then W_K
        if (!solve_B(hs + st.GQ, hs + st.CQ, BQ)) return fail();
        if (!solve_B(hs + st.GK, hs + st.CK, BK)) return fail();
        for (int e = tid; e < rs * ds; e += nt) { hs[st.BQp + e] = 0.f; hs[st.BKp + e] = 0.f; }
        __syncthreads();
        if (!solve_W(hs + st.GQ, hs + st.CQ, BK, lk, hs + st.W)) return fail();
        return;
    }
    if (stage == 1) {
        // after the K pass: new C_K, G_AK; W_Q for the Q pass
        reduce_into(hs + st.CK, hs + st.GK, misc + PF_DAK, nullptr);
        if (!solve_W(hs + st.GK, hs + st.CK, BQ, lq, hs + st.W)) return fail();
        return;
    }
    // stage 2: after the Q pass -> objective, convergence, next sweep's B and W_K
    reduce_into(hs + st.CQ, hs + st.GQ, misc + PF_DAQ, nullptr);
    // non-finite factors (prefill.py:216-218)
    __shared__ int s_bad;
    if (tid == 0) s_bad = 0;
    __syncthreads();
    for (int e = tid; e < ds * rs; e += nt)
        if (!isfinite(hs[st.CQ + e]) || !isfinite(hs[st.CK + e])) s_bad = 1;
    if (tid == 0 && !(isfinite(misc[PF_DAQ]) && isfinite(misc[PF_DAK]))) s_bad = 1;
    __syncthreads();
    if (s_bad) {
        if (tid == 0) { set_status(P.status, LRQK_ST_NONFINITE); misc[PF_ACTIVE] = 0.f; }
        return;
    }
    if (P.want_objective) {
        const float obj = objective();
        if (tid == 0) P.objective[(size_t)h * (P.max_iter + 1) + sweep + 1] = obj;
    }
    // _factor_delta (prefill.py:184-194)
    __shared__ float s_db[2];
    if (tid < 64) {
        const int side = tid >> 5, lane = tid & 31;
        const float *Bn = side ? BK : BQ;
        const float *Bo = hs + (side ? st.BKp : st.BQp);
        float acc = 0.f;
        for (int e = lane; e < rs * ds; e += 32) { const float df = Bn[e] - Bo[e]; acc = fmaf(df, df, acc); }
        acc = warp_sum(acc);
        if (lane == 0) s_db[side] = acc;
    }
    __syncthreads();
    const double lr = (double)D.l * r, rd = (double)r * d;
    const double delta = ((double)misc[PF_DAQ] / lr + (double)misc[PF_DAK] / lr + (double)s_db[0] / rd +
                          (double)s_db[1] / rd) / 4.0;
    const bool conv = delta <= (double)P.tol;
    const bool last = conv || (sweep + 1 >= P.max_iter);
    if (tid == 0) {
        P.sweeps[h] = sweep + 1;
        P.converged[h] = conv ? 1 : 0;
    }
    __syncthreads();
    if (last) {
        if (tid == 0) misc[PF_ACTIVE] = 0.f;
        return;
    }
    // next sweep: B from the new A's (start of sweep s+1), keep the old B's
    for (int e = tid; e < rs * ds; e += nt) { hs[st.BQp + e] = BQ[e]; hs[st.BKp + e] = BK[e]; }
    __syncthreads();
    if (!solve_B(hs + st.GQ, hs + st.CQ, BQ)) return fail();
    if (!solve_B(hs + st.GK, hs + st.CK, BK)) return fail();
    if (!solve_W(hs + st.GQ, hs + st.CQ, BK, lk, hs + st.W)) return fail();
}

__global__ void pf_init_kernel(const PfDims D, lrqk_prefill_t P) {
    const int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= D.H) return;
    const PfState st = pf_state(D);
    float *misc = P.scratch + (size_t)h * D.head_sz + st.misc;
    for (int i = 0; i < kPfMisc; ++i) misc[i] = 0.f;
    misc[PF_ACTIVE] = 1.f;
    P.sweeps[h] = 0;
    P.converged[h] = 0;
    if (P.objective)
        for (int i = 0; i <= P.max_iter; ++i) P.objective[(size_t)h * (P.max_iter + 1) + i] = __int_as_float(0x7fc00000);
}

static PfDims pf_dims(const lrqk_prefill_t &P, int nsm) {
    PfDims D;
    D.H = P.n_heads;
    D.group = P.group > 0 ? P.group : 1;
    D.l = P.len;
    D.d = P.head_dim;
    D.ds = P.dim_stride;
    D.r = P.rank;
    D.rs = P.rank_stride;
    const int nchunks = (P.len + kPfRows - 1) / kPfRows;
    int nb = (2 * nsm + D.H - 1) / D.H;  // about two waves over all heads
    nb = nb < 1 ? 1 : nb;
    D.NB = nb < nchunks ? nb : nchunks;
    if (D.NB < 1) D.NB = 1;
    D.psz = (size_t)D.ds * D.rs + (size_t)D.rs * D.rs + 2;
    D.head_sz = (size_t)D.NB * D.psz + 5 * (size_t)D.ds * D.rs + 2 * (size_t)D.rs * D.rs + kPfMisc;
    D.head_sz = (D.head_sz + 3) & ~(size_t)3;
    return D;
}

extern int num_sms();

static bool pf_mma_enabled() {
    static const bool on = [] { const char *e = getenv("LRQK_PREFILL_MMA"); return !(e && e[0] == '0'); }();
    return on;
}

size_t prefill_scratch_floats(const lrqk_prefill_t &P) {
    PfDims D = pf_dims(P, num_sms());
    return (size_t)D.H * D.head_sz + (P.want_objective ? (size_t)(D.H + D.H / D.group) * D.ds * D.ds : 0);
}

int launch_prefill(const lrqk_prefill_t &P, cudaStream_t st) {
    if (P.rank_stride % 4 || P.dim_stride % 4 || P.rank > P.head_dim || P.rank_stride > 64 || P.dim_stride > 256)
        return LRQK_EUNSUPPORTED;
    const PfDims D = pf_dims(P, num_sms());
    pf_init_kernel<<<(D.H + 127) / 128, 128, 0, st>>>(D, P);
    const size_t pass_smem = ((size_t)kPfRows * (D.ds + 4) + (size_t)kPfRows * (D.rs + 4) + (size_t)D.ds * D.rs +
                              (size_t)kPfThreads * 16 + 64) * sizeof(float);
    const size_t solve_smem = (2 * (size_t)D.rs * (D.rs + 1) + (size_t)D.rs * D.ds + 64) * sizeof(float);
    dim3 pgrid(D.NB, D.H);
    const bool bf = P.dtype == LRQK_BF16;
    const bool mma = bf && D.ds == kPfD && (D.rs == 16 || D.rs == 32 || D.rs == 64) && pf_mma_enabled();
    auto pass = [&](const void *X, int is_k, float *A, int update, int want_x2) {
        if (mma) {
            const __nv_bfloat16 *Xb = reinterpret_cast<const __nv_bfloat16 *>(X);
#define LRQK_PF_MMA(RSV)                                                                             \
    do {                                                                                             \
        auto fn = pf_pass_mma_kernel<RSV>;                                                           \
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pf_mma_smem<RSV>()); \
        fn<<<pgrid, kPfThreads, pf_mma_smem<RSV>(), st>>>(D, Xb, is_k, A, A, update, want_x2, P.scratch); \
    } while (0)
            if (D.rs == 16) LRQK_PF_MMA(16);
            else if (D.rs == 32) LRQK_PF_MMA(32);
            else LRQK_PF_MMA(64);
#undef LRQK_PF_MMA
        } else if (bf) {
            auto fn = pf_pass_kernel<__nv_bfloat16>;
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pass_smem);
            fn<<<pgrid, kPfThreads, pass_smem, st>>>(D, reinterpret_cast<const __nv_bfloat16 *>(X), is_k, A, A,
                                                    update, want_x2, P.scratch);
        } else {
            auto fn = pf_pass_kernel<float>;
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pass_smem);
            fn<<<pgrid, kPfThreads, pass_smem, st>>>(D, reinterpret_cast<const float *>(X), is_k, A, A, update,
                                                    want_x2, P.scratch);
        }
    };
    cudaFuncSetAttribute(pf_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)solve_smem);
    if (P.want_objective) {
        float *gbase = P.scratch + (size_t)D.H * D.head_sz;
        float *gq = gbase, *gk = gbase + (size_t)D.H * D.ds * D.ds;
        const int nk = D.H / D.group;
        if (bf) {
            pf_gram_dd_kernel<__nv_bfloat16><<<dim3(D.ds, D.H), 128, 0, st>>>(D, reinterpret_cast<const __nv_bfloat16 *>(P.Q), D.H, gq);
            pf_gram_dd_kernel<__nv_bfloat16><<<dim3(D.ds, nk), 128, 0, st>>>(D, reinterpret_cast<const __nv_bfloat16 *>(P.K), nk, gk);
        } else {
            pf_gram_dd_kernel<float><<<dim3(D.ds, D.H), 128, 0, st>>>(D, reinterpret_cast<const float *>(P.Q), D.H, gq);
            pf_gram_dd_kernel<float><<<dim3(D.ds, nk), 128, 0, st>>>(D, reinterpret_cast<const float *>(P.K), nk, gk);
        }
        pf_qk2_kernel<<<D.H, 256, 0, st>>>(D, gq, gk, P.scratch);
    }
    // init passes: reductions of the initial A's
    pass(P.Q, 0, P.A_Q, 0, 1);
    pf_solve_kernel<<<D.H, kPfThreads, solve_smem, st>>>(D, P, 3, 0);
    pass(P.K, 1, P.A_K, 0, 1);
    pf_solve_kernel<<<D.H, kPfThreads, solve_smem, st>>>(D, P, 4, 0);
    for (int s = 0; s < P.max_iter; ++s) {
        pass(P.K, 1, P.A_K, 1, 0);
        pf_solve_kernel<<<D.H, kPfThreads, solve_smem, st>>>(D, P, 1, s);
        pass(P.Q, 0, P.A_Q, 1, 0);
        pf_solve_kernel<<<D.H, kPfThreads, solve_smem, st>>>(D, P, 2, s);
    }
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

}  // namespace lrqk
