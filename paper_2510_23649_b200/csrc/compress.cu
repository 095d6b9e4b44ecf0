// K2: per-token compression (q_hat, k_hat), B line-search update and the
// append of (k_hat -> proxy store, k/v -> slow tier / slot).
//
// ref: decode.py:79-184 (khat_initial_guess, update_qhat, update_khat,
//      decode_compress, _line_search_step, update_projections),
//      cache.py:199-214 (append_token), session.py:95-98 (order).
//
// The reference solves, per token (decode.py:84-119),
//     q_hat = solve(P + l1 k_hat^T k_hat,  q B_Q^T + l1 qk k_hat + l2 (q K_res^T) A_res)
//     k_hat = solve(R + l1 q_hat^T q_hat,  k B_K^T + l1 qk q_hat)
// with P = B_Q B_Q^T + l2 A_res^T A_res and R = B_K B_K^T.  Everything in
// those systems except q, k themselves is fixed once step t-1 has finished
// (its selection Omega_{t-1} and its B update), because
//     (q K_res^T) A_res = q (A_res^T K_res)^T = q Y^T.
// So the work is split in two kernels:
//   compress_prepare (K2p, after step t-1's selection; off the critical
//     path, on a side stream in the captured engine step):
//       Y = A_res^T K_res, G = A_res^T A_res over Omega_{t-1};
//       P, R, their inverses (Gauss-Jordan; P, R kept for the fallback);
//       W = B_Q + l2 Y,  Z_Q = P^-1 W,  Z_K = R^-1 B_K.
//   compress (K2c, per token, critical path):
//       y_q = q Z_Q^T = m P^-1 (m = q W^T),  y_k = k Z_K^T = k_hat0 (decode.py:79-81),
//       then the alternation through the closed form of the rank-1-updated
//       systems  x (S + l1 v^T v) = b + l1 qk v
//           =>   x = y + u * l1 (qk - y.v) / (1 + l1 v.u),   u = v S^-1,
//       the exact line-search B update and the appends.
// Algebraically this is the reference's computation; the Gauss-Jordan sweep
// (no pivoting) succeeds exactly when the matrix is numerically SPD, i.e.
// when the reference's Cholesky does.  If P or R is not SPD, K2c solves each
// full system directly with the reference's jitter retry (linalg.py:80-91).
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "mma_common.cuh"

namespace lrqk {

constexpr int kCompressThreads = 256;
constexpr int kSub = 64;  // rows staged per sub-chunk in the prepare reduction

struct CompressArgs {
    lrqk_layer_t L;
    const void *q, *k, *v;
    int update_b;
    int defer_b;  // leave the B update to the next compress_prepare (cluster path)
};

// Per-head precompute ("pre" buffer) written by K2p, read by K2c.
struct PreLayout {
    int Pinv, Rinv, P, R, ZQ, ZK, W, flags, X, total;
};
__host__ __device__ inline PreLayout pre_layout(int R, int d) {
    PreLayout p;
    int o = 0;
    p.Pinv = o; o += R * R;
    p.Rinv = o; o += R * R;
    p.P = o; o += R * R;
    p.R = o; o += R * R;
    p.ZQ = o; o += R * d;
    p.ZK = o; o += R * d;
    p.W = o; o += R * d;
    p.flags = o; o += 4;   // okP, okR, B update pending
    p.X = o; o += 2 * d + 2 * R;  // deferred B update: q, k, q_hat, k_hat of the step
    p.total = (o + 3) & ~3;
    return p;
}
struct PreLayoutOrder {  // compress_kernel bulk-copies Pinv|Rinv and ZQ|ZK as pairs
    static constexpr bool kPairs = true;
};
// Per-head reduction scratch of K2p: chunk partials [Y (R*d) | G (R*R)] + the
// prep block's B_Q B_Q^T.
__host__ __device__ inline int compress_chunks_dev(const lrqk_layer_t &L) { return (L.s_cap + kRedRows - 1) / kRedRows; }
__host__ __device__ inline size_t red_head_floats(int R, int d, int nchunks) {
    return (size_t)nchunks * (R * d + R * R) + R * R;
}

// ---------------------------------------------------------------------------
// Block-wide Gauss-Jordan inverse of an R x R SPD matrix in shared memory
// (R = rank_stride, a power of two; rows/columns beyond the true rank hold
// the identity, which leaves the leading block's inverse and its SPD-ness
// unchanged).  Thread t owns E consecutive elements of one row; the matrix
// ping-pongs between b0 and b1 so each pivot costs a single barrier.  No
// pivoting: every pivot is > 0 exactly when the matrix is numerically SPD,
// i.e. when the reference's Cholesky succeeds (linalg.py:81).  Returns false
// (block-uniformly) otherwise.  R is even, so the inverse ends up in b0.
// ---------------------------------------------------------------------------
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
        if (!(p > 0.f) || !isfinite(p)) return false;  // block-uniform
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
    if (act) {
#pragma unroll
        for (int e = 0; e < E; ++e) M[i * ld + c0 + e] = own[e];
    }
    __syncthreads();
    return true;
}

// In-place inverse of the padded R x R matrix in M (row stride ld); on
// failure M is left in an undefined state.
__device__ bool block_gj(float *M, int R, int ld, float *s_rc) {
    const int nn = R * R;
    if (nn >= 16 * kCompressThreads) return block_gj_t<16>(M, R, ld, s_rc);
    if (nn >= 4 * kCompressThreads) return block_gj_t<4>(M, R, ld, s_rc);
    return block_gj_t<1>(M, R, ld, s_rc);
}

// Both inverses of the finish kernel (R and P) in one Gauss-Jordan sweep:
// one barrier per pivot for the pair.  s_rc: 512 floats.  ok[m] is
// block-uniform; a failed matrix stops updating, the other goes on.
template <int E>
__device__ void block_gj2_t(float *M0, float *M1, int R, int ld, float *s_rc, bool (&ok)[2]) {
    const int tid = threadIdx.x;
    const int e0 = tid * E;
    const bool act = e0 < R * R;
    const int i = act ? e0 / R : 0, c0 = act ? e0 - (e0 / R) * R : 0;
    float own[2][E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        own[0][e] = act ? M0[i * ld + c0 + e] : 0.f;
        own[1][e] = act ? M1[i * ld + c0 + e] : 0.f;
    }
    ok[0] = ok[1] = true;
    __syncthreads();
    for (int k = 0; k < R; ++k) {
        float *buf = s_rc + (k & 1) * 256;  // [m][row 64 | col 64]
        if (act) {
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                if (i == k) {
#pragma unroll
                    for (int e = 0; e < E; ++e) buf[m * 128 + c0 + e] = own[m][e];
                }
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if (c0 + e == k) buf[m * 128 + 64 + i] = own[m][e];
            }
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            const float *rowb = buf + m * 128, *colb = rowb + 64;
            const float p = rowb[k];
            if (!(p > 0.f) || !isfinite(p)) ok[m] = false;  // block-uniform
            if (act && ok[m]) {
                const float ip = __frcp_rn(p);
                const float f = colb[i] * ip;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int j = c0 + e;
                    const float piv = rowb[j];
                    if (i == k) own[m][e] = (j == k) ? ip : own[m][e] * ip;
                    else own[m][e] = (j == k) ? -f : fmaf(-f, piv, own[m][e]);
                }
            }
        }
    }
    if (act) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (ok[0]) M0[i * ld + c0 + e] = own[0][e];
            if (ok[1]) M1[i * ld + c0 + e] = own[1][e];
        }
    }
    __syncthreads();
}
__device__ void block_gj2(float *M0, float *M1, int R, int ld, float *s_rc, bool (&ok)[2]) {
    const int nn = R * R;
    if (nn >= 16 * kCompressThreads) block_gj2_t<16>(M0, M1, R, ld, s_rc, ok);
    else if (nn >= 4 * kCompressThreads) block_gj2_t<4>(M0, M1, R, ld, s_rc, ok);
    else block_gj2_t<1>(M0, M1, R, ld, s_rc, ok);
}

// Fill b0 with M (r x r, row stride ldm) + jit on the diagonal, padded with
// the identity to R x R (stride ld).  Whole block; ends with a barrier.
__device__ void fill_padded(float *b0, const float *M, int ldm, int r, int R, int ld, float jit) {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
        const int i = e / R, j = e - i * R;
        float v;
        if (i < r && j < r) v = M[i * ldm + j] + (i == j ? jit : 0.f);
        else v = (i == j) ? 1.f : 0.f;
        b0[i * ld + j] = v;
    }
    __syncthreads();
}

// Solve x M = rhs directly (M SPD r x r) with the reference's single jitter
// retry (linalg.py:80-91).  Returns 0 ok, 1 ok after jitter, 2 failed.
__device__ int solve_spd_direct(const float *M, int ldm, int r, int R, int ld, const float *rhs, float *x,
                                float *b0, float *s_rc) {
    // attempt 0: M as given; then the reference's jitter 1e-10 (tr/r + 1)
    // (linalg.py:83-87), floored at fp32 resolution.  A rank-deficient M that
    // the reference factors in fp64 carries O(n u |M|) rounding in fp32, which
    // can exceed that floor, so the fp32 retry escalates the floor x16 up to
    // three more times (to ~5e-4 dmax) before reporting SolveFailedError.
    for (int attempt = 0; attempt < 5; ++attempt) {
        float jit = 0.f;
        if (attempt >= 1) {
            float tr = 0.f, dmax = 0.f;
            for (int i = 0; i < r; ++i) { tr += M[i * ldm + i]; dmax = fmaxf(dmax, fabsf(M[i * ldm + i])); }
            jit = fmaxf(1e-10f * (tr / r + 1.f), dmax * 1.2e-7f * (float)(1 << (4 * (attempt - 1))));
        }
        fill_padded(b0, M, ldm, r, R, ld, jit);
        if (block_gj(b0, R, ld, s_rc)) {
            for (int j = threadIdx.x; j < r; j += blockDim.x) {
                float acc = 0.f;
                for (int i = 0; i < r; ++i) acc = fmaf(rhs[i], b0[i * ld + j], acc);
                x[j] = acc;
            }
            __syncthreads();
            return attempt ? 1 : 0;
        }
    }
    return 2;
}

// Stage a [rows][d] fp32 matrix from global into shared (row stride ldx,
// d and ldx multiples of 4) with all loads of a thread issued together.
__device__ void stage_rows_f32(float *dst, int ldx, const float *src, int rows, int d) {
    const int n4 = rows * d / 4;
    const float4 *s4 = reinterpret_cast<const float4 *>(src);
    constexpr int U = 8;
    const int d4 = d / 4;
    if ((int)blockDim.x % d4 == 0) {  // fixed column per thread: no divisions in the loop
        const int c = (int)threadIdx.x % d4, rstep = blockDim.x / d4;
        for (int p0 = threadIdx.x / d4; p0 < rows; p0 += rstep * U) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (p0 + u * rstep < rows) v[u] = __ldcg(s4 + (p0 + u * rstep) * d4 + c);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (p0 + u * rstep < rows) *reinterpret_cast<float4 *>(dst + (p0 + u * rstep) * ldx + c * 4) = v[u];
        }
        return;
    }
    for (int base = threadIdx.x; base < n4; base += blockDim.x * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = base + u * blockDim.x;
            if (e < n4) v[u] = __ldcg(s4 + e);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = base + u * blockDim.x;
            if (e < n4) {
                const int p = (e * 4) / d, i = e * 4 - p * d;
                *reinterpret_cast<float4 *>(dst + p * ldx + i) = v[u];
            }
        }
    }
}

// y[j] = sum_i v[i] * S[i*ld + j]   (one warp, n <= 64)
LRQK_DEV void warp_vecmat(const float *v, const float *S, int n, int ld, float *y) {
    const int lane = threadIdx.x & 31;
    for (int j = lane; j < n; j += 32) {
        float acc0 = 0.f, acc1 = 0.f;
        int i = 0;
        for (; i + 1 < n; i += 2) {
            acc0 = fmaf(v[i], S[i * ld + j], acc0);
            acc1 = fmaf(v[i + 1], S[(i + 1) * ld + j], acc1);
        }
        if (i < n) acc0 = fmaf(v[i], S[i * ld + j], acc0);
        y[j] = acc0 + acc1;
    }
    __syncwarp();
}
LRQK_DEV float warp_dot(const float *a, const float *b, int n) {
    const int lane = threadIdx.x & 31;
    float acc = 0.f;
    for (int j = lane; j < n; j += 32) acc = fmaf(a[j], b[j], acc);
    return warp_sum(acc);
}

// X X^T for X (r x d in shared, row stride ldx) through upper-triangular
// 4x4 register tiles, each tile's d range split in two; result mirrored into
// out (row stride ldo) so it is exactly symmetric (linalg.py:53-54).
__device__ void gram_rows(const float *X, int r, int d, int ldx, float *out, int ldo, float *tmp) {
    const int RB = (r + 3) / 4;
    const int NP = RB * (RB + 1) / 2;
    const int halves = (2 * NP <= (int)blockDim.x) ? 2 : 1;
    const int dh = d / halves;
    for (int w = threadIdx.x; w < NP * halves; w += blockDim.x) {
        const int pair = w % NP, hf = w / NP;
        int pb = 0, rem = pair;
        while (rem >= RB - pb) { rem -= RB - pb; ++pb; }
        const int qb = pb + rem;
        float acc[16] = {};
        const int i0 = hf * dh, i1 = i0 + dh;
        for (int i = i0; i < i1; ++i) {
            float xp[4], xq[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                xp[u] = (pb * 4 + u < r) ? X[(pb * 4 + u) * ldx + i] : 0.f;
                xq[u] = (qb * 4 + u < r) ? X[(qb * 4 + u) * ldx + i] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u * 4 + v] = fmaf(xp[u], xq[v], acc[u * 4 + v]);
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) tmp[(hf * NP + pair) * 16 + e] = acc[e];
    }
    __syncthreads();
    for (int w = threadIdx.x; w < NP * 16; w += blockDim.x) {
        const int pair = w / 16, uv = w - pair * 16;
        int pb = 0, rem = pair;
        while (rem >= RB - pb) { rem -= RB - pb; ++pb; }
        const int qb = pb + rem;
        const int p = pb * 4 + uv / 4, q = qb * 4 + (uv & 3);
        float s = tmp[pair * 16 + uv];
        if (halves == 2) s += tmp[(NP + pair) * 16 + uv];
        if (p < r && q < r && (pb < qb || p <= q)) {
            out[p * ldo + q] = s;
            out[q * ldo + p] = s;
        }
    }
    __syncthreads();
}

// The two grams X0 X0^T and X1 X1^T in one pass (one barrier pair, twice the
// threads busy); tmp holds 4 * NP * 16 floats.
__device__ void gram_rows2(const float *X0, const float *X1, int r, int d, int ldx, float *out0, float *out1, int ldo,
                           float *tmp) {
    const int RB = (r + 3) / 4;
    const int NP = RB * (RB + 1) / 2;
    const int halves = (4 * NP <= (int)blockDim.x) ? 2 : 1;
    const int dh = d / halves;
    for (int w = threadIdx.x; w < 2 * NP * halves; w += blockDim.x) {
        const int mat = w / (NP * halves), w2 = w - mat * NP * halves;
        const int pair = w2 % NP, hf = w2 / NP;
        const float *X = mat ? X1 : X0;
        int pb = 0, rem = pair;
        while (rem >= RB - pb) { rem -= RB - pb; ++pb; }
        const int qb = pb + rem;
        float acc[16] = {};
        const int i0 = hf * dh, i1 = i0 + dh;
#pragma unroll 4
        for (int i = i0; i < i1; ++i) {
            float xp[4], xq[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                xp[u] = (pb * 4 + u < r) ? X[(pb * 4 + u) * ldx + i] : 0.f;
                xq[u] = (qb * 4 + u < r) ? X[(qb * 4 + u) * ldx + i] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u * 4 + v] = fmaf(xp[u], xq[v], acc[u * 4 + v]);
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) tmp[((mat * halves + hf) * NP + pair) * 16 + e] = acc[e];
    }
    __syncthreads();
    for (int w = threadIdx.x; w < 2 * NP * 16; w += blockDim.x) {
        const int mat = w / (NP * 16), w2 = w - mat * NP * 16;
        const int pair = w2 / 16, uv = w2 - pair * 16;
        int pb = 0, rem = pair;
        while (rem >= RB - pb) { rem -= RB - pb; ++pb; }
        const int qb = pb + rem;
        const int p = pb * 4 + uv / 4, q = qb * 4 + (uv & 3);
        float sv = tmp[(mat * halves * NP + pair) * 16 + uv];
        if (halves == 2) sv += tmp[((mat * 2 + 1) * NP + pair) * 16 + uv];
        float *out = mat ? out1 : out0;
        if (p < r && q < r && (pb < qb || p <= q)) {
            out[p * ldo + q] = sv;
            out[q * ldo + p] = sv;
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// K2p reduce on tensor cores (bf16 storage): per 64-row sub-chunk of Omega,
//     Y += A_sub^T K_sub   (M = r, N = d, K = 64)      G += A_sub^T A_sub
// with mma.sync m16n8k16 bf16 x bf16 -> fp32.  Products of bf16 values are
// exact in fp32, so this equals the fp32 CUDA-core accumulation up to
// summation order.  Rows are gathered into shared memory with cp.async
// (16-byte LDGSTS) into two buffers, so the next sub-chunk's gather overlaps
// the current sub-chunk's MMAs; fragments come from ldmatrix.trans.
// ---------------------------------------------------------------------------

__device__ void prepare_reduce_mma(const lrqk_layer_t &L, int bh, int row0, int nrow, const __nv_bfloat16 *kbase,
                                   const __nv_bfloat16 *proxy, bool host, float *part, uint8_t *smem,
                                   int *s_ridx = nullptr, int *s_rproxy = nullptr, int nbuf = 2) {
    const int d = L.dim_stride, R = L.rank_stride;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ldk = d * 2 + 16, lda = R * 2 + 16;  // bytes
    const int stage = mma_stage_bytes(R, d);
    // the proxy rows from the row-major copy when the layer keeps one
    const __nv_bfloat16 *arows = L.proxy_rowmajor
        ? reinterpret_cast<const __nv_bfloat16 *>(L.proxy_rowmajor) + (size_t)bh * L.t_max * R : nullptr;
    const int *ridx = L.res_idx + (size_t)bh * L.s_cap + row0;
    const int *rslot = L.res_slot + (size_t)bh * L.s_cap + row0;
    const int MT = R / 16;            // m tiles (rank rows)
    const int NTW = d / 64;           // n tiles of 8 columns per warp (d / 8 / 8 warps)
    const int GT = (R / 16) * (R / 8);  // G tiles
    float yacc[4][4][4];              // [m tile][n tile of this warp][frag]
    float gacc[4][4];                 // up to 4 G tiles per warp
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b2 = 0; b2 < 4; ++b2)
#pragma unroll
            for (int c = 0; c < 4; ++c) { yacc[a][b2][c] = 0.f; gacc[a][c] = 0.f; }
    const int nsub = (nrow + kMmaRows - 1) / kMmaRows;
    if (s_ridx != nullptr) {  // this slice's row indices, one round trip
        for (int j = tid; j < nrow; j += blockDim.x) s_ridx[j] = host ? rslot[j] : ridx[j];
        if (host) for (int j = tid; j < nrow; j += blockDim.x) s_rproxy[j] = ridx[j];
        __syncthreads();
        trace(17);
    }
    auto issue = [&](int sub) {
        uint8_t *buf = smem + (sub % nbuf) * stage;
        uint8_t *kb_s = buf, *ab_s = buf + kMmaRows * ldk;
        const int s0 = sub * kMmaRows;
        const int ns = min(kMmaRows, nrow - s0);
        const int kp = d / 8, ap = R / 8;  // 16-byte packs per row
        for (int e = tid; e < kMmaRows * (kp + ap); e += blockDim.x) {
            if (e < kMmaRows * kp) {
                const int j = e / kp, pk = e - j * kp;
                if (j < ns) {
                    const int src = s_ridx ? s_ridx[s0 + j] : (host ? rslot[s0 + j] : ridx[s0 + j]);
                    cp_async16(kb_s + j * ldk + pk * 16, kbase + (size_t)src * d + pk * 8);
                } else {
                    *reinterpret_cast<uint4 *>(kb_s + j * ldk + pk * 16) = make_uint4(0, 0, 0, 0);
                }
            } else {
                const int e2 = e - kMmaRows * kp;
                const int j = e2 / ap, pk = e2 - j * ap;
                if (j < ns) {
                    const int x = s_ridx ? (host ? s_rproxy[s0 + j] : s_ridx[s0 + j]) : ridx[s0 + j];
                    cp_async16(ab_s + j * lda + pk * 16,
                               arows ? arows + (size_t)x * R + pk * 8 : proxy + proxy_pack_offset(x, pk, ap) * 8);
                }
                else *reinterpret_cast<uint4 *>(ab_s + j * lda + pk * 16) = make_uint4(0, 0, 0, 0);
            }
        }
        cp_async_commit();
    };
    // nbuf - 1 sub-chunk gathers stay in flight: the gather of sub + nbuf - 1
    // goes out as soon as sub's data has landed, into the buffer freed by sub - 1
    for (int sub = 0; sub < min(nbuf - 1, nsub); ++sub) issue(sub);
    for (int sub = 0; sub < nsub; ++sub) {
        const int ahead = min(nsub - sub - 1, nbuf - 2);  // groups allowed to stay pending
        if (ahead >= 2) cp_async_wait<2>();
        else if (ahead == 1) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncthreads();
        if (sub + nbuf - 1 < nsub) issue(sub + nbuf - 1);
        if (sub == 0) trace(18);
        const uint8_t *buf = smem + (sub % nbuf) * stage;
        const uint8_t *kb_s = buf, *ab_s = buf + kMmaRows * ldk;
        const int q = lane >> 3, i8 = lane & 7;
#pragma unroll
        for (int ks = 0; ks < kMmaRows; ks += 16) {
            // A fragments (A_mat[m][k] = A_sm[k][m]) for every m tile
            uint32_t af[4][4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                if (mt >= MT) break;
                const int m0 = mt * 16 + ((q & 1) ? 8 : 0), k0 = ks + ((q & 2) ? 8 : 0);
                ldsm_x4_trans(af[mt], ab_s + (k0 + i8) * lda + m0 * 2);
            }
            // Y: this warp's n tiles (columns warp*8*NTW ...)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                if (nt >= NTW) break;
                const int n0 = (warp * NTW + nt) * 8;
                uint32_t bfr[2];
                const int k0 = ks + ((lane >> 3) & 1) * 8;  // lanes 0-7: k 0-7, 8-15: k 8-15
                ldsm_x2_trans(bfr, kb_s + (k0 + i8) * ldk + n0 * 2);
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) {
                    if (mt >= MT) break;
                    mma_bf16_16816(yacc[mt][nt], af[mt], bfr);
                }
            }
            // G tiles owned by this warp: tile g = warp + 8*w2
#pragma unroll
            for (int w2 = 0; w2 < 4; ++w2) {
                const int gtile = warp + 8 * w2;
                if (gtile >= GT) break;
                const int mt = gtile / (R / 8), n0 = (gtile % (R / 8)) * 8;
                uint32_t bfr[2];
                const int k0 = ks + ((lane >> 3) & 1) * 8;
                ldsm_x2_trans(bfr, ab_s + (k0 + i8) * lda + n0 * 2);
                mma_bf16_16816(gacc[w2], af[mt], bfr);
            }
        }
        __syncthreads();
    }
    trace(19);
    // accumulator fragments -> partial (Y row-major R x d, then G R x R)
    const int fr = lane >> 2, fc = (lane & 3) * 2;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
        if (mt >= MT) break;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            if (nt >= NTW) break;
            const int n0 = (warp * NTW + nt) * 8;
            float *y = part + (mt * 16 + fr) * d + n0 + fc;
            *reinterpret_cast<float2 *>(y) = make_float2(yacc[mt][nt][0], yacc[mt][nt][1]);
            *reinterpret_cast<float2 *>(y + 8 * d) = make_float2(yacc[mt][nt][2], yacc[mt][nt][3]);
        }
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

// ---------------------------------------------------------------------------
// Hit/miss accounting of the HBM policy (cache.py:190-195, 63-74), off the
// decode critical path: compress_prepare runs after the step's selection on
// a side stream.  res_bits holds the fast tier before the fetch, Omega_{t-1};
// the new token t is never in it, so
//     hits = 1 + #{x in Omega_t : x in Omega_{t-1}},  miss = |Omega_t| - hits,
// then res_bits becomes Omega_t.  After lrqk_seed_prompt the bitmap already
// equals Omega (M_BITS_FRESH) and nothing is counted.
// ---------------------------------------------------------------------------
__device__ void count_hits_hbm(const lrqk_layer_t &L, int bh, int n, float *scratch) {
    int *meta = L.sel_meta + (size_t)bh * kMetaInts;
    const int words = (L.t_max + 31) >> 5;
    uint32_t *bits = L.res_bits + (size_t)bh * words;
    const int *idx = L.res_idx + (size_t)bh * L.s_cap;
    __syncthreads();
    const bool fresh = meta[M_BITS_FRESH] != 0;
    // every thread has read the flag before thread 0 may clear it below
    // (compute-sanitizer synccheck caught warps taking different branches)
    __syncthreads();
    if (!fresh) {
        // all index loads of a thread in flight together, then the bit loads
        constexpr int UH = 8;
        int hit = 0;
        for (int i0 = 0; i0 < n; i0 += blockDim.x * UH) {
            int xs[UH];
            uint32_t ws[UH];
#pragma unroll
            for (int u = 0; u < UH; ++u) {
                const int i = i0 + u * blockDim.x + threadIdx.x;
                xs[u] = i < n ? __ldcg(idx + i) : -1;
            }
#pragma unroll
            for (int u = 0; u < UH; ++u) ws[u] = xs[u] >= 0 ? __ldcg(bits + (xs[u] >> 5)) : 0u;
#pragma unroll
            for (int u = 0; u < UH; ++u) hit += xs[u] >= 0 ? (int)((ws[u] >> (xs[u] & 31)) & 1u) : 0;
        }
        int *s_red = reinterpret_cast<int *>(scratch);
        int hits;
        block_exclusive_scan(hit, s_red, &hits);
        for (int w = threadIdx.x; w < words; w += blockDim.x) bits[w] = 0u;
        __syncthreads();
        if (threadIdx.x == 0) {
            const int miss = n - (hits + 1);
            L.c_miss[bh] += miss;
            L.c_total[bh] += n;
            L.step_miss[bh] = miss;
            L.step_total[bh] = n;
        }
        for (int i0 = 0; i0 < n; i0 += blockDim.x * UH) {
            int xs[UH];
#pragma unroll
            for (int u = 0; u < UH; ++u) {
                const int i = i0 + u * blockDim.x + threadIdx.x;
                xs[u] = i < n ? __ldcg(idx + i) : -1;
            }
#pragma unroll
            for (int u = 0; u < UH; ++u)
                if (xs[u] >= 0) atomicOr(bits + (xs[u] >> 5), 1u << (xs[u] & 31));
        }
    } else if (threadIdx.x == 0) {
        meta[M_BITS_FRESH] = 0;
    }
}

// ---------------------------------------------------------------------------
// K2p: compress_prepare
// ---------------------------------------------------------------------------
template <typename T> constexpr bool kUseMma = false;
template <> constexpr bool kUseMma<__nv_bfloat16> = true;

template <typename T>
__global__ void __launch_bounds__(kCompressThreads, 2)
prepare_kernel(const lrqk_layer_t L) {
    extern __shared__ __align__(16) float smem[];
    __shared__ int s_flag;
    __shared__ float s_rc[256];
    const int bh = blockIdx.y;
    const int b = bh / L.n_q_heads, h = bh - b * L.n_q_heads;
    const int G = L.n_q_heads / L.n_kv_heads, g = h / G;
    const int d = L.dim_stride, R = L.rank_stride, r = L.rank;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int nchunks = gridDim.x - 1;
    const int n_prev = L.res_cnt[bh];
    const bool host = L.policy == LRQK_SLOW_HOST;
    const size_t kv_rows = ((size_t)b * L.n_kv_heads + g) * L.t_max;
    const T *proxy = reinterpret_cast<const T *>(L.proxy) + (size_t)bh * L.t_max * R;
    const T *arows = L.proxy_rowmajor ? reinterpret_cast<const T *>(L.proxy_rowmajor) + (size_t)bh * L.t_max * R
                                      : nullptr;
    const T *kbase = host ? reinterpret_cast<const T *>(L.slot_k) + (size_t)bh * L.n_slots * d
                          : reinterpret_cast<const T *>(L.slow_k) + kv_rows * d;
    float *hs = L.red_scratch + (size_t)bh * red_head_floats(R, d, nchunks);
    float *pre = L.pre + (size_t)bh * pre_layout(R, d).total;
    const PreLayout PL = pre_layout(R, d);
    const float *BQg = L.B_Q + (size_t)bh * R * d;
    const float *BKg = L.B_K + (size_t)bh * R * d;
    const int ldB = d + 4, ldM = R + 4;
    constexpr int N = Pack<T>::N;

    trace(10);
    if ((int)blockIdx.x < nchunks && kUseMma<T> && R >= 16 && d >= 64) {
        const int row0 = blockIdx.x * kRedRows;
        const int nrow = max(0, min(kRedRows, n_prev - row0));
        prepare_reduce_mma(L, bh, row0, nrow, reinterpret_cast<const __nv_bfloat16 *>(kbase),
                           reinterpret_cast<const __nv_bfloat16 *>(proxy), host,
                           hs + (size_t)blockIdx.x * (R * d + R * R), reinterpret_cast<uint8_t *>(smem));
        trace(11);
    } else if ((int)blockIdx.x < nchunks) {
        // ---- reduce: Y = A^T K and G = A^T A over this chunk of Omega ------
        const int row0 = blockIdx.x * kRedRows;
        const int nrow = max(0, min(kRedRows, n_prev - row0));
        const int ldA = R + 4;
        float *sK = smem;                    // [kSub][ldB]
        float *sA = sK + kSub * ldB;         // [kSub][ldA]
        float *sRed = sA + kSub * ldA;       // gram groups
        const int *ridx = L.res_idx + (size_t)bh * L.s_cap + row0;
        const int *rslot = L.res_slot + (size_t)bh * L.s_cap + row0;
        // Y = A^T K: 8 (p) x 4 (i) register tiles; rows split over RG groups
        const int ntl = (R / 8) * (d / 4);
        const int RG = ntl >= kCompressThreads ? 1 : kCompressThreads / ntl;
        const int tgrp = tid / ntl;                  // row group (RG > 1)
        float yacc[2][32];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int e = 0; e < 32; ++e) yacc[a][e] = 0.f;
        const int RB = R / 4, NP = RB * (RB + 1) / 2;
        const int NG = max(1, kCompressThreads / NP);
        float gacc[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) gacc[e] = 0.f;
        for (int s0 = 0; s0 < nrow; s0 += kSub) {
            const int ns = min(kSub, nrow - s0);
            __syncthreads();
            // stage K rows and A rows (all loads of a thread issued together)
            const int kp = d / N, ap = R / N;
            const int tot = ns * (kp + ap);
            constexpr int U = 8;
            for (int base = tid; base < tot; base += kCompressThreads * U) {
                uint4 v[U];
                int dst[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int e = base + u * kCompressThreads;
                    dst[u] = -1;
                    if (e < tot) {
                        if (e < ns * kp) {
                            const int j = e / kp, pk = e - j * kp;
                            const int src = host ? rslot[s0 + j] : ridx[s0 + j];
                            v[u] = *reinterpret_cast<const uint4 *>(kbase + (size_t)src * d + pk * N);
                            dst[u] = j * ldB + pk * N;
                        } else {
                            const int e2 = e - ns * kp;
                            const int j = e2 / ap, pk = e2 - j * ap;
                            v[u] = *reinterpret_cast<const uint4 *>(
                                arows ? arows + (size_t)ridx[s0 + j] * R + pk * N
                                      : proxy + proxy_pack_offset(ridx[s0 + j], pk, ap) * N);
                            dst[u] = (1 << 30) | (j * ldA + pk * N);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (dst[u] < 0) continue;
                    float x[N];
                    unpack16<T>(v[u], x);
                    float *o = (dst[u] & (1 << 30)) ? sA + (dst[u] & ~(1 << 30)) : sK + dst[u];
#pragma unroll
                    for (int i = 0; i < N; ++i) o[i] = x[i];
                }
            }
            __syncthreads();
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const int tI = (RG > 1) ? tid % ntl : tid + a * kCompressThreads;
                if ((RG > 1 && a > 0) || tI >= ntl) break;
                const int p0 = (tI / (d / 4)) * 8, i0 = (tI % (d / 4)) * 4;
                for (int j = (RG > 1 ? tgrp : 0); j < ns; j += RG) {
                    const float4 kv = *reinterpret_cast<const float4 *>(sK + j * ldB + i0);
                    const float4 a0 = *reinterpret_cast<const float4 *>(sA + j * ldA + p0);
                    const float4 a1 = *reinterpret_cast<const float4 *>(sA + j * ldA + p0 + 4);
                    const float ks[4] = {kv.x, kv.y, kv.z, kv.w};
                    const float as[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
                    for (int u = 0; u < 8; ++u)
#pragma unroll
                        for (int w2 = 0; w2 < 4; ++w2) yacc[a][u * 4 + w2] = fmaf(as[u], ks[w2], yacc[a][u * 4 + w2]);
                }
            }
            // G += A^T A (upper 4x4 tiles, row groups)
            if (tid < NP * NG) {
                const int pair = tid % NP, grp = tid / NP;
                int pb = 0, rem = pair;
                while (rem >= RB - pb) { rem -= RB - pb; ++pb; }
                const int qb = pb + rem;
                for (int j = grp; j < ns; j += NG) {
                    const float *arow = sA + j * ldA;
                    float a4[4], b4[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) { a4[u] = arow[pb * 4 + u]; b4[u] = arow[qb * 4 + u]; }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int w2 = 0; w2 < 4; ++w2) gacc[u * 4 + w2] = fmaf(a4[u], b4[w2], gacc[u * 4 + w2]);
                }
            }
        }
        trace(11);
        float *part = hs + (size_t)blockIdx.x * (R * d + R * R);
        if (RG == 1) {
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const int tI = tid + a * kCompressThreads;
                if (tI >= ntl) break;
                const int p0 = (tI / (d / 4)) * 8, i0 = (tI % (d / 4)) * 4;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    *reinterpret_cast<float4 *>(part + (p0 + u) * d + i0) =
                        make_float4(yacc[a][u * 4], yacc[a][u * 4 + 1], yacc[a][u * 4 + 2], yacc[a][u * 4 + 3]);
            }
        } else {
            // sum the RG row groups through shared memory (reuses the staging area)
            __syncthreads();
            float *red = smem;  // [RG][R*d]
            const int tI = tid % ntl;
            const int p0 = (tI / (d / 4)) * 8, i0 = (tI % (d / 4)) * 4;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                *reinterpret_cast<float4 *>(red + (size_t)tgrp * R * d + (p0 + u) * d + i0) =
                    make_float4(yacc[0][u * 4], yacc[0][u * 4 + 1], yacc[0][u * 4 + 2], yacc[0][u * 4 + 3]);
            __syncthreads();
            for (int e4 = tid; e4 < R * d / 4; e4 += kCompressThreads) {
                float4 acc = reinterpret_cast<const float4 *>(red)[e4];
                for (int gI = 1; gI < RG; ++gI) {
                    const float4 v = reinterpret_cast<const float4 *>(red + (size_t)gI * R * d)[e4];
                    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
                }
                reinterpret_cast<float4 *>(part)[e4] = acc;
            }
        }
        __syncthreads();
        if (tid < NP * NG) {
#pragma unroll
            for (int e = 0; e < 16; ++e) sRed[tid * 16 + e] = gacc[e];
        }
        __syncthreads();
        for (int e = tid; e < NP * 16; e += kCompressThreads) {
            float acc = 0.f;
            for (int gI = 0; gI < NG; ++gI) acc += sRed[(gI * NP) * 16 + e];
            const int pair = e / 16, uw = e - pair * 16;
            int pb = 0, rem = pair;
            while (rem >= RB - pb) { rem -= RB - pb; ++pb; }
            const int qb = pb + rem;
            part[R * d + (pb * 4 + uw / 4) * R + qb * 4 + (uw & 3)] = acc;  // tiles with pb <= qb
        }
    } else {
        // ---- prep: R = B_K B_K^T, R^-1, Z_K = R^-1 B_K, B_Q B_Q^T -----------
        float *sBQ = smem;                   // [R][ldB]
        float *sBK = sBQ + R * ldB;          // [R][ldB]
        float *b0 = sBK + R * ldB;           // [R][ldM]
        float *tmp = b0 + R * ldM;           // gram scratch
        stage_rows_f32(sBQ, ldB, BQg, R, d);
        stage_rows_f32(sBK, ldB, BKg, R, d);
        for (int e = tid; e < R * R; e += blockDim.x) {  // identity padding
            const int i = e / R, j = e - i * R;
            if (i >= r || j >= r) b0[i * ldM + j] = (i == j) ? 1.f : 0.f;
        }
        __syncthreads();
        gram_rows(sBK, r, d, ldB, b0, ldM, tmp);                       // R (exactly symmetric)
        gram_rows(sBQ, r, d, ldB, hs + (size_t)nchunks * (R * d + R * R), R, tmp);  // B_Q B_Q^T
        for (int e = tid; e < R * R; e += blockDim.x) {
            const int i = e / R, j = e - i * R;
            pre[PL.R + e] = (i < r && j < r) ? b0[i * ldM + j] : 0.f;
        }
        __syncthreads();
        const bool ok = block_gj(b0, R, ldM, s_rc);
        if (ok) {
            for (int e = tid; e < R * R; e += blockDim.x) {
                const int i = e / R, j = e - i * R;
                pre[PL.Rinv + e] = (i < r && j < r) ? b0[i * ldM + j] : 0.f;
            }
            // Z_K = R^-1 B_K  (r x d)
            for (int e = tid; e < R * d; e += blockDim.x) {
                const int p = e / d, i = e - p * d;
                float acc = 0.f;
                if (p < r)
                    for (int q = 0; q < r; ++q) acc = fmaf(b0[p * ldM + q], sBK[q * ldB + i], acc);
                pre[PL.ZK + e] = acc;
            }
        }
        if (tid == 0) pre[PL.flags + 1] = ok ? 1.f : 0.f;
        if (!host) count_hits_hbm(L, bh, n_prev, s_rc);
    }
    trace((int)blockIdx.x < nchunks ? 12 : 13);
    if (!last_arrival(L.counters + (size_t)bh * kCounterInts + C_PREPARE, gridDim.x, &s_flag)) return;
    trace(14);

    // ---- finish: P, P^-1, W, Z_Q ---------------------------------------------
    float *sW = smem;                    // [R][ldB]   W = B_Q + l2 Y
    float *b0 = sW + R * ldB;            // [R][ldM]
    const float l2 = L.lambda_2;
    const bool have_res = n_prev > 0;
    {
        const float4 *bq4 = reinterpret_cast<const float4 *>(BQg);
        const int n4 = R * d / 4;
        for (int e4 = tid; e4 < n4; e4 += blockDim.x) {
            float4 acc = __ldcg(bq4 + e4);
            if (have_res) {
                float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int ch = 0; ch < nchunks; ++ch) {
                    const float4 v = __ldcg(reinterpret_cast<const float4 *>(hs + (size_t)ch * (R * d + R * R)) + e4);
                    y.x += v.x; y.y += v.y; y.z += v.z; y.w += v.w;
                }
                acc.x = fmaf(l2, y.x, acc.x); acc.y = fmaf(l2, y.y, acc.y);
                acc.z = fmaf(l2, y.z, acc.z); acc.w = fmaf(l2, y.w, acc.w);
            }
            const int p = (e4 * 4) / d, i = e4 * 4 - p * d;
            *reinterpret_cast<float4 *>(sW + p * ldB + i) = acc;
            *reinterpret_cast<float4 *>(pre + PL.W + e4 * 4) = acc;
        }
        const float *RQ = hs + (size_t)nchunks * (R * d + R * R);
        for (int e = tid; e < R * R; e += blockDim.x) {
            const int pi = e / R, qi = e - pi * R;
            float v;
            if (pi < r && qi < r) {
                const int a0 = min(pi, qi), c0 = max(pi, qi);
                float gs = 0.f;
                if (have_res)
                    for (int ch = 0; ch < nchunks; ++ch)
                        gs += __ldcg(hs + (size_t)ch * (R * d + R * R) + R * d + a0 * R + c0);
                v = __ldcg(RQ + pi * R + qi) + (have_res ? l2 * gs : 0.f);
                pre[PL.P + e] = v;
            } else {
                v = (pi == qi) ? 1.f : 0.f;
                pre[PL.P + e] = 0.f;
            }
            b0[pi * ldM + qi] = v;
        }
    }
    __syncthreads();
    trace(15);
    const bool okP = block_gj(b0, R, ldM, s_rc);
    if (okP) {
        for (int e = tid; e < R * R; e += blockDim.x) {
            const int i = e / R, j = e - i * R;
            pre[PL.Pinv + e] = (i < r && j < r) ? b0[i * ldM + j] : 0.f;
        }
        for (int e = tid; e < R * d; e += blockDim.x) {  // Z_Q = P^-1 W
            const int p = e / d, i = e - p * d;
            float acc = 0.f;
            if (p < r)
                for (int q = 0; q < r; ++q) acc = fmaf(b0[p * ldM + q], sW[q * ldB + i], acc);
            pre[PL.ZQ + e] = acc;
        }
    }
    trace(16);
    if (tid == 0) pre[PL.flags + 0] = okP ? 1.f : 0.f;
    (void)warp;
}

// ---------------------------------------------------------------------------
// K2p in two short kernels (bf16 storage):
//  prepare_reduce_cluster_kernel -- one cluster of kPcCtas CTAs per head;
//    every CTA gathers its slice of Omega_t and reduces it on the tensor
//    cores into shared memory (Y_c = A^T K, G_c = A^T A); CTA 0 sums the
//    slices over distributed shared memory in rank order (deterministic)
//    and writes Y | G for the head.
//  prepare_finish_kernel -- one block per head: R = B_K B_K^T,
//    P = B_Q B_Q^T + l2 G, W = B_Q + l2 Y, P^-1, R^-1 (what compress needs
//    besides q and k), and the HBM-policy hit/miss count.
// Both are brief, so the precompute barely competes with the decode chain
// it overlaps on the side stream.
// ---------------------------------------------------------------------------
// The line-search B update of decode.py:150-184 for both sides, on B rows
// staged in shared memory (row stride ldB): resid = x_hat B - x,
// eta = (resid . s) / (s . s) with s = |x_hat|^2 resid (0 under the
// reference's floor), B -= eta x_hat^T resid.  X = [q | k | q_hat | k_hat].
// Writes the updated rows back to B_Q / B_K and eta.  scratch: 4 * d + 2 * R floats.
__device__ void apply_deferred_b_update(const lrqk_layer_t &L, int bh, const float *X, float *sBQ, float *sBK,
                                        int ldB, float *scratch, float *s_red) {
    const int d = L.dim_stride, R = L.rank_stride, r = L.rank;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float *resid = scratch;  // [2][d]
    {   // X to shared memory once: the loops below read it repeatedly
        float *xs = scratch + 2 * d;
        for (int i = tid; i < 2 * d + 2 * R; i += blockDim.x) xs[i] = __ldcg(X + i);
        __syncthreads();
        X = xs;
    }
    for (int w = tid; w < 2 * d; w += blockDim.x) {
        const int side = w / d, i = w - side * d;
        const float *xh = X + 2 * d + side * R;
        const float *Bm = side ? sBK : sBQ;
        float a0 = 0.f, a1 = 0.f;
        int p = 0;
        for (; p + 1 < r; p += 2) {
            a0 = fmaf(xh[p], Bm[p * ldB + i], a0);
            a1 = fmaf(xh[p + 1], Bm[(p + 1) * ldB + i], a1);
        }
        if (p < r) a0 = fmaf(xh[p], Bm[p * ldB + i], a0);
        resid[w] = a0 + a1 - X[side * d + i];
    }
    __syncthreads();
    if (warp < 2) {
        const int side = warp;
        const float *xh = X + 2 * d + side * R;
        float nx = 0.f;
        for (int p = lane; p < r; p += 32) nx = fmaf(xh[p], xh[p], nx);
        nx = warp_sum(nx);
        float ss = 0.f;
        for (int i = lane; i < d; i += 32) ss = fmaf(resid[side * d + i], resid[side * d + i], ss);
        ss = warp_sum(ss);
        const float num = nx * ss, den = nx * num;
        if (lane == 0) s_red[side] = (den <= 1e-14f * (1.f + fabsf(num))) ? 0.f : num / den;
    }
    __syncthreads();
    {   // B -= eta x_hat^T resid, float4 columns; rows 0..r-1 of B_Q then of B_K
        const int d4 = d / 4, rstep = blockDim.x / d4;  // d4 divides blockDim (d is a power of two <= 4 * blockDim)
        const int i = (tid - (tid / d4) * d4) * 4;
        for (int rr = tid / d4; rr < 2 * r; rr += rstep) {
            const int side = rr >= r, p = rr - side * r;
            const float c = s_red[side] * X[2 * d + side * R + p];
            float *Bm = (side ? sBK : sBQ) + p * ldB + i;
            const float *rs = resid + side * d + i;
            float4 v = *reinterpret_cast<float4 *>(Bm);
            v.x -= c * rs[0]; v.y -= c * rs[1]; v.z -= c * rs[2]; v.w -= c * rs[3];
            *reinterpret_cast<float4 *>(Bm) = v;
            *reinterpret_cast<float4 *>((side ? L.B_K : L.B_Q) + (size_t)bh * R * d + p * d + i) = v;
        }
    }
    if (tid < 2) L.eta[(size_t)bh * 2 + tid] = s_red[tid];
    __syncthreads();
}

constexpr int kPcCtas = 8;
constexpr int kPcBufs = 4;  // gather buffers per CTA (kPcBufs - 1 sub-chunks in flight)

__host__ __device__ inline size_t pc_part_floats(int R, int d) { return (size_t)R * d + (size_t)R * R; }

__device__ __forceinline__ void prepare_reduce_body(const lrqk_layer_t &L, int yg_slots, int bh) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) float smem[];
    const int crank = (int)cluster.block_rank();
    const int b = bh / L.n_q_heads, h = bh - b * L.n_q_heads;
    const int G = L.n_q_heads / L.n_kv_heads, g = h / G;
    const int d = L.dim_stride, R = L.rank_stride;
    const int n = L.res_cnt[bh];
    if (L.sel_meta[(size_t)bh * kMetaInts + M_YG] > 0) return;  // select_attend reduced this head already
    const bool host = L.policy == LRQK_SLOW_HOST;
    const size_t kv_rows = ((size_t)b * L.n_kv_heads + g) * L.t_max;
    const __nv_bfloat16 *proxy = reinterpret_cast<const __nv_bfloat16 *>(L.proxy) + (size_t)bh * L.t_max * R;
    const __nv_bfloat16 *kbase = host ? reinterpret_cast<const __nv_bfloat16 *>(L.slot_k) + (size_t)bh * L.n_slots * d
                                      : reinterpret_cast<const __nv_bfloat16 *>(L.slow_k) + kv_rows * d;
    const size_t PF = pc_part_floats(R, d);
    float *part = smem;  // [R*d | R*R]  Y_c | G_c
    trace(10);
    const int chunk = (n + kPcCtas - 1) / kPcCtas;
    const int row0 = crank * chunk, nrow = max(0, min(chunk, n - row0));
    int *s_ridx = reinterpret_cast<int *>(reinterpret_cast<uint8_t *>(part + PF) + kPcBufs * mma_stage_bytes(R, d));
    prepare_reduce_mma(L, bh, row0, nrow, kbase, proxy, host, part, reinterpret_cast<uint8_t *>(part + PF),
                       s_ridx, s_ridx + chunk, kPcBufs);
    trace(11);
    cluster.sync();
    {   // every CTA sums one slice of Y | G over the cluster, in rank order
        float *dst = L.red_scratch + (size_t)bh * yg_slots * PF;
        const size_t per = (PF + kPcCtas - 1) / kPcCtas;
        const size_t e0 = crank * per, e1 = min(PF, e0 + per);
        const float *src[kPcCtas];
#pragma unroll
        for (int c = 0; c < kPcCtas; ++c) src[c] = cluster.map_shared_rank(part, c);
        for (size_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
            float v[kPcCtas];
#pragma unroll
            for (int c = 0; c < kPcCtas; ++c) v[c] = src[c][e];
            float acc = 0.f;
#pragma unroll
            for (int c = 0; c < kPcCtas; ++c) acc += v[c];
            dst[e] = acc;
        }
    }
    cluster.sync();  // the other CTAs' shared memory stays alive until here
    trace(12);
}

__device__ __forceinline__ void prepare_finish_body(const lrqk_layer_t &L, int yg_slots) {
    extern __shared__ __align__(16) float smem[];
    __shared__ float s_rc[512];
    const int bh = blockIdx.x;
    const int d = L.dim_stride, R = L.rank_stride, r = L.rank;
    const int tid = threadIdx.x;
    const int n = L.res_cnt[bh];
    const bool host = L.policy == LRQK_SLOW_HOST;
    const PreLayout PL = pre_layout(R, d);
    float *pre = L.pre + (size_t)bh * PL.total;
    // Y | G: the sum of the partial slots select_attend wrote (M_YG), or the
    // cluster reduce's slot 0
    const size_t PF = yg_part_floats(R, d);
    float *YG = L.red_scratch + (size_t)bh * yg_slots * PF;
    int *meta = L.sel_meta + (size_t)bh * kMetaInts;
    const int nyg = meta[M_YG];
    if (nyg > 1 && meta[M_YG_FOLD] == 0) {  // slots summed in order; 8 slots' loads in flight per float4
        const size_t PF4 = PF / 4;
        float4 *YG4 = reinterpret_cast<float4 *>(YG);
        for (size_t e4 = tid; e4 < PF4; e4 += blockDim.x) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int c0 = 0; c0 < nyg; c0 += 8) {
                float4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (c0 + u < nyg) v[u] = __ldcg(YG4 + (size_t)(c0 + u) * PF4 + e4);
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (c0 + u < nyg) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
            }
            YG4[e4] = acc;
        }
        __syncthreads();
    }
    const int nadd = meta[M_YG_ADD];
    if (nadd > 0) {  // the threshold-bin winners select_attend left to this kernel
        __syncthreads();
        yg_rows_small(L, reinterpret_cast<const __nv_bfloat16 *>(L.slow_k) +
                             ((size_t)(bh / L.n_q_heads) * L.n_kv_heads + (bh % L.n_q_heads) / (L.n_q_heads / L.n_kv_heads)) *
                                 L.t_max * d,
                      reinterpret_cast<const __nv_bfloat16 *>(L.proxy) + (size_t)bh * L.t_max * R,
                      L.res_idx + (size_t)bh * L.s_cap + meta[M_NABOVE], nadd, smem, YG);
    }
    __syncthreads();
    if (tid == 0) { meta[M_YG] = 0; meta[M_YG_ADD] = 0; meta[M_YG_FOLD] = 0; }
    const int ldB = d + 4, ldM = R + 4;
    const int RB = R / 4, NP = RB * (RB + 1) / 2;
    float *sBQ = smem;                   // [R][ldB]
    float *sBK = sBQ + R * ldB;          // [R][ldB]
    float *b0 = sBK + R * ldB;           // [R][ldM]  R, then R^-1
    float *b1 = b0 + R * ldM;            // [R][ldM]  P, then P^-1
    float *tmp = b1 + R * ldM;           // [4 * NP * 16] gram scratch
    trace(13);
    if (!host) count_hits_hbm(L, bh, n, s_rc);
    trace(35);
    stage_rows_f32(sBQ, ldB, L.B_Q + (size_t)bh * R * d, R, d);
    stage_rows_f32(sBK, ldB, L.B_K + (size_t)bh * R * d, R, d);
    if (pre[PL.flags + 2] != 0.f) {  // the step's deferred line-search B update
        __syncthreads();
        trace(36);
        apply_deferred_b_update(L, bh, pre + PL.X, sBQ, sBK, ldB, tmp, s_rc);
        if (tid == 0) pre[PL.flags + 2] = 0.f;
    }
    trace(37);
    for (int e = tid; e < R * R; e += blockDim.x) {  // identity padding
        const int i = e / R, j = e - i * R;
        if (i >= r || j >= r) { b0[i * ldM + j] = (i == j) ? 1.f : 0.f; b1[i * ldM + j] = (i == j) ? 1.f : 0.f; }
    }
    __syncthreads();
    gram_rows2(sBK, sBQ, r, d, ldB, b0, b1, ldM, tmp);  // R (exactly symmetric), B_Q B_Q^T
    trace(38);
    const float l2 = L.lambda_2;
    const bool have_res = n > 0;
    const float *Gs = YG + (size_t)R * d;
    for (int e = tid; e < R * R; e += blockDim.x) {
        const int i = e / R, j = e - i * R;
        const bool in = i < r && j < r;
        float pv = 0.f;
        if (in) {
            pv = b1[i * ldM + j] + (have_res ? l2 * __ldcg(Gs + min(i, j) * R + max(i, j)) : 0.f);
            b1[i * ldM + j] = pv;
        }
        pre[PL.P + e] = pv;
        pre[PL.R + e] = in ? b0[i * ldM + j] : 0.f;
    }
    for (int e4 = tid; e4 < R * d / 4; e4 += blockDim.x) {  // W = B_Q + l2 Y
        const int p2 = (e4 * 4) / d, i = e4 * 4 - p2 * d;
        float4 acc = *reinterpret_cast<const float4 *>(sBQ + p2 * ldB + i);
        if (have_res) {
            const float4 y = __ldcg(reinterpret_cast<const float4 *>(YG) + e4);
            acc.x = fmaf(l2, y.x, acc.x); acc.y = fmaf(l2, y.y, acc.y);
            acc.z = fmaf(l2, y.z, acc.z); acc.w = fmaf(l2, y.w, acc.w);
        }
        *reinterpret_cast<float4 *>(pre + PL.W + e4 * 4) = acc;
    }
    __syncthreads();
    trace(14);
    bool okRP[2];
    block_gj2(b0, b1, R, ldM, s_rc, okRP);
    const bool okR = okRP[0], okP = okRP[1];
    for (int e = tid; e < R * R; e += blockDim.x) {
        const int i = e / R, j = e - i * R;
        const bool in = i < r && j < r;
        if (okR) pre[PL.Rinv + e] = in ? b0[i * ldM + j] : 0.f;
        if (okP) pre[PL.Pinv + e] = in ? b1[i * ldM + j] : 0.f;
    }
    if (tid == 0) {
        pre[PL.flags + 0] = okP ? 1.f : 0.f;
        pre[PL.flags + 1] = okR ? 1.f : 0.f;
    }
    trace(16);
}

// one layer (struct by value) or a batch of layers (device array, layer =
// blockIdx.z): every layer's precompute is only needed by its next step, so
// the engine runs all layers' compress_prepare together at the end of a step
__global__ void __cluster_dims__(kPcCtas, 1, 1) __launch_bounds__(kCompressThreads, 2)
prepare_reduce_cluster_kernel(const lrqk_layer_t L, int yg_slots) { prepare_reduce_body(L, yg_slots, blockIdx.y); }
__global__ void __cluster_dims__(kPcCtas, 1, 1) __launch_bounds__(kCompressThreads, 2)
prepare_reduce_cluster_layers_kernel(const lrqk_layer_t *Ls, int n_layers, int yg_slots) {
    // persistent clusters over (layer, head): heads that select_attend
    // already reduced (the common case) are skipped: one parallel flag read
    // per blockDim items, compacted in item order (identical in every CTA of
    // the cluster, so the cluster stays on the same item)
    __shared__ int s_items[kCompressThreads];
    __shared__ int s_scan[32];
    trace(8);
    const int BH = Ls[0].batch * Ls[0].n_q_heads;
    const int n_mine = (n_layers * BH - (int)blockIdx.y + (int)gridDim.y - 1) / (int)gridDim.y;
    for (int k0 = 0; k0 < n_mine; k0 += blockDim.x) {
        const int k = k0 + threadIdx.x;
        const int item = blockIdx.y + k * gridDim.y;
        bool need = false;
        if (k < n_mine) {
            const int *meta = Ls[item / BH].sel_meta + (size_t)(item % BH) * kMetaInts;
            need = __ldcg(meta + M_YG) <= 0;
        }
        int tot;
        const int pos = block_exclusive_scan(need ? 1 : 0, s_scan, &tot);
        if (need) s_items[pos] = item;
        __syncthreads();
        for (int j = 0; j < tot; ++j) {
            const int it = s_items[j];
            prepare_reduce_body(Ls[it / BH], yg_slots, it % BH);
            __syncthreads();
        }
    }
    trace(9);
}
__global__ void __launch_bounds__(kCompressThreads)
prepare_finish_kernel(const lrqk_layer_t L, int yg_slots) { prepare_finish_body(L, yg_slots); }
__global__ void __launch_bounds__(kCompressThreads, 4)
prepare_finish_layers_kernel(const lrqk_layer_t *Ls, int yg_slots) {
    trace(7);
    prepare_finish_body(Ls[blockIdx.z], yg_slots);
}

static bool pc_enabled() {
    static const bool on = [] { const char *e = getenv("LRQK_PREPARE_CLUSTER"); return !(e && e[0] == '0'); }();
    return on;
}

// compress_prepare runs as cluster reduce + finish kernels (which also apply
// the deferred B update) for bf16 storage with rank >= 16, d >= 64
static bool cluster_prepare_path(const lrqk_layer_t &L) {
    return L.dtype == LRQK_BF16 && L.rank_stride >= 16 && L.dim_stride >= 64 && pc_enabled();
}

static size_t prepare_reduce_smem_bytes(const lrqk_layer_t &L) {
    const int d = L.dim_stride, R = L.rank_stride;
    const size_t chunk = ((size_t)L.s_cap + kPcCtas - 1) / kPcCtas;
    return pc_part_floats(R, d) * sizeof(float) + kPcBufs * (size_t)mma_stage_bytes(R, d) + 2 * chunk * sizeof(int);
}
static size_t prepare_finish_smem_bytes(const lrqk_layer_t &L) {
    const size_t d = L.dim_stride, R = L.rank_stride;
    const size_t ldB = d + 4, ldM = R + 4, RB = R / 4, NP = RB * (RB + 1) / 2;
    const size_t scratch = 4 * NP * 16 > 4 * d + 2 * R ? 4 * NP * 16 : 4 * d + 2 * R;
    const size_t main = 2 * R * ldB + 2 * R * ldM + scratch;
    const size_t small_yg = (size_t)kMmaRows * (d + R);  // yg_rows_small's fp32 staging of the bin-D rows
    return (main > small_yg ? main : small_yg) * sizeof(float);
}

// ---------------------------------------------------------------------------
// K2c: compress (one block per head)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kCompressThreads)
compress_kernel(const CompressArgs args) {
    const lrqk_layer_t &L = args.L;
    extern __shared__ __align__(16) float smem[];
    __shared__ float s_scalar[8];
    __shared__ int s_bad;
    __shared__ float s_rc[256];
    __shared__ __align__(8) uint64_t s_bar;
    const int bh = blockIdx.x;
    const int b = bh / L.n_q_heads, h = bh - b * L.n_q_heads;
    const int G = L.n_q_heads / L.n_kv_heads, g = h / G;
    const int d = L.dim_stride, R = L.rank_stride, r = L.rank;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    trace(0);
    const PreLayout PL = pre_layout(R, d);
    const float *pre = L.pre + (size_t)bh * PL.total;
    const size_t head_rows = (size_t)bh * L.t_max;
    const size_t kv_rows = ((size_t)b * L.n_kv_heads + g) * L.t_max;
    const T *qrow = reinterpret_cast<const T *>(args.q) + (size_t)bh * d;
    const T *krow = reinterpret_cast<const T *>(args.k) + ((size_t)b * L.n_kv_heads + g) * d;
    const T *vrow = reinterpret_cast<const T *>(args.v) + ((size_t)b * L.n_kv_heads + g) * d;
    // Staged operands, unpadded: B_Q, B_K | P^-1, R^-1 | Z_Q, Z_K arrive with
    // four 1-D bulk copies on one mbarrier (the pre layout keeps each pair
    // contiguous), issued before anything else so the whole 72 KB lands in
    // one memory round trip.
    const int ldB = d, ldM = R;
    float *sBQ = smem;                   // [R][d]
    float *sBK = sBQ + R * d;            // [R][d]
    float *sPi = sBK + R * d;            // [R][R]  P^-1 (P in the fallback)
    float *sRi = sPi + R * R;            // [R][R]  R^-1 (R in the fallback)
    float *sW = sRi + R * R;             // [R][d]  W = B_Q + l2 A_res^T K_res
    float *b0 = sW + R * d;              // [R][R]  fallback scratch
    float *sM = b0 + R * R;              // [R][R]  fallback system
    float *vq = sM + R * R;              // [d]
    float *vk = vq + d;                  // [d]
    float *yq = vk + d;                  // [R]
    float *yk = yq + R;                  // [R]
    float *qh = yk + R;                  // [R]
    float *kh = qh + R;                  // [R]
    float *u = kh + R;                   // [R]
    float *prevc = u + R;                // [2R]
    float *resid = prevc + 2 * R;        // [2][d]
    static_assert(PreLayoutOrder::kPairs, "pre layout keeps Pinv|Rinv adjacent");
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint32_t mat = (uint32_t)(R * d * 4), sq = (uint32_t)(R * R * 4);
        mbar_expect_tx(&s_bar, 3 * mat + 2 * sq);
        bulk_g2s(sBQ, L.B_Q + (size_t)bh * R * d, mat, &s_bar);
        bulk_g2s(sBK, L.B_K + (size_t)bh * R * d, mat, &s_bar);
        bulk_g2s(sPi, pre + PL.Pinv, 2 * sq, &s_bar);
        bulk_g2s(sW, pre + PL.W, mat, &s_bar);
        s_bad = 0;
    }
    // B_Q/B_K and pre were written by the previous step (older than this
    // kernel's predecessor); q/k/v and ctx_len may come from the predecessor
    pdl_wait();
    pdl_trigger();
    const bool okP = __ldcg(pre + PL.flags + 0) != 0.f;
    const bool okR = __ldcg(pre + PL.flags + 1) != 0.f;
    const bool fast = okP && okR;
    const int t = L.ctx_len[b];
    __syncthreads();
    if (t >= L.t_max) {
        mbar_wait(&s_bar, 0);  // no bulk copy may still target this block's smem
        if (tid == 0) set_status(L.status, LRQK_ST_CAPACITY);
        return;
    }
    for (int i = tid; i < d; i += blockDim.x) {
        vq[i] = to_float<T>(qrow[i]);
        vk[i] = to_float<T>(krow[i]);
        if (!isfinite(vq[i]) || !isfinite(vk[i]) || !isfinite(to_float<T>(vrow[i]))) s_bad = 1;
    }
    mbar_wait(&s_bar, 0);
    if (!fast) {  // rare: the direct solves need P, R instead of P^-1, R^-1
        for (int e = tid; e < R * R; e += blockDim.x) {
            sPi[e] = __ldcg(pre + PL.P + e);
            sRi[e] = __ldcg(pre + PL.R + e);
        }
    }
    __syncthreads();
    if (s_bad) {  // ref: linalg.py:32-33 via as_row (session.py:94)
        if (tid == 0) set_status(L.status, LRQK_ST_NONFINITE);
        return;
    }
    trace(1);
    // ---- m_q = q W^T, m_k = k B_K^T, qk; then y_q = m_q P^-1, y_k = m_k R^-1 ---
    // one 8-lane group per output row; 32 groups per block
    {
        const int grp = tid >> 3, gl = tid & 7;
        // trip count is uniform across each warp (the shuffles below need all lanes)
        for (int o0 = 0; o0 < 2 * r + 1; o0 += kCompressThreads / 8) {
            const int o = o0 + grp;
            const bool valid = o < 2 * r + 1;
            float acc = 0.f;
            if (valid) {
                const float *x = o < r ? sW + o * ldB : (o < 2 * r ? sBK + (o - r) * ldB : vq);
                const float *y = o < r ? vq : vk;
                for (int i = gl * 4; i < d; i += 32) {
                    const float4 xv = *reinterpret_cast<const float4 *>(x + i);
                    const float4 yv = *reinterpret_cast<const float4 *>(y + i);
                    acc = fmaf(xv.x, yv.x, fmaf(xv.y, yv.y, fmaf(xv.z, yv.z, fmaf(xv.w, yv.w, acc))));
                }
            }
            acc += __shfl_xor_sync(0xffffffffu, acc, 4);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            if (valid && gl == 0) {
                if (o < r) yq[o] = acc;
                else if (o < 2 * r) yk[o - r] = acc;
                else s_scalar[0] = acc;
            }
        }
    }
    __syncthreads();
    if (fast) {  // y_q = m_q P^-1 (warp 0), y_k = m_k R^-1 = k_hat0 (warp 1), decode.py:79-108
        if (warp < 2) {
            const float *mv = warp == 0 ? yq : yk;
            const float *S = warp == 0 ? sPi : sRi;
            float *dstv = warp == 0 ? u : prevc;
            warp_vecmat(mv, S, r, ldM, dstv);
            for (int i = lane; i < r; i += 32) (warp == 0 ? yq : yk)[i] = dstv[i];
        }
        __syncthreads();
    }
    trace(2);
    const float qk = s_scalar[0];
    const float l1 = L.lambda_1;
    const int max_iter = L.max_iter;
    if (fast && r <= 32) {
        // the alternation, one warp: lane j keeps column j of P^-1 and R^-1 in
        // registers, vectors are distributed one component per lane
        if (warp == 0) {
            float pc[32], rc2[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                pc[i] = (i < r && lane < r) ? sPi[i * ldM + lane] : 0.f;
                rc2[i] = (i < r && lane < r) ? sRi[i * ldM + lane] : 0.f;
            }
            const float yqv = lane < r ? yq[lane] : 0.f;
            const float ykv = lane < r ? yk[lane] : 0.f;
            float khv = ykv, qhv = 0.f, pq = 0.f, pk = 0.f;
            for (int it = 0; it < max_iter; ++it) {
                float uv = 0.f;                      // u = k_hat P^-1
#pragma unroll
                for (int i = 0; i < 32; ++i) uv = fmaf(__shfl_sync(0xffffffffu, khv, i), pc[i], uv);
                float alpha = yqv * khv, c = uv * khv;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    alpha += __shfl_xor_sync(0xffffffffu, alpha, o);
                    c += __shfl_xor_sync(0xffffffffu, c, o);
                }
                qhv = fmaf(l1 * (qk - alpha) / (1.f + l1 * c), uv, yqv);   // decode.py:84-108
                float wv = 0.f;                      // w = q_hat R^-1
#pragma unroll
                for (int i = 0; i < 32; ++i) wv = fmaf(__shfl_sync(0xffffffffu, qhv, i), rc2[i], wv);
                float beta = ykv * qhv, e2 = wv * qhv;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    beta += __shfl_xor_sync(0xffffffffu, beta, o);
                    e2 += __shfl_xor_sync(0xffffffffu, e2, o);
                }
                khv = fmaf(l1 * (qk - beta) / (1.f + l1 * e2), wv, ykv);   // decode.py:111-119
                const float dq = qhv - pq, dk = khv - pk;
                const float dsum = warp_sum(dq * dq + dk * dk);
                pq = qhv;
                pk = khv;
                if (it > 0 && dsum / (2.f * r) <= L.tol) break;            // decode.py:143-146
            }
            qh[lane] = lane < r ? qhv : 0.f;
            kh[lane] = lane < r ? khv : 0.f;
            for (int i = 32 + lane; i < R; i += 32) { qh[i] = 0.f; kh[i] = 0.f; }
        }
        __syncthreads();
    } else if (fast) {
        if (warp == 0) {
            for (int i = lane; i < r; i += 32) kh[i] = yk[i];
            __syncwarp();
            for (int it = 0; it < max_iter; ++it) {
                warp_vecmat(kh, sPi, r, ldM, u);
                const float alpha = warp_dot(yq, kh, r), c = warp_dot(u, kh, r);
                const float coef = l1 * (qk - alpha) / (1.f + l1 * c);
                for (int i = lane; i < r; i += 32) qh[i] = fmaf(coef, u[i], yq[i]);
                __syncwarp();
                warp_vecmat(qh, sRi, r, ldM, u);
                const float beta = warp_dot(yk, qh, r), e2 = warp_dot(u, qh, r);
                const float coef2 = l1 * (qk - beta) / (1.f + l1 * e2);
                for (int i = lane; i < r; i += 32) kh[i] = fmaf(coef2, u[i], yk[i]);
                __syncwarp();
                float dsum = 0.f;
                for (int i = lane; i < r; i += 32) {
                    const float dq = qh[i] - prevc[i], dk = kh[i] - prevc[r + i];
                    dsum += dq * dq + dk * dk;
                }
                dsum = warp_sum(dsum);
                const bool stop = it > 0 && dsum / (2.f * r) <= L.tol;
                for (int i = lane; i < r; i += 32) { prevc[i] = qh[i]; prevc[r + i] = kh[i]; }
                __syncwarp();
                if (stop) break;
            }
            for (int i = r + lane; i < R; i += 32) { qh[i] = 0.f; kh[i] = 0.f; }
        }
        __syncthreads();
    } else {
        // ---- fallback: the reference's direct solves with jitter retry -----
        // sZQ holds W, so yq = m = q W^T;  yk = k B_K^T;  sPi = P, sRi = R
        int jitter = 0;
        int rc = solve_spd_direct(sRi, ldM, r, R, ldM, yk, kh, b0, s_rc);  // k_hat0
        if (rc == 2) { if (tid == 0) set_status(L.status, LRQK_ST_SOLVE_FAILED); return; }
        jitter |= rc;
        for (int it = 0; it < max_iter; ++it) {
            for (int e = tid; e < r * r; e += blockDim.x) {
                const int pi = e / r, qi = e - pi * r;
                sM[pi * ldM + qi] = sPi[pi * ldM + qi] + l1 * kh[pi] * kh[qi];
            }
            for (int p = tid; p < r; p += blockDim.x) u[p] = yq[p] + l1 * qk * kh[p];
            __syncthreads();
            rc = solve_spd_direct(sM, ldM, r, R, ldM, u, qh, b0, s_rc);
            if (rc == 2) { if (tid == 0) set_status(L.status, LRQK_ST_SOLVE_FAILED); return; }
            jitter |= rc;
            for (int e = tid; e < r * r; e += blockDim.x) {
                const int pi = e / r, qi = e - pi * r;
                sM[pi * ldM + qi] = sRi[pi * ldM + qi] + l1 * qh[pi] * qh[qi];
            }
            for (int p = tid; p < r; p += blockDim.x) u[p] = yk[p] + l1 * qk * qh[p];
            __syncthreads();
            // note: yk here is k B_K^T (the rhs), not k_hat0
            rc = solve_spd_direct(sM, ldM, r, R, ldM, u, kh, b0, s_rc);
            if (rc == 2) { if (tid == 0) set_status(L.status, LRQK_ST_SOLVE_FAILED); return; }
            jitter |= rc;
            if (tid == 0) {
                float dsum = 0.f;
                for (int i = 0; i < r; ++i) {
                    const float dq = qh[i] - prevc[i], dk = kh[i] - prevc[r + i];
                    dsum += dq * dq + dk * dk;
                }
                s_scalar[1] = (it > 0 && dsum / (2.f * r) <= L.tol) ? 1.f : 0.f;
                for (int i = 0; i < r; ++i) { prevc[i] = qh[i]; prevc[r + i] = kh[i]; }
            }
            __syncthreads();
            if (s_scalar[1] != 0.f) break;
        }
        for (int i = r + tid; i < R; i += blockDim.x) { qh[i] = 0.f; kh[i] = 0.f; }
        if (tid == 0) set_status(L.status, LRQK_ST_FALLBACK | (jitter ? LRQK_ST_JITTERED : 0u));
        __syncthreads();
    }
    trace(3);
    if (args.update_b && args.defer_b) {
        // The line-search B update (decode.py:150-184) only feeds the next
        // step: hand q, k, q_hat, k_hat to compress_prepare, which applies it
        // off the decode critical path.
        float *X = L.pre + (size_t)bh * PL.total + PL.X;
        for (int i = tid; i < d; i += blockDim.x) { X[i] = vq[i]; X[d + i] = vk[i]; }
        for (int i = tid; i < R; i += blockDim.x) { X[2 * d + i] = qh[i]; X[2 * d + R + i] = kh[i]; }
        if (tid == 0) L.pre[(size_t)bh * PL.total + PL.flags + 2] = 1.f;
        s_scalar[2] = s_scalar[3] = 0.f;
    } else {

    // ---------------- line-search B update (decode.py:150-184), both sides --
    // resid = x_hat B - x ; s = x_hat grad = |x_hat|^2 resid ; eta = (resid.s)/(s.s)
    for (int w = tid; w < 2 * d; w += blockDim.x) {
        const int side = w / d, i = w - side * d;
        const float *xh = side ? kh : qh;
        const float *Bm = side ? sBK : sBQ;
        float a0 = 0.f, a1 = 0.f;
        int p = 0;
        for (; p + 1 < r; p += 2) {
            a0 = fmaf(xh[p], Bm[p * ldB + i], a0);
            a1 = fmaf(xh[p + 1], Bm[(p + 1) * ldB + i], a1);
        }
        if (p < r) a0 = fmaf(xh[p], Bm[p * ldB + i], a0);
        resid[w] = a0 + a1 - (side ? vk[i] : vq[i]);
    }
    __syncthreads();
    trace(5);
    if (warp < 2) {
        const int side = warp;
        const float *xh = side ? kh : qh;
        const float nx = warp_dot(xh, xh, r);
        // s = x_hat grad = |x_hat|^2 resid, so num = |x|^2 |resid|^2 and
        // den = |x|^4 |resid|^2 (decode.py:150-166, with its underflow floor)
        float ss = 0.f;
        for (int i = lane; i < d; i += 32) ss = fmaf(resid[side * d + i], resid[side * d + i], ss);
        ss = warp_sum(ss);
        const float num = nx * ss, den = nx * num;
        if (lane == 0) s_scalar[2 + side] = (den <= 1e-14f * (1.f + fabsf(num))) ? 0.f : num / den;
    }
    __syncthreads();
    trace(6);
    if (args.update_b) {
        const int n4 = r * d / 4;
        for (int w = tid; w < 2 * n4; w += blockDim.x) {
            const int side = w / n4, e4 = w - side * n4;
            const float eta = s_scalar[2 + side];
            if (eta == 0.f) continue;
            const int p = (e4 * 4) / d, i = e4 * 4 - p * d;
            const float *Bm = side ? sBK : sBQ;
            const float *xh = side ? kh : qh;
            const float c = eta * xh[p];
            const float *rs = resid + side * d + i;
            float4 o;
            o.x = Bm[p * ldB + i] - c * rs[0];
            o.y = Bm[p * ldB + i + 1] - c * rs[1];
            o.z = Bm[p * ldB + i + 2] - c * rs[2];
            o.w = Bm[p * ldB + i + 3] - c * rs[3];
            *reinterpret_cast<float4 *>((side ? L.B_K : L.B_Q) + (size_t)bh * R * d + p * d + i) = o;
        }
    }
    }  // immediate B update
    trace(4);

    // ---------------- outputs and appends ---------------------------------
    for (int i = tid; i < R; i += blockDim.x) {
        L.q_hat[(size_t)bh * R + i] = qh[i];
        L.k_hat[(size_t)bh * R + i] = kh[i];
    }
    if (warp == 0) {  // |q_hat|: the selection scales its threshold hint by it (select_common.cuh)
        float a = 0.f;
        for (int i = lane; i < R; i += 32) a = fmaf(qh[i], qh[i], a);
        a = warp_sum(a);
        if (lane == 0) L.sel_meta[(size_t)bh * kMetaInts + M_QN] = __float_as_int(sqrtf(a));
    }
    if (tid == 0 && !(args.update_b && args.defer_b)) {
        L.eta[(size_t)bh * 2 + 0] = s_scalar[2];
        L.eta[(size_t)bh * 2 + 1] = s_scalar[3];
    }
    {   // append k_hat to the proxy store (cache.py:211), interleaved layout
        constexpr int N = Pack<T>::N;
        const int apacks = R / N;
        T *base = reinterpret_cast<T *>(L.proxy) + head_rows * R;
        for (int i = tid; i < R; i += blockDim.x)
            base[proxy_pack_offset(t, i / N, apacks) * N + (i % N)] = from_float<T>(kh[i]);
        if (L.proxy_rowmajor) {  // and to its row-major copy (the gathers read that one)
            T *rm = reinterpret_cast<T *>(L.proxy_rowmajor) + (head_rows + t) * R;
            for (int i = tid; i < R; i += blockDim.x) rm[i] = from_float<T>(kh[i]);
        }
    }
    if (h % G == 0) {  // append k, v once per KV head (cache.py:209-210)
        T *dk = reinterpret_cast<T *>(L.slow_k) + (kv_rows + t) * d;
        T *dv = reinterpret_cast<T *>(L.slow_v) + (kv_rows + t) * d;
        for (int i = tid; i < d; i += blockDim.x) { dk[i] = krow[i]; dv[i] = vrow[i]; }
    }
    if (L.policy == LRQK_SLOW_HOST) {  // the new row also lands in this head's spare slot
        const int slot = L.spare_slot[bh];
        T *sk = reinterpret_cast<T *>(L.slot_k) + ((size_t)bh * L.n_slots + slot) * d;
        T *sv = reinterpret_cast<T *>(L.slot_v) + ((size_t)bh * L.n_slots + slot) * d;
        for (int i = tid; i < d; i += blockDim.x) { sk[i] = krow[i]; sv[i] = vrow[i]; }
    }
    (void)nwarps;
}

int compress_chunks(const lrqk_layer_t &L) { return (L.s_cap + kRedRows - 1) / kRedRows; }

int score_tma_parts(const lrqk_layer_t &L);
// Y|G partial slots per head: the legacy reduce's chunks, or one per score
// part plus one (select_attend)
int yg_slots(const lrqk_layer_t &L) { return std::max(compress_chunks(L) + 1, score_tma_parts(L) + 1); }
size_t compress_scratch_floats_per_head(const lrqk_layer_t &L) {
    return (size_t)yg_slots(L) * yg_part_floats(L.rank_stride, L.dim_stride);
}
size_t compress_pre_floats_per_head(const lrqk_layer_t &L) {
    return pre_layout(L.rank_stride, L.dim_stride).total;
}

static size_t prepare_smem_bytes(const lrqk_layer_t &L) {
    const size_t d = L.dim_stride, R = L.rank_stride;
    const size_t RB = R / 4, NP = RB * (RB + 1) / 2;
    const size_t NG = NP >= (size_t)kCompressThreads ? 1 : kCompressThreads / NP;
    const size_t ldB = d + 4, ldM = R + 4;
    const size_t a = std::max(std::max(((size_t)kSub * ldB + (size_t)kSub * (R + 4) + NG * NP * 16) * sizeof(float),
                                       (size_t)8192 * sizeof(float)),
                              (size_t)2 * mma_stage_bytes((int)R, (int)d));
    const size_t p = (2 * R * ldB + R * ldM + 2 * NP * 16) * sizeof(float);
    const size_t f = (R * ldB + R * ldM) * sizeof(float);
    return std::max(a, std::max(p, f));
}
static size_t compress_smem_bytes(const lrqk_layer_t &L) {
    const size_t d = L.dim_stride, R = L.rank_stride;
    return (3 * R * d + 4 * R * R + 4 * d + 7 * R) * sizeof(float);
}

int launch_prepare(const lrqk_layer_t &L, cudaStream_t st);
int yg_slots(const lrqk_layer_t &L);
int num_sms();
int launch_prepare_layers(const lrqk_layer_t *dev_layers, const lrqk_layer_t *host_layers, int n_layers,
                          cudaStream_t st) {
    const lrqk_layer_t &L = host_layers[0];
    if (cluster_prepare_path(L)) {
        const size_t s1 = prepare_reduce_smem_bytes(L), s2 = prepare_finish_smem_bytes(L);
        cudaFuncSetAttribute(prepare_reduce_cluster_layers_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
        cudaFuncSetAttribute(prepare_finish_layers_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
        const int n_items = L.batch * L.n_q_heads * n_layers;
        const int clusters = std::max(1, std::min(n_items, num_sms() * 2 / kPcCtas));
        prepare_reduce_cluster_layers_kernel<<<dim3(kPcCtas, clusters), kCompressThreads, s1, st>>>(
            dev_layers, n_layers, yg_slots(L));
        prepare_finish_layers_kernel<<<dim3(L.batch * L.n_q_heads, 1, n_layers), kCompressThreads, s2, st>>>(
            dev_layers, yg_slots(L));
        return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
    }
    for (int i = 0; i < n_layers; ++i) {
        const int rc = launch_prepare(host_layers[i], st);
        if (rc) return rc;
    }
    return LRQK_OK;
}

int launch_prepare(const lrqk_layer_t &L, cudaStream_t st) {
    if (cluster_prepare_path(L)) {
        const size_t s1 = prepare_reduce_smem_bytes(L), s2 = prepare_finish_smem_bytes(L);
        cudaFuncSetAttribute(prepare_reduce_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
        cudaFuncSetAttribute(prepare_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
        prepare_reduce_cluster_kernel<<<dim3(kPcCtas, L.batch * L.n_q_heads), kCompressThreads, s1, st>>>(L, yg_slots(L));
        prepare_finish_kernel<<<L.batch * L.n_q_heads, kCompressThreads, s2, st>>>(L, yg_slots(L));
        return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
    }
    dim3 grid(compress_chunks(L) + 1, L.batch * L.n_q_heads);
    const size_t smem = prepare_smem_bytes(L);
    if (L.dtype == LRQK_BF16) {
        cudaFuncSetAttribute(prepare_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        prepare_kernel<__nv_bfloat16><<<grid, kCompressThreads, smem, st>>>(L);
    } else {
        cudaFuncSetAttribute(prepare_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        prepare_kernel<float><<<grid, kCompressThreads, smem, st>>>(L);
    }
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

int launch_compress(const lrqk_layer_t &L, const void *q, const void *k, const void *v, int update_b,
                    cudaStream_t st) {
    CompressArgs a{L, q, k, v, update_b, cluster_prepare_path(L) ? 1 : 0};
    const size_t smem = compress_smem_bytes(L);
    if (L.dtype == LRQK_BF16) {
        cudaFuncSetAttribute(compress_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_kernel(compress_kernel<__nv_bfloat16>, L.batch * L.n_q_heads, kCompressThreads, smem, st, true, a);
    } else {
        cudaFuncSetAttribute(compress_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_kernel(compress_kernel<float>, L.batch * L.n_q_heads, kCompressThreads, smem, st, true, a);
    }
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

}  // namespace lrqk
