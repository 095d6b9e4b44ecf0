// K2: per-token compression (q_hat, k_hat), B line-search update and the
// append of (k_hat -> proxy store, k/v -> slow tier / slot).
//
// ref: decode.py:79-184 (khat_initial_guess, update_qhat, update_khat,
//      decode_compress, _line_search_step, update_projections),
//      cache.py:199-214 (append_token), session.py:95-98 (order).
//
// Layout of the work: grid.y = B*Hq (one reference session per y), grid.x =
// chunks of kRedRows rows of the previous resident set Omega_{t-1}.  Each
// block reduces its rows' contribution to
//     G_res = A_res^T A_res          (r x r)       decode.py:106
//     m_res = (q K_res^T) A_res      (1 x r)       decode.py:105
// into a partial; the last block of the head to arrive sums the partials and
// runs the r x r algebra:
//   * R = B_K B_K^T and P = B_Q B_Q^T + l2 G_res are inverted once by an
//     in-place Gauss-Jordan sweep (no pivoting; every pivot > 0 <=> SPD,
//     exactly the condition under which the reference's Cholesky succeeds);
//   * every q_hat / k_hat solve of the alternation is then the closed form
//     of a rank-1-updated SPD system,
//        x (S + l1 v^T v) = b + l1 qk v
//        =>  x = y + u * l1 (qk - y.v) / (1 + l1 v.u),  y = b S^-1, u = v S^-1,
//     which is algebraically the reference's solve_spd(M, RHS) with
//     M = S + l1 v^T v (decode.py:100-108, 115-119);
//   * if either base matrix is not numerically SPD the block falls back to
//     solving each full system directly with the reference's jitter retry
//     (linalg.py:80-91).
#include "common.cuh"

namespace lrqk {

constexpr int kCompressThreads = 256;

struct CompressArgs {
    lrqk_layer_t L;
    const void *q, *k, *v;
    int update_b;
};

// ---------------------------------------------------------------------------
// small dense helpers operating on shared memory, whole block participates
// ---------------------------------------------------------------------------

// In-place Gauss-Jordan inverse of an n x n SPD matrix stored with row
// stride ld.  Returns false if a pivot is not > 0 (or non-finite).
__device__ bool gj_inverse(float *A, int n, int ld, float *s_piv) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int k = 0; k < n; ++k) {
        __syncthreads();
        float p = A[k * ld + k];
        if (!(p > 0.f) || !isfinite(p)) return false;  // uniform across block
        float ip = 1.f / p;
        // read phase: each thread computes its new values in registers
        float nv[24];
        int cnt = 0;
        for (int e = tid; e < n * n; e += nt) {
            int i = e / n, j = e - i * n;
            float aij = A[i * ld + j];
            float r;
            if (i == k && j == k) r = ip;
            else if (i == k) r = aij * ip;
            else if (j == k) r = -aij * ip;
            else r = aij - A[i * ld + k] * A[k * ld + j] * ip;
            nv[cnt++] = r;
        }
        __syncthreads();
        cnt = 0;
        for (int e = tid; e < n * n; e += nt) {
            int i = e / n, j = e - i * n;
            A[i * ld + j] = nv[cnt++];
        }
    }
    __syncthreads();
    (void)s_piv;
    return true;
}

// Solve x M = rhs (M SPD n x n, row stride ld, not modified) by Gauss-Jordan
// on a scratch copy; on failure retry once with the reference jitter
// 1e-10 (tr(M)/n + 1) (linalg.py:80-91).  x written to `x` (n floats).
// Returns 0 ok, 1 jittered ok, 2 failed.
__device__ int solve_spd_direct(const float *M, int n, int ld, const float *rhs, float *x,
                                float *work /* n*(n+1) floats */) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int w = n + 1;
    for (int attempt = 0; attempt < 2; ++attempt) {
        float jit = 0.f;
        if (attempt == 1) {
            float tr = 0.f;
            for (int i = 0; i < n; ++i) tr += M[i * ld + i];
            jit = 1e-10f * (tr / n + 1.f);
            // float(1e-10) jitter is below fp32 resolution of most diagonals;
            // keep the reference constant but never less than one ulp step.
            float dmax = 0.f;
            for (int i = 0; i < n; ++i) dmax = fmaxf(dmax, fabsf(M[i * ld + i]));
            jit = fmaxf(jit, dmax * 1.2e-7f);
        }
        __syncthreads();
        // augmented [M^T | rhs^T]: solving M^T x^T = rhs^T == x M = rhs (M symmetric)
        for (int e = tid; e < n * w; e += nt) {
            int i = e / w, j = e - i * w;
            work[e] = (j < n) ? M[j * ld + i] + ((i == j) ? jit : 0.f) : rhs[i];
        }
        __syncthreads();
        bool ok = true;
        for (int k = 0; k < n && ok; ++k) {
            float p = work[k * w + k];
            __syncthreads();
            if (!(p > 0.f) || !isfinite(p)) { ok = false; break; }
            float ip = 1.f / p;
            float nv[24];
            int cnt = 0;
            for (int e = tid; e < n * w; e += nt) {
                int i = e / w, j = e - i * w;
                float a = work[e];
                nv[cnt++] = (i == k) ? a * ip : a - work[i * w + k] * work[k * w + j] * ip;
            }
            __syncthreads();
            cnt = 0;
            for (int e = tid; e < n * w; e += nt) work[e] = nv[cnt++];
            __syncthreads();
        }
        if (ok) {
            for (int i = tid; i < n; i += nt) x[i] = work[i * w + n];
            __syncthreads();
            return attempt;
        }
    }
    return 2;
}

// y[j] = sum_i v[i] * S[i*ld + j]   (one warp, n <= 64)
LRQK_DEV void warp_vecmat(const float *v, const float *S, int n, int ld, float *y) {
    const int lane = threadIdx.x & 31;
    for (int j = lane; j < n; j += 32) {
        float acc = 0.f;
        for (int i = 0; i < n; ++i) acc = fmaf(v[i], S[i * ld + j], acc);
        y[j] = acc;
    }
    __syncwarp();
}
LRQK_DEV float warp_dot(const float *a, const float *b, int n) {
    const int lane = threadIdx.x & 31;
    float acc = 0.f;
    for (int j = lane; j < n; j += 32) acc = fmaf(a[j], b[j], acc);
    return warp_sum(acc);
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kCompressThreads)
compress_kernel(const CompressArgs args) {
    const lrqk_layer_t &L = args.L;
    extern __shared__ __align__(16) float smem[];
    __shared__ int s_flag;
    __shared__ int s_scan[32];

    const int bh = blockIdx.y;
    const int b = bh / L.n_q_heads, h = bh - b * L.n_q_heads;
    const int G = L.n_q_heads / L.n_kv_heads;
    const int g = h / G;
    const int d = L.dim_stride, R = L.rank_stride, r = L.rank;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int t = L.ctx_len[b];
    if (t >= L.t_max) {  // no room for the new token
        if (blockIdx.x == 0 && tid == 0) set_status(L.status, LRQK_ST_CAPACITY);
        return;
    }
    const int n_prev = L.res_cnt[bh];
    const size_t head_rows = (size_t)bh * L.t_max;
    const size_t kv_rows = ((size_t)b * L.n_kv_heads + g) * L.t_max;
    const T *proxy = reinterpret_cast<const T *>(L.proxy) + head_rows * R;
    const bool host = (L.policy == LRQK_SLOW_HOST);
    const T *kres_base = host ? reinterpret_cast<const T *>(L.slot_k) + (size_t)bh * L.n_slots * d
                              : reinterpret_cast<const T *>(L.slow_k) + kv_rows * d;
    const T *qrow = reinterpret_cast<const T *>(args.q) + (size_t)bh * d;
    const T *krow = reinterpret_cast<const T *>(args.k) + ((size_t)b * L.n_kv_heads + g) * d;
    const T *vrow = reinterpret_cast<const T *>(args.v) + ((size_t)b * L.n_kv_heads + g) * d;

    // ---------------- phase A: partial G_res, m_res over this chunk ---------
    float *sq = smem;                    // [d]
    float *sS = sq + d;                  // [kRedRows]
    float *sA = sS + kRedRows;           // [kRedRows][R+1]
    const int ldA = R + 1;
    for (int i = tid; i < d; i += blockDim.x) sq[i] = to_float<T>(qrow[i]);
    const int row0 = blockIdx.x * kRedRows;
    const int nrow = max(0, min(kRedRows, n_prev - row0));
    __syncthreads();
    {
        constexpr int N = Pack<T>::N;
        constexpr int U = 8;  // rows in flight per lane group
        // K_res rows: lanes-per-row LPR covering d in 16-byte packs
        const int packs = d / N;
        const int lpr = packs < 32 ? packs : 32;
        const int ppl = packs / lpr;  // packs per lane (1 or 2)
        const int rpw = 32 / lpr;     // rows per warp step
        const int sub = lane / lpr, sl = lane - sub * lpr;
        const int step = nwarps * rpw;
        const int *ridx = L.res_idx + (size_t)bh * L.s_cap + row0;
        const int *rslot = L.res_slot + (size_t)bh * L.s_cap + row0;
        for (int base = warp * rpw + sub; base < nrow + sub; base += step * U) {
            float x[U][2][N];
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int j = base + uu * step;
                if (j < nrow) {
                    const int src = host ? rslot[j] : ridx[j];
                    const T *kr = kres_base + (size_t)src * d;
#pragma unroll
                    for (int pp = 0; pp < 2; ++pp)
                        if (pp < ppl) Pack<T>::load(kr + (sl + pp * lpr) * N, x[uu][pp]);
                }
            }
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int j = base + uu * step;
                float part = 0.f;
                if (j < nrow) {
#pragma unroll
                    for (int pp = 0; pp < 2; ++pp)
                        if (pp < ppl) {
                            const float *qq = sq + (sl + pp * lpr) * N;
#pragma unroll
                            for (int e = 0; e < N; ++e) part = fmaf(x[uu][pp][e], qq[e], part);
                        }
                }
                for (int o = lpr / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                if (j < nrow && sl == 0) sS[j] = part;
            }
        }
        // A_res rows -> shared (fp32)
        const int apacks = R / N;
        const int total_a = nrow * apacks;
        for (int e0 = tid; e0 < total_a; e0 += blockDim.x * 4) {
            float xa[4][N];
#pragma unroll
            for (int uu = 0; uu < 4; ++uu) {
                const int e = e0 + uu * blockDim.x;
                if (e < total_a) {
                    const int j = e / apacks, p = e - j * apacks;
                    Pack<T>::load(proxy + (size_t)ridx[j] * R + p * N, xa[uu]);
                }
            }
#pragma unroll
            for (int uu = 0; uu < 4; ++uu) {
                const int e = e0 + uu * blockDim.x;
                if (e < total_a) {
                    const int j = e / apacks, p = e - j * apacks;
#pragma unroll
                    for (int i = 0; i < N; ++i) sA[j * ldA + p * N + i] = xa[uu][i];
                }
            }
        }
    }
    __syncthreads();
    float *part_out = L.red_scratch + ((size_t)bh * gridDim.x + blockIdx.x) * (size_t)(R * R + R);
    {
        // upper-triangular 4x4 blocks of G, rows split into groups
        const int RB = R / 4;
        const int NP = RB * (RB + 1) / 2;
        const int NG = max(1, (int)blockDim.x / NP);
        float *sRed = sA + kRedRows * ldA;  // [NG][NP*16] partial blocks
        if (tid < NP * NG) {
            const int pair = tid % NP, grp = tid / NP;
            // decode pair -> (pb, qb) with pb <= qb
            int pb = 0, rem = pair;
            while (rem >= RB - pb) { rem -= RB - pb; ++pb; }
            const int qb = pb + rem;
            float acc[4][4] = {};
            for (int j = grp; j < nrow; j += NG) {
                const float *a = sA + j * ldA;
                float ap[4], aq[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) { ap[u] = a[pb * 4 + u]; aq[u] = a[qb * 4 + u]; }
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int w2 = 0; w2 < 4; ++w2) acc[u][w2] = fmaf(ap[u], aq[w2], acc[u][w2]);
            }
            float *dst = sRed + ((size_t)grp * NP + pair) * 16;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int w2 = 0; w2 < 4; ++w2) dst[u * 4 + w2] = acc[u][w2];
        }
        // m_res partial
        for (int p = tid; p < R; p += blockDim.x) {
            float acc = 0.f;
            for (int j = 0; j < nrow; ++j) acc = fmaf(sS[j], sA[j * ldA + p], acc);
            part_out[R * R + p] = acc;
        }
        __syncthreads();
        for (int e = tid; e < NP * 16; e += blockDim.x) {
            float acc = 0.f;
            for (int gI = 0; gI < NG; ++gI) acc += sRed[(size_t)gI * NP * 16 + e];
            const int pair = e / 16, uw = e - pair * 16;
            int pb = 0, rem = pair;
            while (rem >= RB - pb) { rem -= RB - pb; ++pb; }
            const int qb = pb + rem;
            const int pi = pb * 4 + uw / 4, qi = qb * 4 + (uw & 3);
            part_out[pi * R + qi] = acc;  // only entries with block(pi) <= block(qi)
        }
    }
    if (!last_arrival(L.counters + (size_t)bh * kCounterInts + C_COMPRESS, gridDim.x, &s_flag)) return;

    // ---------------- phase B (one block per head) --------------------------
    const int ldM = R + 1;
    float *sBQ = smem;                   // [R][d+1]
    float *sBK = sBQ + R * (d + 1);      // [R][d+1]
    float *sP = sBK + R * (d + 1);       // [R][ldM]  -> P, then P^-1
    float *sRK = sP + R * ldM;           // [R][ldM]  -> R, then R^-1
    float *sRQ = sRK + R * ldM;          // [R][ldM]  B_Q B_Q^T (kept for fallback)
    float *vq = sRQ + R * ldM;           // [d]
    float *vk = vq + d;                  // [d]
    float *vv = vk + d;                  // [d]
    float *bq = vv + d;                  // [R]  q B_Q^T
    float *bk = bq + R;                  // [R]  k B_K^T
    float *mres = bk + R;                // [R]
    float *yq = mres + R;                // [R]
    float *yk = yq + R;                  // [R]
    float *qh = yk + R;                  // [R]
    float *kh = qh + R;                  // [R]
    float *u = kh + R;                   // [R]
    float *prevc = u + R;                // [2R]
    float *resid = prevc + 2 * R;        // [d]
    float *work = resid + d;             // [R*(R+1)] fallback scratch
    __shared__ float s_scalar[8];
    __shared__ int s_bad;

    const float *BQg = L.B_Q + (size_t)bh * R * d;
    const float *BKg = L.B_K + (size_t)bh * R * d;
    for (int e = tid; e < R * d; e += blockDim.x) {
        const int p = e / d, i = e - p * d;
        sBQ[p * (d + 1) + i] = BQg[e];
        sBK[p * (d + 1) + i] = BKg[e];
    }
    if (tid == 0) s_bad = 0;
    __syncthreads();
    for (int i = tid; i < d; i += blockDim.x) {
        vq[i] = to_float<T>(qrow[i]);
        vk[i] = to_float<T>(krow[i]);
        vv[i] = to_float<T>(vrow[i]);
        if (!isfinite(vq[i]) || !isfinite(vk[i]) || !isfinite(vv[i])) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) {  // ref: linalg.py:32-33 via as_row (session.py:94)
        if (tid == 0) set_status(L.status, LRQK_ST_NONFINITE);
        return;
    }
    // dots over d, one warp per output, lanes split d:  RQ, RK (upper), bq, bk, qk
    {
        const int nUp = r * (r + 1) / 2;
        const int total = 2 * nUp + 2 * r + 1;
        for (int o = warp; o < total; o += nwarps) {
            const float *x, *y;
            int kind, pi = 0, qi = 0;
            if (o < 2 * nUp) {
                kind = o < nUp ? 0 : 1;
                int rem = kind ? o - nUp : o;
                while (rem >= r - pi) { rem -= r - pi; ++pi; }
                qi = pi + rem;
                const float *Bm = kind ? sBK : sBQ;
                x = Bm + pi * (d + 1);
                y = Bm + qi * (d + 1);
            } else if (o < 2 * nUp + 2 * r) {
                const int e = o - 2 * nUp;
                kind = e < r ? 2 : 3;
                pi = kind == 2 ? e : e - r;
                x = (kind == 2 ? sBQ : sBK) + pi * (d + 1);
                y = kind == 2 ? vq : vk;
            } else {
                kind = 4;
                x = vq;
                y = vk;
            }
            float acc = 0.f;
            for (int i = lane; i < d; i += 32) acc = fmaf(x[i], y[i], acc);
            acc = warp_sum(acc);
            if (lane == 0) {
                if (kind == 0) { sRQ[pi * ldM + qi] = acc; sRQ[qi * ldM + pi] = acc; }
                else if (kind == 1) { sRK[pi * ldM + qi] = acc; sRK[qi * ldM + pi] = acc; }
                else if (kind == 2) bq[pi] = acc;
                else if (kind == 3) bk[pi] = acc;
                else s_scalar[0] = acc;
            }
        }
    }
    __syncthreads();
    // reduce the compression partials: P = RQ + l2 G_res, m = bq + l2 m_res
    const int nchunks = gridDim.x;
    const float *parts = L.red_scratch + (size_t)bh * nchunks * (size_t)(R * R + R);
    const bool have_res = n_prev > 0;
    const float l1 = L.lambda_1, l2 = L.lambda_2;
    for (int e = tid; e < r * r; e += blockDim.x) {
        const int pi = e / r, qi = e - pi * r;
        const int a = min(pi, qi), c = max(pi, qi);
        // partials hold the entry at (a, c) when block(a) <= block(c)
        float gsum = 0.f;
        if (have_res)
            for (int ch = 0; ch < nchunks; ++ch) gsum += __ldcg(parts + (size_t)ch * (R * R + R) + a * R + c);
        sP[pi * ldM + qi] = sRQ[pi * ldM + qi] + (have_res ? l2 * gsum : 0.f);
    }
    for (int p = tid; p < r; p += blockDim.x) {
        float msum = 0.f;
        if (have_res)
            for (int ch = 0; ch < nchunks; ++ch) msum += __ldcg(parts + (size_t)ch * (R * R + R) + R * R + p);
        mres[p] = bq[p] + (have_res ? l2 * msum : 0.f);
    }
    __syncthreads();
    const float qk = s_scalar[0];

    // copy R = B_K B_K^T aside for inversion (sRK is inverted in place; keep
    // the original in `work` region? we re-derive it on fallback instead)
    bool okP = gj_inverse(sP, r, ldM, nullptr);
    bool okR = okP ? gj_inverse(sRK, r, ldM, nullptr) : false;
    int jitter_flag = 0;
    const int max_iter = L.max_iter;

    if (okP && okR) {
        // fast path: two base inverses, rank-1 closed forms
        if (warp == 0) {
            warp_vecmat(bk, sRK, r, ldM, yk);      // k_hat0 = (k B_K^T) R^-1  (decode.py:79-81)
            warp_vecmat(mres, sP, r, ldM, yq);     // y_q = m P^-1
            for (int i = lane; i < r; i += 32) kh[i] = yk[i];
            __syncwarp();
            for (int it = 0; it < max_iter; ++it) {
                // q_hat (decode.py:84-108)
                warp_vecmat(kh, sP, r, ldM, u);
                float alpha = warp_dot(yq, kh, r), c = warp_dot(u, kh, r);
                float coef = l1 * (qk - alpha) / (1.f + l1 * c);
                for (int i = lane; i < r; i += 32) qh[i] = yq[i] + coef * u[i];
                __syncwarp();
                // k_hat (decode.py:111-119)
                warp_vecmat(qh, sRK, r, ldM, u);
                float beta = warp_dot(yk, qh, r), e2 = warp_dot(u, qh, r);
                float coef2 = l1 * (qk - beta) / (1.f + l1 * e2);
                for (int i = lane; i < r; i += 32) kh[i] = yk[i] + coef2 * u[i];
                __syncwarp();
                // stop rule (decode.py:143-146): mean squared change of [q_hat, k_hat]
                float dsum = 0.f;
                for (int i = lane; i < r; i += 32) {
                    float dq = qh[i] - prevc[i], dk = kh[i] - prevc[r + i];
                    dsum += dq * dq + dk * dk;
                }
                dsum = warp_sum(dsum);
                bool stop = it > 0 && dsum / (2.f * r) <= L.tol;
                for (int i = lane; i < r; i += 32) { prevc[i] = qh[i]; prevc[r + i] = kh[i]; }
                __syncwarp();
                if (stop) break;
            }
        }
        __syncthreads();
    } else {
        // fallback: the reference's direct solves with jitter retry
        // rebuild R (it may have been partially inverted)
        __syncthreads();
        for (int o = warp; o < r * r; o += nwarps) {
            const int pi = o / r, qi = o - pi * r;
            float acc = 0.f;
            for (int i = lane; i < d; i += 32) acc = fmaf(sBK[pi * (d + 1) + i], sBK[qi * (d + 1) + i], acc);
            acc = warp_sum(acc);
            if (lane == 0) sRK[pi * ldM + qi] = acc;
        }
        // rebuild P base
        for (int e = tid; e < r * r; e += blockDim.x) {
            const int pi = e / r, qi = e - pi * r;
            const int a = min(pi, qi), c = max(pi, qi);
            float gsum = 0.f;
            if (have_res)
                for (int ch = 0; ch < nchunks; ++ch) gsum += __ldcg(parts + (size_t)ch * (R * R + R) + a * R + c);
            sP[pi * ldM + qi] = sRQ[pi * ldM + qi] + (have_res ? l2 * gsum : 0.f);
        }
        __syncthreads();
        float *Mt = sRQ;  // reuse as the full system matrix
        int rc = solve_spd_direct(sRK, r, ldM, bk, kh, work);
        if (rc == 2) { if (tid == 0) set_status(L.status, LRQK_ST_SOLVE_FAILED); return; }
        jitter_flag |= rc;
        for (int it = 0; it < max_iter; ++it) {
            __syncthreads();
            for (int e = tid; e < r * r; e += blockDim.x) {
                const int pi = e / r, qi = e - pi * r;
                Mt[pi * ldM + qi] = sP[pi * ldM + qi] + l1 * kh[pi] * kh[qi];
            }
            for (int p = tid; p < r; p += blockDim.x) u[p] = mres[p] + l1 * qk * kh[p];
            __syncthreads();
            rc = solve_spd_direct(Mt, r, ldM, u, qh, work);
            if (rc == 2) { if (tid == 0) set_status(L.status, LRQK_ST_SOLVE_FAILED); return; }
            jitter_flag |= rc;
            __syncthreads();
            for (int e = tid; e < r * r; e += blockDim.x) {
                const int pi = e / r, qi = e - pi * r;
                Mt[pi * ldM + qi] = sRK[pi * ldM + qi] + l1 * qh[pi] * qh[qi];
            }
            for (int p = tid; p < r; p += blockDim.x) u[p] = bk[p] + l1 * qk * qh[p];
            __syncthreads();
            rc = solve_spd_direct(Mt, r, ldM, u, kh, work);
            if (rc == 2) { if (tid == 0) set_status(L.status, LRQK_ST_SOLVE_FAILED); return; }
            jitter_flag |= rc;
            __syncthreads();
            if (tid == 0) {
                float dsum = 0.f;
                for (int i = 0; i < r; ++i) {
                    float dq = qh[i] - prevc[i], dk = kh[i] - prevc[r + i];
                    dsum += dq * dq + dk * dk;
                }
                s_scalar[1] = (it > 0 && dsum / (2.f * r) <= L.tol) ? 1.f : 0.f;
                for (int i = 0; i < r; ++i) { prevc[i] = qh[i]; prevc[r + i] = kh[i]; }
            }
            __syncthreads();
            if (s_scalar[1] != 0.f) break;
        }
        if (jitter_flag && tid == 0) set_status(L.status, LRQK_ST_JITTERED);
    }
    __syncthreads();
    // zero the padded tail of the compressed rows
    for (int i = r + tid; i < R; i += blockDim.x) { qh[i] = 0.f; kh[i] = 0.f; }
    __syncthreads();

    // ---------------- line-search B update (decode.py:150-184) -------------
    // resid = x_hat B - x ; s = x_hat grad = |x_hat|^2 resid ; eta = (resid.s)/(s.s)
    for (int side = 0; side < 2; ++side) {
        const float *xh = side ? kh : qh;
        const float *x = side ? vk : vq;
        float *Bm = side ? sBK : sBQ;
        for (int i = tid; i < d; i += blockDim.x) {
            float acc = 0.f;
            for (int p = 0; p < r; ++p) acc = fmaf(xh[p], Bm[p * (d + 1) + i], acc);
            resid[i] = acc - x[i];
        }
        __syncthreads();
        if (warp == 0) {
            float nx = warp_dot(xh, xh, r);
            double num = 0.0, den = 0.0;
            for (int i = lane; i < d; i += 32) {
                double s = (double)nx * (double)resid[i];
                num += (double)resid[i] * s;
                den += s * s;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                num += __shfl_xor_sync(0xffffffffu, num, o);
                den += __shfl_xor_sync(0xffffffffu, den, o);
            }
            if (lane == 0) {
                double eta = (den <= 1e-14 * (1.0 + fabs(num))) ? 0.0 : num / den;
                s_scalar[2 + side] = (float)eta;
            }
        }
        __syncthreads();
        const float eta = s_scalar[2 + side];
        if (args.update_b && eta != 0.f) {
            float *Bg = side ? (L.B_K + (size_t)bh * R * d) : (L.B_Q + (size_t)bh * R * d);
            for (int e = tid; e < r * d; e += blockDim.x) {
                const int p = e / d, i = e - p * d;
                Bg[p * d + i] = Bm[p * (d + 1) + i] - eta * (xh[p] * resid[i]);
            }
        }
        __syncthreads();
    }

    // ---------------- outputs and appends ---------------------------------
    for (int i = tid; i < R; i += blockDim.x) {
        L.q_hat[(size_t)bh * R + i] = qh[i];
        L.k_hat[(size_t)bh * R + i] = kh[i];
    }
    if (tid == 0) {
        L.eta[(size_t)bh * 2 + 0] = s_scalar[2];
        L.eta[(size_t)bh * 2 + 1] = s_scalar[3];
    }
    // append k_hat to the proxy store (cache.py:211)
    {
        T *dst = reinterpret_cast<T *>(L.proxy) + (head_rows + t) * R;
        for (int i = tid; i < R; i += blockDim.x) dst[i] = from_float<T>(kh[i]);
    }
    // append k, v to the slow tier once per KV head (cache.py:209-210)
    if (h % G == 0) {
        T *dk = reinterpret_cast<T *>(L.slow_k) + (kv_rows + t) * d;
        T *dv = reinterpret_cast<T *>(L.slow_v) + (kv_rows + t) * d;
        for (int i = tid; i < d; i += blockDim.x) { dk[i] = krow[i]; dv[i] = vrow[i]; }
    }
    // host policy: the new row also lands in this head's spare slot
    if (host) {
        const int slot = L.spare_slot[bh];
        T *sk = reinterpret_cast<T *>(L.slot_k) + ((size_t)bh * L.n_slots + slot) * d;
        T *sv = reinterpret_cast<T *>(L.slot_v) + ((size_t)bh * L.n_slots + slot) * d;
        for (int i = tid; i < d; i += blockDim.x) { sk[i] = krow[i]; sv[i] = vrow[i]; }
    }
}

size_t compress_smem_bytes(const lrqk_layer_t &L) {
    const size_t d = L.dim_stride, R = L.rank_stride;
    const size_t RB = R / 4, NP = RB * (RB + 1) / 2;
    const size_t NG = NP >= kCompressThreads ? 1 : kCompressThreads / NP;
    size_t a = (d + kRedRows + (size_t)kRedRows * (R + 1) + NG * NP * 16) * sizeof(float);
    size_t bsz = (2 * R * (d + 1) + 3 * R * (R + 1) + 4 * d + 10 * R + R * (R + 1)) * sizeof(float);
    return a > bsz ? a : bsz;
}

int compress_chunks(const lrqk_layer_t &L) { return (L.s_cap + kRedRows - 1) / kRedRows; }

int launch_compress(const lrqk_layer_t &L, const void *q, const void *k, const void *v, int update_b,
                    cudaStream_t st) {
    CompressArgs a{L, q, k, v, update_b};
    dim3 grid(compress_chunks(L), L.batch * L.n_q_heads);
    size_t smem = compress_smem_bytes(L);
    if (L.dtype == LRQK_BF16) {
        auto fn = compress_kernel<__nv_bfloat16>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        fn<<<grid, kCompressThreads, smem, st>>>(a);
    } else {
        auto fn = compress_kernel<float>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        fn<<<grid, kCompressThreads, smem, st>>>(a);
    }
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

}  // namespace lrqk
