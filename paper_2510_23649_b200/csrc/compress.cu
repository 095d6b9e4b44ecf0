// K2: per-token compression (q_hat, k_hat), B line-search update and the
// append of (k_hat -> proxy store, k/v -> slow tier / slot).
//
// ref: decode.py:79-184 (khat_initial_guess, update_qhat, update_khat,
//      decode_compress, _line_search_step, update_projections),
//      cache.py:199-214 (append_token), session.py:95-98 (order).
//
// Work layout: grid.y = B*Hq (one reference session per y).  Along grid.x,
//   blocks 0..n_chunks-1  ("reduce" blocks) each take kRedRows rows of the
//       previous resident set Omega_{t-1} and produce partial sums of
//           G_res = A_res^T A_res            (decode.py:106)
//           m_res = (q K_res^T) A_res        (decode.py:105)
//   block n_chunks       ("prep" block) works concurrently on everything that
//       does not depend on Omega_{t-1}:  R = B_K B_K^T, its inverse,
//       k_hat0 = (k B_K^T) R^-1 (decode.py:79-81), B_Q B_Q^T, q B_Q^T, q.k.
// The last block of the head to arrive ("finish") forms
//   P = B_Q B_Q^T + l2 G_res, inverts it, and runs the alternation with the
// closed form of a rank-1-updated SPD system
//        x (S + l1 v^T v) = b + l1 qk v
//        =>  x = y + u * l1 (qk - y.v) / (1 + l1 v.u),  y = b S^-1, u = v S^-1,
// which is algebraically the reference's solve_spd(M, RHS) with
// M = S + l1 v^T v (decode.py:100-108, 115-119).  Inverses come from an
// in-place Gauss-Jordan sweep without pivoting: every pivot is > 0 exactly
// when the matrix is numerically SPD, i.e. when the reference's Cholesky
// succeeds.  If P or R is not SPD the finish block solves each full system
// directly with the reference's single jitter retry (linalg.py:80-91).
#include <algorithm>

#include "common.cuh"

namespace lrqk {

constexpr int kCompressThreads = 256;
constexpr int kMaxElems = 16;  // GJ elements per thread: r^2 / 256 for r <= 64

struct CompressArgs {
    lrqk_layer_t L;
    const void *q, *k, *v;
    int update_b;
};

// Per-head prep area inside red_scratch, after the chunk partials.
struct PrepLayout {
    int RQ, Rinv, bq, bk, yk, misc, total;
};
__host__ __device__ inline PrepLayout prep_layout(int R) {
    PrepLayout p;
    int o = 0;
    p.RQ = o; o += R * R;
    p.Rinv = o; o += R * R;
    p.bq = o; o += R;
    p.bk = o; o += R;
    p.yk = o; o += R;
    p.misc = o; o += 4;  // qk, R-is-SPD flag, non-finite flag
    p.total = o;
    return p;
}
__host__ __device__ inline size_t red_head_floats(int R, int nchunks) {
    return (size_t)nchunks * (R * R + R) + prep_layout(R).total;
}

// ---------------------------------------------------------------------------
// An n x n matrix (n <= 64) spread over the block's registers: slot s of a
// thread holds element e = tid + s*blockDim.x (row-major); its (row, col) is
// decoded once into `ij` (-1 marks an unused slot).
// Gauss-Jordan inversion in place: row k and column k travel through
// double-buffered shared vectors, so each pivot costs one barrier.  inverse()
// returns false (uniformly) if a pivot is not > 0, i.e. exactly when the
// matrix is not numerically SPD.
// ---------------------------------------------------------------------------
struct RegMat {
    float a[kMaxElems];
    int ij[kMaxElems];  // (i << 8) | j, or -1

    __device__ void init(int n) {
#pragma unroll
        for (int s = 0; s < kMaxElems; ++s) {
            const int e = threadIdx.x + s * blockDim.x;
            ij[s] = e < n * n ? (((e / n) << 8) | (e % n)) : -1;
        }
    }
    __device__ void load(const float *M, int ld, float diag_add = 0.f) {
#pragma unroll
        for (int s = 0; s < kMaxElems; ++s) {
            if (ij[s] < 0) break;
            const int i = ij[s] >> 8, j = ij[s] & 255;
            a[s] = M[i * ld + j] + (i == j ? diag_add : 0.f);
        }
    }
    __device__ void store(float *M, int ld) const {
#pragma unroll
        for (int s = 0; s < kMaxElems; ++s) {
            if (ij[s] < 0) break;
            M[(ij[s] >> 8) * ld + (ij[s] & 255)] = a[s];
        }
    }
    __device__ bool inverse(int n, float *s_rc /* 256 floats */) {
        for (int k = 0; k < n; ++k) {
            float *row = s_rc + (k & 1) * 128;
            float *col = row + 64;
#pragma unroll
            for (int s = 0; s < kMaxElems; ++s) {
                if (ij[s] < 0) break;
                const int i = ij[s] >> 8, j = ij[s] & 255;
                if (i == k) row[j] = a[s];
                if (j == k) col[i] = a[s];
            }
            __syncthreads();
            const float p = row[k];
            if (!(p > 0.f) || !isfinite(p)) return false;
            const float ip = 1.f / p;
#pragma unroll
            for (int s = 0; s < kMaxElems; ++s) {
                if (ij[s] < 0) break;
                const int i = ij[s] >> 8, j = ij[s] & 255;
                if (i == k && j == k) a[s] = ip;
                else if (i == k) a[s] *= ip;
                else if (j == k) a[s] = -a[s] * ip;
                else a[s] = fmaf(-col[i] * ip, row[j], a[s]);
            }
        }
        __syncthreads();
        return true;
    }
};

// Solve x M = rhs directly (M SPD n x n, row stride ld) with the reference's
// single jitter retry.  Returns 0 ok, 1 ok after jitter, 2 failed.
__device__ int solve_spd_direct(const float *M, int n, int ld, const float *rhs, float *x, float *work,
                                float *s_rc) {
    RegMat m;
    m.init(n);
    for (int attempt = 0; attempt < 2; ++attempt) {
        float jit = 0.f;
        if (attempt == 1) {
            float tr = 0.f, dmax = 0.f;
            for (int i = 0; i < n; ++i) { tr += M[i * ld + i]; dmax = fmaxf(dmax, fabsf(M[i * ld + i])); }
            // 1e-10 (tr/n + 1) as the reference, floored at fp32 resolution
            jit = fmaxf(1e-10f * (tr / n + 1.f), dmax * 1.2e-7f);
        }
        m.load(M, ld, jit);
        __syncthreads();
        if (m.inverse(n, s_rc)) {
            m.store(work, n);
            __syncthreads();
            for (int j = threadIdx.x; j < n; j += blockDim.x) {
                float acc = 0.f;
                for (int i = 0; i < n; ++i) acc = fmaf(rhs[i], work[i * n + j], acc);
                x[j] = acc;
            }
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

// ---------------------------------------------------------------------------
// reduce blocks: partial G_res (upper 4x4 tiles) and m_res of kRedRows rows
// ---------------------------------------------------------------------------
template <typename T, int LPR, int PPL>
__device__ void reduce_chunk(const lrqk_layer_t &L, const T *qrow, const T *kres_base, const T *proxy, bool host,
                             int bh, int row0, int nrow, float *part_out, float *smem) {
    constexpr int N = Pack<T>::N;
    constexpr int RPW = 32 / LPR;
    constexpr int NW = kCompressThreads / 32;
    constexpr int STEPS = kRedRows / (NW * RPW);
    constexpr int SR = STEPS < 8 ? STEPS : 8;  // rows in flight per lane group
    const int d = L.dim_stride, R = L.rank_stride;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sub = lane / LPR, sl = lane - sub * LPR;
    const int ldA = R + 1;
    float *sq = smem;                        // [d]
    float *sS = sq + d;                      // [kRedRows]
    float *sA = sS + kRedRows;               // [kRedRows][R+1]
    int *sIdx = reinterpret_cast<int *>(sA + kRedRows * ldA);  // gather row (slot or index)
    int *sPx = sIdx + kRedRows;              // proxy row (index)
    float *sRed = reinterpret_cast<float *>(sPx + kRedRows);
    for (int i = tid; i < d; i += blockDim.x) sq[i] = to_float<T>(qrow[i]);
    const int *ridx = L.res_idx + (size_t)bh * L.s_cap + row0;
    const int *rslot = L.res_slot + (size_t)bh * L.s_cap + row0;
    for (int j = tid; j < nrow; j += blockDim.x) {
        const int x = ridx[j];
        sPx[j] = x;
        sIdx[j] = host ? rslot[j] : x;
    }
    __syncthreads();
    // A_res rows: issue the loads first, consume after the K dots
    const int apacks = R / N;
    constexpr int AU = 4;
    uint4 ax[AU];
    const int total_a = nrow * apacks;
#pragma unroll
    for (int u = 0; u < AU; ++u) {
        const int e = tid + u * kCompressThreads;
        if (e < total_a) {
            const int j = e / apacks, p = e - j * apacks;
            ax[u] = *reinterpret_cast<const uint4 *>(proxy + proxy_pack_offset(sPx[j], p, apacks) * N);
        }
    }
    // K_res rows: q . K_res[j]
    for (int s0 = 0; s0 < STEPS; s0 += SR) {
        uint4 kx[SR][PPL];
#pragma unroll
        for (int s = 0; s < SR; ++s) {
            const int j = ((s0 + s) * NW + warp) * RPW + sub;
            if (j < nrow) {
                const T *kr = kres_base + (size_t)sIdx[j] * d;
#pragma unroll
                for (int pp = 0; pp < PPL; ++pp)
                    kx[s][pp] = *reinterpret_cast<const uint4 *>(kr + (sl + pp * LPR) * N);
            } else {
#pragma unroll
                for (int pp = 0; pp < PPL; ++pp) kx[s][pp] = make_uint4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int s = 0; s < SR; ++s) {
            const int j = ((s0 + s) * NW + warp) * RPW + sub;
            float part = 0.f;
#pragma unroll
            for (int pp = 0; pp < PPL; ++pp) {
                float x[N];
                unpack16<T>(kx[s][pp], x);
                const float *qq = sq + (sl + pp * LPR) * N;
#pragma unroll
                for (int e = 0; e < N; ++e) part = fmaf(x[e], qq[e], part);
            }
            part = group_sum<LPR>(part);
            if (j < nrow && sl == 0) sS[j] = part;
        }
    }
#pragma unroll
    for (int u = 0; u < AU; ++u) {
        const int e = tid + u * kCompressThreads;
        if (e < total_a) {
            const int j = e / apacks, p = e - j * apacks;
            float x[N];
            unpack16<T>(ax[u], x);
#pragma unroll
            for (int i = 0; i < N; ++i) sA[j * ldA + p * N + i] = x[i];
        }
    }
    for (int e = tid + AU * kCompressThreads; e < total_a; e += kCompressThreads) {
        const int j = e / apacks, p = e - j * apacks;
        float x[N];
        Pack<T>::load(proxy + proxy_pack_offset(sPx[j], p, apacks) * N, x);
#pragma unroll
        for (int i = 0; i < N; ++i) sA[j * ldA + p * N + i] = x[i];
    }
    __syncthreads();
    // upper-triangular 4x4 tiles of G over the chunk's rows
    const int RB = R / 4;
    const int NP = RB * (RB + 1) / 2;
    const int NG = max(1, kCompressThreads / NP);
    if (tid < NP * NG) {
        const int pair = tid % NP, grp = tid / NP;
        int pb = 0, rem = pair;
        while (rem >= RB - pb) { rem -= RB - pb; ++pb; }
        const int qb = pb + rem;
        float acc[16] = {};
        for (int j = grp; j < nrow; j += NG) {
            const float *a = sA + j * ldA;
            float ap[4], aq[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { ap[u] = a[pb * 4 + u]; aq[u] = a[qb * 4 + u]; }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int w2 = 0; w2 < 4; ++w2) acc[u * 4 + w2] = fmaf(ap[u], aq[w2], acc[u * 4 + w2]);
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) sRed[(grp * NP + pair) * 16 + e] = acc[e];
    }
    for (int p = tid; p < R; p += kCompressThreads) {
        float acc0 = 0.f, acc1 = 0.f;
        int j = 0;
        for (; j + 1 < nrow; j += 2) {
            acc0 = fmaf(sS[j], sA[j * ldA + p], acc0);
            acc1 = fmaf(sS[j + 1], sA[(j + 1) * ldA + p], acc1);
        }
        if (j < nrow) acc0 = fmaf(sS[j], sA[j * ldA + p], acc0);
        part_out[R * R + p] = acc0 + acc1;
    }
    __syncthreads();
    for (int e = tid; e < NP * 16; e += kCompressThreads) {
        float acc = 0.f;
        for (int gI = 0; gI < NG; ++gI) acc += sRed[(gI * NP) * 16 + e];
        const int pair = e / 16, uw = e - pair * 16;
        int pb = 0, rem = pair;
        while (rem >= RB - pb) { rem -= RB - pb; ++pb; }
        const int qb = pb + rem;
        part_out[(pb * 4 + uw / 4) * R + qb * 4 + (uw & 3)] = acc;  // tiles with pb <= qb
    }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <typename T, int LPR, int PPL>
__global__ void __launch_bounds__(kCompressThreads)
compress_kernel(const CompressArgs args) {
    const lrqk_layer_t &L = args.L;
    extern __shared__ __align__(16) float smem[];
    __shared__ int s_flag;
    __shared__ float s_rc[256];
    __shared__ float s_scalar[8];
    __shared__ int s_bad;

    const int bh = blockIdx.y;
    const int b = bh / L.n_q_heads, h = bh - b * L.n_q_heads;
    const int G = L.n_q_heads / L.n_kv_heads;
    const int g = h / G;
    const int d = L.dim_stride, R = L.rank_stride, r = L.rank;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int t = L.ctx_len[b];
    if (t >= L.t_max) {
        if (blockIdx.x == 0 && tid == 0) set_status(L.status, LRQK_ST_CAPACITY);
        return;
    }
    const int nchunks = gridDim.x - 1;
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
    float *hs = L.red_scratch + (size_t)bh * red_head_floats(R, nchunks);
    const PrepLayout PL = prep_layout(R);
    float *prep = hs + (size_t)nchunks * (R * R + R);
    const int ldM = R + 1;

    if ((int)blockIdx.x < nchunks) {
        const int row0 = blockIdx.x * kRedRows;
        const int nrow = max(0, min(kRedRows, n_prev - row0));
        reduce_chunk<T, LPR, PPL>(L, qrow, kres_base, proxy, host, bh, row0, nrow,
                                  hs + (size_t)blockIdx.x * (R * R + R), smem);
    } else {
        // ---------------- prep block: the Omega-independent algebra ---------
        float *sBQ = smem;                   // [R][d+1]
        float *sBK = sBQ + R * (d + 1);      // [R][d+1]
        float *sR = sBK + R * (d + 1);       // [R][ldM]
        float *vq = sR + R * ldM;            // [d]
        float *vk = vq + d;                  // [d]
        float *bk = vk + d;                  // [R]
        float *tmp = bk + R;                 // gram scratch
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
            if (!isfinite(vq[i]) || !isfinite(vk[i]) || !isfinite(to_float<T>(vrow[i]))) s_bad = 1;
        }
        __syncthreads();
        gram_rows(sBK, r, d, d + 1, sR, ldM, tmp);            // R = B_K B_K^T
        gram_rows(sBQ, r, d, d + 1, prep + PL.RQ, R, tmp);    // B_Q B_Q^T
        for (int o = tid; o < 2 * r + 1; o += blockDim.x) {    // q B_Q^T, k B_K^T, q.k
            const float *x = o < r ? sBQ + o * (d + 1) : (o < 2 * r ? sBK + (o - r) * (d + 1) : vq);
            const float *y = o < r ? vq : vk;
            float a0 = 0.f, a1 = 0.f;
            for (int i = 0; i < d; i += 2) {
                a0 = fmaf(x[i], y[i], a0);
                a1 = fmaf(x[i + 1], y[i + 1], a1);
            }
            const float s = a0 + a1;
            if (o < r) prep[PL.bq + o] = s;
            else if (o < 2 * r) { prep[PL.bk + o - r] = s; bk[o - r] = s; }
            else prep[PL.misc + 0] = s;
        }
        __syncthreads();
        RegMat m;
        m.init(r);
        m.load(sR, ldM);
        const bool ok = m.inverse(r, s_rc);
        if (ok) {
            m.store(prep + PL.Rinv, R);
            m.store(sR, ldM);
        }
        __syncthreads();
        if (ok && warp == 0) warp_vecmat(bk, sR, r, ldM, prep + PL.yk);  // k_hat0
        if (tid == 0) {
            prep[PL.misc + 1] = ok ? 1.f : 0.f;
            prep[PL.misc + 2] = s_bad ? 1.f : 0.f;
        }
    }
    if (!last_arrival(L.counters + (size_t)bh * kCounterInts + C_COMPRESS, gridDim.x, &s_flag)) return;

    // ================= finish (one block per head) ==========================
    float *sP = smem;                    // [R][ldM]  P, then P^-1
    float *sRi = sP + R * ldM;           // [R][ldM]  R^-1 (R in the fallback)
    float *vq = sRi + R * ldM;           // [d]
    float *vk = vq + d;                  // [d]
    float *bk = vk + d;                  // [R]
    float *mres = bk + R;                // [R]
    float *yq = mres + R;                // [R]
    float *yk = yq + R;                  // [R]
    float *qh = yk + R;                  // [R]
    float *kh = qh + R;                  // [R]
    float *u = kh + R;                   // [R]
    float *prevc = u + R;                // [2R]
    float *resid = prevc + 2 * R;        // [2][d]
    float *work = resid + 2 * d;         // [R*(R+1)] fallback
    float *sM = work + R * (R + 1);      // [R][ldM] fallback system
    const float l1 = L.lambda_1, l2 = L.lambda_2;
    if (__ldcg(prep + PL.misc + 2) != 0.f) {  // ref: linalg.py:32-33 via as_row (session.py:94)
        if (tid == 0) set_status(L.status, LRQK_ST_NONFINITE);
        return;
    }
    const bool have_res = n_prev > 0;
    const float qk = __ldcg(prep + PL.misc + 0);
    const bool okR = __ldcg(prep + PL.misc + 1) != 0.f;
    for (int i = tid; i < d; i += blockDim.x) {
        vq[i] = to_float<T>(qrow[i]);
        vk[i] = to_float<T>(krow[i]);
    }
    // P = B_Q B_Q^T + l2 G_res ; m = q B_Q^T + l2 m_res
    for (int e = tid; e < r * r; e += blockDim.x) {
        const int pi = e / r, qi = e - pi * r;
        const int a0 = min(pi, qi), c0 = max(pi, qi);
        float g0 = 0.f, g1 = 0.f;
        if (have_res) {
            int ch = 0;
            for (; ch + 1 < nchunks; ch += 2) {
                g0 += __ldcg(hs + (size_t)ch * (R * R + R) + a0 * R + c0);
                g1 += __ldcg(hs + (size_t)(ch + 1) * (R * R + R) + a0 * R + c0);
            }
            if (ch < nchunks) g0 += __ldcg(hs + (size_t)ch * (R * R + R) + a0 * R + c0);
        }
        sP[pi * ldM + qi] = __ldcg(prep + PL.RQ + pi * R + qi) + (have_res ? l2 * (g0 + g1) : 0.f);
    }
    for (int p = tid; p < r; p += blockDim.x) {
        float m0 = 0.f, m1 = 0.f;
        if (have_res) {
            int ch = 0;
            for (; ch + 1 < nchunks; ch += 2) {
                m0 += __ldcg(hs + (size_t)ch * (R * R + R) + R * R + p);
                m1 += __ldcg(hs + (size_t)(ch + 1) * (R * R + R) + R * R + p);
            }
            if (ch < nchunks) m0 += __ldcg(hs + (size_t)ch * (R * R + R) + R * R + p);
        }
        mres[p] = __ldcg(prep + PL.bq + p) + (have_res ? l2 * (m0 + m1) : 0.f);
        bk[p] = __ldcg(prep + PL.bk + p);
        yk[p] = okR ? __ldcg(prep + PL.yk + p) : 0.f;
    }
    if (okR)
        for (int e = tid; e < r * r; e += blockDim.x) {
            const int pi = e / r, qi = e - pi * r;
            sRi[pi * ldM + qi] = __ldcg(prep + PL.Rinv + pi * R + qi);
        }
    __syncthreads();
    bool okP = false;
    if (okR) {
        RegMat m;
        m.init(r);
        m.load(sP, ldM);
        okP = m.inverse(r, s_rc);
        if (okP) m.store(sP, ldM);  // on failure sP still holds P
        __syncthreads();
    }
    const int max_iter = L.max_iter;
    if (okP) {
        if (warp == 0) {
            warp_vecmat(mres, sP, r, ldM, yq);     // y_q = m P^-1
            for (int i = lane; i < r; i += 32) kh[i] = yk[i];
            __syncwarp();
            for (int it = 0; it < max_iter; ++it) {
                warp_vecmat(kh, sP, r, ldM, u);    // q_hat (decode.py:84-108)
                const float alpha = warp_dot(yq, kh, r), c = warp_dot(u, kh, r);
                const float coef = l1 * (qk - alpha) / (1.f + l1 * c);
                for (int i = lane; i < r; i += 32) qh[i] = fmaf(coef, u[i], yq[i]);
                __syncwarp();
                warp_vecmat(qh, sRi, r, ldM, u);   // k_hat (decode.py:111-119)
                const float beta = warp_dot(yk, qh, r), e2 = warp_dot(u, qh, r);
                const float coef2 = l1 * (qk - beta) / (1.f + l1 * e2);
                for (int i = lane; i < r; i += 32) kh[i] = fmaf(coef2, u[i], yk[i]);
                __syncwarp();
                float dsum = 0.f;                  // stop rule (decode.py:143-146)
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
        }
        __syncthreads();
    } else {
        // ---- fallback: the reference's direct solves with jitter retry -----
        const float *BKg = L.B_K + (size_t)bh * R * d;
        for (int o = warp; o < r * r; o += nwarps) {  // R = B_K B_K^T again
            const int pi = o / r, qi = o - pi * r;
            float acc = 0.f;
            for (int i = lane; i < d; i += 32) acc = fmaf(BKg[pi * d + i], BKg[qi * d + i], acc);
            acc = warp_sum(acc);
            if (lane == 0) sRi[pi * ldM + qi] = acc;
        }
        __syncthreads();
        int jitter = 0;
        int rc = solve_spd_direct(sRi, r, ldM, bk, kh, work, s_rc);  // k_hat0
        if (rc == 2) { if (tid == 0) set_status(L.status, LRQK_ST_SOLVE_FAILED); return; }
        jitter |= rc;
        for (int it = 0; it < max_iter; ++it) {
            __syncthreads();
            for (int e = tid; e < r * r; e += blockDim.x) {
                const int pi = e / r, qi = e - pi * r;
                sM[pi * ldM + qi] = sP[pi * ldM + qi] + l1 * kh[pi] * kh[qi];
            }
            for (int p = tid; p < r; p += blockDim.x) u[p] = mres[p] + l1 * qk * kh[p];
            __syncthreads();
            rc = solve_spd_direct(sM, r, ldM, u, qh, work, s_rc);
            if (rc == 2) { if (tid == 0) set_status(L.status, LRQK_ST_SOLVE_FAILED); return; }
            jitter |= rc;
            __syncthreads();
            for (int e = tid; e < r * r; e += blockDim.x) {
                const int pi = e / r, qi = e - pi * r;
                sM[pi * ldM + qi] = sRi[pi * ldM + qi] + l1 * qh[pi] * qh[qi];
            }
            for (int p = tid; p < r; p += blockDim.x) u[p] = bk[p] + l1 * qk * qh[p];
            __syncthreads();
            rc = solve_spd_direct(sM, r, ldM, u, kh, work, s_rc);
            if (rc == 2) { if (tid == 0) set_status(L.status, LRQK_ST_SOLVE_FAILED); return; }
            jitter |= rc;
            __syncthreads();
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
        if (tid == 0) set_status(L.status, LRQK_ST_FALLBACK | (jitter ? LRQK_ST_JITTERED : 0u));
    }
    __syncthreads();
    for (int i = r + tid; i < R; i += blockDim.x) { qh[i] = 0.f; kh[i] = 0.f; }
    __syncthreads();

    // ---------------- line-search B update (decode.py:150-184), both sides --
    // resid = x_hat B - x ; s = x_hat grad = |x_hat|^2 resid ; eta = (resid.s)/(s.s)
    const float *BQg = L.B_Q + (size_t)bh * R * d;
    const float *BKg = L.B_K + (size_t)bh * R * d;
    for (int w = tid; w < 2 * d; w += blockDim.x) {
        const int side = w / d, i = w - side * d;
        const float *xh = side ? kh : qh;
        const float *Bm = side ? BKg : BQg;
        float acc = 0.f;
        for (int p = 0; p < r; ++p) acc = fmaf(xh[p], __ldcg(Bm + p * d + i), acc);
        resid[w] = acc - (side ? vk[i] : vq[i]);
    }
    __syncthreads();
    if (warp < 2) {
        const int side = warp;
        const float *xh = side ? kh : qh;
        const float nx = warp_dot(xh, xh, r);
        double num = 0.0, den = 0.0;
        for (int i = lane; i < d; i += 32) {
            const double rr = (double)resid[side * d + i];
            const double s = (double)nx * rr;
            num += rr * s;
            den += s * s;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            num += __shfl_xor_sync(0xffffffffu, num, o);
            den += __shfl_xor_sync(0xffffffffu, den, o);
        }
        if (lane == 0) s_scalar[2 + side] = (den <= 1e-14 * (1.0 + fabs(num))) ? 0.f : (float)(num / den);
    }
    __syncthreads();
    if (args.update_b) {
        for (int w = tid; w < 2 * r * d; w += blockDim.x) {
            const int side = w / (r * d), e = w - side * r * d;
            const float eta = s_scalar[2 + side];
            if (eta == 0.f) continue;
            const int p = e / d, i = e - p * d;
            float *Bg = (side ? L.B_K : L.B_Q) + (size_t)bh * R * d;
            const float *xh = side ? kh : qh;
            Bg[p * d + i] = __ldcg(Bg + p * d + i) - eta * (xh[p] * resid[side * d + i]);
        }
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
    {   // append k_hat to the proxy store (cache.py:211), interleaved layout
        constexpr int N = Pack<T>::N;
        const int apacks = R / N;
        T *base = reinterpret_cast<T *>(L.proxy) + head_rows * R;
        for (int i = tid; i < R; i += blockDim.x)
            base[proxy_pack_offset(t, i / N, apacks) * N + (i % N)] = from_float<T>(kh[i]);
    }
    if (h % G == 0) {  // append k, v once per KV head (cache.py:209-210)
        T *dk = reinterpret_cast<T *>(L.slow_k) + (kv_rows + t) * d;
        T *dv = reinterpret_cast<T *>(L.slow_v) + (kv_rows + t) * d;
        for (int i = tid; i < d; i += blockDim.x) { dk[i] = krow[i]; dv[i] = vrow[i]; }
    }
    if (host) {  // the new row also lands in this head's spare slot
        const int slot = L.spare_slot[bh];
        T *sk = reinterpret_cast<T *>(L.slot_k) + ((size_t)bh * L.n_slots + slot) * d;
        T *sv = reinterpret_cast<T *>(L.slot_v) + ((size_t)bh * L.n_slots + slot) * d;
        for (int i = tid; i < d; i += blockDim.x) { sk[i] = krow[i]; sv[i] = vrow[i]; }
    }
}

int compress_chunks(const lrqk_layer_t &L) { return (L.s_cap + kRedRows - 1) / kRedRows; }

size_t compress_scratch_floats_per_head(const lrqk_layer_t &L) {
    return red_head_floats(L.rank_stride, compress_chunks(L));
}

size_t compress_smem_bytes(const lrqk_layer_t &L) {
    const size_t d = L.dim_stride, R = L.rank_stride;
    const size_t RB = R / 4, NP = RB * (RB + 1) / 2;
    const size_t NG = NP >= (size_t)kCompressThreads ? 1 : kCompressThreads / NP;
    const size_t a = (d + kRedRows + (size_t)kRedRows * (R + 1) + 2 * kRedRows + NG * NP * 16) * sizeof(float);
    const size_t p = (2 * R * (d + 1) + R * (R + 1) + 2 * d + R + 2 * NP * 16) * sizeof(float);
    const size_t f = (4 * R * (R + 1) + 4 * d + 9 * R) * sizeof(float);
    return std::max(a, std::max(p, f));
}

template <typename T>
static int launch_compress_t(const CompressArgs &a, cudaStream_t st) {
    const lrqk_layer_t &L = a.L;
    constexpr int N = Pack<T>::N;
    const int packs = L.dim_stride / N;
    const int lpr = packs < 32 ? packs : 32;
    const int ppl = packs / lpr;
    dim3 grid(compress_chunks(L) + 1, L.batch * L.n_q_heads);
    const size_t smem = compress_smem_bytes(L);
#define LRQK_CMP(LP, PP)                                                                   \
    do {                                                                                   \
        auto fn = compress_kernel<T, LP, PP>;                                              \
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
        fn<<<grid, kCompressThreads, smem, st>>>(a);                                       \
    } while (0)
    if (ppl == 1) {
        switch (lpr) {
            case 1: LRQK_CMP(1, 1); break;
            case 2: LRQK_CMP(2, 1); break;
            case 4: LRQK_CMP(4, 1); break;
            case 8: LRQK_CMP(8, 1); break;
            case 16: LRQK_CMP(16, 1); break;
            case 32: LRQK_CMP(32, 1); break;
            default: return LRQK_EUNSUPPORTED;
        }
    } else if (ppl == 2 && lpr == 32) {
        LRQK_CMP(32, 2);
    } else {
        return LRQK_EUNSUPPORTED;
    }
#undef LRQK_CMP
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

int launch_compress(const lrqk_layer_t &L, const void *q, const void *k, const void *v, int update_b,
                    cudaStream_t st) {
    CompressArgs a{L, q, k, v, update_b};
    return L.dtype == LRQK_BF16 ? launch_compress_t<__nv_bfloat16>(a, st) : launch_compress_t<float>(a, st);
}

}  // namespace lrqk
