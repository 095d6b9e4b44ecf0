// K1: the prefill joint rank-r factorisation, in Gram space on the tensor
// cores.
//
// ref: prefill.py:142-230 (lagrangian_value, update_B, update_AK, update_AQ,
//      _factor_delta, prefill_run), linalg.py:63-93 (solve_spd).
//
// Every product of the reference sweep is associated so that X (Q or K)
// enters only through its d x d Gram GX = X^T X and, once, through the init
// cross term C0 = X^T A0:
//
//   after the first A update, A_X = X W_X for a d x r matrix W_X, so
//   C_X = X^T A_X = GX W_X,  G_AX = A_X^T A_X = W_X^T GX W_X,
//   ||A_X' - A_X||^2 = tr(dW^T GX dW),
//   ||X - A_X B_X||^2 = tr(GX) - 2<B_X^T, C_X> + <G_AX, B_X B_X^T>,
//   ||Q K^T - A_Q A_K^T||^2 = <GQ, GK> - 2<C_Q, C_K> + <G_AQ, G_AK>
//   (the reference's own Gram-trace expansion, prefill.py:150-153).
//
// So the whole factorisation streams each prompt matrix exactly twice:
//
//   K1g  pf_gram_kernel      one TMA -> tcgen05 pass per head:
//                            D1 = X^T X (128 x 128) and D2 = X^T Y (Y = the
//                            bf16 hi|lo split of A0), fp32 accumulators in
//                            TMEM, split over row slabs
//   K1c  pf_combine_kernel   slab partials -> float64 GX, C0, G0 = A0^T A0
//   K1s  pf_solve_kernel     one block per query head: every sweep of the
//                            reference in float64 on d x r / r x r matrices
//                            (Cholesky with the reference's jitter retry),
//                            the objective trajectory and the convergence
//                            test; writes B_Q, B_K and W_Q, W_K
//   K1m  pf_mat_kernel       one TMA -> tcgen05 pass: A_Q = Q W_Q and
//                            A_K = K W_K, one K tile serving all the query
//                            heads of its GQA group (N = heads x 2r)
//
// Precision.  bf16 X is exact on the tensor core.  fp32 X is split into bf16
// hi + lo (|X - hi - lo| <= 2^-17 |X|) and every product takes both parts;
// fp32 factors (A0, W) are split the same way.  Accumulation is fp32 in
// TMEM, slab sums and all the d-space algebra are float64.
#include <cudaTypedefs.h>
#include <string.h>

#include <algorithm>

#include "tc_common.cuh"

namespace lrqk {

constexpr int kTile = 128;                 // rows per TMA tile
constexpr int kBlkBytes = kTile * 128;     // one 64-column SW128 block of a tile
constexpr int kMaxMapW = 128;              // widest TMA'd tensor (columns)
constexpr int kGramThreads = 128;
constexpr int kMatThreads = 192;           // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kSolveThreads = 1024;
constexpr int kMaxStages = 6;
constexpr int kEpiStride = 36;                 // pf_mat staged epilogue: padded row (floats)
constexpr int kEpiWarpFloats = 32 * kEpiStride;
constexpr int kEpiBytes = 1024 + 4 * kEpiWarpFloats * 4;  // barrier room + four warp buffers
constexpr int kWorkMats = 10;              // float64 d x r work matrices per head (solver)

enum PfMap { MQ = 0, MQL = 1, MK = 2, MKL = 3, MYQ = 4, MYK = 5, kNumMaps = 6 };

struct PfMaps {
    CUtensorMap m[kNumMaps];
};

struct PfGeom {
    int H, Hk, group, l, d, ds, r, rs;
    int parts;   // 1: bf16 X, 2: fp32 X as bf16 hi + lo
    int direct;  // bf16 X TMA'd in place
    int XW, YW;  // TMA'd widths (64 or 128) of X and of Y = [A0 hi | A0 lo | 0]
    int shared;  // one A0 for every head (the reference's randn draw)
    int NY;      // Y tensors per side
    int NQU, NKU, NU, S, PW, tiles;
    int NMU, HPU, nsub, Nmax;  // materialize units, heads per K unit, K sub-units per KV head, max N
    size_t off_x[4], off_y[2], off_part, off_gq, off_cq, off_gk, off_ck, off_g0q, off_g0k, off_w, off_work, total;
};

// one Gram unit: D1 = X^T X, D2 = X^T [Y1 | Y2]
struct GUnit {
    int xm, xh, y1m, y1h, y2m, y2h;
};

__host__ __device__ inline int map_width(const PfGeom &G, int m) {
    return m < 0 ? 0 : (m >= MYQ ? G.YW : G.XW);
}

__host__ __device__ inline GUnit gram_unit(const PfGeom &G, int u) {
    GUnit U{-1, 0, -1, 0, -1, 0};
    const int nq = G.NQU * G.parts, nk = G.NKU * G.parts;
    if (u < nq + nk) {
        const bool kside = u >= nq;
        const int v = kside ? u - nq : u;
        const int i = v / G.parts, part = v % G.parts;
        const int xh = kside ? (G.shared ? i : i / G.group) : i;
        const int yh = G.shared ? 0 : i;
        const int mx = kside ? MK : MQ, mxl = kside ? MKL : MQL, my = kside ? MYK : MYQ;
        if (G.parts == 1) U = GUnit{mx, xh, my, yh, -1, 0};
        else if (part == 0) U = GUnit{mx, xh, mxl, xh, my, yh};
        else U = GUnit{mxl, xh, my, yh, -1, 0};
    } else {
        const int g = u - nq - nk;
        U = g < G.NY ? GUnit{MYQ, g, -1, 0, -1, 0} : GUnit{MYK, g - G.NY, -1, 0, -1, 0};
    }
    return U;
}

// ---------------------------------------------------------------------------
// K1g: D1 = X^T X, D2 = X^T Y over one slab of rows of one unit
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kGramThreads, 1)
pf_gram_kernel(const __grid_constant__ PfMaps maps, const PfGeom G, float *__restrict__ part, int budget) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int u = blockIdx.x / G.S, s = blockIdx.x % G.S;
    const GUnit U = gram_unit(G, u);
    const int xw = map_width(G, U.xm), w1 = map_width(G, U.y1m), w2 = map_width(G, U.y2m);
    const int nxb = xw / 64, nyb = (w1 + w2) / 64, ny = w1 + w2;
    const int stage_bytes = (2 + nyb) * kBlkBytes;
    const int nst = min(kMaxStages, budget / stage_bytes);
    const uint32_t ncols = 128 + ny <= 256 ? 256 : 512;  // D1 | D2 (two CTAs per SM fit at 256)
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + nst * stage_bytes);
    uint64_t *empty = full + kMaxStages;
    uint64_t *done = empty + kMaxStages;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(done + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t0 = (int)((long long)G.tiles * s / G.S), t1 = (int)((long long)G.tiles * (s + 1) / G.S);

    if (nxb == 1) {  // X narrower than the 128-row M: the upper block stays zero
        for (int st = 0; st < nst; ++st)
            for (int e = threadIdx.x; e < kBlkBytes / 16; e += blockDim.x)
                reinterpret_cast<uint4 *>(sm + st * stage_bytes + kBlkBytes)[e] = make_uint4(0, 0, 0, 0);
        tc::fence_proxy_async();
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tc::tma_prefetch(&maps.m[U.xm]);
        if (U.y1m >= 0) tc::tma_prefetch(&maps.m[U.y1m]);
        if (U.y2m >= 0) tc::tma_prefetch(&maps.m[U.y2m]);
    }
    if (warp == 2) tc::tmem_alloc(tslot, ncols);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = *tslot;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer ----------------------------------------------------
        const uint64_t pol_x = l2_policy_evict_first(), pol_y = l2_policy_evict_last();
        for (int t = t0, i = 0; t < t1; ++t, ++i) {
            const int st = i % nst;
            mbar_wait(empty + st, ((i / nst) & 1) ^ 1);
            uint8_t *base = sm + st * stage_bytes;
            mbar_expect_tx(full + st, (nxb + nyb) * kBlkBytes);
            for (int b = 0; b < nxb; ++b)
                tc::tma_load_3d(base + b * kBlkBytes, &maps.m[U.xm], b * 64, t * kTile, U.xh, full + st, pol_x);
            uint8_t *yb = base + 2 * kBlkBytes;
            for (int b = 0; b < w1 / 64; ++b, yb += kBlkBytes)
                tc::tma_load_3d(yb, &maps.m[U.y1m], b * 64, t * kTile, U.y1h, full + st,
                                U.y1m >= MYQ ? pol_y : pol_x);
            for (int b = 0; b < w2 / 64; ++b, yb += kBlkBytes)
                tc::tma_load_3d(yb, &maps.m[U.y2m], b * 64, t * kTile, U.y2h, full + st, pol_y);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer: X^T (MN-major A) against X and Y (MN-major B) --------
        const uint32_t id1 = tc::idesc_bf16(128, 128, true, true);
        const uint32_t id2 = tc::idesc_bf16(128, ny > 0 ? ny : 16, true, true);
        for (int t = t0, i = 0; t < t1; ++t, ++i) {
            const int st = i % nst;
            mbar_wait(full + st, (i / nst) & 1);
            tc::fence_after();
            const uint32_t base = smem_u32(sm + st * stage_bytes);
#pragma unroll
            for (int k = 0; k < kTile / 16; ++k) {
                const uint64_t ax = tc::desc_sw128(base + k * 2048, kBlkBytes, 1024);
                const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
                tc::mma_bf16(tm, ax, ax, id1, acc);
                if (ny) {
                    const uint64_t by = tc::desc_sw128(base + 2 * kBlkBytes + k * 2048, kBlkBytes, 1024);
                    tc::mma_bf16(tm + 128, ax, by, id2, acc);
                }
            }
            tc::mma_commit(empty + st);
        }
        tc::mma_commit(done);
    }
    __syncwarp();
    // ---- epilogue: every warp drains its 32 TMEM lanes (rows of D) ---------
    mbar_wait(done, 0);
    tc::fence_after();
    const int row = warp * 32 + lane;
    float *dst = part + ((size_t)blockIdx.x * kTile + row) * G.PW;
    const uint32_t lane_addr = tm + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 128 + ny; c += 32) {
        float v[32];
        tc::tmem_ld32(lane_addr + c, v);
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4 *>(dst + c + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 2) tc::tmem_dealloc(tm, ncols);
}

// ---------------------------------------------------------------------------
// K1c: slab partials -> float64 GX (mirrored), C0, G0
// ---------------------------------------------------------------------------
LRQK_DEV double slab_sum(const PfGeom &G, const float *part, int u, int row, int col) {
    double s = 0.0;
    const float *p = part + ((size_t)u * G.S * kTile + row) * G.PW + col;
    for (int k = 0; k < G.S; ++k) s += (double)p[(size_t)k * kTile * G.PW];  // fixed order
    return s;
}

__global__ void pf_combine_kernel(const PfGeom G, const float *__restrict__ part, uint8_t *scr) {
    const int RS = G.rs;
    const long long nG = (long long)kTile * kTile, nC = (long long)kTile * RS, n0 = (long long)RS * RS;
    const long long sQ = (long long)G.NQU * (nG + nC), sK = (long long)G.NKU * (nG + nC);
    const long long total = sQ + sK + 2LL * G.NY * n0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        if (e < sQ + sK) {
            const bool kside = e >= sQ;
            long long v = kside ? e - sQ : e;
            const int nunits = kside ? G.NKU : G.NQU;
            const int ubase = kside ? G.NQU * G.parts : 0;
            double *gx = reinterpret_cast<double *>(scr + (kside ? G.off_gk : G.off_gq));
            double *cx = reinterpret_cast<double *>(scr + (kside ? G.off_ck : G.off_cq));
            if (v < nunits * nG) {
                const int h = (int)(v / nG), ij = (int)(v % nG), i = ij / kTile, j = ij % kTile;
                const int a = min(i, j), b = max(i, j);  // gram is exactly symmetric (linalg.py:53-54)
                const int u = ubase + h * G.parts;
                double s = slab_sum(G, part, u, a, b);
                if (G.parts == 2) {
                    // hi^T lo occupies D2 columns [0, XW) only; X is zero past XW
                    if (b < G.XW) s += slab_sum(G, part, u, a, 128 + b) + slab_sum(G, part, u, b, 128 + a);
                    s += slab_sum(G, part, u + 1, a, b);
                }
                gx[(size_t)h * nG + ij] = s;
            } else {
                v -= nunits * nG;
                const int h = (int)(v / nC), ip = (int)(v % nC), i = ip / RS, p = ip % RS;
                const int u = ubase + h * G.parts;
                double s;
                if (G.parts == 1) s = slab_sum(G, part, u, i, 128 + p) + slab_sum(G, part, u, i, 128 + RS + p);
                else
                    s = slab_sum(G, part, u, i, 128 + G.XW + p) + slab_sum(G, part, u, i, 128 + G.XW + RS + p) +
                        slab_sum(G, part, u + 1, i, 128 + p) + slab_sum(G, part, u + 1, i, 128 + RS + p);
                cx[(size_t)h * nC + ip] = s;
            }
        } else {
            long long v = e - sQ - sK;
            const int y = (int)(v / n0), pq = (int)(v % n0), p = pq / RS, q = pq % RS;
            const int a = min(p, q), b = max(p, q);
            const int u = (G.NQU + G.NKU) * G.parts + y;
            const double s = slab_sum(G, part, u, a, b) + slab_sum(G, part, u, a, RS + b) +
                             slab_sum(G, part, u, RS + a, b) + slab_sum(G, part, u, RS + a, RS + b);
            const bool kside = y >= G.NY;
            double *g0 = reinterpret_cast<double *>(scr + (kside ? G.off_g0k : G.off_g0q));
            g0[(size_t)(kside ? y - G.NY : y) * n0 + pq] = s;
        }
    }
}

// ---------------------------------------------------------------------------
// K1s: the reference sweep in d-space, float64, one block per query head
// ---------------------------------------------------------------------------
// Block-wide product out(i, j) = sum_k a(i, k) b(k, j) with compile-time
// shapes: 2 x 2 register tiles (rows i, i + M/2; columns j, j + N/2, so
// adjacent lanes touch adjacent columns).  When there are fewer tiles than
// threads, KS lanes of one warp (lane bits above the tile bits) split the k
// range in chunks of CW rows -- slice s takes rows s*CW.. of every KS*CW --
// and combine with shuffles in a fixed order.  With the padded shared-memory
// strides of pf_solve (odd: C rows R + 1, B rows D + 1) the two slices a
// half-warp holds read rows 8 apart, i.e. the other 8 banks.
template <int M, int N, int K, class FA, class FB, class FO>
LRQK_DEV void tile_mm(FA a, FB b, FO o) {
    static_assert(M % 2 == 0 && N % 2 == 0, "even shapes");
    constexpr int TN = N / 2, NTILE = (M / 2) * TN;
    constexpr int KS = NTILE >= kSolveThreads ? 1 : (NTILE * 2 >= kSolveThreads ? 2 : (NTILE * 4 >= kSolveThreads ? 4 : 8));
    constexpr int TOTAL = NTILE * KS, TPW = 32 / KS;  // tiles per warp
    constexpr int CW = K / KS < 8 ? K / KS : 8;
    static_assert(TOTAL % 32 == 0 && K % (KS * CW) == 0, "whole warps and chunks");
#pragma unroll 1
    for (int t = threadIdx.x; t < TOTAL; t += kSolveThreads) {
        const int lane = t & 31, sl = lane / TPW, tile = (t >> 5) * TPW + lane % TPW;
        const int i0 = tile / TN, j0 = tile % TN, i1 = i0 + M / 2, j1 = j0 + N / 2;
        double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
#pragma unroll 1
        for (int kc = sl * CW; kc < K; kc += KS * CW) {
#pragma unroll
            for (int u = 0; u < CW; ++u) {
                const int k = kc + u;
                const double x0 = a(i0, k), x1 = a(i1, k), y0 = b(k, j0), y1 = b(k, j1);
                a00 = fma(x0, y0, a00);
                a01 = fma(x0, y1, a01);
                a10 = fma(x1, y0, a10);
                a11 = fma(x1, y1, a11);
            }
        }
#pragma unroll
        for (int off = TPW; off < 32; off <<= 1) {
            a00 += __shfl_xor_sync(0xffffffffu, a00, off);
            a01 += __shfl_xor_sync(0xffffffffu, a01, off);
            a10 += __shfl_xor_sync(0xffffffffu, a10, off);
            a11 += __shfl_xor_sync(0xffffffffu, a11, off);
        }
        if (sl == 0) {
            o(i0, j0, a00);
            o(i0, j1, a01);
            o(i1, j0, a10);
            o(i1, j1, a11);
        }
    }
    __syncthreads();
}

// block sum of NV values at once (fixed order: deterministic)
template <int NV>
LRQK_DEV void block_sums(double (&v)[NV], double *red) {
#pragma unroll
    for (int j = 0; j < NV; ++j)
        for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
    // then every warp sums the per-warp partials with the same shuffle tree
    constexpr int nw = kSolveThreads / 32;
    static_assert(nw == 32, "one partial per lane");
    const int lane = threadIdx.x & 31;
    if (lane == 0)
#pragma unroll
        for (int j = 0; j < NV; ++j) red[j * 32 + (threadIdx.x >> 5)] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        double t = red[j * 32 + lane];
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        v[j] = t;
    }
    __syncthreads();
}

// In-place inverse of the SPD matrix M (R x R, rank r, identity-padded past r)
// by Gauss-Jordan without pivoting, one barrier per pivot.  On an SPD matrix
// every pivot is positive exactly when the reference's Cholesky succeeds (the
// pivots are the squared Cholesky diagonal), so a non-positive pivot is the
// LinAlgError of linalg.py:81 and triggers the same single retry with
// M + 1e-10 (tr(M)/r + 1) I (linalg.py:84-91).
// Returns 0 ok, 1 jittered, 2 failed, 3 non-finite M.
template <int R>
__device__ int spd_inverse_f64(double *M, int r, double *W, double *rc, double *red) {
    double s2[2] = {0.0, 0.0};
    for (int e = threadIdx.x; e < R * R; e += kSolveThreads) {
        const int i = e / R, j = e % R;
        s2[0] += isfinite(M[e]) ? 0.0 : 1.0;
        if (i == j && i < r) s2[1] += M[e];
    }
    block_sums<2>(s2, red);
    if (s2[0] != 0.0) return 3;
    const double tr = s2[1];
    for (int attempt = 0; attempt < 2; ++attempt) {
        const double jit = attempt ? 1e-10 * (tr / r + 1.0) : 0.0;
        __syncthreads();  // a failed attempt's last pivot reads are done before rc is refilled
        for (int e = threadIdx.x; e < R * R; e += kSolveThreads) {
            const int i = e / R, j = e % R;
            const double v = (i < r && j < r) ? M[e] + (i == j ? jit : 0.0) : (i == j ? 1.0 : 0.0);
            W[e] = v;
            if (i == 0) rc[j] = v;  // pivot row / column of step 0
            if (j == 0) rc[64 + i] = v;
        }
        __syncthreads();
        bool ok = true;
#pragma unroll 1
        for (int k = 0; k < R; ++k) {
            // the pivot row / column of step k were written by their owners
            // during step k - 1; the next step's go to the other buffer
            const double *row = rc + (k & 1) * 128, *col = row + 64;
            double *nrow = rc + ((k + 1) & 1) * 128, *ncol = nrow + 64;
            const double p = row[k];
            if (!(p > 0.0)) { ok = false; break; }  // block-uniform
            const double ip = 1.0 / p;
            for (int e = threadIdx.x; e < R * R; e += kSolveThreads) {
                const int i = e / R, j = e % R;
                const double a = W[e];
                const double f = col[i] * ip;
                const double v = i == k ? (j == k ? ip : a * ip) : (j == k ? -f : fma(-f, row[j], a));
                W[e] = v;
                if (i == k + 1) nrow[j] = v;
                if (j == k + 1) ncol[i] = v;
            }
            __syncthreads();
        }
        if (ok) {
            for (int e = threadIdx.x; e < R * R; e += kSolveThreads) {  // exact symmetry
                const int i = e / R, j = e % R;
                M[e] = i <= j ? W[e] : W[j * R + i];
            }
            __syncthreads();
            return attempt;
        }
    }
    return 2;
}

// Padded shapes: D = 128 rows of d (zero past d), R = rank_stride columns of
// r (zero past r); the inverses see the identity past r, so every padded
// entry stays exactly zero and the true blocks are the reference's algebra.
template <int R>
__global__ void __launch_bounds__(kSolveThreads)
pf_solve_kernel(const PfGeom G, lrqk_prefill_t P, uint8_t *scr) {
    constexpr int D = kTile;
    extern __shared__ __align__(16) double sd[];
    const int h = blockIdx.x, tid = threadIdx.x, nt = kSolveThreads;
    const int r = G.r, d = G.d;
    const double lq = P.lambda_q, lk = P.lambda_k;
    double *GAQ = sd, *GAK = GAQ + R * R, *Mm = GAK + R * R, *Wg = Mm + R * R, *BBq = Wg + R * R, *BBk = BBq + R * R;
    double *rc = BBk + R * R, *red = rc + 256;
    const int ku = G.shared ? h / G.group : h;
    const int yq = G.shared ? 0 : h;
    const double *__restrict__ GQ = reinterpret_cast<const double *>(scr + G.off_gq) + (size_t)h * D * D;
    const double *__restrict__ GK = reinterpret_cast<const double *>(scr + G.off_gk) + (size_t)ku * D * D;
    const double *__restrict__ CQ0 = reinterpret_cast<const double *>(scr + G.off_cq) + (size_t)h * D * R;
    const double *__restrict__ CK0 = reinterpret_cast<const double *>(scr + G.off_ck) + (size_t)ku * D * R;
    const double *__restrict__ G0Q = reinterpret_cast<const double *>(scr + G.off_g0q) + (size_t)yq * R * R;
    const double *__restrict__ G0K = reinterpret_cast<const double *>(scr + G.off_g0k) + (size_t)yq * R * R;
    // float64 work: C, W are D x R; B are R x D
    double *wk = reinterpret_cast<double *>(scr + G.off_work) + (size_t)h * kWorkMats * D * R;
    double *Cq = wk, *Ck = Cq + D * R, *Wq = Ck + D * R, *Wk = Wq + D * R, *Wn = Wk + D * R, *Dt = Wn + D * R;
    double *Bq = Dt + D * R, *Bk = Bq + D * R, *Boq = Bk + D * R, *Bok = Boq + D * R;
    // C_Q, C_K, B_Q, B_K and the new W live in shared memory when they fit
    // (rank stride <= 32): the products of update_B / update_W read them many
    // times.  Their rows are padded to an odd stride (LC, LB) so the
    // transposed reads of update_B (lanes walking down a column) hit 16
    // different banks; the other work matrices keep the dense global layout.
    constexpr bool kSm = R <= 32;
    constexpr int LC = kSm ? R + 1 : R, LB = kSm ? D + 1 : D;
    if constexpr (kSm) {
        double *sm5 = red + 5 * 32;
        Cq = sm5; Ck = Cq + D * LC; Wn = Ck + D * LC; Bq = Wn + D * LC; Bk = Bq + R * LB;
    }
    auto cix = [](int i, int p) { return i * LC + p; };  // C, Wn (D x R)
    auto bix = [](int p, int i) { return p * LB + i; };  // B (R x D)
    float *Wout = reinterpret_cast<float *>(scr + G.off_w);  // [2][H][128][RS] fp32 (Q then K)
    float *obj = P.objective ? P.objective + (size_t)h * (P.max_iter + 1) : nullptr;

    // Gram-trace constants <GQ, GK>, tr GQ, tr GK, tr G0Q, tr G0K
    double c5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int e = tid; e < D * D; e += nt) {
        c5[0] += GQ[e] * GK[e];
        if (e / D == e % D) { c5[1] += GQ[e]; c5[2] += GK[e]; }
    }
    for (int p = tid; p < R; p += nt) { c5[3] += G0Q[p * R + p]; c5[4] += G0K[p * R + p]; }
    block_sums<5>(c5, red);
    const double qk2 = c5[0], tq = c5[1], tk = c5[2], trg0q = c5[3], trg0k = c5[4];
    for (int e = tid; e < D * R; e += nt) {
        const int i = e / R, p = e % R;
        Cq[cix(i, p)] = CQ0[e];
        Ck[cix(i, p)] = CK0[e];
        Bq[bix(p, i)] = 0.0;
        Bk[bix(p, i)] = 0.0;
    }
    for (int e = tid; e < R * R; e += nt) { GAQ[e] = G0Q[e]; GAK[e] = G0K[e]; BBq[e] = 0.0; BBk[e] = 0.0; }
    __syncthreads();

    // lagrangian_value (prefill.py:142-158) from the Gram-space quantities;
    // BBq = B_Q B_Q^T and BBk = B_K B_K^T are current whenever it runs
    auto objective = [&]() -> double {
        double v4[4] = {0.0, 0.0, 0.0, 0.0};  // cross, approx, q-resid, k-resid
        for (int e = tid; e < D * R; e += nt) {
            const int i = e / R, p = e % R, c = cix(i, p), b = bix(p, i);
            v4[0] += Cq[c] * Ck[c];
            v4[2] -= 2.0 * Bq[b] * Cq[c];
            v4[3] -= 2.0 * Bk[b] * Ck[c];
        }
        for (int e = tid; e < R * R; e += nt) {
            v4[1] += GAQ[e] * GAK[e];
            v4[2] += GAQ[e] * BBq[e];
            v4[3] += GAK[e] * BBk[e];
        }
        block_sums<4>(v4, red);
        return 0.5 * fmax(qk2 - 2.0 * v4[0] + v4[1], 0.0) + 0.5 * lq * (v4[2] + tq) + 0.5 * lk * (v4[3] + tk);
    };
    auto fail = [&](uint32_t bit) {
        if (tid == 0) set_status(P.status, bit);
    };
    auto inverse = [&](double *Mx) -> bool {
        const int rc2 = spd_inverse_f64<R>(Mx, r, Wg, rc, red);
        if (rc2 >= 2) { fail(rc2 == 3 ? LRQK_ST_NONFINITE : LRQK_ST_SOLVE_FAILED); return false; }
        if (rc2 == 1) fail(LRQK_ST_JITTERED);
        return true;
    };
    // B = G_A^-1 C^T (update_B, prefill.py:161-163), then B B^T
    auto update_B = [&](const double *GA, const double *Cx, double *B, double *BB) -> bool {
        for (int e = tid; e < R * R; e += nt) Mm[e] = GA[e];
        __syncthreads();
        if (!inverse(Mm)) return false;
        tile_mm<R, D, R>([&](int p, int q) { return Mm[p * R + q]; }, [&](int q, int i) { return Cx[cix(i, q)]; },
                         [&](int p, int i, double v) { B[bix(p, i)] = v; });
        tile_mm<R, R, D>([&](int p, int i) { return B[bix(p, i)]; }, [&](int i, int q) { return B[bix(q, i)]; },
                         [&](int p, int q, double v) { BB[p * R + q] = v; });
        return true;
    };
    // Wn = (Cx + lam B^T)(G_A + lam B B^T)^-1 (update_AK / update_AQ, prefill.py:166-181)
    auto update_W = [&](const double *GA, const double *Cx, const double *B, const double *BB, double lam) -> bool {
        for (int e = tid; e < R * R; e += nt) Mm[e] = GA[e] + lam * BB[e];
        __syncthreads();
        if (!inverse(Mm)) return false;
        tile_mm<D, R, R>([&](int i, int q) { return Cx[cix(i, q)] + lam * B[bix(q, i)]; },
                         [&](int q, int p) { return Mm[q * R + p]; }, [&](int i, int p, double v) { Wn[cix(i, p)] = v; });
        return true;
    };
    // after Wn: new C = GX W, G_A = W^T C, and ||A' - A||^2 (sweep 1: against A0)
    auto advance = [&](const double *__restrict__ GX, double *W, double *Cx, double *GA, const double *C0,
                       double trg0, bool first) -> double {
        double dv[1] = {0.0};
        if (first) {
            tile_mm<D, R, D>([&](int i, int j) { return GX[i * D + j]; }, [&](int j, int p) { return Wn[cix(j, p)]; },
                             [&](int i, int p, double v) { Cx[cix(i, p)] = v; });
            for (int e = tid; e < D * R; e += nt) {
                const int c = cix(e / R, e % R);
                dv[0] += Wn[c] * (Cx[c] - 2.0 * C0[e]);
                W[e] = Wn[c];
            }
            block_sums<1>(dv, red);
            dv[0] += trg0;
        } else {
            for (int e = tid; e < D * R; e += nt) W[e] = Wn[cix(e / R, e % R)] - W[e];  // dW
            __syncthreads();
            tile_mm<D, R, D>([&](int i, int j) { return GX[i * D + j]; }, [&](int j, int p) { return W[j * R + p]; },
                             [&](int i, int p, double v) { Dt[i * R + p] = v; });
            for (int e = tid; e < D * R; e += nt) {
                const int c = cix(e / R, e % R);
                dv[0] += W[e] * Dt[e];
                Cx[c] += Dt[e];
                W[e] = Wn[c];
            }
            block_sums<1>(dv, red);
        }
        tile_mm<R, R, D>([&](int p, int i) { return W[i * R + p]; }, [&](int i, int q) { return Cx[cix(i, q)]; },
                         [&](int p, int q, double v) { Mm[p * R + q] = v; });
        for (int e = tid; e < R * R; e += nt) GA[e] = 0.5 * (Mm[e] + Mm[(e % R) * R + e / R]);
        __syncthreads();
        return fmax(dv[0], 0.0);
    };

    if (obj) {
        const double o = objective();
        if (tid == 0) {
            obj[0] = (float)o;
            for (int i = 1; i <= P.max_iter; ++i) obj[i] = __int_as_float(0x7fc00000);
        }
    }
    int sweeps = 0, conv = 0, ok = 1;
    for (int s = 0; s < P.max_iter; ++s) {
        for (int e = tid; e < R * D; e += nt) {
            const int b = bix(e / D, e % D);
            Boq[e] = Bq[b];
            Bok[e] = Bk[b];
        }
        __syncthreads();
        if (!update_B(GAQ, Cq, Bq, BBq) || !update_B(GAK, Ck, Bk, BBk)) { ok = 0; break; }
        if (!update_W(GAQ, Cq, Bk, BBk, lk)) { ok = 0; break; }
        const double dak = advance(GK, Wk, Ck, GAK, CK0, trg0k, s == 0);
        if (!update_W(GAK, Ck, Bq, BBq, lq)) { ok = 0; break; }
        const double daq = advance(GQ, Wq, Cq, GAQ, CQ0, trg0q, s == 0);
        ++sweeps;
        double v3[3] = {0.0, 0.0, 0.0};  // ||dB_Q||^2, ||dB_K||^2, non-finite count
        for (int e = tid; e < R * D; e += nt) {
            const int bi = bix(e / D, e % D);
            const double a = Bq[bi] - Boq[e], b = Bk[bi] - Bok[e];
            v3[0] += a * a;
            v3[1] += b * b;
            v3[2] += (isfinite(Wq[e]) && isfinite(Wk[e])) ? 0.0 : 1.0;
        }
        block_sums<3>(v3, red);
        // non-finite factors (prefill.py:216-218)
        if (v3[2] != 0.0 || !isfinite(dak) || !isfinite(daq) || !isfinite(v3[0]) || !isfinite(v3[1])) {
            fail(LRQK_ST_NONFINITE);
            ok = 0;
            break;
        }
        if (obj) {
            const double o = objective();
            if (tid == 0) obj[s + 1] = (float)o;
        }
        // _factor_delta (prefill.py:184-194): mean over the four factors
        const double lr = (double)G.l * r, rd = (double)r * d;
        const double delta = (daq / lr + dak / lr + v3[0] / rd + v3[1] / rd) / 4.0;
        if (delta <= (double)P.tol) { conv = 1; break; }
    }
    if (tid == 0) { P.sweeps[h] = sweeps; P.converged[h] = conv; }
    // outputs: B (fp32, [RS][ds]) and W for the materialize pass
    float *BQo = P.B_Q + (size_t)h * R * G.ds, *BKo = P.B_K + (size_t)h * R * G.ds;
    for (int e = tid; e < R * G.ds; e += nt) {
        const int p = e / G.ds, i = e % G.ds;
        BQo[e] = ok ? (float)Bq[bix(p, i)] : 0.f;
        BKo[e] = ok ? (float)Bk[bix(p, i)] : 0.f;
    }
    float *WQo = Wout + (size_t)h * D * R, *WKo = Wout + ((size_t)G.H + h) * D * R;
    for (int e = tid; e < D * R; e += nt) {
        const bool in = ok && sweeps > 0;
        WQo[e] = in ? (float)Wq[e] : 0.f;
        WKo[e] = in ? (float)Wk[e] : 0.f;
    }
}

// ---------------------------------------------------------------------------
// K1m: A = X W for the query heads of one unit (TMA -> tcgen05 -> TMEM ->
// fp32 rows), double-buffered accumulators
// ---------------------------------------------------------------------------
__host__ __device__ inline void mat_unit(const PfGeom &G, int u, int &kside, int &xh, int &h0, int &nh) {
    if (u < G.H) { kside = 0; xh = u; h0 = u; nh = 1; return; }
    const int v = u - G.H, g = v / G.nsub, sb = v % G.nsub;
    kside = 1;
    xh = g;
    h0 = g * G.group + sb * G.HPU;
    nh = min(G.HPU, G.group - sb * G.HPU);
}

__global__ void __launch_bounds__(kMatThreads, 1)
pf_mat_kernel(const __grid_constant__ PfMaps maps, const PfGeom G, const float *__restrict__ W, float *A_Q, float *A_K,
              int u0, int S2, int budget, int staged) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int u = u0 + blockIdx.x / S2, s = blockIdx.x % S2;
    int kside, xh, h0, nh;
    mat_unit(G, u, kside, xh, h0, nh);
    const int RS = G.rs, N = nh * 2 * RS;  // accumulator columns: per head [hi-part | lo-part]
    const int nxb = G.XW / 64, npart = G.parts;
    const int stage_bytes = npart * 2 * kBlkBytes;
    const int wbytes = 2 * (kside ? G.Nmax : 2 * RS) * 128;  // W^T split, K-major SW128: [2 d-blocks][N rows][128 B]
    const int nst = min(kMaxStages, (budget - wbytes) / stage_bytes);
    uint8_t *sW = sm + nst * stage_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(sW + wbytes);
    uint64_t *empty = full + kMaxStages;
    uint64_t *tfull = empty + kMaxStages;
    uint64_t *tempty = tfull + 2;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t0 = (int)((long long)G.tiles * s / S2), t1 = (int)((long long)G.tiles * (s + 1) / S2);
    const uint32_t ncols = N <= 16 ? 32 : (N <= 32 ? 64 : (N <= 64 ? 128 : (N <= 128 ? 256 : 512)));
    const int mx = kside ? MK : MQ, mxl = kside ? MKL : MQL;

    // stage W^T (rows n = head j, column c of [hi | lo]; K = d) with the swizzle
    const float *Wsrc = W + ((size_t)(kside ? G.H : 0) + h0) * kTile * RS;
    for (int e = threadIdx.x; e < N * (kTile / 8); e += blockDim.x) {
        const int n = e / (kTile / 8), ch = e % (kTile / 8);  // 8 d-values per 16-B chunk
        const int j = n / (2 * RS), c = n % (2 * RS), p = c % RS, lo = c >= RS;
        uint32_t pk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            __nv_bfloat16 v2[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const float w = Wsrc[((size_t)j * kTile + ch * 8 + q * 2 + t) * RS + p];
                const __nv_bfloat16 hi = __float2bfloat16_rn(w);
                v2[t] = lo ? __float2bfloat16_rn(w - __bfloat162float(hi)) : hi;
            }
            pk[q] = (uint32_t)__bfloat16_as_ushort(v2[0]) | ((uint32_t)__bfloat16_as_ushort(v2[1]) << 16);
        }
        const int kb = ch / 8, c16 = ch % 8;
        *reinterpret_cast<uint4 *>(sW + kb * N * 128 + n * 128 + ((c16 ^ (n & 7)) * 16)) =
            make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
    if (nxb == 1)  // X narrower than 128 columns: its upper K block is zero
        for (int st = 0; st < nst; ++st)
            for (int pp = 0; pp < npart; ++pp)
                for (int e = threadIdx.x; e < kBlkBytes / 16; e += blockDim.x)
                    reinterpret_cast<uint4 *>(sm + st * stage_bytes + (pp * 2 + 1) * kBlkBytes)[e] = make_uint4(0, 0, 0, 0);
    tc::fence_proxy_async();
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(tfull + i, 1); mbar_init(tempty + i, 4); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tc::tma_prefetch(&maps.m[mx]);
        if (npart == 2) tc::tma_prefetch(&maps.m[mxl]);
    }
    if (warp == 1) tc::tmem_alloc(tslot, ncols);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = *tslot;

    if (warp == 0 && lane == 0) {
        const uint64_t pol = l2_policy_evict_first();
        for (int t = t0, i = 0; t < t1; ++t, ++i) {
            const int st = i % nst;
            mbar_wait(empty + st, ((i / nst) & 1) ^ 1);
            uint8_t *base = sm + st * stage_bytes;
            mbar_expect_tx(full + st, npart * nxb * kBlkBytes);
            for (int pp = 0; pp < npart; ++pp)
                for (int b = 0; b < nxb; ++b)
                    tc::tma_load_3d(base + (pp * 2 + b) * kBlkBytes, &maps.m[pp ? mxl : mx], b * 64, t * kTile, xh,
                                    full + st, pol);
        }
    } else if (warp == 1 && lane == 0) {
        const uint32_t id = tc::idesc_bf16(128, N, false, false);
        const uint32_t wb = smem_u32(sW);
        for (int t = t0, i = 0; t < t1; ++t, ++i) {
            const int st = i % nst, ab = i & 1;
            mbar_wait(tempty + ab, ((i >> 1) & 1) ^ 1);
            mbar_wait(full + st, (i / nst) & 1);
            tc::fence_after();
            const uint32_t base = smem_u32(sm + st * stage_bytes);
            for (int pp = 0; pp < npart; ++pp)
#pragma unroll
                for (int k = 0; k < kTile / 16; ++k) {
                    const uint32_t koff = (k >> 2) * kBlkBytes + (k & 3) * 32;
                    const uint64_t ad = tc::desc_sw128(base + pp * 2 * kBlkBytes + koff, 16, 1024);
                    const uint64_t bd = tc::desc_sw128(wb + (k >> 2) * N * 128 + (k & 3) * 32, 16, 1024);
                    tc::mma_bf16(tm + ab * (ncols / 2), ad, bd, id, (pp > 0 || k > 0) ? 1u : 0u);
                }
            tc::mma_commit(empty + st);
            tc::mma_commit(tfull + ab);
        }
    } else if (warp >= 2) {
        // ---- epilogue: rows of this warp's TMEM lane quarter -----------------
        const int q4 = warp & 3, row = q4 * 32 + lane;
        float *Aout = kside ? A_K : A_Q;
        for (int t = t0, i = 0; t < t1; ++t, ++i) {
            const int ab = i & 1;
            mbar_wait(tfull + ab, (i >> 1) & 1);
            tc::fence_after();
            const uint32_t ta = tm + ab * (ncols / 2) + ((uint32_t)(q4 * 32) << 16);
            const int grow = t * kTile + row;
            for (int j = 0; j < nh; ++j) {
                float *dst = Aout + ((size_t)(h0 + j) * G.l + grow) * RS;
                if (RS >= 32 && staged) {
                    // rows through a padded per-warp buffer so that each store
                    // instruction writes four whole 128-B row segments
                    float *eb = reinterpret_cast<float *>(sm + budget + 1024) + q4 * kEpiWarpFloats;
                    for (int c0 = 0; c0 < RS; c0 += 32) {
                        float hi[32], lo[32];
                        tc::tmem_ld32(ta + j * 2 * RS + c0, hi);
                        tc::tmem_ld32(ta + j * 2 * RS + RS + c0, lo);
#pragma unroll
                        for (int p = 0; p < 32; p += 4)
                            *reinterpret_cast<float4 *>(eb + lane * kEpiStride + p) =
                                make_float4(hi[p] + lo[p], hi[p + 1] + lo[p + 1], hi[p + 2] + lo[p + 2], hi[p + 3] + lo[p + 3]);
                        __syncwarp();
#pragma unroll
                        for (int m = 0; m < 8; ++m) {
                            const int rr = 4 * m + (lane >> 3), cc = (lane & 7) * 4;
                            const int gr = t * kTile + q4 * 32 + rr;
                            if (gr < G.l)
                                *reinterpret_cast<float4 *>(Aout + ((size_t)(h0 + j) * G.l + gr) * RS + c0 + cc) =
                                    *reinterpret_cast<const float4 *>(eb + rr * kEpiStride + cc);
                        }
                        __syncwarp();
                    }
                } else if (RS >= 32) {
                    for (int c0 = 0; c0 < RS; c0 += 32) {
                        float hi[32], lo[32];
                        tc::tmem_ld32(ta + j * 2 * RS + c0, hi);
                        tc::tmem_ld32(ta + j * 2 * RS + RS + c0, lo);
                        if (grow < G.l)
#pragma unroll
                            for (int p = 0; p < 32; p += 4)
                                *reinterpret_cast<float4 *>(dst + c0 + p) =
                                    make_float4(hi[p] + lo[p], hi[p + 1] + lo[p + 1], hi[p + 2] + lo[p + 2], hi[p + 3] + lo[p + 3]);
                    }
                } else if (RS == 16) {  // one head = [hi 16 | lo 16]
                    float v[32];
                    tc::tmem_ld32(ta + j * 32, v);
                    if (grow < G.l)
#pragma unroll
                        for (int p = 0; p < 16; p += 4)
                            *reinterpret_cast<float4 *>(dst + p) =
                                make_float4(v[p] + v[16 + p], v[p + 1] + v[17 + p], v[p + 2] + v[18 + p], v[p + 3] + v[19 + p]);
                } else {  // RS == 8: one head = [hi 8 | lo 8]
                    float v[16];
                    tc::tmem_ld16(ta + j * 16, v);
                    if (grow < G.l)
#pragma unroll
                        for (int p = 0; p < 8; p += 4)
                            *reinterpret_cast<float4 *>(dst + p) =
                                make_float4(v[p] + v[8 + p], v[p + 1] + v[9 + p], v[p + 2] + v[10 + p], v[p + 3] + v[11 + p]);
                }
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty + ab);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tm, ncols);
}

// ---------------------------------------------------------------------------
// bf16 operand preparation: X (fp32 split hi/lo, or bf16 widened to 64
// columns) and Y = [A0 hi | A0 lo | 0] (width YW)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void pf_split_kernel(const T *__restrict__ X, int rows, int cols, int ld, int ow,
                                __nv_bfloat16 *__restrict__ hi, __nv_bfloat16 *__restrict__ lo) {
    const long long n = (long long)rows * ow;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const long long rI = e / ow;
        const int c = (int)(e % ow);
        const float v = c < cols ? to_float<T>(X[rI * ld + c]) : 0.f;
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        hi[e] = h;
        if (lo) lo[e] = __float2bfloat16_rn(v - __bfloat162float(h));
    }
}

__global__ void pf_ysplit_kernel(const float *__restrict__ A, int rows, int r, int RS, int YW, __nv_bfloat16 *__restrict__ Y) {
    // Y = [A hi | A lo | 0]: one thread per row and 8-column chunk
    const int cpr = YW / 8;
    const long long n = (long long)rows * cpr;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const long long rI = e / cpr;
        const int c0 = (int)(e - rI * cpr) * 8;
        uint32_t pk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint16_t h2[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int c = c0 + 2 * q + t;
                float v = 0.f;
                if (c < 2 * RS && c % RS < r) {
                    const float a = A[rI * RS + c % RS];
                    const __nv_bfloat16 hi = __float2bfloat16_rn(a);
                    v = c < RS ? __bfloat162float(hi) : a - __bfloat162float(hi);
                }
                h2[t] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
            }
            pk[q] = (uint32_t)h2[0] | ((uint32_t)h2[1] << 16);
        }
        *reinterpret_cast<uint4 *>(Y + rI * YW + c0) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
extern int num_sms();

static int pick_slabs(int units, int tiles, int nsm) {  // nsm: resident block slots
    // the smallest slab count whose last wave of one-block-per-SM is >= 85 % full
    int best = 1;
    double best_eff = -1.0;
    for (int w = 1; w <= 16; ++w) {
        int s = (w * nsm + units - 1) / units;
        s = std::max(1, std::min(s, tiles));
        const long long blocks = (long long)units * s;
        const long long waves = (blocks + nsm - 1) / nsm;
        const double eff = (double)blocks / (double)(waves * nsm);
        if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
        if (eff >= 0.85 || s == tiles) break;
    }
    return best;
}

static size_t al(size_t x) { return (x + 1023) & ~(size_t)1023; }

static bool pf_geom(const lrqk_prefill_t &P, PfGeom &G) {
    G.H = P.n_heads;
    G.group = P.group > 0 ? P.group : 1;
    G.Hk = G.H / G.group;
    G.l = P.len;
    G.d = P.head_dim;
    G.ds = P.dim_stride;
    G.r = P.rank;
    G.rs = P.rank_stride;
    if (G.ds > 128 || G.ds < 8 || G.ds % 8 || G.rs > 64 || G.rs < 8 || (G.rs & (G.rs - 1)) || G.r > G.d || G.r > G.rs || G.d > G.ds)
        return false;
    G.parts = P.dtype == LRQK_BF16 ? 1 : 2;
    G.direct = P.dtype == LRQK_BF16 && (G.ds == 64 || G.ds == 128);
    G.XW = G.ds > 64 ? 128 : 64;
    G.YW = 2 * G.rs > 64 ? 128 : 64;
    G.shared = P.A_Q0 && P.init_shared ? 1 : 0;
    G.NY = G.shared ? 1 : G.H;
    G.NQU = G.H;
    G.NKU = G.shared ? G.Hk : G.H;
    G.NU = (G.NQU + G.NKU) * G.parts + 2 * G.NY;
    G.tiles = (G.l + kTile - 1) / kTile;
    const int nsm = num_sms();
    G.S = pick_slabs(G.NU, G.tiles, nsm * (G.parts == 1 ? 2 : 1));
    G.PW = 128 + (G.parts == 2 ? G.XW + G.YW : G.YW);
    G.HPU = std::max(1, std::min(G.group, 256 / (2 * G.rs)));
    G.nsub = (G.group + G.HPU - 1) / G.HPU;
    G.NMU = G.H + G.Hk * G.nsub;
    G.Nmax = std::max(2 * G.rs, G.HPU * 2 * G.rs);
    size_t o = 0;
    const size_t xq = (size_t)G.H * G.l * G.XW * 2, xk = (size_t)G.Hk * G.l * G.XW * 2;
    const bool own_x = !G.direct;
    for (int i = 0; i < 4; ++i) G.off_x[i] = 0;
    if (own_x) {
        G.off_x[0] = o; o = al(o + xq);
        G.off_x[2] = o; o = al(o + xk);
        if (G.parts == 2) {
            G.off_x[1] = o; o = al(o + xq);
            G.off_x[3] = o; o = al(o + xk);
        }
    }
    const size_t ysz = (size_t)G.NY * G.l * G.YW * 2;
    G.off_y[0] = o; o = al(o + ysz);
    G.off_y[1] = o; o = al(o + ysz);
    G.off_part = o; o = al(o + (size_t)G.NU * G.S * kTile * G.PW * 4);
    G.off_gq = o; o = al(o + (size_t)G.NQU * kTile * kTile * 8);
    G.off_cq = o; o = al(o + (size_t)G.NQU * kTile * G.rs * 8);
    G.off_gk = o; o = al(o + (size_t)G.NKU * kTile * kTile * 8);
    G.off_ck = o; o = al(o + (size_t)G.NKU * kTile * G.rs * 8);
    G.off_g0q = o; o = al(o + (size_t)G.NY * G.rs * G.rs * 8);
    G.off_g0k = o; o = al(o + (size_t)G.NY * G.rs * G.rs * 8);
    G.off_w = o; o = al(o + (size_t)2 * G.H * kTile * G.rs * 4);
    G.off_work = o; o = al(o + (size_t)G.H * kWorkMats * kTile * G.rs * 8);
    G.total = o + 1024;
    return true;
}

size_t prefill_scratch_floats(const lrqk_prefill_t &P) {
    PfGeom G;
    if (!pf_geom(P, G)) return 0;
    return (G.total + 3) / 4;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// [heads][rows][width] bf16, boxes of 64 columns x 128 rows, SW128
static bool make_map(CUtensorMap *m, const void *base, int heads, int rows, int width) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)width, (cuuint64_t)rows, (cuuint64_t)heads};
    const cuuint64_t strides[2] = {(cuuint64_t)width * 2, (cuuint64_t)rows * width * 2};
    const cuuint32_t box[3] = {64, (cuuint32_t)kTile, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int launch_prefill(const lrqk_prefill_t &P, cudaStream_t st) {
    PfGeom G;
    if (!pf_geom(P, G)) return LRQK_EUNSUPPORTED;
    uint8_t *scr = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(P.scratch) + 1023) & ~(uintptr_t)1023);
    // ---- operands ----------------------------------------------------------
    const int Hk = G.Hk;
    const void *xq = P.Q, *xk = P.K, *xql = nullptr, *xkl = nullptr;
    if (!G.direct) {
        auto split = [&](const void *X, int heads, uint8_t *hi, uint8_t *lo) {
            const long long n = (long long)heads * G.l * G.XW;
            const int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
            if (P.dtype == LRQK_BF16)
                pf_split_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16 *>(X),
                                                                      heads * G.l, G.d, G.ds, G.XW,
                                                                      reinterpret_cast<__nv_bfloat16 *>(hi), nullptr);
            else
                pf_split_kernel<float><<<grid, 256, 0, st>>>(reinterpret_cast<const float *>(X), heads * G.l, G.d,
                                                              G.ds, G.XW, reinterpret_cast<__nv_bfloat16 *>(hi),
                                                              reinterpret_cast<__nv_bfloat16 *>(lo));
        };
        split(P.Q, G.H, scr + G.off_x[0], G.parts == 2 ? scr + G.off_x[1] : nullptr);
        split(P.K, Hk, scr + G.off_x[2], G.parts == 2 ? scr + G.off_x[3] : nullptr);
        xq = scr + G.off_x[0];
        xk = scr + G.off_x[2];
        xql = G.parts == 2 ? scr + G.off_x[1] : nullptr;
        xkl = G.parts == 2 ? scr + G.off_x[3] : nullptr;
    }
    const float *a0q = P.A_Q0 ? P.A_Q0 : P.A_Q, *a0k = P.A_K0 ? P.A_K0 : P.A_K;
    {
        const long long n = (long long)G.NY * G.l * (G.YW / 8);
        const int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
        pf_ysplit_kernel<<<grid, 256, 0, st>>>(a0q, G.NY * G.l, G.r, G.rs, G.YW,
                                               reinterpret_cast<__nv_bfloat16 *>(scr + G.off_y[0]));
        pf_ysplit_kernel<<<grid, 256, 0, st>>>(a0k, G.NY * G.l, G.r, G.rs, G.YW,
                                               reinterpret_cast<__nv_bfloat16 *>(scr + G.off_y[1]));
    }
    PfMaps maps;
    memset(&maps, 0, sizeof(maps));
    bool ok = make_map(&maps.m[MQ], xq, G.H, G.l, G.XW) && make_map(&maps.m[MK], xk, Hk, G.l, G.XW) &&
              make_map(&maps.m[MYQ], scr + G.off_y[0], G.NY, G.l, G.YW) &&
              make_map(&maps.m[MYK], scr + G.off_y[1], G.NY, G.l, G.YW);
    if (G.parts == 2)
        ok = ok && make_map(&maps.m[MQL], xql, G.H, G.l, G.XW) && make_map(&maps.m[MKL], xkl, Hk, G.l, G.XW);
    if (!ok) return LRQK_ECUDA;
    // ---- K1g -----------------------------------------------------------------
    // bf16: two CTAs per SM (TMEM 256 columns, 2 stages of X|Y each); fp32: one
    const int gbudget = G.parts == 1 ? 96 * 1024 : 200 * 1024;
    const size_t gsm = gbudget + 2048;
    cudaFuncSetAttribute(pf_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 2048);
    float *part = reinterpret_cast<float *>(scr + G.off_part);
    pf_gram_kernel<<<G.NU * G.S, kGramThreads, gsm, st>>>(maps, G, part, gbudget);
    // ---- K1c -----------------------------------------------------------------
    {
        const long long tot = (long long)(G.NQU + G.NKU) * kTile * (kTile + G.rs) + 2LL * G.NY * G.rs * G.rs;
        const int grid = (int)std::min<long long>((tot + 255) / 256, 148LL * 8);
        pf_combine_kernel<<<grid, 256, 0, st>>>(G, part, scr);
    }
    // ---- K1s -----------------------------------------------------------------
    // the R x R work, the reduction scratch, and (rank stride <= 32) five D x R
    // work matrices kept on chip
    const size_t ssm = (6 * (size_t)G.rs * G.rs + 256 + 5 * 32 + (G.rs <= 32 ? 3 * (size_t)kTile * (G.rs + 1) + 2 * (size_t)G.rs * (kTile + 1) : 0)) *
                       sizeof(double);
#define LRQK_PF_SOLVE(RV)                                                                               \
    do {                                                                                                \
        cudaFuncSetAttribute(pf_solve_kernel<RV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm); \
        pf_solve_kernel<RV><<<G.H, kSolveThreads, ssm, st>>>(G, P, scr);                                \
    } while (0)
    if (G.rs == 8) LRQK_PF_SOLVE(8);
    else if (G.rs == 16) LRQK_PF_SOLVE(16);
    else if (G.rs == 32) LRQK_PF_SOLVE(32);
    else LRQK_PF_SOLVE(64);
#undef LRQK_PF_SOLVE
    // ---- K1m -----------------------------------------------------------------
    // query heads: two CTAs per SM for bf16 (N = 2r, W^T 16 KB, 2 stages);
    // K heads: one CTA per SM, one K tile for up to 256 / 2r heads of its group
    cudaFuncSetAttribute(pf_mat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 2048 + kEpiBytes);
    const float *Wsp = reinterpret_cast<const float *>(scr + G.off_w);
    const int nsm = num_sms();
    if (P.A_Q) {  // NULL (with a separate init): the query factor is not materialised
        // bf16: 80 KB = W^T (16 KB) + two 32-KB stages, so two CTAs fit with their epilogue staging
        const int budget = G.parts == 1 ? 80 * 1024 : 200 * 1024;
        const int S2 = pick_slabs(G.H, G.tiles, nsm * (G.parts == 1 ? 2 : 1));
        pf_mat_kernel<<<G.H * S2, kMatThreads, budget + 2048 + kEpiBytes, st>>>(maps, G, Wsp, P.A_Q, P.A_K, 0, S2,
                                                                                budget, 1);
    }
    {
        const int nk = G.Hk * G.nsub, S2 = pick_slabs(nk, G.tiles, nsm);
        pf_mat_kernel<<<nk * S2, kMatThreads, 200 * 1024 + 2048 + kEpiBytes, st>>>(maps, G, Wsp, P.A_Q, P.A_K, G.H,
                                                                                   S2, 200 * 1024, 1);
    }
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

}  // namespace lrqk
