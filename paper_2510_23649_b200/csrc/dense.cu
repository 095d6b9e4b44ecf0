// Float64 dense kernels behind the drop-in linear-algebra entry points of the
// reference (pkg/src/lrqk/linalg.py:48-110, prefill.py:142-253,
// decode.py:79-119).  The reference computes these in float64 with numpy /
// LAPACK; the B200 runs them in float64 too (full-rate FP64 on sm_100), so
// the drop-in functions agree with the reference to ~1e-12 and take the same
// branches (Cholesky failure -> jitter retry -> SolveFailedError).
//
// These are the per-call API kernels.  The fused decode / prefill path uses
// its own fp32/bf16 kernels (compress.cu, prefill.cu).
//
//   gemm_f64      C = alpha op(A) op(B) + beta C, row-major, 64x64 tiles,
//                 deterministic split-K (partials reduced in a fixed order)
//   mirror_f64    copy the strict upper triangle onto the lower one
//                 (linalg.py:48-55: gram is exactly symmetric)
//   dot_f64       sum_i a_i b_i, two fixed-order passes (fro_norm_sq,
//                 the Gram-trace inner products of lagrangian_value)
//   axpby_f64     y = alpha [* *s] x + beta y
//   chol_f64      Cholesky of an r x r SPD matrix (lower triangle read, as
//                 LAPACK potrf); on a non-positive pivot one retry with
//                 M + 1e-10 (tr(M)/r + 1) I; status bits as errors.py
//   subst_f64     X M = RHS row by row: L y = rhs, L^T x = y
//   topk_f64      k largest of n float64 scores, ties -> lower index,
//                 ascending output (linalg.py:96-110), on order-preserving
//                 64-bit keys (radix select, one block)
#include "common.cuh"

namespace lrqk {

constexpr int kGT = 64;   // gemm tile (M and N)
constexpr int kGK = 16;   // gemm k step
constexpr double kJitterEps = 1e-10;  // linalg.py:19

// ---------------------------------------------------------------------------
// GEMM
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
gemm_f64_kernel(int ta, int tb, int m, int n, int k, int kchunk, const double *__restrict__ A, int lda,
                const double *__restrict__ B, int ldb, double *__restrict__ part, double alpha, double beta,
                double *__restrict__ C, int ldc, int direct) {
    __shared__ double As[kGK][kGT + 1];
    __shared__ double Bs[kGK][kGT + 1];
    const int tid = threadIdx.x;
    const int m0 = blockIdx.y * kGT, n0 = blockIdx.x * kGT;
    const int k0 = blockIdx.z * kchunk, k1 = min(k, k0 + kchunk);
    const int tr = (tid / 16) * 4, tc = (tid % 16) * 4;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int kk = k0; kk < k1; kk += kGK) {
        // A tile: rows m0..m0+63, cols kk..kk+15 of op(A)
        for (int e = tid; e < kGT * kGK; e += 256) {
            int i, p;
            if (ta) { p = e / kGT; i = e % kGT; } else { i = e / kGK; p = e % kGK; }
            const int gi = m0 + i, gp = kk + p;
            double v = 0.0;
            if (gi < m && gp < k1) v = ta ? A[(size_t)gp * lda + gi] : A[(size_t)gi * lda + gp];
            As[p][i] = v;
        }
        for (int e = tid; e < kGT * kGK; e += 256) {
            int j, p;
            if (tb) { j = e / kGK; p = e % kGK; } else { p = e / kGT; j = e % kGT; }
            const int gj = n0 + j, gp = kk + p;
            double v = 0.0;
            if (gj < n && gp < k1) v = tb ? B[(size_t)gj * ldb + gp] : B[(size_t)gp * ldb + gj];
            Bs[p][j] = v;
        }
        __syncthreads();
#pragma unroll
        for (int p = 0; p < kGK; ++p) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[p][tr + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[p][tc + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gi = m0 + tr + i, gj = n0 + tc + j;
            if (gi >= m || gj >= n) continue;
            if (direct) {
                double *c = C + (size_t)gi * ldc + gj;
                *c = beta == 0.0 ? alpha * acc[i][j] : fma(alpha, acc[i][j], beta * *c);
            } else {
                part[((size_t)blockIdx.z * m + gi) * n + gj] = acc[i][j];
            }
        }
}

__global__ void gemm_reduce_kernel(int m, int n, int splits, const double *__restrict__ part, double alpha,
                                   double beta, double *__restrict__ C, int ldc) {
    const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (size_t)m * n) return;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[(size_t)z * m * n + e];  // fixed order: deterministic
    const int i = (int)(e / n), j = (int)(e % n);
    double *c = C + (size_t)i * ldc + j;
    *c = beta == 0.0 ? alpha * s : fma(alpha, s, beta * *c);
}

size_t gemm_f64_workspace(int m, int n, int k) {
    const int tiles = ((m + kGT - 1) / kGT) * ((n + kGT - 1) / kGT);
    if (tiles >= 148 || k <= 512) return 0;
    int splits = min(64, max(1, (296 + tiles - 1) / tiles));
    splits = min(splits, (k + 255) / 256);
    return splits > 1 ? (size_t)splits * m * n * sizeof(double) : 0;
}

int launch_gemm_f64(int ta, int tb, int m, int n, int k, double alpha, const double *A, int lda, const double *B,
                    int ldb, double beta, double *C, int ldc, void *work, size_t work_bytes, cudaStream_t st) {
    if (m == 0 || n == 0) return LRQK_OK;
    const size_t need = gemm_f64_workspace(m, n, k);
    int splits = 1;
    if (need && work && work_bytes >= need) splits = (int)(need / ((size_t)m * n * sizeof(double)));
    const int kchunk = splits > 1 ? ((k + splits - 1) / splits + kGK - 1) / kGK * kGK : max(k, 1);
    splits = splits > 1 ? (k + kchunk - 1) / kchunk : 1;
    dim3 grid((n + kGT - 1) / kGT, (m + kGT - 1) / kGT, splits);
    gemm_f64_kernel<<<grid, 256, 0, st>>>(ta, tb, m, n, k, kchunk, A, lda, B, ldb, (double *)work, alpha, beta, C,
                                          ldc, splits == 1);
    if (splits > 1) {
        const size_t tot = (size_t)m * n;
        gemm_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(m, n, splits, (const double *)work, alpha,
                                                                          beta, C, ldc);
    }
    return cudaPeekAtLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

// ---------------------------------------------------------------------------
// exact symmetry: lower := upper (linalg.py:53-54)
// ---------------------------------------------------------------------------
__global__ void mirror_f64_kernel(double *G, int r, int ldg) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= r * r) return;
    const int i = e / r, j = e % r;
    if (i > j) G[(size_t)i * ldg + j] = G[(size_t)j * ldg + i];
}

int launch_mirror_f64(double *G, int r, int ldg, cudaStream_t st) {
    if (r <= 1) return LRQK_OK;
    mirror_f64_kernel<<<(r * r + 255) / 256, 256, 0, st>>>(G, r, ldg);
    return cudaPeekAtLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

// ---------------------------------------------------------------------------
// dot product, fixed reduction order: 256 block partials, then one block
// ---------------------------------------------------------------------------
constexpr int kDotBlocks = 256;

__device__ double block_sum_f64(double v, double *sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    __syncthreads();
    return t;
}

__global__ void __launch_bounds__(256) dot_f64_kernel(const double *__restrict__ a, const double *__restrict__ b,
                                                      long long n, double *__restrict__ part) {
    __shared__ double sh[8];
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        s = fma(a[i], b[i], s);
    s = block_sum_f64(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(256) dot_finish_kernel(const double *__restrict__ part, int np, double *out) {
    __shared__ double sh[8];
    double s = threadIdx.x < np ? part[threadIdx.x] : 0.0;
    s = block_sum_f64(s, sh);
    if (threadIdx.x == 0) *out = s;
}

int launch_dot_f64(const double *a, const double *b, long long n, double *out, double *work, cudaStream_t st) {
    dot_f64_kernel<<<kDotBlocks, 256, 0, st>>>(a, b, n, work);
    dot_finish_kernel<<<1, 256, 0, st>>>(work, kDotBlocks, out);
    return cudaPeekAtLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

// ---------------------------------------------------------------------------
// y = alpha [* s] x + beta y
// ---------------------------------------------------------------------------
__global__ void axpby_f64_kernel(long long n, double alpha, const double *s, const double *x, double beta,
                                 double *y) {
    const double a = s ? alpha * *s : alpha;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = beta == 0.0 ? a * x[i] : fma(a, x[i], beta * y[i]);
}

int launch_axpby_f64(long long n, double alpha, const double *s, const double *x, double beta, double *y,
                     cudaStream_t st) {
    if (n <= 0) return LRQK_OK;
    const int blocks = (int)min((n + 255) / 256, (long long)1184);
    axpby_f64_kernel<<<blocks, 256, 0, st>>>(n, alpha, s, x, beta, y);
    return cudaPeekAtLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

// ---------------------------------------------------------------------------
// SPD right-solve X M = RHS (linalg.py:63-93)
// work: [r*r] Cholesky factor | [1] flag (1: factor usable)
// ---------------------------------------------------------------------------
__device__ bool chol_attempt(const double *M, int ldm, double *Lf, int r, double jitter, double *sh) {
    // left-looking column Cholesky on the lower triangle (what potrf reads)
    __shared__ int s_fail;
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    for (int j = 0; j < r; ++j) {
        double part = 0.0;
        for (int p = threadIdx.x; p < j; p += blockDim.x) part = fma(Lf[(size_t)j * r + p], Lf[(size_t)j * r + p], part);
        const double sq = block_sum_f64(part, sh);
        if (threadIdx.x == 0) {
            const double dj = M[(size_t)j * ldm + j] + jitter - sq;
            if (!(dj > 0.0)) s_fail = 1;
            else Lf[(size_t)j * r + j] = sqrt(dj);
        }
        __syncthreads();
        if (s_fail) return false;
        const double ljj = Lf[(size_t)j * r + j];
        for (int i = j + 1 + threadIdx.x; i < r; i += blockDim.x) {
            double s = M[(size_t)i * ldm + j];
            for (int p = 0; p < j; ++p) s = fma(-Lf[(size_t)i * r + p], Lf[(size_t)j * r + p], s);
            Lf[(size_t)i * r + j] = s / ljj;
        }
        __syncthreads();
    }
    return true;
}

__global__ void __launch_bounds__(256) chol_f64_kernel(const double *M, int r, int ldm, double *work,
                                                       uint32_t *status) {
    __shared__ double sh[8];
    __shared__ int s_bad;
    double *Lf = work;
    if (threadIdx.x == 0) { s_bad = 0; work[(size_t)r * r] = 0.0; }
    __syncthreads();
    // non-finite M -> NonFiniteError (linalg.py:71-72)
    for (int e = threadIdx.x; e < r * r; e += blockDim.x)
        if (!isfinite(M[(size_t)(e / r) * ldm + e % r])) s_bad = 1;
    __syncthreads();
    if (s_bad) {
        if (threadIdx.x == 0) set_status(status, LRQK_ST_NONFINITE);
        return;
    }
    if (chol_attempt(M, ldm, Lf, r, 0.0, sh)) {
        if (threadIdx.x == 0) work[(size_t)r * r] = 1.0;
        return;
    }
    // one retry with jitter 1e-10 (trace(M)/r + 1) on the diagonal (linalg.py:83-87)
    double tr = 0.0;
    for (int j = threadIdx.x; j < r; j += blockDim.x) tr += M[(size_t)j * ldm + j];
    tr = block_sum_f64(tr, sh);
    __shared__ double s_jit;
    if (threadIdx.x == 0) s_jit = kJitterEps * (tr / r + 1.0);
    __syncthreads();
    if (chol_attempt(M, ldm, Lf, r, s_jit, sh)) {
        if (threadIdx.x == 0) { work[(size_t)r * r] = 1.0; set_status(status, LRQK_ST_JITTERED); }
    } else if (threadIdx.x == 0) {
        set_status(status, LRQK_ST_SOLVE_FAILED);
    }
}

__global__ void __launch_bounds__(128) subst_f64_kernel(const double *RHS, int n, int ldr, int r, const double *work,
                                                        double *X, int ldx, uint32_t *status) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const double *Lf = work;
    const double *b = RHS + (size_t)row * ldr;
    bool finite = true;
    for (int j = 0; j < r; ++j) finite &= (bool)isfinite(b[j]);
    if (!finite) { set_status(status, LRQK_ST_NONFINITE); return; }
    if (work[(size_t)r * r] != 1.0) return;   // factorisation failed: no output
    double *x = X + (size_t)row * ldx;
    // L y = b (y stored in x), then L^T x = y
    for (int j = 0; j < r; ++j) {
        double s = b[j];
        for (int p = 0; p < j; ++p) s = fma(-Lf[(size_t)j * r + p], x[p], s);
        x[j] = s / Lf[(size_t)j * r + j];
    }
    for (int j = r - 1; j >= 0; --j) {
        double s = x[j];
        for (int p = j + 1; p < r; ++p) s = fma(-Lf[(size_t)p * r + j], x[p], s);
        x[j] = s / Lf[(size_t)j * r + j];
    }
}

int launch_solve_spd_f64(const double *M, int r, int ldm, const double *RHS, int n, int ldr, double *X, int ldx,
                         double *work, uint32_t *status, cudaStream_t st) {
    chol_f64_kernel<<<1, 256, 0, st>>>(M, r, ldm, work, status);
    if (n > 0) subst_f64_kernel<<<(n + 127) / 128, 128, 0, st>>>(RHS, n, ldr, r, work, X, ldx, status);
    return cudaPeekAtLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

// ---------------------------------------------------------------------------
// top-k of float64 scores (linalg.py:96-110): order-preserving 64-bit keys,
// 8-bit radix select from the top byte down (one block), then an ascending
// compaction: winners are every key above the threshold key plus the
// lowest-index rows equal to it.  -0.0 compares equal to +0.0 (numpy).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t key64(double x) {
    uint64_t u = (uint64_t)__double_as_longlong(x);
    if (u == 0x8000000000000000ull) u = 0ull;
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void __launch_bounds__(1024) topk_f64_kernel(const double *__restrict__ s, int n, int k,
                                                        int32_t *__restrict__ out) {
    __shared__ int hist[256];
    __shared__ uint64_t s_prefix, s_mask;
    __shared__ int s_need, s_eq_take, s_cnt;
    __shared__ int wtot[32];
    const int tid = threadIdx.x;
    if (tid == 0) { s_prefix = 0; s_mask = 0; s_need = k; }
    __syncthreads();
    // find the k-th largest key byte by byte
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const uint64_t pre = s_prefix, msk = s_mask;
        for (int i = tid; i < n; i += blockDim.x) {
            const uint64_t kk = key64(s[i]);
            if ((kk & msk) == pre) atomicAdd(&hist[(kk >> shift) & 255], 1);
        }
        __syncthreads();
        if (tid == 0) {
            int need = s_need, b = 255;
            for (; b > 0; --b) {
                if (hist[b] >= need) break;
                need -= hist[b];
            }
            s_need = need;
            s_prefix = pre | ((uint64_t)b << shift);
            s_mask = msk | (255ull << shift);
        }
        __syncthreads();
    }
    const uint64_t thr = s_prefix;
    // rows equal to thr: the first s_need of them (lowest indices) win
    if (tid == 0) { s_eq_take = s_need; s_cnt = 0; }
    __syncthreads();
    // ascending compaction in index order, chunk by chunk
    int eq_seen = 0;  // running count of equal keys before this chunk (uniform)
    int written = 0;
    for (int base = 0; base < n; base += blockDim.x) {
        const int i = base + tid;
        const uint64_t kk = i < n ? key64(s[i]) : 0ull;
        const int is_eq = (i < n && kk == thr) ? 1 : 0;
        int eq_tot;
        const int eq_before = block_exclusive_scan(is_eq, wtot, &eq_tot);
        const int win = (i < n) && (kk > thr || (is_eq && eq_seen + eq_before < s_eq_take));
        int w_tot;
        const int pos = block_exclusive_scan(win, wtot, &w_tot);
        if (win) out[written + pos] = i;
        written += w_tot;
        eq_seen += eq_tot;
    }
}

int launch_topk_f64(const double *s, int n, int k, int32_t *out, cudaStream_t st) {
    if (n <= 0 || k <= 0) return LRQK_OK;
    topk_f64_kernel<<<1, 1024, 0, st>>>(s, n, k, out);
    return cudaPeekAtLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

}  // namespace lrqk
