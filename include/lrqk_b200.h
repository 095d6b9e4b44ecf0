/*
 * lrqk_b200.h -- C-ABI of the B200-native LRQK decode-time sparse-attention
 * path (arXiv 2510.23649).  Plain pointers, sizes and a cudaStream_t passed
 * as void*; no torch or C++ types cross this boundary.
 *
 * The reference exposes this path as a Python function API over float64
 * numpy arrays (pkg/src/lrqk/__init__.py:10-82); it has no FFI of its own.
 * Each entry point below names the reference function(s) it replaces.  The
 * Python host mirror (paper_2510_23649_b200/) binds this header with ctypes;
 * INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - "layer" = one attention layer's decode state for B sequences x Hq query
 *    heads (GQA: Hkv key/value heads, G = Hq / Hkv query heads per KV head).
 *    Every (sequence, query head) pair is one reference DecodeSession
 *    (session.py:62-131); K/V rows are stored once per KV head, while proxy
 *    rows, B factors, selections and counters are per query head
 *    (SURVEY.md Appendix A.11).
 *  - All buffers are caller-allocated (sizes: lrqk_layer_buffer_bytes).  The
 *    library never allocates device memory.
 *  - Row vectors are padded to dim_stride / rank_stride elements (multiples
 *    of 8); padding must be zero.  head_dim / rank are the true sizes used for
 *    the 1/sqrt(d) scale and for the r x r solves.
 *  - Return value: 0 on success, else an LRQK_E* code for argument / launch
 *    errors.  Numerical conditions found on the device (non-finite input,
 *    SPD solve failed after jitter, index out of range) are OR-ed into the
 *    device status word `status` and read with lrqk_read_status().
 */
#ifndef LRQK_B200_H
#define LRQK_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LRQK_ABI_VERSION 2

/* storage dtypes */
#define LRQK_F32 0
#define LRQK_BF16 1

/* slow-tier placement ("physical cache policy") */
#define LRQK_SLOW_HBM 0  /* full K/V history in HBM; selected rows gathered by index   */
#define LRQK_SLOW_HOST 1 /* full K/V history in mapped pinned host memory; GPU holds   */
                         /* only the selected rows in per-head slots; misses over PCIe */

/* return codes */
#define LRQK_OK 0
#define LRQK_EINVAL 1
#define LRQK_ECUDA 2
#define LRQK_EUNSUPPORTED 3

/* device status bits (ref: errors.py:4-9, cache.py:183-189) */
#define LRQK_ST_NONFINITE 1u     /* NonFiniteError                         */
#define LRQK_ST_SOLVE_FAILED 2u  /* SolveFailedError (jitter retry failed) */
#define LRQK_ST_INDEX_RANGE 4u   /* IndexError (selection out of range)    */
#define LRQK_ST_CAPACITY 8u      /* store capacity t_max exhausted          */
#define LRQK_ST_JITTERED 16u     /* informational: a jittered solve ran     */
#define LRQK_ST_FALLBACK 32u     /* informational: direct-solve fallback ran */
#define LRQK_ST_BARRIER 64u      /* a per-head barrier of lrqk_score_attend timed out (never expected) */

typedef struct lrqk_layer {
    /* ---- shapes / configuration ---- */
    int32_t batch, n_q_heads, n_kv_heads;
    int32_t head_dim, dim_stride;
    int32_t rank, rank_stride;
    int32_t t_max;                 /* tokens the stores can hold            */
    int32_t k_budget, lite_budget; /* ref: SessionConfig.k_budget/lite_budget */
    int32_t s_cap;                 /* k_budget + lite_budget                */
    int32_t n_slots;               /* s_cap + 1 (slots per head, host policy) */
    int32_t cand_cap;              /* radix-select candidate capacity / head */
    int32_t dtype;                 /* LRQK_F32 | LRQK_BF16                  */
    int32_t policy;                /* LRQK_SLOW_HBM | LRQK_SLOW_HOST        */
    int32_t max_iter;              /* ref: DecodeConfig.max_iter            */
    float lambda_1, lambda_2, tol; /* ref: DecodeConfig                     */

    /* ---- persistent state ---- */
    void *proxy;                   /* A_K store [B,Hq,t_max,rank_stride] dtype  (cache.py proxy store) */
    float *B_Q, *B_K;              /* [B,Hq,rank_stride,dim_stride] f32           */
    void *slow_k, *slow_v;         /* [B,Hkv,t_max,dim_stride] dtype (device or mapped host) */
    void *slot_k, *slot_v;         /* [B,Hq,n_slots,dim_stride] dtype (host policy only)     */
    int32_t *ctx_len;              /* [B] tokens stored; the new token gets index ctx_len[b]  */
    int32_t *res_idx;              /* [B,Hq,s_cap] fast-tier index set Omega_t: ascending under   */
                                   /* LRQK_SLOW_HOST; under LRQK_SLOW_HBM unordered (certain     */
                                   /* winners | threshold-bin winners | lite window)            */
    int32_t *res_slot;             /* [B,Hq,s_cap] slot of each resident row (host policy)   */
    int32_t *res_cnt;              /* [B,Hq]                                                 */
    int32_t *spare_slot;           /* [B,Hq] free slot that receives the next appended row   */
    int32_t *miss_idx, *miss_slot; /* [B,Hq,s_cap] rows to fetch this step (host policy)     */
    int32_t *miss_cnt;             /* [B,Hq]                                                 */
    int64_t *c_miss, *c_total;     /* [B,Hq] cumulative counters (cache.py:63-74)            */
    int32_t *step_miss, *step_total; /* [B,Hq] this step's counts (StepReport)               */

    /* ---- per-step scratch ---- */
    float *q_hat, *k_hat;          /* [B,Hq,rank_stride]                      */
    float *eta;                    /* [B,Hq,2] line-search steps (eta_Q, eta_K) */
    uint32_t *keys;                /* [B,Hq,t_max] order-preserving score keys */
    uint32_t *hist;                /* [B,Hq,3,2048] coarse | fine / part counts | hint window (zero between steps) */
    int32_t *sel_meta;             /* [B,Hq,48] selection state (incl. the persistent threshold hint; common.cuh Meta) */
    int32_t *sure_idx;             /* [B,Hq,select_parts,k_budget]            */
    uint64_t *cand;                /* [B,Hq,cand_cap]                          */
    float *red_scratch;            /* [B,Hq,red_chunks,rank_stride*(rank_stride+1)] */
    float *attn_scratch;           /* [B,Hq,attn_splits,dim_stride+2]          */
    int32_t *counters;             /* [B,Hq,8] arrival counters, zero between steps */
    uint32_t *status;              /* [1] device status word                  */

    /* ---- persistent precompute of the next step's compression (K2p) ---- */
    float *pre;                    /* [B,Hq,pre_floats]: P^-1, R^-1, P, R, Z_Q, Z_K, W, flags */

    /* ---- per-step scratch of the fused score/selection path ---- */
    uint64_t *fcand;               /* [B*Hq*score_parts, 1025] per-part window suffix counts (lrqk_score) */
    int32_t *fcnt;                 /* [B*Hq*score_parts] certain winners before each part (offsets)  */

    /* ---- persistent residency bitmap (HBM policy hit/miss accounting) ---- */
    uint32_t *res_bits;            /* [B,Hq,ceil(t_max/32)] bit x set <=> x in the fast tier      */

    /* ---- per-step scratch: rows whose score key clears the candidate bound ---- */
    uint32_t *cmask;               /* [B,Hq,ceil(t_max/32)] one bit per row (lrqk_score)          */

    /* ---- persistent: row-major copy of the proxy store (optional, may be NULL) ---- */
    void *proxy_rowmajor;          /* [B,Hq,t_max,rank_stride] dtype: the same A_K rows, one contiguous */
                                   /* rank_stride run per row, kept by lrqk_decode_compress's append;   */
                                   /* the selected rows' gathers read it (one 64-byte run per row      */
                                   /* at r=32 bf16 instead of rank_stride/8 scattered 16-byte packs)   */
} lrqk_layer_t;

/* Sizes (bytes) of every buffer in lrqk_layer_t for the given configuration,
 * written to out[] in the order of lrqk_buffer_names().  Returns the count. */
int lrqk_layer_buffer_bytes(const lrqk_layer_t *cfg, size_t *out, int max_out);
const char *lrqk_buffer_names(void);
int lrqk_abi_version(void);
int lrqk_red_chunks(const lrqk_layer_t *cfg);
int lrqk_attn_splits(const lrqk_layer_t *cfg);

/* Prompt seeding: proxy[0..l) and slow K/V[0..l) must already hold the
 * prompt; sets ctx_len=l, fast tier = last lite_budget prompt rows, zeroes
 * counters/hist, fills slots (host policy).  ref: cache.py:114-124. */
int lrqk_seed_prompt(const lrqk_layer_t *L, int32_t prompt_len, void *stream);

/* Precompute, from the current fast-tier set Omega and B factors, everything
 * the next token's compression needs except q and k (A_res^T K_res,
 * A_res^T A_res, the r x r inverses, Z_Q, Z_K).  Runs after lrqk_select of
 * the previous step (after lrqk_gather_misses in the host policy) and after
 * lrqk_seed_prompt; may overlap the rest of the step on a side stream.
 * ref: decode.py:84-119 (the q/k-independent parts of update_qhat/khat). */
int lrqk_compress_prepare(const lrqk_layer_t *L, void *stream);

/* lrqk_compress_prepare for n_layers identically shaped layers in one
 * launch: dev_layers is a device copy of host_layers[0..n_layers).  A
 * layer's precompute is only consumed by its next decode step, so an engine
 * runs this once per step after the last layer. */
int lrqk_compress_prepare_layers(const lrqk_layer_t *dev_layers, const lrqk_layer_t *host_layers, int32_t n_layers,
                                 void *stream);

/* Per-token compression + B line-search update + append of k_hat/k/v.
 * With bf16 storage (rank >= 16, d >= 64) the B update only feeds the next
 * step, so it is deferred: the next lrqk_compress_prepare(_layers) applies
 * it before forming the next step's systems (eta is written then). 
 * ref: decode.py:122-184 (decode_compress, update_projections),
 *      cache.py:199-214 (append_token), session.py:95-98.
 * q [B,Hq,dim_stride], k/v [B,Hkv,dim_stride] dtype. */
int lrqk_decode_compress(const lrqk_layer_t *L, const void *q, const void *k, const void *v,
                         int update_b, void *stream);

/* Proxy scores over tokens 0..t (incl. the just-appended row) as
 * order-preserving keys + per-head radix histogram.  ref: cache.py:141-146. */
int lrqk_score(const lrqk_layer_t *L, void *stream);

/* Top-k + lite-window selection fused with hit/miss accounting and slot
 * replacement.  ref: cache.py:149-196, linalg.py:96-110. */
int lrqk_select(const lrqk_layer_t *L, void *stream);

/* Fused selection + attention for the heads whose score pass located the
 * k-th largest key in its threshold window (the common case, HBM policy):
 * writes Omega_t to res_idx and the attention's softmax partials for those
 * heads; lrqk_select skips them and lrqk_attention only merges their
 * partials into out.  Launch it right after lrqk_score, and lrqk_attention
 * after it.  ref: cache.py:149-171, attention.py:23-34. */
int lrqk_select_attend(const lrqk_layer_t *L, const void *q, float *out, void *stream);

/* lrqk_score + lrqk_select_attend as ONE kernel (HBM policy, dim_stride
 * 128): each head's blocks meet at per-head barriers, so a head selects and
 * attends as soon as its own parts have streamed; its softmax partials are
 * merged into out by lrqk_attention (launch it after lrqk_select, as after
 * lrqk_select_attend).  Heads off the hint-window path this step are left
 * to lrqk_select / lrqk_attention as after lrqk_score.  Returns
 * LRQK_EUNSUPPORTED (nothing launched) for layouts it does not cover or when
 * its grid cannot be co-resident; run lrqk_score + lrqk_select_attend then.
 * ref: cache.py:141-171, linalg.py:96-110, attention.py:23-34. */
int lrqk_score_attend(const lrqk_layer_t *L, const void *q, float *out, void *stream);

/* Process-wide switch for lrqk_score_attend / lrqk_decode_step: 0 runs the
 * split path (lrqk_score + lrqk_select_attend) everywhere; returns the
 * previous setting.  Default on (environment LRQK_FUSED=0: off). */
int lrqk_set_fused(int on);

/* Host policy: copy this step's missed K/V rows from the pinned host slow
 * tier into their slots (zero-copy PCIe reads) as a pass of its own.
 * Optional: lrqk_attention fetches the misses lrqk_select marked (slot bit
 * 30) itself, overlapped with the hit rows, and lrqk_decode_step relies on
 * that; after this call lrqk_attention reads every row from its slot.
 * ref: cache.py:193-194. */
int lrqk_gather_misses(const lrqk_layer_t *L, void *stream);

/* Exact softmax attention over the selected rows; out [B,Hq,dim_stride] f32.
 * ref: attention.py:23-34, session.py:101-102. */
int lrqk_attention(const lrqk_layer_t *L, const void *q, float *out, void *stream);

/* One whole decode step of one layer (compress, score_attend -- or score +
 * select_attend --, select, gather, attention, compress_prepare -- the reference's order,
 * session.py:90-104); advance!=0 also bumps ctx_len. */
int lrqk_decode_step(const lrqk_layer_t *L, const void *q, const void *k, const void *v,
                     float *out, int advance, void *stream);

/* ctx_len[b] += 1 for every sequence (end of a multi-layer step). */
int lrqk_advance(int32_t *ctx_len, int32_t batch, void *stream);

/* Standalone proxy scores for the drop-in proxy_scores(q_hat, store):
 * scores[h, i] = store[h, i, :] . q_hat[h, :], n_heads independent rows.  */
int lrqk_proxy_scores_f32(const void *store, int32_t dtype, const float *q_hat, float *scores,
                          int32_t n_heads, int32_t n_rows, int32_t rank_stride, void *stream);

/* Standalone selection for the drop-in select_active(scores, t, k, lite):
 * scores [n_heads, t+1] f32 -> omega [n_heads, s_cap] ascending, count. */
int lrqk_select_scores(const float *scores, int32_t n_heads, int32_t t, int32_t k_budget,
                       int32_t lite_budget, int32_t *omega, int32_t *omega_cnt,
                       void *workspace, size_t workspace_bytes, void *stream);
size_t lrqk_select_scores_workspace(int32_t n_heads, int32_t t, int32_t k_budget, int32_t lite_budget);

/* Standalone exact attention over explicit fp32 rows (drop-in
 * exact_attention, attention.py:23-34): q [H][ld], K/V [H][n][ld];
 * out [H][ld], weights [H][n] (may be NULL). */
int lrqk_attention_rows(const float *q, const float *K, const float *V, int32_t n_heads, int32_t n_rows,
                        int32_t head_dim, int32_t ld, float *out, float *weights, void *stream);

/* Hit/miss accounting of an explicit selection against an ascending
 * resident set (drop-in fetch_and_merge, cache.py:174-196):
 * out3 = {misses, selected, any index outside [0, size)}. */
int lrqk_count_misses(const int32_t *resident, int32_t n_resident, const int32_t *omega, int32_t n_selected,
                      int32_t size, int32_t *out3, void *stream);

/* Standalone exact line-search step on one B factor (drop-in
 * update_projections, decode.py:150-184): x_hat [H][r], B [H][r][d],
 * x [H][d] -> B_out, grad (may be NULL) [H][r][d], eta [H]. */
int lrqk_line_search(const float *x_hat, const float *B, const float *x, int32_t n_heads, int32_t rank,
                     int32_t dim, float *B_out, float *grad, float *eta, void *stream);

/* ---- float64 dense kernels of the drop-in linear algebra ------------------
 * The reference computes these in float64 (numpy / LAPACK); so do these
 * kernels, so the per-call drop-in functions (gram, solve_spd, fro_norm_sq,
 * update_B/AK/AQ, lagrangian_value, factor_residuals, khat_initial_guess,
 * update_qhat/khat, topk_indices) agree with it to rounding.  Row-major,
 * device pointers, caller-allocated outputs and workspaces. */

/* C = alpha op(A) op(B) + beta C; op = transpose when trans_* != 0.
 * work (may be NULL: no split-K) of lrqk_gemm_f64_workspace() bytes.
 * ref: the `@` products of prefill.py:142-181, decode.py:79-119. */
int lrqk_gemm_f64(int32_t trans_a, int32_t trans_b, int32_t m, int32_t n, int32_t k, double alpha, const double *A,
                  int32_t lda, const double *B, int32_t ldb, double beta, double *C, int32_t ldc, void *work,
                  size_t work_bytes, void *stream);
size_t lrqk_gemm_f64_workspace(int32_t m, int32_t n, int32_t k);

/* Copy the strict upper triangle of the r x r matrix G onto the lower one
 * (gram's exact symmetry, linalg.py:48-55). */
int lrqk_symmetrize_f64(double *G, int32_t r, int32_t ldg, void *stream);

/* *out = sum a[i] b[i] (device scalar), fixed reduction order; work >= 256
 * doubles.  ref: fro_norm_sq linalg.py:58-60 and the Gram-trace inner
 * products of lagrangian_value prefill.py:150-153. */
int lrqk_dot_f64(const double *a, const double *b, int64_t n, double *out, double *work, void *stream);

/* y = alpha * (*alpha_scale if non-NULL) * x + beta * y. */
int lrqk_axpby_f64(int64_t n, double alpha, const double *alpha_scale, const double *x, double beta, double *y,
                   void *stream);

/* X M = RHS for X (n x r), M r x r symmetric positive (semi)definite, lower
 * triangle read.  Cholesky; on failure one retry with 1e-10 (tr(M)/r + 1) on
 * the diagonal (sets LRQK_ST_JITTERED); still failing -> LRQK_ST_SOLVE_FAILED
 * and X untouched; non-finite M or RHS -> LRQK_ST_NONFINITE.  work: r*r + 1
 * doubles.  ref: solve_spd linalg.py:63-93. */
int lrqk_solve_spd_f64(const double *M, int32_t r, int32_t ldm, const double *RHS, int32_t n, int32_t ldr, double *X,
                       int32_t ldx, double *work, uint32_t *status, void *stream);

/* Indices of the k largest of n float64 scores, ascending, ties toward the
 * lower index (k < n; out holds k ints).  ref: topk_indices linalg.py:96-110. */
int lrqk_topk_f64(const double *scores, int32_t n, int32_t k, int32_t *out, void *stream);

/* ---- prefill factorisation (ref: prefill.py:197-230) ---- */
typedef struct lrqk_prefill {
    int32_t n_heads;        /* independent (Q,K) problems                     */
    int32_t group;          /* query heads sharing one K (GQA); K index = h / group */
    int32_t len, head_dim, dim_stride, rank, rank_stride;
    int32_t dtype;          /* dtype of Q, K                                  */
    int32_t max_iter;
    float lambda_q, lambda_k, tol;
    int32_t want_objective; /* record the Lagrangian after init and each sweep */
    const void *Q;          /* [n_heads, len, dim_stride]                     */
    const void *K;          /* [n_heads/group, len, dim_stride]               */
    float *A_Q, *A_K;       /* [n_heads, len, rank_stride] in: init, out: factors;
                             * A_Q may be NULL when A_Q0 is given: the query
                             * factor is then not materialised (decode reads
                             * only A_K, B_Q, B_K) */
    float *B_Q, *B_K;       /* [n_heads, rank_stride, dim_stride] out         */
    float *objective;       /* [n_heads, max_iter+1] (NaN where not reached)  */
    int32_t *sweeps;        /* [n_heads]                                      */
    int32_t *converged;     /* [n_heads]                                      */
    float *scratch;         /* lrqk_prefill_scratch_bytes()                   */
    uint32_t *status;
    /* Optional separate init factors.  NULL: the init is read from A_Q/A_K
     * (in/out, [n_heads, len, rank_stride]).  Non-NULL: read from here,
     * [len, rank_stride] when init_shared (one draw for every head, as the
     * reference's randn init, prefill.py:124-127), else
     * [n_heads, len, rank_stride].                                        */
    const float *A_Q0, *A_K0;
    int32_t init_shared;
} lrqk_prefill_t;

size_t lrqk_prefill_scratch_bytes(const lrqk_prefill_t *P);
int lrqk_prefill_factorize(const lrqk_prefill_t *P, void *stream);

/* Copy the status word to host memory (synchronises the stream). */
int lrqk_read_status(const uint32_t *status, uint32_t *host_out, void *stream);

/* ---- SURVEY §8(b) entry-point names -------------------------------------
 * The scope table names a minimum export list; these are those names over
 * the entry points above (same semantics, same status codes). */

/* Total device bytes of one layer's buffers (the sum of
 * lrqk_layer_buffer_bytes), 0 for an invalid configuration. */
size_t lrqk_workspace_size(const lrqk_layer_t *cfg);

/* Proxy scores over A_K[0..t] (k_hat_t was appended by
 * lrqk_decode_compress) = lrqk_score.  ref: cache.py:141-146, 211. */
int lrqk_score_append(const lrqk_layer_t *L, void *stream);

/* Fast-tier update after the selection: the host policy copies the step's
 * missed rows into their slots (= lrqk_gather_misses); the HBM policy's
 * residency/counter update is folded into lrqk_compress_prepare, so this is
 * a no-op for it.  ref: cache.py:174-196. */
int lrqk_cache_update(const lrqk_layer_t *L, void *stream);

/* The layer's status word to host (= lrqk_read_status(L->status, ...)). */
int lrqk_get_status(const lrqk_layer_t *L, uint32_t *host_out, void *stream);

/* CacheStats counters to host: c_miss and c_total, [B, Hq] int64 each
 * (synchronises the stream).  ref: cache.py:63-81. */
int lrqk_counters(const lrqk_layer_t *L, int64_t *c_miss_out, int64_t *c_total_out, void *stream);

/* Name of the last CUDA error seen by the library (thread-local). */
const char *lrqk_last_error(void);

/* ABI self-checks for binders: sizeof(lrqk_layer_t), sizeof(lrqk_prefill_t). */
size_t lrqk_sizeof_layer(void);
size_t lrqk_sizeof_prefill(void);

/* Pinned, mapped, portable host memory for the LRQK_SLOW_HOST slow tier
 * (cudaHostAlloc); lrqk_host_device_ptr returns the device alias. */
void *lrqk_host_alloc(size_t bytes);
void lrqk_host_free(void *p);
void *lrqk_host_device_ptr(void *p);

/* Development tracing of kernel phases (%globaltimer records). */
int lrqk_trace_enable(int on);
int lrqk_trace_read(unsigned long long *out, int cap);

#ifdef __cplusplus
}
#endif
#endif /* LRQK_B200_H */
