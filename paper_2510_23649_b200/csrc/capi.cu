// extern "C" boundary of liblrqk_b200.so (declared in include/lrqk_b200.h).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace lrqk {
int launch_compress(const lrqk_layer_t &L, const void *q, const void *k, const void *v, int update_b, cudaStream_t st);
int compress_chunks(const lrqk_layer_t &L);
size_t compress_scratch_floats_per_head(const lrqk_layer_t &L);
size_t compress_pre_floats_per_head(const lrqk_layer_t &L);
int launch_prepare(const lrqk_layer_t &L, cudaStream_t st);
int launch_prepare_layers(const lrqk_layer_t *dev_layers, const lrqk_layer_t *host_layers, int n_layers, cudaStream_t st);
int launch_score(const lrqk_layer_t &L, const float *ext_scores, cudaStream_t st);
int launch_select(const lrqk_layer_t &L, cudaStream_t st);
int launch_gather(const lrqk_layer_t &L, cudaStream_t st);
int launch_attention(const lrqk_layer_t &L, const void *q, float *out, cudaStream_t st);
int attn_splits(const lrqk_layer_t &L);
int select_sure_rows(const lrqk_layer_t &L);
int score_part_rows(const lrqk_layer_t &L);
int attn_scratch_slots(const lrqk_layer_t &L);
int launch_select_attend(const lrqk_layer_t &L, const void *q, float *out, cudaStream_t st);
int launch_score_attend(const lrqk_layer_t &L, const void *q, float *out, cudaStream_t st);
int launch_seed(const lrqk_layer_t &L, int prompt_len, cudaStream_t st);
int launch_advance(int32_t *ctx_len, int n, cudaStream_t st);
int launch_proxy_scores(const void *store, int dtype, const float *qh, float *out, int n_heads, int n_rows, int R,
                        cudaStream_t st);
int launch_fill_int(int32_t *p, int n, int v, cudaStream_t st);
int launch_attention_rows(const float *q, const float *K, const float *V, int H, int n, int d, int ld, float *out,
                          float *weights, cudaStream_t st);
int launch_count_misses(const int32_t *resident, int n_res, const int32_t *omega, int n_sel, int size, int32_t *out,
                        cudaStream_t st);
int launch_line_search(const float *xh, const float *B, const float *x, int H, int r, int d, float *B_out,
                       float *grad, float *eta, cudaStream_t st);
size_t prefill_scratch_floats(const lrqk_prefill_t &P);
int launch_prefill(const lrqk_prefill_t &P, cudaStream_t st);
int launch_gemm_f64(int ta, int tb, int m, int n, int k, double alpha, const double *A, int lda, const double *B,
                    int ldb, double beta, double *C, int ldc, void *work, size_t work_bytes, cudaStream_t st);
size_t gemm_f64_workspace(int m, int n, int k);
int launch_mirror_f64(double *G, int r, int ldg, cudaStream_t st);
int launch_dot_f64(const double *a, const double *b, long long n, double *out, double *work, cudaStream_t st);
int launch_axpby_f64(long long n, double alpha, const double *s, const double *x, double beta, double *y,
                     cudaStream_t st);
int launch_solve_spd_f64(const double *M, int r, int ldm, const double *RHS, int n, int ldr, double *X, int ldx,
                         double *work, uint32_t *status, cudaStream_t st);
int launch_topk_f64(const double *s, int n, int k, int32_t *out, cudaStream_t st);
}  // namespace lrqk

using namespace lrqk;

bool lrqk::pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("LRQK_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

static thread_local char g_err[256] = "";

static int check(int rc) {
    if (rc == LRQK_ECUDA) {
        cudaError_t e = cudaGetLastError();
        snprintf(g_err, sizeof g_err, "%s", cudaGetErrorString(e));
    }
    return rc;
}

static bool pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

static int validate(const lrqk_layer_t *L) {
    if (!L) return LRQK_EINVAL;
    if (L->batch < 1 || L->n_q_heads < 1 || L->n_kv_heads < 1 || L->n_q_heads % L->n_kv_heads) return LRQK_EINVAL;
    if (L->head_dim < 1 || L->head_dim > L->dim_stride || L->rank < 1 || L->rank > L->rank_stride) return LRQK_EINVAL;
    if (!pow2(L->dim_stride) || L->dim_stride < 8 || L->dim_stride > 256) return LRQK_EUNSUPPORTED;
    if (!pow2(L->rank_stride) || L->rank_stride < 8 || L->rank_stride > 64) return LRQK_EUNSUPPORTED;
    if (L->k_budget < 1 || L->lite_budget < 1 || L->s_cap != L->k_budget + L->lite_budget) return LRQK_EINVAL;
    if (L->t_max < 32 || L->t_max % 32 || L->t_max >= (1 << 21)) return LRQK_EUNSUPPORTED;
    if (L->s_cap > 8192) return LRQK_EUNSUPPORTED;
    if (L->dtype != LRQK_F32 && L->dtype != LRQK_BF16) return LRQK_EINVAL;
    if (L->policy == LRQK_SLOW_HOST && L->n_slots != L->s_cap + 1) return LRQK_EINVAL;
    if (L->cand_cap < 1) return LRQK_EINVAL;
    return LRQK_OK;
}

extern "C" {

int lrqk_abi_version(void) { return LRQK_ABI_VERSION; }
size_t lrqk_sizeof_layer(void) { return sizeof(lrqk_layer_t); }
size_t lrqk_sizeof_prefill(void) { return sizeof(lrqk_prefill_t); }

void *lrqk_host_alloc(size_t bytes) {
    void *p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
        snprintf(g_err, sizeof g_err, "%s", cudaGetErrorString(cudaGetLastError()));
        return nullptr;
    }
    return p;
}
void lrqk_host_free(void *p) {
    if (p) cudaFreeHost(p);
}
void *lrqk_host_device_ptr(void *p) {
    void *d = nullptr;
    if (cudaHostGetDevicePointer(&d, p, 0) != cudaSuccess) return nullptr;
    return d;
}
const char *lrqk_last_error(void) { return g_err; }

const char *lrqk_buffer_names(void) {
    return "proxy,B_Q,B_K,slow_k,slow_v,slot_k,slot_v,ctx_len,res_idx,res_slot,res_cnt,spare_slot,miss_idx,"
           "miss_slot,miss_cnt,c_miss,c_total,step_miss,step_total,q_hat,k_hat,eta,keys,hist,sel_meta,sure_idx,"
           "cand,red_scratch,attn_scratch,counters,status,pre,fcand,fcnt,res_bits,cmask,proxy_rowmajor";
}

int lrqk_red_chunks(const lrqk_layer_t *L) { return compress_chunks(*L); }
int lrqk_attn_splits(const lrqk_layer_t *L) { return attn_splits(*L); }

int lrqk_layer_buffer_bytes(const lrqk_layer_t *L, size_t *out, int max_out) {
    if (validate(L) != LRQK_OK) return -1;
    const size_t B = L->batch, Hq = L->n_q_heads, Hkv = L->n_kv_heads, BH = B * Hq;
    const size_t e = L->dtype == LRQK_BF16 ? 2 : 4;
    const size_t T = L->t_max, d = L->dim_stride, R = L->rank_stride, S = L->s_cap;
    const bool host = L->policy == LRQK_SLOW_HOST;
    const size_t slots = host ? (size_t)L->n_slots : 0;
    const size_t v[] = {
        BH * T * R * e,                 // proxy
        BH * R * d * 4,                 // B_Q
        BH * R * d * 4,                 // B_K
        B * Hkv * T * d * e,            // slow_k (host memory when policy=HOST)
        B * Hkv * T * d * e,            // slow_v
        BH * slots * d * e,             // slot_k
        BH * slots * d * e,             // slot_v
        B * 4,                          // ctx_len
        BH * S * 4,                     // res_idx
        BH * S * 4,                     // res_slot
        BH * 4,                         // res_cnt
        BH * 4,                         // spare_slot
        BH * S * 4,                     // miss_idx
        BH * S * 4,                     // miss_slot
        BH * 4,                         // miss_cnt
        BH * 8,                         // c_miss
        BH * 8,                         // c_total
        BH * 4,                         // step_miss
        BH * 4,                         // step_total
        BH * R * 4,                     // q_hat
        BH * R * 4,                     // k_hat
        BH * 2 * 4,                     // eta
        BH * T * 4,                     // keys
        BH * kHistLevels * kHistBins * 4,  // hist (coarse | fine | hint window)
        BH * kMetaInts * 4,             // sel_meta
        (size_t)select_sure_rows(*L) * (size_t)L->k_budget * 4,  // sure_idx (per select part in mode 3)
        BH * (size_t)L->cand_cap * 8,   // cand
        BH * compress_scratch_floats_per_head(*L) * 4,       // red_scratch
        BH * (size_t)attn_scratch_slots(*L) * (d + 2) * 4,  // attn_scratch (attention splits / fused parts)
        BH * kCounterInts * 4,          // counters
        4,                              // status
        BH * compress_pre_floats_per_head(*L) * 4,  // pre
        (size_t)score_part_rows(*L) * kCandPart * 8,    // fcand
        (size_t)score_part_rows(*L) * 4,                // fcnt
        BH * (size_t)((L->t_max + 31) / 32) * 4,        // res_bits
        BH * (size_t)((L->t_max + 31) / 32) * 4,        // cmask
        BH * T * R * e,                                 // proxy_rowmajor
    };
    const int n = (int)(sizeof v / sizeof v[0]);
    for (int i = 0; i < n && i < max_out; ++i) out[i] = v[i];
    return n;
}

int lrqk_seed_prompt(const lrqk_layer_t *L, int32_t prompt_len, void *stream) {
    int rc = validate(L);
    if (rc) return rc;
    if (prompt_len < 1 || prompt_len > L->t_max) return LRQK_EINVAL;
    int rc2 = check(launch_seed(*L, prompt_len, (cudaStream_t)stream));
    if (rc2) return rc2;
    return check(launch_prepare(*L, (cudaStream_t)stream));
}

int lrqk_compress_prepare(const lrqk_layer_t *L, void *stream) {
    int rc = validate(L);
    if (rc) return rc;
    return check(launch_prepare(*L, (cudaStream_t)stream));
}

int lrqk_compress_prepare_layers(const lrqk_layer_t *dev_layers, const lrqk_layer_t *host_layers, int32_t n_layers,
                                 void *stream) {
    if (!dev_layers || !host_layers || n_layers < 1) return LRQK_EINVAL;
    for (int i = 0; i < n_layers; ++i) {
        const int rc = validate(&host_layers[i]);
        if (rc) return rc;
        const lrqk_layer_t &a = host_layers[i], &b = host_layers[0];
        if (a.batch != b.batch || a.n_q_heads != b.n_q_heads || a.dim_stride != b.dim_stride ||
            a.rank_stride != b.rank_stride || a.s_cap != b.s_cap || a.dtype != b.dtype || a.policy != b.policy)
            return LRQK_EINVAL;  // one launch covers identically shaped layers
    }
    return check(launch_prepare_layers(dev_layers, host_layers, n_layers, (cudaStream_t)stream));
}

int lrqk_decode_compress(const lrqk_layer_t *L, const void *q, const void *k, const void *v, int update_b,
                         void *stream) {
    int rc = validate(L);
    if (rc) return rc;
    if (!q || !k || !v) return LRQK_EINVAL;
    return check(launch_compress(*L, q, k, v, update_b, (cudaStream_t)stream));
}

int lrqk_score(const lrqk_layer_t *L, void *stream) {
    int rc = validate(L);
    if (rc) return rc;
    return check(launch_score(*L, nullptr, (cudaStream_t)stream));
}

int lrqk_select(const lrqk_layer_t *L, void *stream) {
    int rc = validate(L);
    if (rc) return rc;
    return check(launch_select(*L, (cudaStream_t)stream));
}

int lrqk_gather_misses(const lrqk_layer_t *L, void *stream) {
    int rc = validate(L);
    if (rc) return rc;
    return check(launch_gather(*L, (cudaStream_t)stream));
}

int lrqk_select_attend(const lrqk_layer_t *L, const void *q, float *out, void *stream) {
    int rc = validate(L);
    if (rc) return rc;
    if (!q || !out) return LRQK_EINVAL;
    return check(launch_select_attend(*L, q, out, (cudaStream_t)stream));
}

// LRQK_FUSED=0 (or lrqk_set_fused(0)) turns the fused score/select/attend
// kernel off: A/B runs, and tests of the split path
static int g_fused = -1;
static bool fused_enabled() {
    if (g_fused < 0) {
        const char *e = getenv("LRQK_FUSED");
        g_fused = (e && e[0] == '0') ? 0 : 1;
    }
    return g_fused != 0;
}

int lrqk_set_fused(int on) {
    const int prev = fused_enabled() ? 1 : 0;
    g_fused = on ? 1 : 0;
    return prev;
}

int lrqk_score_attend(const lrqk_layer_t *L, const void *q, float *out, void *stream) {
    int rc = validate(L);
    if (rc) return rc;
    if (!q || !out) return LRQK_EINVAL;
    if (!fused_enabled()) return LRQK_EUNSUPPORTED;
    return check(launch_score_attend(*L, q, out, (cudaStream_t)stream));
}

int lrqk_attention(const lrqk_layer_t *L, const void *q, float *out, void *stream) {
    int rc = validate(L);
    if (rc) return rc;
    if (!q || !out) return LRQK_EINVAL;
    return check(launch_attention(*L, q, out, (cudaStream_t)stream));
}

int lrqk_decode_step(const lrqk_layer_t *L, const void *q, const void *k, const void *v, float *out, int advance,
                     void *stream) {
    int rc = validate(L);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if ((rc = check(launch_compress(*L, q, k, v, 1, st)))) return rc;
    rc = fused_enabled() ? launch_score_attend(*L, q, out, st) : LRQK_EUNSUPPORTED;
    if (rc == LRQK_EUNSUPPORTED) {
        if ((rc = check(launch_score(*L, nullptr, st)))) return rc;
        if ((rc = check(launch_select_attend(*L, q, out, st)))) return rc;
    } else if ((rc = check(rc))) {
        return rc;
    }
    if ((rc = check(launch_select(*L, st)))) return rc;
    // host policy: the attention kernel fetches this step's misses itself (K5b fused)
    if ((rc = check(launch_attention(*L, q, out, st)))) return rc;
    if ((rc = check(launch_prepare(*L, st)))) return rc;
    if (advance) rc = check(launch_advance(L->ctx_len, L->batch, st));
    return rc;
}

int lrqk_advance(int32_t *ctx_len, int32_t batch, void *stream) {
    if (!ctx_len || batch < 1) return LRQK_EINVAL;
    return check(launch_advance(ctx_len, batch, (cudaStream_t)stream));
}

int lrqk_proxy_scores_f32(const void *store, int32_t dtype, const float *q_hat, float *scores, int32_t n_heads,
                          int32_t n_rows, int32_t rank_stride, void *stream) {
    if (!store || !q_hat || !scores || n_heads < 1 || n_rows < 0 || rank_stride < 1) return LRQK_EINVAL;
    if (n_rows == 0) return LRQK_OK;
    return check(launch_proxy_scores(store, dtype, q_hat, scores, n_heads, n_rows, rank_stride, (cudaStream_t)stream));
}

// Workspace carve-up for the standalone selection.
struct SelWs {
    lrqk_layer_t L;
    size_t bytes;
};
static SelWs sel_layout(int32_t n_heads, int32_t t, int32_t k_budget, int32_t lite_budget, char *base) {
    SelWs w;
    memset(&w.L, 0, sizeof w.L);
    lrqk_layer_t &L = w.L;
    L.batch = n_heads;
    L.n_q_heads = 1;
    L.n_kv_heads = 1;
    L.head_dim = 8;
    L.dim_stride = 8;
    L.rank = 8;
    L.rank_stride = 8;
    L.t_max = ((t + 1 + 31) / 32) * 32;
    L.k_budget = k_budget;
    L.lite_budget = lite_budget;
    L.s_cap = k_budget + lite_budget;
    L.n_slots = L.s_cap + 1;
    L.cand_cap = 8192;
    L.dtype = LRQK_F32;
    L.policy = LRQK_SLOW_HBM;
    size_t off = 0;
    auto take = [&](size_t n) -> char * {
        char *p = base ? base + off : nullptr;
        off += (n + 255) & ~(size_t)255;
        return p;
    };
    const size_t BH = n_heads;
    L.ctx_len = (int32_t *)take(BH * 4);
    L.res_cnt = (int32_t *)take(BH * 4);
    L.res_idx = (int32_t *)take(BH * L.s_cap * 4);
    L.res_slot = L.res_idx;
    L.c_miss = (int64_t *)take(BH * 8);
    L.c_total = (int64_t *)take(BH * 8);
    L.step_miss = (int32_t *)take(BH * 4);
    L.step_total = (int32_t *)take(BH * 4);
    L.keys = (uint32_t *)take(BH * L.t_max * 4);
    L.hist = (uint32_t *)take(BH * kHistLevels * kHistBins * 4);
    L.sel_meta = (int32_t *)take(BH * kMetaInts * 4);
    L.sure_idx = (int32_t *)take((size_t)select_sure_rows(L) * (size_t)k_budget * 4);
    L.cand = (uint64_t *)take(BH * (size_t)L.cand_cap * 8);
    L.counters = (int32_t *)take(BH * kCounterInts * 4);
    L.status = (uint32_t *)take(4);
    w.bytes = off;
    return w;
}

size_t lrqk_select_scores_workspace(int32_t n_heads, int32_t t, int32_t k_budget, int32_t lite_budget) {
    return sel_layout(n_heads, t, k_budget, lite_budget, nullptr).bytes;
}

int lrqk_select_scores(const float *scores, int32_t n_heads, int32_t t, int32_t k_budget, int32_t lite_budget,
                       int32_t *omega, int32_t *omega_cnt, void *workspace, size_t workspace_bytes, void *stream) {
    if (!scores || !omega || !omega_cnt || !workspace || n_heads < 1 || t < 0 || k_budget < 1 || lite_budget < 1)
        return LRQK_EINVAL;
    SelWs w = sel_layout(n_heads, t, k_budget, lite_budget, (char *)workspace);
    if (workspace_bytes < w.bytes) return LRQK_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(workspace, 0, w.bytes, st);
    lrqk_layer_t &L = w.L;
    int rc;
    if ((rc = check(launch_fill_int(L.ctx_len, n_heads, t, st)))) return rc;
    if ((rc = check(launch_score(L, scores, st)))) return rc;
    if ((rc = check(launch_select(L, st)))) return rc;
    if (cudaMemcpyAsync(omega, L.res_idx, (size_t)n_heads * L.s_cap * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return check(LRQK_ECUDA);
    if (cudaMemcpyAsync(omega_cnt, L.res_cnt, (size_t)n_heads * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return check(LRQK_ECUDA);
    return LRQK_OK;
}

int lrqk_attention_rows(const float *q, const float *K, const float *V, int32_t n_heads, int32_t n_rows,
                        int32_t head_dim, int32_t ld, float *out, float *weights, void *stream) {
    if (!q || !K || !V || !out || n_heads < 1 || n_rows < 1 || head_dim < 1 || ld < head_dim) return LRQK_EINVAL;
    return check(launch_attention_rows(q, K, V, n_heads, n_rows, head_dim, ld, out, weights, (cudaStream_t)stream));
}

int lrqk_count_misses(const int32_t *resident, int32_t n_resident, const int32_t *omega, int32_t n_selected,
                      int32_t size, int32_t *out3, void *stream) {
    if (!omega || !out3 || n_resident < 0 || n_selected < 0) return LRQK_EINVAL;
    return check(launch_count_misses(resident, n_resident, omega, n_selected, size, out3, (cudaStream_t)stream));
}

int lrqk_line_search(const float *x_hat, const float *B, const float *x, int32_t n_heads, int32_t rank,
                     int32_t dim, float *B_out, float *grad, float *eta, void *stream) {
    if (!x_hat || !B || !x || !B_out || !eta || n_heads < 1 || rank < 1 || dim < 1) return LRQK_EINVAL;
    return check(launch_line_search(x_hat, B, x, n_heads, rank, dim, B_out, grad, eta, (cudaStream_t)stream));
}

size_t lrqk_prefill_scratch_bytes(const lrqk_prefill_t *P) {
    if (!P) return 0;
    return prefill_scratch_floats(*P) * sizeof(float);
}

int lrqk_prefill_factorize(const lrqk_prefill_t *P, void *stream) {
    if (!P || P->n_heads < 1 || P->len < 1 || !P->Q || !P->K || !(P->A_Q || P->A_Q0) || !P->A_K || !P->B_Q || !P->B_K ||
        !P->scratch || !P->sweeps || !P->converged || P->max_iter < 1)
        return LRQK_EINVAL;
    if (P->want_objective && !P->objective) return LRQK_EINVAL;
    if (P->group < 1 || P->n_heads % P->group) return LRQK_EINVAL;
    return check(launch_prefill(*P, (cudaStream_t)stream));
}

int lrqk_read_status(const uint32_t *status, uint32_t *host_out, void *stream) {
    if (!status || !host_out) return LRQK_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemcpyAsync(host_out, status, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess) return check(LRQK_ECUDA);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check(LRQK_ECUDA);
    return LRQK_OK;
}

size_t lrqk_workspace_size(const lrqk_layer_t *cfg) {
    size_t sizes[64];
    const int n = lrqk_layer_buffer_bytes(cfg, sizes, 64);
    if (n <= 0) return 0;
    size_t tot = 0;
    for (int i = 0; i < n; ++i) tot += sizes[i];
    return tot;
}

int lrqk_score_append(const lrqk_layer_t *L, void *stream) { return lrqk_score(L, stream); }

int lrqk_cache_update(const lrqk_layer_t *L, void *stream) { return lrqk_gather_misses(L, stream); }

int lrqk_get_status(const lrqk_layer_t *L, uint32_t *host_out, void *stream) {
    if (!L) return LRQK_EINVAL;
    return lrqk_read_status(L->status, host_out, stream);
}

int lrqk_counters(const lrqk_layer_t *L, int64_t *c_miss_out, int64_t *c_total_out, void *stream) {
    int rc = validate(L);
    if (rc) return rc;
    if (!c_miss_out || !c_total_out || !L->c_miss || !L->c_total) return LRQK_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)L->batch * L->n_q_heads * sizeof(int64_t);
    if (cudaMemcpyAsync(c_miss_out, L->c_miss, n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(c_total_out, L->c_total, n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return check(LRQK_ECUDA);
    return LRQK_OK;
}

}  // extern "C"

// ---- development tracing (see common.cuh) --------------------------------
namespace lrqk {
__device__ int g_lrqk_trace_on = 0;
__device__ unsigned long long g_lrqk_trace[kTraceCap][2];
}  // namespace lrqk

extern "C" int lrqk_trace_enable(int on) {
    if (cudaMemcpyToSymbol(lrqk::g_lrqk_trace_on, &on, sizeof(int)) != cudaSuccess) return LRQK_ECUDA;
    void *p = nullptr;
    if (cudaGetSymbolAddress(&p, lrqk::g_lrqk_trace) != cudaSuccess) return LRQK_ECUDA;
    if (cudaMemset(p, 0, sizeof(unsigned long long) * 2 * lrqk::kTraceCap) != cudaSuccess) return LRQK_ECUDA;
    return cudaDeviceSynchronize() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

// Copies the recorded (tag<<48 | block, %globaltimer) pairs, compacted, to out.
extern "C" int lrqk_trace_read(unsigned long long *out, int cap) {
    static unsigned long long buf[lrqk::kTraceCap][2];
    if (cudaMemcpyFromSymbol(buf, lrqk::g_lrqk_trace, sizeof buf) != cudaSuccess) return -1;
    int n = 0;
    for (int i = 0; i < lrqk::kTraceCap && n < cap; ++i) {
        if (buf[i][1] == 0) continue;
        out[2 * n] = buf[i][0];
        out[2 * n + 1] = buf[i][1];
        ++n;
    }
    return n;
}

// ---- float64 dense kernels (dense.cu) ----------------------------------------
int lrqk_gemm_f64(int32_t trans_a, int32_t trans_b, int32_t m, int32_t n, int32_t k, double alpha, const double *A,
                  int32_t lda, const double *B, int32_t ldb, double beta, double *C, int32_t ldc, void *work,
                  size_t work_bytes, void *stream) {
    if (m < 0 || n < 0 || k < 0 || !C || (k > 0 && (!A || !B))) return LRQK_EINVAL;
    if (lda < (trans_a ? m : k) || ldb < (trans_b ? k : n) || ldc < n) return LRQK_EINVAL;
    return check(lrqk::launch_gemm_f64(trans_a, trans_b, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, work,
                                       work_bytes, (cudaStream_t)stream));
}
size_t lrqk_gemm_f64_workspace(int32_t m, int32_t n, int32_t k) { return lrqk::gemm_f64_workspace(m, n, k); }

int lrqk_symmetrize_f64(double *G, int32_t r, int32_t ldg, void *stream) {
    if (!G || r < 0 || ldg < r) return LRQK_EINVAL;
    return check(lrqk::launch_mirror_f64(G, r, ldg, (cudaStream_t)stream));
}

int lrqk_dot_f64(const double *a, const double *b, int64_t n, double *out, double *work, void *stream) {
    if (!a || !b || !out || !work || n < 0) return LRQK_EINVAL;
    return check(lrqk::launch_dot_f64(a, b, n, out, work, (cudaStream_t)stream));
}

int lrqk_axpby_f64(int64_t n, double alpha, const double *alpha_scale, const double *x, double beta, double *y,
                   void *stream) {
    if (n < 0 || (n > 0 && (!x || !y))) return LRQK_EINVAL;
    return check(lrqk::launch_axpby_f64(n, alpha, alpha_scale, x, beta, y, (cudaStream_t)stream));
}

int lrqk_solve_spd_f64(const double *M, int32_t r, int32_t ldm, const double *RHS, int32_t n, int32_t ldr, double *X,
                       int32_t ldx, double *work, uint32_t *status, void *stream) {
    if (!M || !work || !status || r < 1 || ldm < r || n < 0 || (n > 0 && (!RHS || !X || ldr < r || ldx < r)))
        return LRQK_EINVAL;
    return check(lrqk::launch_solve_spd_f64(M, r, ldm, RHS, n, ldr, X, ldx, work, status, (cudaStream_t)stream));
}

int lrqk_topk_f64(const double *scores, int32_t n, int32_t k, int32_t *out, void *stream) {
    if (!scores || !out || n < 0 || k < 1 || k >= n + 1) return LRQK_EINVAL;
    return check(lrqk::launch_topk_f64(scores, n, k, out, (cudaStream_t)stream));
}
