// K6: gather-fused exact attention over the selected rows
//     (attention.py:23-34, session.py:101-102)
// K5b: host-policy miss gather from the pinned host slow tier (cache.py:193-194)
// plus prompt seeding (cache.py:114-124) and small utilities.
#include "common.cuh"
#include "attend_common.cuh"

namespace lrqk {

constexpr int kAttnThreads = 128;

struct AttnArgs {
    lrqk_layer_t L;
    const void *q;
    float *out;
    int yg_slots;  // red_scratch slots per head (compress.cu yg_slots)
    int slots;     // attn_scratch partial slots per head (attn_scratch_slots): the
                   // stride select_attend_kernel uses too, so heads of the two
                   // paths in one step never write each other's partials
};

// A mode-5 head's blocks other than split 0 have no rows to attend; they sum
// select_attend's Y|G slot partials (in slot order, as the finish kernel
// would) into slot 0, each block one float4 slice, so the end-of-step finish
// kernel reads one slot instead of parts + 1.
__device__ void fold_yg_slots(const lrqk_layer_t &L, int bh, int yg_slots, int blk, int nblk) {
    const int *meta = L.sel_meta + (size_t)bh * kMetaInts;
    const int nyg = meta[M_YG];
    if (nyg <= 1) return;
    const size_t PF4 = yg_part_floats(L.rank_stride, L.dim_stride) / 4;
    float4 *YG4 = reinterpret_cast<float4 *>(L.red_scratch + (size_t)bh * yg_slots * PF4 * 4);
    const size_t per = (PF4 + nblk - 1) / nblk, e0 = (size_t)blk * per, e1 = min(PF4, e0 + per);
    for (size_t e4 = e0 + threadIdx.x; e4 < e1; e4 += blockDim.x) {
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
    if (blk == 0 && threadIdx.x == 0) const_cast<int *>(meta)[M_YG_FOLD] = 1;
}

// Output of a head whose selection ran in score_attend_kernel: its P
// partials (slot stride attn_slots_dev(P)) merged by one block.
__device__ void merge_score_attend_partials(const lrqk_layer_t &L, int bh, float *out) {
    __shared__ float s_w[64], s_red[2];
    const int d = L.dim_stride;
    const int np = L.sel_meta[(size_t)bh * kMetaInts + M_ATT_PARTS];
    const float *parts = L.attn_scratch + (size_t)bh * attn_slots_dev(L, np) * (size_t)(d + 2);
    merge_partials(parts, np, d, out + (size_t)bh * d, s_w, s_red);
}

// One block = one split of kAttnRows selected rows of one (b, h).  Lanes are
// grouped LPR per row (16-byte packs across d); each group runs an online
// softmax over its rows; groups, warps and finally splits are merged with the
// usual (max, sum, acc) rescaling.  The last split block of a head merges the
// split partials and writes the output.
// Output of a head whose selection ran in select_attend_kernel: its
// parts + 1 partials (max, sum, acc[d]; log2 domain) merged by one block.
__device__ void merge_select_attend_partials(const lrqk_layer_t &L, int bh, float *out) {
    __shared__ float s_w[64], s_red[2];
    const int d = L.dim_stride;
    const int np = L.sel_meta[(size_t)bh * kMetaInts + M_ATT_PARTS];
    const float *parts = L.attn_scratch + (size_t)bh * attn_slots_dev(L, np - 1) * (size_t)(d + 2);
    merge_partials(parts, np, d, out + (size_t)bh * d, s_w, s_red);
    trace(39);
}

template <typename T, int LPR, int PPL>
__global__ void __launch_bounds__(kAttnThreads)
attention_kernel(const AttnArgs a) {
    const lrqk_layer_t &L = a.L;
    constexpr int N = Pack<T>::N;
    constexpr int RPW = 32 / LPR;
    constexpr int U = 8;
    constexpr int NW = kAttnThreads / 32;
    __shared__ float s_m[NW * RPW], s_l[NW * RPW];
    __shared__ int s_flag;
    extern __shared__ __align__(16) float s_acc[];  // [NW*RPW][d]
    const int bh = blockIdx.y, split = blockIdx.x;
    const int b = bh / L.n_q_heads, h = bh - b * L.n_q_heads;
    const int G = L.n_q_heads / L.n_kv_heads, g = h / G;
    const int d = L.dim_stride;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sub = lane / LPR, sl = lane - sub * LPR;
    trace(30);
    pdl_wait();
    pdl_trigger();
    const int mode = L.sel_meta[(size_t)bh * kMetaInts + M_MODE];
    if (mode == 5) {
        // select_attend_kernel left parts + 1 softmax partials: merge them
        if (split == 0) merge_select_attend_partials(L, bh, a.out);
        else if (a.yg_slots > 0) fold_yg_slots(L, bh, a.yg_slots, split - 1, gridDim.x - 1);
        return;
    }
    if (mode == 6) {
        // score_attend_kernel left P softmax partials: split 0 merges them into
        // the output, the other splits fold its Y|G slots
        if (split == 0) merge_score_attend_partials(L, bh, a.out);
        if (a.yg_slots > 0 && (split > 0 || gridDim.x == 1))
            fold_yg_slots(L, bh, a.yg_slots, gridDim.x == 1 ? 0 : split - 1, gridDim.x == 1 ? 1 : gridDim.x - 1);
        return;
    }
    const int S = L.res_cnt[bh];
    const bool host = L.policy == LRQK_SLOW_HOST;
    const T *kb, *vb;
    if (host) {
        kb = reinterpret_cast<const T *>(L.slot_k) + (size_t)bh * L.n_slots * d;
        vb = reinterpret_cast<const T *>(L.slot_v) + (size_t)bh * L.n_slots * d;
    } else {
        const size_t kv_rows = ((size_t)b * L.n_kv_heads + g) * L.t_max;
        kb = reinterpret_cast<const T *>(L.slow_k) + kv_rows * d;
        vb = reinterpret_cast<const T *>(L.slow_v) + kv_rows * d;
    }
    const int *src = (host ? L.res_slot : L.res_idx) + (size_t)bh * L.s_cap;
    // scale folded into log2 domain: p = 2^(x*c - m), c = log2(e)/sqrt(head_dim)
    const float c = 1.4426950408889634f * rsqrtf((float)L.head_dim);
    float qv[PPL][N];
    {
        const T *qr = reinterpret_cast<const T *>(a.q) + (size_t)bh * d;
#pragma unroll
        for (int pp = 0; pp < PPL; ++pp) Pack<T>::load(qr + (sl + pp * LPR) * N, qv[pp]);
    }
    float m = -INFINITY, l = 0.f;
    float acc[PPL][N];
#pragma unroll
    for (int pp = 0; pp < PPL; ++pp)
#pragma unroll
        for (int e = 0; e < N; ++e) acc[pp][e] = 0.f;
    const int r0 = split * kAttnRows, r1 = min(S, r0 + kAttnRows);
    const int step = NW * RPW;
    // the split's row offsets, staged once (one dependent round trip).  Host
    // policy: rows missed this step (slot | kSlotMiss) are read from the
    // pinned host tier here, zero-copy over PCIe, in the same loads as the
    // hits' HBM slot rows (K5b overlapped with the hits), then stored into
    // their slots; s_tok holds their token index (-1: a hit)
    __shared__ int s_src[kAttnRows];
    __shared__ int s_tok[kAttnRows];
    const T *hk = nullptr, *hv = nullptr;
    if (host) {
        const size_t kv_rows = ((size_t)b * L.n_kv_heads + g) * L.t_max;
        hk = reinterpret_cast<const T *>(L.slow_k) + kv_rows * d;
        hv = reinterpret_cast<const T *>(L.slow_v) + kv_rows * d;
    }
    for (int j = tid; j < r1 - r0; j += blockDim.x) {
        const int sv = src[r0 + j];
        s_src[j] = sv & ~kSlotMiss;
        s_tok[j] = (host && (sv & kSlotMiss)) ? L.res_idx[(size_t)bh * L.s_cap + r0 + j] : -1;
        if (s_tok[j] >= 0) L.res_slot[(size_t)bh * L.s_cap + r0 + j] = sv & ~kSlotMiss;  // fetched below
    }
    __syncthreads();
    // scores of U rows per lane group in flight, K and V kept packed until used
    for (int base = r0 + warp * RPW + sub; base < r1 + sub; base += step * U) {
        uint4 kx[U][PPL], vx[U][PPL];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = base + u * step;
            if (j < r1) {
                const int tok = s_tok[j - r0];
                const T *kr = tok >= 0 ? hk + (size_t)tok * d : kb + (size_t)s_src[j - r0] * d;
                const T *vr = tok >= 0 ? hv + (size_t)tok * d : vb + (size_t)s_src[j - r0] * d;
#pragma unroll
                for (int pp = 0; pp < PPL; ++pp) {
                    kx[u][pp] = *reinterpret_cast<const uint4 *>(kr + (sl + pp * LPR) * N);
                    vx[u][pp] = *reinterpret_cast<const uint4 *>(vr + (sl + pp * LPR) * N);
                }
            } else {
#pragma unroll
                for (int pp = 0; pp < PPL; ++pp) { kx[u][pp] = make_uint4(0, 0, 0, 0); vx[u][pp] = make_uint4(0, 0, 0, 0); }
            }
        }
        if (host) {  // this step's misses -> their fast-tier slots
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = base + u * step;
                if (j < r1 && s_tok[j - r0] >= 0) {
                    const size_t row = (size_t)s_src[j - r0] * d;
#pragma unroll
                    for (int pp = 0; pp < PPL; ++pp) {
                        *reinterpret_cast<uint4 *>(const_cast<T *>(kb) + row + (sl + pp * LPR) * N) = kx[u][pp];
                        *reinterpret_cast<uint4 *>(const_cast<T *>(vb) + row + (sl + pp * LPR) * N) = vx[u][pp];
                    }
                }
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
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = (base + u * step < r1) ? x[u] * c : -INFINITY;
        float mx = m;
#pragma unroll
        for (int u = 0; u < U; ++u) mx = fmaxf(mx, x[u]);
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
    trace(31);
    // per-group partials to shared
    const int gidx = warp * RPW + sub;
    if (sl == 0) { s_m[gidx] = m; s_l[gidx] = l; }
#pragma unroll
    for (int pp = 0; pp < PPL; ++pp)
#pragma unroll
        for (int e = 0; e < N; ++e) s_acc[gidx * d + (sl + pp * LPR) * N + e] = acc[pp][e];
    __syncthreads();
    // merge groups -> split partial
    float *part = L.attn_scratch + ((size_t)bh * a.slots + split) * (size_t)(d + 2);
    float M = -INFINITY;
    for (int i = 0; i < NW * RPW; ++i) M = fmaxf(M, s_m[i]);
    for (int i = tid; i < d; i += blockDim.x) {
        float sacc = 0.f;
        for (int gI = 0; gI < NW * RPW; ++gI)
            if (s_m[gI] != -INFINITY) sacc += s_acc[gI * d + i] * exp2f(s_m[gI] - M);
        part[2 + i] = sacc;
    }
    if (tid == 0) {
        float sl2 = 0.f;
        for (int gI = 0; gI < NW * RPW; ++gI)
            if (s_m[gI] != -INFINITY) sl2 += s_l[gI] * exp2f(s_m[gI] - M);
        part[0] = M;
        part[1] = sl2;
    }
    trace(32);
    if (!last_arrival(L.counters + (size_t)bh * kCounterInts + C_ATTN, gridDim.x, &s_flag)) return;
    trace(33);
    // merge the splits of this head
    __shared__ float s_ms[64], s_w[64];
    __shared__ float s_den;
    const int nsp = gridDim.x;
    const float *parts = L.attn_scratch + (size_t)bh * a.slots * (size_t)(d + 2);
    for (int sp = tid; sp < nsp; sp += blockDim.x) {
        s_ms[sp] = __ldcg(parts + (size_t)sp * (d + 2));
        s_w[sp] = __ldcg(parts + (size_t)sp * (d + 2) + 1);
    }
    __syncthreads();
    if (tid == 0) {
        float MM = -INFINITY;
        for (int sp = 0; sp < nsp; ++sp) MM = fmaxf(MM, s_ms[sp]);
        float den = 0.f;
        for (int sp = 0; sp < nsp; ++sp) {
            const float w = s_ms[sp] != -INFINITY ? exp2f(s_ms[sp] - MM) : 0.f;
            den = fmaf(s_w[sp], w, den);
            s_ms[sp] = w;  // now the split weight
        }
        s_den = den;
    }
    __syncthreads();
    const float inv = 1.f / s_den;
    for (int i = tid; i < d; i += blockDim.x) {
        float o0 = 0.f, o1 = 0.f;
        int sp = 0;
        for (; sp + 1 < nsp; sp += 2) {
            o0 = fmaf(__ldcg(parts + (size_t)sp * (d + 2) + 2 + i), s_ms[sp], o0);
            o1 = fmaf(__ldcg(parts + (size_t)(sp + 1) * (d + 2) + 2 + i), s_ms[sp + 1], o1);
        }
        if (sp < nsp) o0 = fmaf(__ldcg(parts + (size_t)sp * (d + 2) + 2 + i), s_ms[sp], o0);
        a.out[(size_t)bh * d + i] = (o0 + o1) * inv;
    }
    trace(34);
}

int attn_splits(const lrqk_layer_t &L) { return (L.s_cap + kAttnRows - 1) / kAttnRows; }
int score_tma_parts(const lrqk_layer_t &L);
int attn_scratch_slots(const lrqk_layer_t &L) { return max(attn_splits(L), score_tma_parts(L) + 1); }

template <typename T>
static int launch_attention_t(const AttnArgs &a, cudaStream_t st) {
    const lrqk_layer_t &L = a.L;
    constexpr int N = Pack<T>::N;
    const int packs = L.dim_stride / N;
    dim3 grid(attn_splits(L), L.batch * L.n_q_heads);
    const int lpr = packs < 32 ? packs : 32;
    const int ppl = packs / lpr;
    const size_t smem = (size_t)(kAttnThreads / 32) * (32 / lpr) * L.dim_stride * sizeof(float);
#define LRQK_ATTN(LP, PP)                                                                        \
    do {                                                                                         \
        auto fn = attention_kernel<T, LP, PP>;                                                   \
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
        launch_kernel(fn, grid, kAttnThreads, smem, st, true, a);                                \
    } while (0)
    if (ppl == 1) {
        switch (lpr) {
            case 1: LRQK_ATTN(1, 1); break;
            case 2: LRQK_ATTN(2, 1); break;
            case 4: LRQK_ATTN(4, 1); break;
            case 8: LRQK_ATTN(8, 1); break;
            case 16: LRQK_ATTN(16, 1); break;
            case 32: LRQK_ATTN(32, 1); break;
            default: return LRQK_EUNSUPPORTED;
        }
    } else if (ppl == 2 && lpr == 32) {
        LRQK_ATTN(32, 2);
    } else {
        return LRQK_EUNSUPPORTED;
    }
#undef LRQK_ATTN
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

int yg_slots(const lrqk_layer_t &L);
int attn_scratch_slots(const lrqk_layer_t &L);
int launch_attention(const lrqk_layer_t &L, const void *q, float *out, cudaStream_t st) {
    AttnArgs a{L, q, out, L.red_scratch ? yg_slots(L) : 0, attn_scratch_slots(L)};
    return L.dtype == LRQK_BF16 ? launch_attention_t<__nv_bfloat16>(a, st) : launch_attention_t<float>(a, st);
}

// ---------------------------------------------------------------------------
// K5b: missed rows, pinned host -> slots.  One warp copies 16-byte packs of
// several rows at once so that enough PCIe reads are in flight.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
gather_misses_kernel(const lrqk_layer_t L) {
    const int bh = blockIdx.y;
    const int b = bh / L.n_q_heads, h = bh - b * L.n_q_heads;
    const int G = L.n_q_heads / L.n_kv_heads, g = h / G;
    const int n = L.miss_cnt[bh];
    const size_t row_bytes = (size_t)L.dim_stride * (L.dtype == LRQK_BF16 ? 2 : 4);
    const int packs = (int)(row_bytes / 16);
    const size_t kv_rows = ((size_t)b * L.n_kv_heads + g) * L.t_max;
    const uint4 *sk = reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(L.slow_k) + kv_rows * row_bytes);
    const uint4 *sv = reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(L.slow_v) + kv_rows * row_bytes);
    uint4 *dk = reinterpret_cast<uint4 *>(reinterpret_cast<char *>(L.slot_k) + (size_t)bh * L.n_slots * row_bytes);
    uint4 *dv = reinterpret_cast<uint4 *>(reinterpret_cast<char *>(L.slot_v) + (size_t)bh * L.n_slots * row_bytes);
    const int *mi = L.miss_idx + (size_t)bh * L.s_cap;
    const int *ms = L.miss_slot + (size_t)bh * L.s_cap;
    const int total = n * packs;
    if (blockIdx.x == 0)  // the rows are in their slots after this kernel: plain slot indices
        for (int i = threadIdx.x; i < L.res_cnt[bh]; i += blockDim.x)
            L.res_slot[(size_t)bh * L.s_cap + i] &= ~kSlotMiss;
    constexpr int U = 4;
    for (int e0 = blockIdx.x * blockDim.x * U + threadIdx.x; e0 < total; e0 += gridDim.x * blockDim.x * U) {
        uint4 kx[U], vx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < total) {
                const int j = e / packs, p = e - j * packs;
                const size_t off = (size_t)mi[j] * packs + p;
                kx[u] = sk[off];
                vx[u] = sv[off];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < total) {
                const int j = e / packs, p = e - j * packs;
                const size_t off = (size_t)ms[j] * packs + p;
                dk[off] = kx[u];
                dv[off] = vx[u];
            }
        }
    }
}

int launch_gather(const lrqk_layer_t &L, cudaStream_t st) {
    if (L.policy != LRQK_SLOW_HOST) return LRQK_OK;
    const int row_bytes = L.dim_stride * (L.dtype == LRQK_BF16 ? 2 : 4);
    const int per_head = L.s_cap * (row_bytes / 16);
    const int gx = max(1, min(16, (per_head + 1023) / 1024));
    gather_misses_kernel<<<dim3(gx, L.batch * L.n_q_heads), 256, 0, st>>>(L);
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

// ---------------------------------------------------------------------------
// prompt seeding: fast tier = last lite_budget prompt rows (cache.py:114-124)
// ---------------------------------------------------------------------------
__global__ void seed_kernel(const lrqk_layer_t L, int prompt_len) {
    const int bh = blockIdx.x;
    const int b = bh / L.n_q_heads, h = bh - b * L.n_q_heads;
    const int G = L.n_q_heads / L.n_kv_heads, g = h / G;
    const int lo = max(0, prompt_len - L.lite_budget);
    const int n = prompt_len - lo;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        L.res_idx[(size_t)bh * L.s_cap + i] = lo + i;
        if (L.policy == LRQK_SLOW_HOST) L.res_slot[(size_t)bh * L.s_cap + i] = i;
    }
    if (threadIdx.x == 0) {
        L.res_cnt[bh] = n;
        L.c_miss[bh] = 0;
        L.c_total[bh] = 0;
        L.step_miss[bh] = 0;
        L.step_total[bh] = 0;
        if (L.policy == LRQK_SLOW_HOST) L.spare_slot[bh] = n;
        if (h == 0) L.ctx_len[b] = prompt_len;
    }
    for (int i = threadIdx.x; i < kHistLevels * kHistBins; i += blockDim.x)
        L.hist[(size_t)bh * kHistLevels * kHistBins + i] = 0u;
    for (int i = threadIdx.x; i < kMetaInts; i += blockDim.x)
        L.sel_meta[(size_t)bh * kMetaInts + i] = i == M_BITS_FRESH ? 1 : 0;
    if (L.res_bits) {  // residency bitmap = the prompt's lite rows
        uint32_t *bits = L.res_bits + (size_t)bh * ((L.t_max + 31) / 32);
        for (int w = threadIdx.x; w < (L.t_max + 31) / 32; w += blockDim.x) {
            uint32_t v = 0u;
            for (int j = 0; j < 32; ++j) {
                const int x = w * 32 + j;
                if (x >= lo && x < prompt_len) v |= 1u << j;
            }
            bits[w] = v;
        }
    }
    for (int i = threadIdx.x; i < kCounterInts; i += blockDim.x) L.counters[(size_t)bh * kCounterInts + i] = 0;
    if (L.policy == LRQK_SLOW_HOST) {
        const size_t row_bytes = (size_t)L.dim_stride * (L.dtype == LRQK_BF16 ? 2 : 4);
        const int packs = (int)(row_bytes / 16);
        const size_t kv_rows = ((size_t)b * L.n_kv_heads + g) * L.t_max;
        const uint4 *sk = reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(L.slow_k) + kv_rows * row_bytes);
        const uint4 *sv = reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(L.slow_v) + kv_rows * row_bytes);
        uint4 *dk = reinterpret_cast<uint4 *>(reinterpret_cast<char *>(L.slot_k) + (size_t)bh * L.n_slots * row_bytes);
        uint4 *dv = reinterpret_cast<uint4 *>(reinterpret_cast<char *>(L.slot_v) + (size_t)bh * L.n_slots * row_bytes);
        for (int e = threadIdx.x; e < n * packs; e += blockDim.x) {
            const int j = e / packs, p = e - j * packs;
            dk[(size_t)j * packs + p] = sk[(size_t)(lo + j) * packs + p];
            dv[(size_t)j * packs + p] = sv[(size_t)(lo + j) * packs + p];
        }
    }
}

int launch_seed(const lrqk_layer_t &L, int prompt_len, cudaStream_t st) {
    seed_kernel<<<L.batch * L.n_q_heads, 256, 0, st>>>(L, prompt_len);
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

__global__ void advance_kernel(int32_t *ctx_len, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) ctx_len[i] += 1;
}
int launch_advance(int32_t *ctx_len, int n, cudaStream_t st) {
    advance_kernel<<<(n + 255) / 256, 256, 0, st>>>(ctx_len, n);
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

// standalone proxy scores (float out) for the drop-in proxy_scores()
template <typename T>
__global__ void proxy_scores_kernel(const T *store, const float *qh, float *out, int n_heads, int n_rows, int R) {
    const int h = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rows) return;
    const T *row = store + ((size_t)h * n_rows + i) * R;
    const float *q = qh + (size_t)h * R;
    float s = 0.f;
    for (int p = 0; p < R; ++p) s = fmaf(to_float<T>(row[p]), q[p], s);
    out[(size_t)h * n_rows + i] = s;
}
int launch_proxy_scores(const void *store, int dtype, const float *qh, float *out, int n_heads, int n_rows, int R,
                        cudaStream_t st) {
    dim3 grid((n_rows + 255) / 256, n_heads);
    if (dtype == LRQK_BF16)
        proxy_scores_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16 *>(store), qh,
                                                                 out, n_heads, n_rows, R);
    else
        proxy_scores_kernel<float><<<grid, 256, 0, st>>>(reinterpret_cast<const float *>(store), qh, out, n_heads,
                                                         n_rows, R);
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

__global__ void fill_int_kernel(int32_t *p, int n, int v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
int launch_fill_int(int32_t *p, int n, int v, cudaStream_t st) {
    if (n <= 0) return LRQK_OK;
    fill_int_kernel<<<(n + 255) / 256, 256, 0, st>>>(p, n, v);
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

}  // namespace lrqk

namespace lrqk {
// ---------------------------------------------------------------------------
// Standalone exact attention over explicit rows (drop-in exact_attention,
// attention.py:23-34): one block per head, logits -> max -> exp -> weights
// -> output.  Rows are fp32 [H][n][ld]; outputs [H][ld] and weights [H][n].
// ---------------------------------------------------------------------------
__global__ void attention_rows_kernel(const float *q, const float *K, const float *V, int n, int d, int ld,
                                      float scale, float *out, float *weights) {
    extern __shared__ float w[];  // [n]
    __shared__ float red[32];
    const int h = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const float *qh = q + (size_t)h * ld;
    const float *Kh = K + (size_t)h * n * ld;
    const float *Vh = V + (size_t)h * n * ld;
    // logits, one warp per row
    for (int j = warp; j < n; j += nw) {
        float acc = 0.f;
        for (int i = lane; i < d; i += 32) acc = fmaf(qh[i], Kh[(size_t)j * ld + i], acc);
        acc = warp_sum(acc);
        if (lane == 0) w[j] = acc * scale;
    }
    __syncthreads();
    float m = -INFINITY;
    for (int j = tid; j < n; j += blockDim.x) m = fmaxf(m, w[j]);
    m = warp_max(m);
    if (lane == 0) red[warp] = m;
    __syncthreads();
    if (tid < 32) {
        float v = tid < nw ? red[tid] : -INFINITY;
        v = warp_max(v);
        if (tid == 0) red[0] = v;
    }
    __syncthreads();
    m = red[0];
    __syncthreads();
    float sacc = 0.f;
    for (int j = tid; j < n; j += blockDim.x) {
        const float e = expf(w[j] - m);
        w[j] = e;
        sacc += e;
    }
    sacc = warp_sum(sacc);
    if (lane == 0) red[warp] = sacc;
    __syncthreads();
    if (tid < 32) {
        float v = tid < nw ? red[tid] : 0.f;
        v = warp_sum(v);
        if (tid == 0) red[0] = v;
    }
    __syncthreads();
    const float inv = 1.f / red[0];
    for (int j = tid; j < n; j += blockDim.x) {
        w[j] *= inv;
        if (weights) weights[(size_t)h * n + j] = w[j];
    }
    __syncthreads();
    for (int i = tid; i < d; i += blockDim.x) {
        float o = 0.f;
        for (int j = 0; j < n; ++j) o = fmaf(w[j], Vh[(size_t)j * ld + i], o);
        out[(size_t)h * ld + i] = o;
    }
}

int launch_attention_rows(const float *q, const float *K, const float *V, int H, int n, int d, int ld, float *out,
                          float *weights, cudaStream_t st) {
    const size_t smem = (size_t)n * sizeof(float);
    if (smem > 200 * 1024) return LRQK_EUNSUPPORTED;
    cudaFuncSetAttribute(attention_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attention_rows_kernel<<<H, 256, smem, st>>>(q, K, V, n, d, ld, rsqrtf((float)d), out, weights);
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

// ---------------------------------------------------------------------------
// Hit/miss accounting for an explicit selection (drop-in fetch_and_merge,
// cache.py:174-196): resident (ascending, n_res) vs omega (n_sel, any order,
// unique); outputs [miss, selected, out_of_range].  One block.
// ---------------------------------------------------------------------------
__global__ void count_misses_kernel(const int32_t *resident, int n_res, const int32_t *omega, int n_sel, int size,
                                    int32_t *out) {
    __shared__ int s_miss, s_bad;
    if (threadIdx.x == 0) { s_miss = 0; s_bad = 0; }
    __syncthreads();
    int miss = 0, bad = 0;
    for (int i = threadIdx.x; i < n_sel; i += blockDim.x) {
        const int x = omega[i];
        if (x < 0 || x >= size) bad = 1;
        int lo = 0, hi = n_res - 1, found = 0;
        while (lo <= hi) {
            const int mid = (lo + hi) >> 1;
            const int v = resident[mid];
            if (v == x) { found = 1; break; }
            if (v < x) lo = mid + 1; else hi = mid - 1;
        }
        miss += found ? 0 : 1;
    }
    atomicAdd(&s_miss, miss);
    if (bad) atomicOr(&s_bad, 1);
    __syncthreads();
    if (threadIdx.x == 0) { out[0] = s_miss; out[1] = n_sel; out[2] = s_bad; }
}

int launch_count_misses(const int32_t *resident, int n_res, const int32_t *omega, int n_sel, int size, int32_t *out,
                        cudaStream_t st) {
    count_misses_kernel<<<1, 256, 0, st>>>(resident, n_res, omega, n_sel, size, out);
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}
}  // namespace lrqk

namespace lrqk {
// ---------------------------------------------------------------------------
// Standalone exact line-search step on one B factor (drop-in
// update_projections, decode.py:150-184): per head h,
//   resid = x_hat B - x, grad = x_hat^T resid, s = x_hat grad,
//   eta = (resid.s)/(s.s) (0 when s.s <= 1e-14 (1 + |resid.s|)),
//   B_out = B - eta grad.   Shapes: x_hat [H][r], B [H][r][d], x [H][d].
// ---------------------------------------------------------------------------
__global__ void line_search_kernel(const float *xh, const float *B, const float *x, int r, int d, float *B_out,
                                   float *grad, float *eta_out) {
    extern __shared__ float sm[];
    float *res = sm;        // [d]
    float *sx = res + d;    // [r]
    __shared__ double s_nd[2][32];
    const int h = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const float *Bh = B + (size_t)h * r * d;
    for (int p = tid; p < r; p += blockDim.x) sx[p] = xh[(size_t)h * r + p];
    __syncthreads();
    float nx = 0.f;
    for (int p = 0; p < r; ++p) nx = fmaf(sx[p], sx[p], nx);
    double num = 0.0, den = 0.0;
    for (int i = tid; i < d; i += blockDim.x) {
        float acc = 0.f;
        for (int p = 0; p < r; ++p) acc = fmaf(sx[p], Bh[(size_t)p * d + i], acc);
        const float rr = acc - x[(size_t)h * d + i];
        res[i] = rr;
        const double s = (double)nx * rr;
        num += (double)rr * s;
        den += s * s;
    }
    for (int o = 16; o > 0; o >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, o);
        den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    if (lane == 0) { s_nd[0][warp] = num; s_nd[1][warp] = den; }
    __syncthreads();
    double tn = 0.0, td = 0.0;
    for (int w = 0; w < nw; ++w) { tn += s_nd[0][w]; td += s_nd[1][w]; }
    const float eta = (td <= 1e-14 * (1.0 + fabs(tn))) ? 0.f : (float)(tn / td);
    if (tid == 0) eta_out[h] = eta;
    for (int e = tid; e < r * d; e += blockDim.x) {
        const int p = e / d, i = e - p * d;
        const float g = sx[p] * res[i];
        if (grad) grad[(size_t)h * r * d + e] = g;
        B_out[(size_t)h * r * d + e] = Bh[e] - eta * g;
    }
}

int launch_line_search(const float *xh, const float *B, const float *x, int H, int r, int d, float *B_out,
                       float *grad, float *eta, cudaStream_t st) {
    line_search_kernel<<<H, 256, (size_t)(d + r) * sizeof(float), st>>>(xh, B, x, r, d, B_out, grad, eta);
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}
}  // namespace lrqk
