// K4 + K6 fused (selection mode 5, HBM policy): top-k selection straight
// from the score keys and exact softmax attention over the winners, in one
// kernel.  ref: cache.py:149-171 (select_active), linalg.py:96-110
// (topk_indices), attention.py:23-34 (exact_attention), session.py:99-102.
//
// The score kernel (select.cu) has already found, from an exact histogram of
// the keys around the previous step's threshold, the bin D that holds the
// k-th largest key, and for every part p of the head the number of certain
// winners (keys in bins above D) in the parts before it (fcnt).  So each
// block of this kernel owns one part, and in a single pass over its keys it
//   - writes its certain winners, ascending, to res_idx[fcnt[p] + rank],
//   - collects the rows of bin D (a handful) for the last block,
//   - gathers the winners' K/V rows and accumulates an online-softmax
//     partial (max, sum, acc) for its rows.
// The last block of the head ranks bin D (ties -> lower index, as the
// reference), appends those winners and Omega_l = the lite window, adds
// their rows to the softmax, merges the parts' partials and writes the
// output.  Omega_k is stored as [certain winners ascending] ++ [bin-D
// winners ascending]; attention and compression are sums over the set, and
// the host views sort it.  Hit/miss counts are done off the critical path by
// compress_prepare (compress.cu: count_hits_hbm).
#include "common.cuh"
#include "select_common.cuh"
#include "mma_common.cuh"
#include "attend_common.cuh"

namespace lrqk {

int score_tma_parts(const lrqk_layer_t &L);
int yg_slots(const lrqk_layer_t &L);

constexpr int kFThreads = 256;
constexpr int kFRows = kFThreads * 32;  // keys per scan pass: 32 contiguous keys per thread
constexpr int kFList = kCritCap + 64;   // last block: bin-D winners + lite rows

struct FArgs {
    lrqk_layer_t L;
    const void *q;
    float *out;
    int parts;
    int yg_slots;
};

template <typename T, int LPR, int PPL, int YGM>
__global__ void __launch_bounds__(kFThreads, 2)
select_attend_kernel(const FArgs a) {
    const lrqk_layer_t &L = a.L;
    constexpr int N = Pack<T>::N;
    extern __shared__ __align__(128) uint8_t f_smem[];
    int *s_rows = reinterpret_cast<int *>(f_smem);                     // [s_cap] this part's rows / winners
    uint8_t *stage = f_smem + (((size_t)L.s_cap * 4 + 127) & ~(size_t)127);  // K/V/A chunks; later scratch
    __shared__ float s_m[kFThreads / 32], s_l[kFThreads / 32];
    __shared__ int s_scan[32];
    __shared__ int s_flag;
    __shared__ int s_ncrit, s_cbase;
    __shared__ uint64_t s_crit[kFCrit];
    const int P = a.parts;
    const int bh = blockIdx.x / P, part = blockIdx.x - bh * P;
    const int b = bh / L.n_q_heads, h = bh - b * L.n_q_heads;
    const int G = L.n_q_heads / L.n_kv_heads, g = h / G;
    const int d = L.dim_stride, R = L.rank_stride;
    const int tid = threadIdx.x, lane = tid & 31;
    const int sub = lane / LPR, sl = lane - sub * LPR;
    trace(50);
    pdl_wait();
    pdl_trigger();
    const int t = L.ctx_len[b];
    int *meta = L.sel_meta + (size_t)bh * kMetaInts;
    // prefetch this part's candidate-mask words (the score kernel's
    // partition) and the query row together with the meta loads
    const int lite_start = max(0, t + 1 - L.lite_budget);
    const int tpp = (((t + 1 + 31) >> 5) + P - 1) / P;
    const int row0 = min(lite_start, part * tpp * 32), row1 = min(lite_start, (part + 1) * tpp * 32);
    const uint32_t *keys = L.keys + (size_t)bh * L.t_max;
    const int w0 = row0 >> 5, w1 = (row1 + 31) >> 5, nwrd = w1 - w0;
    const int wpt = (nwrd + blockDim.x - 1) / blockDim.x;  // contiguous mask words per thread
    uint32_t wv[4];
    {
        const uint32_t *cmw = L.cmask + (size_t)bh * ((L.t_max + 31) >> 5) + w0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int wi = tid * wpt + u;
            wv[u] = (u < wpt && wi < nwrd) ? __ldcg(cmw + wi) : 0u;
        }
    }
    float qv[PPL][N];
    {
        const T *qr = reinterpret_cast<const T *>(a.q) + (size_t)bh * d;
#pragma unroll
        for (int pp = 0; pp < PPL; ++pp) Pack<T>::load(qr + (sl + pp * LPR) * N, qv[pp]);
    }
    const int mode = meta[M_MODE];
    if (t >= L.t_max || mode != 5) return;  // other heads: select_kernel + attention_kernel
    const uint32_t klo = (uint32_t)meta[M_KLO];
    const int D = meta[M_FBIN];
    const int k_eff = meta[M_K_EFF];
    const int nabove = meta[M_NABOVE];
    int out = __ldcg(L.fcnt + (size_t)bh * P + part);
    int *dst = L.res_idx + (size_t)bh * L.s_cap;
    uint64_t *cand = L.cand + (size_t)bh * L.cand_cap;
    const size_t kv_rows = ((size_t)b * L.n_kv_heads + g) * L.t_max;
    const T *kb = reinterpret_cast<const T *>(L.slow_k) + kv_rows * d;
    const T *vb = reinterpret_cast<const T *>(L.slow_v) + kv_rows * d;
    const T *proxy = reinterpret_cast<const T *>(L.proxy) + (size_t)bh * L.t_max * R;
    const T *arows = L.proxy_rowmajor ? reinterpret_cast<const T *>(L.proxy_rowmajor) + (size_t)bh * L.t_max * R
                                      : nullptr;
    const float c = 1.4426950408889634f * rsqrtf((float)L.head_dim);  // log2(e) / sqrt(d)
    const size_t PF = yg_part_floats(R, d);
    float *yg = L.red_scratch + (size_t)bh * a.yg_slots * PF;
    float m = -INFINITY, l = 0.f;
    float acc[PPL][N];
#pragma unroll
    for (int pp = 0; pp < PPL; ++pp)
#pragma unroll
        for (int e = 0; e < N; ++e) acc[pp][e] = 0.f;
    constexpr bool YG = YGM > 0;
    constexpr int MT = YGM > 0 ? YGM : 1;
    float yacc[MT][2][4], gacc[4][4];
#pragma unroll
    for (int i = 0; i < MT * 8; ++i) yacc[i / 8][(i / 4) & 1][i & 3] = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) gacc[i / 4][i & 3] = 0.f;
    trace(51);

    // ---- this part's winners: ordered write, then attention (+ Y, G) -------
    int nloc = 0;
    if (tid == 0) s_ncrit = 0;
    __syncthreads();
    // Shortlist path: when this step's threshold bin lies above the score
    // kernel's candidate bound, only the rows marked in cmask can win; read
    // their keys instead of the part's whole key range.
    const uint32_t kc = (uint32_t)meta[M_KC];
    bool shortlist = kc != 0xFFFFFFFFu && klo + ((uint32_t)D << kWinShift) >= kc && wpt <= 4;
    if (shortlist) {
        int cnt = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) cnt += __popc(wv[u]);
        int *s_c = reinterpret_cast<int *>(stage) + tid * 16;  // this thread's candidates
        int wu = 0;
        uint32_t rem = wv[0];
        // one round of <= 16 candidates per thread keeps the output order
        // (thread, bit); denser shortlists take the full key scan below
        shortlist = !__syncthreads_or(cnt > 16);
        trace(46);
        if (shortlist) {
            int nc = 0;
            while (nc < 16 && wu < 4) {  // next candidates, ascending
                if (rem == 0u) { if (++wu < 4) rem = wv[wu]; continue; }
                const int bpos = __ffs(rem) - 1;
                rem &= rem - 1u;
                s_c[nc++] = (w0 + tid * wpt + wu) * 32 + bpos;
            }
            trace(47);
            uint32_t kk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) kk[j] = j < nc ? __ldcg(keys + s_c[j]) : 0u;
            uint32_t wmask = 0;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (j >= nc || kk[j] < klo) continue;
                const uint32_t dk = kk[j] - klo;
                if (dk >= kWinKeys || (int)(dk >> kWinShift) > D) {
                    wmask |= 1u << j;
                } else if ((int)(dk >> kWinShift) == D) {
                    const int q = atomicAdd(&s_ncrit, 1);
                    if (q < kFCrit) s_crit[q] = make_comp(kk[j], s_c[j]);
                }
            }
            trace(48);
            int tot;
            int o = nloc + block_exclusive_scan(__popc(wmask), s_scan, &tot);
            trace(49);
            while (wmask) {
                const int j = __ffs(wmask) - 1;
                wmask &= wmask - 1u;
                const int x = s_c[j];
                if (o < L.s_cap) s_rows[o] = x;
                if (out + o < k_eff) dst[out + o] = x;
                ++o;
            }
            nloc += tot;
        }
    }
    for (int base = row0; base < row1 && !shortlist; base += kFRows) {
        uint4 kv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = base + tid * 32 + u * 4;
            kv[u] = i < row1 ? *reinterpret_cast<const uint4 *>(keys + i) : make_uint4(0, 0, 0, 0);
        }
        uint32_t smask = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t kk[4] = {kv[u].x, kv[u].y, kv[u].z, kv[u].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = base + tid * 32 + u * 4 + e;
                if (i < row1 && kk[e] >= klo) {
                    const uint32_t dk = kk[e] - klo;
                    if (dk >= kWinKeys || (int)(dk >> kWinShift) > D) {
                        smask |= 1u << (u * 4 + e);
                    } else if ((int)(dk >> kWinShift) == D) {  // threshold bin: block list first
                        const int q = atomicAdd(&s_ncrit, 1);
                        if (q < kFCrit) s_crit[q] = make_comp(kk[e], i);
                    }
                }
            }
        }
        int tot;
        int o = nloc + block_exclusive_scan(__popc(smask), s_scan, &tot);
        while (smask) {  // thread-contiguous keys: ascending order is (thread, bit)
            const int bpos = __ffs(smask) - 1;
            smask &= smask - 1u;
            const int x = base + tid * 32 + bpos;
            if (o < L.s_cap) s_rows[o] = x;
            if (out + o < k_eff) dst[out + o] = x;
            ++o;
        }
        nloc += tot;
    }
    trace(44);
    {   // this part's threshold-bin rows -> the head's list (one reservation)
        __syncthreads();
        const int nc = s_ncrit;
        if (tid == 0) s_cbase = nc ? atomicAdd(meta + M_CAND, min(nc, kFCrit)) : 0;
        __syncthreads();
        for (int j = tid; j < min(nc, kFCrit); j += blockDim.x)
            if (s_cbase + j < L.cand_cap) cand[s_cbase + j] = s_crit[j];
    }
    trace(45);
    const int nl = t + 1 - lite_start;
    if (part == P - 1) {  // Omega_l = the lite window, attended by the last part
        for (int i = tid; i < nl; i += blockDim.x) {
            dst[k_eff + i] = lite_start + i;
            if (nloc + i < L.s_cap) s_rows[nloc + i] = lite_start + i;
        }
        nloc += nl;
    }
    __syncthreads();
    trace(56);
    attend_reduce_list<T, LPR, PPL, YGM>(L, kb, vb, proxy, arows, s_rows, min(nloc, L.s_cap), qv, c, m, l, acc, stage, yacc,
                                        gacc);
    trace(52);
    if constexpr (YG) mma_write_partial<MT, 2>(yacc, gacc, R, d, yg + (size_t)part * PF);
    trace(57);
    float *s_acc = reinterpret_cast<float *>(stage);  // [nwarps][d]
    float *part_dst = L.attn_scratch + ((size_t)bh * attn_slots_dev(L, P) + part) * (size_t)(d + 2);
    block_partial<T, LPR, PPL>(m, l, acc, d, s_m, s_l, s_acc, part_dst);
    if (!last_arrival(L.counters + (size_t)bh * kCounterInts + C_FUSED, P, &s_flag)) return;
    trace(53);

    // ---- last block: rank bin D, merge -------------------------------------
    const int need2 = k_eff - nabove;
    const int n_crit = __ldcg(meta + M_CAND);
    const int lane_ = tid & 31, warp_ = tid >> 5;
    const bool ok = need2 >= 0 && need2 <= n_crit && n_crit <= L.cand_cap && n_crit <= kCritCap;
    int *s_list = s_rows;  // the winners of bin D
    uint32_t hint = klo + ((uint32_t)(D + 1) << kWinShift);
    int nwin = 0;
    if (!ok) {
        if (tid == 0) set_status(L.status, LRQK_ST_INDEX_RANGE);  // inconsistent selection state (never expected)
    } else if (n_crit <= 32) {
        // one warp: bitonic sort of the composites (descending), then of the
        // winners' indices (ascending), through shuffles
        if (warp_ == 0) {
            uint64_t v = lane_ < n_crit ? __ldcg(cand + lane_) : 0ull;
#pragma unroll
            for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
                for (int j = kk >> 1; j > 0; j >>= 1) {
                    const uint64_t o = __shfl_xor_sync(0xffffffffu, v, j);
                    const bool hi = ((lane_ & kk) == 0) == ((lane_ & j) == 0);  // keep the larger one
                    v = hi ? (v > o ? v : o) : (v < o ? v : o);
                }
            const uint64_t last = __shfl_sync(0xffffffffu, v, max(need2 - 1, 0));
            if (need2 > 0) hint = (uint32_t)(last >> kIdxBits);
            uint32_t ix = lane_ < need2 ? (uint32_t)comp_index(v) : 0xFFFFFFFFu;
#pragma unroll
            for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
                for (int j = kk >> 1; j > 0; j >>= 1) {
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, ix, j);
                    const bool lo = ((lane_ & kk) == 0) == ((lane_ & j) == 0);  // keep the smaller one
                    ix = lo ? min(ix, o) : max(ix, o);
                }
            if (lane_ < need2) {
                dst[nabove + lane_] = (int)ix;
                s_list[lane_] = (int)ix;
            }
        }
        nwin = need2;
    } else {
        int M = 1;
        while (M < n_crit) M <<= 1;
        uint64_t *crit = reinterpret_cast<uint64_t *>(stage);
        for (int i = tid; i < M; i += blockDim.x) crit[i] = i < n_crit ? __ldcg(cand + i) : 0ull;
        __syncthreads();
        block_bitonic(crit, M, true);  // descending composites: ties -> lower index first
        if (need2 > 0) hint = (uint32_t)(crit[need2 - 1] >> kIdxBits);
        int M2 = 1;
        while (M2 < need2) M2 <<= 1;
        for (int i = tid; i < M2; i += blockDim.x) crit[i] = i < need2 ? (uint64_t)comp_index(crit[i]) : ~0ull;
        __syncthreads();
        block_bitonic(crit, M2, false);  // winners by ascending index
        for (int i = tid; i < need2; i += blockDim.x) {
            dst[nabove + i] = (int)crit[i];
            s_list[i] = (int)crit[i];
        }
        nwin = need2;
    }
    __syncthreads();
    trace(55);
#pragma unroll
    for (int pp = 0; pp < PPL; ++pp)
#pragma unroll
        for (int e = 0; e < N; ++e) acc[pp][e] = 0.f;
    m = -INFINITY;
    l = 0.f;
#pragma unroll
    for (int i = 0; i < MT * 8; ++i) yacc[i / 8][(i / 4) & 1][i & 3] = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) gacc[i / 4][i & 3] = 0.f;
    if (nwin > kMmaRows) {
        attend_reduce_list<T, LPR, PPL, YGM>(L, kb, vb, proxy, arows, s_list, nwin, qv, c, m, l, acc, stage, yacc, gacc);
        if constexpr (YG) mma_write_partial<MT, 2>(yacc, gacc, R, d, yg + (size_t)P * PF);
    } else {
        // a handful of rows: attention from registers; Y, G on the CUDA cores
        attend_list<T, LPR, PPL, 1>(kb, vb, s_list, nwin, qv, c, d, m, l, acc);  // compact code: few rows
        // their Y, G contributions are added by the finish kernel (M_YG_ADD)
    }
    // this block's partial goes to slot P; attention_kernel merges the P + 1
    block_partial<T, LPR, PPL>(m, l, acc, d, s_m, s_l, s_acc,
                               L.attn_scratch + ((size_t)bh * attn_slots_dev(L, P) + P) * (size_t)(d + 2));
    trace(58);
    trace(60);
    if (tid == 0) {
        L.res_cnt[bh] = k_eff + (t + 1 - lite_start);
        meta[M_CAND] = 0;
        meta[M_HINT] = (int)hint;
        meta[M_HINT_OK] = 1;
        meta[M_HINT_QN] = __float_as_int(qhat_norm(L, bh));
        // Y|G slots: the P parts (+ the large-bin path's slot P); the few
        // bin-D winners of the common path are added by the finish kernel
        meta[M_YG] = YG ? (nwin > kMmaRows ? P + 1 : P) : 0;
        meta[M_YG_ADD] = YG && nwin <= kMmaRows ? nwin : 0;
        meta[M_ATT_PARTS] = P + 1;
        meta[M_STAT + 5] += 1;
    }
    uint32_t *ghist = L.hist + (size_t)bh * kHistLevels * kHistBins;  // ready for the next step
    for (int i = tid; i < kHistLevels * kHistBins; i += blockDim.x) ghist[i] = 0u;
    trace(54);
}

template <typename T>
static int launch_select_attend_t(const FArgs &a, cudaStream_t st) {
    const lrqk_layer_t &L = a.L;
    constexpr int N = Pack<T>::N;
    const int packs = L.dim_stride / N;
    const int lpr = packs < 32 ? packs : 32;
    const int ppl = packs / lpr;
    // the Y|G reduction rides along for the bf16 rank-16/32/64, d-128 layouts
    const bool yg = sizeof(T) == 2 && (L.rank_stride == 16 || L.rank_stride == 32 || L.rank_stride == 64) &&
                    L.dim_stride == 128;
    const size_t ldk = (size_t)L.dim_stride * sizeof(T) + 16, lda = (size_t)L.rank_stride * 2 + 16;
    const size_t stage = 2 * (2 * kMmaRows * ldk + (yg ? kMmaRows * lda : 0));
    const size_t last = (size_t)kCritCap * 8 > stage ? (size_t)kCritCap * 8 : stage;  // crit sort reuses it
    const size_t tail = ((size_t)(kFThreads / 32) * L.dim_stride + L.dim_stride + 2 + 2 * (size_t)a.parts) * 4;
    const size_t smem = (((size_t)L.s_cap * 4 + 127) & ~(size_t)127) + (last > tail ? last : tail);
    const int grid = L.batch * L.n_q_heads * a.parts;
#define LRQK_F(LP, PP, YG)                                                                        \
    do {                                                                                          \
        auto fn = select_attend_kernel<T, LP, PP, YG>;                                            \
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
        launch_kernel(fn, grid, kFThreads, smem, st, true, a);                                    \
    } while (0)
    if (yg && ppl == 1 && lpr == 16) {
        if constexpr (sizeof(T) == 2) {
            if (L.rank_stride == 64) LRQK_F(16, 1, 4);
            else if (L.rank_stride == 32) LRQK_F(16, 1, 2);
            else LRQK_F(16, 1, 1);
        }
    } else if (ppl == 1) {
        switch (lpr) {
            case 1: LRQK_F(1, 1, 0); break;
            case 2: LRQK_F(2, 1, 0); break;
            case 4: LRQK_F(4, 1, 0); break;
            case 8: LRQK_F(8, 1, 0); break;
            case 16: LRQK_F(16, 1, 0); break;
            case 32: LRQK_F(32, 1, 0); break;
            default: return LRQK_EUNSUPPORTED;
        }
    } else if (ppl == 2 && lpr == 32) {
        LRQK_F(32, 2, 0);
    } else {
        return LRQK_EUNSUPPORTED;
    }
#undef LRQK_F
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

int launch_select_attend(const lrqk_layer_t &L, const void *q, float *out, cudaStream_t st) {
    if (L.policy != LRQK_SLOW_HBM) return LRQK_OK;  // mode 5 is HBM-only
    FArgs a{L, q, out, score_tma_parts(L), yg_slots(L)};
    return L.dtype == LRQK_BF16 ? launch_select_attend_t<__nv_bfloat16>(a, st) : launch_select_attend_t<float>(a, st);
}

}  // namespace lrqk
