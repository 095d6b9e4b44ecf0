// K3: proxy scores fused with the radix histogram (cache.py:141-146)
// K4: top-k + lite-window selection (cache.py:149-171, linalg.py:96-110)
// K5: hit/miss accounting and slot replacement (cache.py:174-196, 63-74)
//
// Selection is exact, including the reference's tie rule: the k largest
// scores win, equal scores prefer the lower index, the result is ascending.
// Scores become order-preserving uint32 keys (-0.0 == +0.0).  The top-k among
// [0, lite_start) is found by a radix select on the 53-bit composite
//     comp = key(32) || (2^21 - 1 - index)(21)
// which is unique per token and orders exactly like (score desc, index asc).
//   pass 1 (fused into the score kernel): histogram of the top 11 key bits;
//   pass 2 (select_scan): tokens above the threshold bin are certain winners,
//           tokens inside it become candidates (key, index);
//   pass 3 (select_finalize, one block per head): exact radix select of the
//           remaining winners among the candidates, ascending compaction via
//           a shared-memory bitmap, then the cache update.
// Degenerate score distributions (threshold bin larger than cand_cap) take an
// exact fallback that radix-selects over the full key array.
#include "common.cuh"

namespace lrqk {

constexpr int kScoreThreads = 256;
constexpr int kScoreChunk = 4096;   // rows per score work item
constexpr int kScanChunk = 8192;    // keys per select_scan work item
constexpr int kFinThreads = 1024;
constexpr int kIdxBits = 21;        // tokens per head < 2^21
constexpr uint32_t kIdxMax = (1u << kIdxBits) - 1u;

LRQK_DEV uint64_t make_comp(uint32_t key, int idx) {
    return ((uint64_t)key << kIdxBits) | (uint64_t)(kIdxMax - (uint32_t)idx);
}
LRQK_DEV int comp_index(uint64_t c) { return (int)(kIdxMax - (uint32_t)(c & kIdxMax)); }

struct ScoreArgs {
    lrqk_layer_t L;
    const float *ext_scores;  // standalone path: precomputed float scores [BH, t+1]
};

// Find D in [0, nbins) with  above(D) < m <= above(D) + hist[D], scanning bins
// from the top.  Whole block participates.  Results in s_out[0]=D, s_out[1]=above.
__device__ void find_crossing(const int *hist, int nbins, int m, int *s_scan, int *s_out) {
    const int nt = blockDim.x;
    const int per = (nbins + nt - 1) / nt;
    const int hi = nbins - 1 - threadIdx.x * per;  // my bins: hi, hi-1, ..., hi-per+1
    int local = 0;
    for (int i = 0; i < per; ++i) {
        const int bin = hi - i;
        if (bin >= 0) local += hist[bin];
    }
    int total;
    int above = block_exclusive_scan(local, s_scan, &total);
    if (above < m && m <= above + local) {
        int acc = above;
        for (int i = 0; i < per; ++i) {
            const int bin = hi - i;
            if (bin < 0) break;
            if (acc + hist[bin] >= m) {
                s_out[0] = bin;
                s_out[1] = acc;
                break;
            }
            acc += hist[bin];
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// K3: score kernel.  TPR = lanes per proxy row (rank_stride*sizeof(T)/16).
// ---------------------------------------------------------------------------
template <typename T, int TPR>
__global__ void __launch_bounds__(kScoreThreads)
score_kernel(const ScoreArgs a) {
    const lrqk_layer_t &L = a.L;
    constexpr int N = Pack<T>::N;
    constexpr int RPW = 32 / TPR;                       // rows per warp step
    constexpr int U = 8;                                // steps in flight
    __shared__ int s_hist[kHistBins];
    __shared__ int s_scan[32];
    __shared__ int s_flag;
    __shared__ int s_out[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int BH = L.batch * L.n_q_heads;
    const int R = L.rank_stride;
    const int nch_max = (L.t_max + kScoreChunk - 1) / kScoreChunk;
    const int sub = lane / TPR, sl = lane - sub * TPR;

    for (int item = blockIdx.x; item < BH * nch_max; item += gridDim.x) {
        const int bh = item / nch_max, ch = item - bh * nch_max;
        const int b = bh / L.n_q_heads;
        const int t = L.ctx_len[b];
        const int n = t + 1;  // scores over tokens 0..t
        const int nch = (n + kScoreChunk - 1) / kScoreChunk;
        if (ch >= nch || t >= L.t_max) continue;
        const int lite_start = max(0, n - L.lite_budget);
        for (int i = tid; i < kHistBins; i += blockDim.x) s_hist[i] = 0;
        __syncthreads();
        const int row0 = ch * kScoreChunk, row1 = min(n, row0 + kScoreChunk);
        uint32_t *keys = L.keys + (size_t)bh * L.t_max;
        if (a.ext_scores == nullptr) {
            float qv[N];
            const float *qh = L.q_hat + (size_t)bh * R + sl * N;
#pragma unroll
            for (int e = 0; e < N; ++e) qv[e] = qh[e];
            const T *base = reinterpret_cast<const T *>(L.proxy) + (size_t)bh * L.t_max * R;
            const int step = (kScoreThreads / 32) * RPW;
            for (int r0 = row0 + warp * RPW + sub; r0 < row1 + sub; r0 += step * U) {
                float x[U][N];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int row = r0 + u * step;
                    if (row < row1) Pack<T>::load_nc(base + (size_t)row * R + sl * N, x[u]);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int row = r0 + u * step;
                    float s = 0.f;
#pragma unroll
                    for (int e = 0; e < N; ++e) s = fmaf(x[u][e], qv[e], s);
                    s = group_sum<TPR>(s);
                    if (sl == 0 && row < row1) {
                        const uint32_t key = score_key(s);
                        keys[row] = key;
                        if (row < lite_start) atomicAdd(&s_hist[key >> (32 - kHistBits)], 1);
                    }
                }
            }
        } else {
            const float *sc = a.ext_scores + (size_t)bh * n;
            for (int row = row0 + tid; row < row1; row += blockDim.x) {
                const uint32_t key = score_key(sc[row]);
                keys[row] = key;
                if (row < lite_start) atomicAdd(&s_hist[key >> (32 - kHistBits)], 1);
            }
        }
        __syncthreads();
        uint32_t *ghist = L.hist + (size_t)bh * kHistBins;
        for (int i = tid; i < kHistBins; i += blockDim.x)
            if (s_hist[i]) atomicAdd(ghist + i, (uint32_t)s_hist[i]);
        int *cnt = L.counters + (size_t)bh * kCounterInts + C_SCORE;
        if (!last_arrival(cnt, nch, &s_flag)) continue;
        // ---- last block of this head: locate the threshold bin -----------
        int *meta = L.sel_meta + (size_t)bh * kMetaInts;
        const int k_eff = min(L.k_budget, lite_start);
        if (lite_start == 0 || k_eff >= lite_start) {
            if (tid == 0) {
                meta[M_MODE] = 1; meta[M_K_EFF] = k_eff; meta[M_LITE] = lite_start;
                meta[M_SURE] = 0; meta[M_CAND] = 0;
            }
            continue;
        }
        for (int i = tid; i < kHistBins; i += blockDim.x) s_hist[i] = (int)__ldcg(ghist + i);
        if (tid == 0) { s_out[0] = -1; s_out[1] = 0; }
        __syncthreads();
        find_crossing(s_hist, kHistBins, k_eff, s_scan, s_out);
        if (tid == 0) {
            const int bin = s_out[0];
            meta[M_THR_BIN] = bin;
            meta[M_N_ABOVE] = s_out[1];
            meta[M_N_BIN] = s_hist[bin];
            meta[M_K_EFF] = k_eff;
            meta[M_LITE] = lite_start;
            meta[M_SURE] = 0;
            meta[M_CAND] = 0;
            meta[M_MODE] = (s_hist[bin] <= L.cand_cap) ? 0 : 2;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// K4a: split the keys below lite_start into certain winners and candidates.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
select_scan_kernel(const lrqk_layer_t L) {
    const int tid = threadIdx.x, lane = tid & 31;
    const int BH = L.batch * L.n_q_heads;
    const int nch_max = (L.t_max + kScanChunk - 1) / kScanChunk;
    for (int item = blockIdx.x; item < BH * nch_max; item += gridDim.x) {
        const int bh = item / nch_max, ch = item - bh * nch_max;
        const int *meta = L.sel_meta + (size_t)bh * kMetaInts;
        if (meta[M_MODE] != 0) continue;
        const int lite_start = meta[M_LITE];
        const int row0 = ch * kScanChunk;
        if (row0 >= lite_start) continue;
        const int row1 = min(lite_start, row0 + kScanChunk);
        const uint32_t thr = (uint32_t)meta[M_THR_BIN];
        const uint32_t *keys = L.keys + (size_t)bh * L.t_max;
        int *sure_cnt = L.sel_meta + (size_t)bh * kMetaInts + M_SURE;
        int *cand_cnt = L.sel_meta + (size_t)bh * kMetaInts + M_CAND;
        int *sure = L.sure_idx + (size_t)bh * L.k_budget;
        uint64_t *cand = L.cand + (size_t)bh * L.cand_cap;
        for (int base = row0; base < row1; base += blockDim.x * 4) {
            uint32_t kv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = base + u * blockDim.x + tid;
                kv[u] = i < row1 ? __ldcg(keys + i) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = base + u * blockDim.x + tid;
                const uint32_t bin = kv[u] >> (32 - kHistBits);
                const bool is_sure = i < row1 && bin > thr;
                const bool is_cand = i < row1 && bin == thr;
                const unsigned ms = __ballot_sync(0xffffffffu, is_sure);
                const unsigned mc = __ballot_sync(0xffffffffu, is_cand);
                if (ms) {
                    int basei = 0;
                    if (lane == 0) basei = atomicAdd(sure_cnt, __popc(ms));
                    basei = __shfl_sync(0xffffffffu, basei, 0);
                    if (is_sure) sure[basei + __popc(ms & ((1u << lane) - 1u))] = i;
                }
                if (mc) {
                    int basei = 0;
                    if (lane == 0) basei = atomicAdd(cand_cnt, __popc(mc));
                    basei = __shfl_sync(0xffffffffu, basei, 0);
                    if (is_cand) cand[basei + __popc(mc & ((1u << lane) - 1u))] = make_comp(kv[u], i);
                }
            }
        }
    }
}

// Radix select over unique composites: returns thr such that exactly m
// elements have comp >= thr.  get(i) yields element i's composite.
template <class Get>
__device__ uint64_t radix_top_m(Get get, int n, int m, int nbits, int *s_hist, int *s_scan, int *s_out) {
    uint64_t prefix = 0;
    int shift = nbits;
    while (shift > 0) {
        const int w = min(kHistBits, shift);
        shift -= w;
        const int nb = 1 << w;
        const int hi_shift = shift + w;
        for (int i = threadIdx.x; i < nb; i += blockDim.x) s_hist[i] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const uint64_t c = get(i);
            if (hi_shift >= 64 || (c >> hi_shift) == (prefix >> hi_shift))
                atomicAdd(&s_hist[(int)((c >> shift) & (uint64_t)(nb - 1))], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) { s_out[0] = 0; s_out[1] = 0; }
        __syncthreads();
        find_crossing(s_hist, nb, m, s_scan, s_out);
        const int D = s_out[0];
        m -= s_out[1];
        prefix |= (uint64_t)D << shift;
        __syncthreads();
    }
    return prefix;
}

// ---------------------------------------------------------------------------
// K4b + K5: finalise the selection of one head and update its cache state.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kFinThreads)
select_finalize_kernel(const lrqk_layer_t L) {
    extern __shared__ __align__(16) uint32_t fsm[];
    __shared__ int s_hist[kHistBins];
    __shared__ int s_scan[32];
    __shared__ int s_out[2];
    __shared__ int s_tot[4];
    const int bh = blockIdx.x;
    const int b = bh / L.n_q_heads;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int t = L.ctx_len[b];
    int *meta = L.sel_meta + (size_t)bh * kMetaInts;
    if (t >= L.t_max) return;
    const int mode = meta[M_MODE];
    const int lite_start = meta[M_LITE];
    const int k_eff = meta[M_K_EFF];
    const int n_words = (lite_start + 31) >> 5;
    const int S = k_eff + (t + 1 - lite_start);  // |omega_k| + |omega_l|
    const bool host = L.policy == LRQK_SLOW_HOST;

    // shared layout: [bitmap n_words][new list s_cap][prev list s_cap][prev slots s_cap]
    //                [new slots s_cap][slot-used bitmap][cand cand_cap (u64)]
    uint32_t *bitmap = fsm;
    int *newl = reinterpret_cast<int *>(bitmap + ((n_words + 3) & ~3));
    int *prevl = newl + L.s_cap;
    int *prevs = prevl + L.s_cap;
    int *news = prevs + L.s_cap;
    uint32_t *slot_used = reinterpret_cast<uint32_t *>(news + L.s_cap);
    const int slot_words = (L.n_slots + 31) >> 5;
    uint64_t *cand_s = reinterpret_cast<uint64_t *>(slot_used + ((slot_words + 3) & ~3));

    // ---- Omega_k -----------------------------------------------------------
    if (mode == 1) {
        for (int i = tid; i < k_eff; i += nt) newl[i] = i;  // everything fits
    } else {
        for (int w = tid; w < n_words; w += nt) bitmap[w] = 0u;
        __syncthreads();
        const uint32_t *keys = L.keys + (size_t)bh * L.t_max;
        if (mode == 0) {
            const int n_sure = meta[M_SURE];
            const int n_cand = meta[M_CAND];
            const int need = k_eff - n_sure;
            const uint64_t *cand = L.cand + (size_t)bh * L.cand_cap;
            for (int i = tid; i < n_cand; i += nt) cand_s[i] = __ldcg(cand + i);
            const int *sure = L.sure_idx + (size_t)bh * L.k_budget;
            for (int i = tid; i < n_sure; i += nt) {
                const int x = __ldcg(sure + i);
                atomicOr(&bitmap[x >> 5], 1u << (x & 31));
            }
            __syncthreads();
            if (need > 0) {
                // all candidates share the top kHistBits key bits
                const int nbits = 32 - kHistBits + kIdxBits;
                const uint64_t lowmask = (1ull << nbits) - 1ull;
                auto get = [&](int i) { return cand_s[i] & lowmask; };
                const uint64_t thr = radix_top_m(get, n_cand, need, nbits, s_hist, s_scan, s_out);
                for (int i = tid; i < n_cand; i += nt) {
                    if ((cand_s[i] & lowmask) >= thr) {
                        const int x = comp_index(cand_s[i]);
                        atomicOr(&bitmap[x >> 5], 1u << (x & 31));
                    }
                }
            }
        } else {
            // exact fallback over the whole key array
            auto get = [&](int i) { return make_comp(__ldcg(keys + i), i); };
            const uint64_t thr = radix_top_m(get, lite_start, k_eff, 32 + kIdxBits, s_hist, s_scan, s_out);
            for (int i = tid; i < lite_start; i += nt)
                if (make_comp(__ldcg(keys + i), i) >= thr) atomicOr(&bitmap[i >> 5], 1u << (i & 31));
        }
        __syncthreads();
        // ascending compaction of the bitmap
        const int per = (n_words + nt - 1) / nt;
        const int w0 = tid * per;
        int local = 0;
        for (int w = w0; w < min(n_words, w0 + per); ++w) local += __popc(bitmap[w]);
        int total;
        int off = block_exclusive_scan(local, s_scan, &total);
        for (int w = w0; w < min(n_words, w0 + per); ++w) {
            uint32_t bits = bitmap[w];
            while (bits) {
                const int bpos = __ffs(bits) - 1;
                bits &= bits - 1u;
                newl[off++] = (w << 5) + bpos;
            }
        }
        if (tid == 0 && total != k_eff) set_status(L.status, LRQK_ST_INDEX_RANGE);
    }
    // ---- Omega_l (always contains t) --------------------------------------
    for (int i = tid; i < t + 1 - lite_start; i += nt) newl[k_eff + i] = lite_start + i;

    // ---- K5: hit/miss against Omega_{t-1} U {t} ---------------------------
    const int n_prev = L.res_cnt[bh];
    int *res_idx = L.res_idx + (size_t)bh * L.s_cap;
    int *res_slot = L.res_slot + (size_t)bh * L.s_cap;
    for (int i = tid; i < n_prev; i += nt) {
        prevl[i] = res_idx[i];
        if (host) prevs[i] = res_slot[i];
    }
    if (host) for (int w = tid; w < slot_words; w += nt) slot_used[w] = 0u;
    __syncthreads();
    const int spare = host ? L.spare_slot[bh] : 0;
    int hits_local = 0;
    for (int i = tid; i < S; i += nt) {
        const int x = newl[i];
        int pos = -1;
        if (x != t) {
            int lo = 0, hi = n_prev - 1;
            while (lo <= hi) {
                const int mid = (lo + hi) >> 1;
                const int v = prevl[mid];
                if (v == x) { pos = mid; break; }
                if (v < x) lo = mid + 1; else hi = mid - 1;
            }
        }
        const bool hit = (x == t) || pos >= 0;
        hits_local += hit;
        if (host) {
            int s = -1;
            if (x == t) s = spare;
            else if (pos >= 0) s = prevs[pos];
            news[i] = s;
            if (s >= 0) atomicOr(&slot_used[s >> 5], 1u << (s & 31));
        }
    }
    int hits;
    block_exclusive_scan(hits_local, s_scan, &hits);
    const int miss = S - hits;
    if (host) {
        __syncthreads();
        // misses in ascending order, paired with free slots in ascending order
        int mloc = 0;
        const int per = (S + nt - 1) / nt;
        const int i0 = tid * per;
        for (int i = i0; i < min(S, i0 + per); ++i) mloc += news[i] < 0;
        int mtot;
        int moff = block_exclusive_scan(mloc, s_scan, &mtot);
        int floc = 0;
        const int fper = (slot_words + nt - 1) / nt;
        const int f0 = tid * fper;
        for (int w = f0; w < min(slot_words, f0 + fper); ++w) {
            uint32_t freew = ~slot_used[w];
            if (w == slot_words - 1 && (L.n_slots & 31)) freew &= (1u << (L.n_slots & 31)) - 1u;
            floc += __popc(freew);
        }
        int ftot;
        int foff = block_exclusive_scan(floc, s_scan, &ftot);
        // free slot list -> prevs (reuse) ; miss positions -> prevl (reuse)
        __syncthreads();
        int *free_list = prevs;
        int *miss_pos = prevl;
        for (int w = f0; w < min(slot_words, f0 + fper); ++w) {
            uint32_t freew = ~slot_used[w];
            if (w == slot_words - 1 && (L.n_slots & 31)) freew &= (1u << (L.n_slots & 31)) - 1u;
            while (freew) {
                const int bpos = __ffs(freew) - 1;
                freew &= freew - 1u;
                free_list[foff++] = (w << 5) + bpos;
            }
        }
        for (int i = i0; i < min(S, i0 + per); ++i)
            if (news[i] < 0) miss_pos[moff++] = i;
        __syncthreads();
        int *mi = L.miss_idx + (size_t)bh * L.s_cap;
        int *ms = L.miss_slot + (size_t)bh * L.s_cap;
        for (int j = tid; j < mtot; j += nt) {
            const int i = miss_pos[j];
            const int s = free_list[j];
            news[i] = s;
            mi[j] = newl[i];
            ms[j] = s;
        }
        __syncthreads();
        if (tid == 0) {
            L.miss_cnt[bh] = mtot;
            L.spare_slot[bh] = (ftot > mtot) ? free_list[mtot] : 0;
            if (ftot <= mtot) set_status(L.status, LRQK_ST_CAPACITY);
        }
        for (int i = tid; i < S; i += nt) res_slot[i] = news[i];
    }
    for (int i = tid; i < S; i += nt) res_idx[i] = newl[i];
    if (tid == 0) {
        L.res_cnt[bh] = S;
        L.c_miss[bh] += miss;
        L.c_total[bh] += S;
        L.step_miss[bh] = miss;
        L.step_total[bh] = S;
        meta[M_SURE] = 0;
        meta[M_CAND] = 0;
    }
    // clear the histogram for the next step
    uint32_t *ghist = L.hist + (size_t)bh * kHistBins;
    for (int i = tid; i < kHistBins; i += nt) ghist[i] = 0u;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

template <typename T>
static int launch_score_t(const ScoreArgs &a, cudaStream_t st) {
    const lrqk_layer_t &L = a.L;
    const int BH = L.batch * L.n_q_heads;
    const int items = BH * ((L.t_max + kScoreChunk - 1) / kScoreChunk);
    const int grid = max(1, min(items, num_sms() * 4));
    const int tpr = L.rank_stride * (int)sizeof(T) / 16;
    switch (tpr) {
        case 1: score_kernel<T, 1><<<grid, kScoreThreads, 0, st>>>(a); break;
        case 2: score_kernel<T, 2><<<grid, kScoreThreads, 0, st>>>(a); break;
        case 4: score_kernel<T, 4><<<grid, kScoreThreads, 0, st>>>(a); break;
        case 8: score_kernel<T, 8><<<grid, kScoreThreads, 0, st>>>(a); break;
        case 16: score_kernel<T, 16><<<grid, kScoreThreads, 0, st>>>(a); break;
        default: return LRQK_EUNSUPPORTED;
    }
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

int launch_score(const lrqk_layer_t &L, const float *ext_scores, cudaStream_t st) {
    ScoreArgs a{L, ext_scores};
    return L.dtype == LRQK_BF16 ? launch_score_t<__nv_bfloat16>(a, st) : launch_score_t<float>(a, st);
}

size_t finalize_smem_bytes(const lrqk_layer_t &L) {
    const size_t n_words = ((size_t)L.t_max + 31) / 32;
    const size_t slot_words = ((size_t)L.n_slots + 31) / 32;
    return ((n_words + 3) & ~(size_t)3) * 4 + 4 * (size_t)L.s_cap * 4 + ((slot_words + 3) & ~(size_t)3) * 4 +
           (size_t)L.cand_cap * 8;
}

int launch_select(const lrqk_layer_t &L, cudaStream_t st) {
    const int BH = L.batch * L.n_q_heads;
    const int items = BH * ((L.t_max + kScanChunk - 1) / kScanChunk);
    const int grid = max(1, min(items, num_sms() * 4));
    select_scan_kernel<<<grid, 256, 0, st>>>(L);
    const size_t smem = finalize_smem_bytes(L);
    cudaFuncSetAttribute(select_finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    select_finalize_kernel<<<BH, kFinThreads, smem, st>>>(L);
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

}  // namespace lrqk
