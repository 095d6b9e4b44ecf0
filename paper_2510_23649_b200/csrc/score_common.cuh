// Proxy-score streaming shared by score_tma_kernel (select.cu, K3) and
// score_attend_kernel (score_attend.cu, K3+K4+K6 fused).  ref: cache.py:141-146.
#pragma once
#include "common.cuh"
#include "select_common.cuh"

namespace lrqk {

// extra sel_meta fields of the mode-0 band (common.cuh holds the first ones)
enum MetaExt : int { M_B_HI = 8, M_B_LO = 9, M_STRIDE = 10, M_S2 = 11 };

constexpr int kSampleRows = 16384;  // histogram rows per head before sampling kicks in

LRQK_DEV int sample_stride(int n_rows) {  // in 32-row tiles
    const int tiles = (n_rows + 31) >> 5;
    const int want = kSampleRows >> 5;
    return tiles <= want ? 1 : (tiles + want - 1) / want;
}

struct ScoreArgs {
    lrqk_layer_t L;
    const float *ext_scores;  // standalone path: precomputed float scores [BH, t+1]
    int parts;                // work items per head
};

// Find D in [0, nbins) with  above(D) < m <= above(D) + hist[D], scanning bins
// from the top (whole block).  s_out[0] = D (or -1 if total < m), s_out[1] = above.
static __device__ __noinline__ void find_crossing(const int *hist, int nbins, int m, int *s_scan, int *s_out) {
    const int nt = blockDim.x;
    const int per = (nbins + nt - 1) / nt;
    const int hi = nbins - 1 - threadIdx.x * per;
    if (threadIdx.x == 0) { s_out[0] = -1; s_out[1] = 0; }
    int local = 0;
    for (int i = 0; i < per; ++i) {
        const int bin = hi - i;
        if (bin >= 0) local += hist[bin];
    }
    int total;
    const int above = block_exclusive_scan(local, s_scan, &total);
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

constexpr int kCW = 8;  // consumer warps

template <int NPK> struct ScoreStages {
    static constexpr int kTileBytes = NPK * 512;
    static constexpr int kStageBytes = kCW * kTileBytes;
    // 64 KB: two score blocks stay co-resident with a compress block (68 KB)
    static constexpr int kStages = (64 * 1024 / kStageBytes) < 2 ? 2 : ((64 * 1024 / kStageBytes) > 6 ? 6 : 64 * 1024 / kStageBytes);
    static constexpr int kSmem = kStages * kStageBytes + 2 * kStages * 8;
};

// Before pdl_wait: the producer lane issues the first pipeline stages, whose
// proxy rows were written by earlier steps (only the tile holding row t is
// appended by this step's compress kernel), so the stream is already in
// flight when q_hat arrives.  Returns the number of stages issued (the
// producer lane only; pass it to score_stream as it0).
template <typename T, int NPK>
LRQK_DEV int score_prefetch_stages(const lrqk_layer_t &L, int bh, int tile0, int tile1, int t, uint8_t *tsm,
                                   uint64_t *full) {
    using SS = ScoreStages<NPK>;
    constexpr int R = NPK * Pack<T>::N;
    const int n_stage_iters = (tile1 - tile0 + kCW - 1) / kCW;
    const uint8_t *src = reinterpret_cast<const uint8_t *>(reinterpret_cast<const T *>(L.proxy) +
                                                           (size_t)bh * L.t_max * R);
    const uint64_t pol_stream = l2_policy_evict_first();
    const int tile_t = t >> 5;
    int it = 0;
    for (; it < SS::kStages && it < n_stage_iters; ++it) {
        const int ta = tile0 + it * kCW, nt = min(kCW, tile1 - ta);
        if (tile_t >= ta && tile_t < ta + nt) break;  // this stage holds the row compress appends
        const uint32_t bytes = (uint32_t)nt * SS::kTileBytes;
        mbar_expect_tx(full + it, bytes);
        bulk_g2s_hint(tsm + it * SS::kStageBytes, src + (size_t)ta * SS::kTileBytes, bytes, full + it, pol_stream);
    }
    return it;
}

// Shared tail of a head's stream (the fused kernel): every part streams the
// first ns tiles of its own range, then the parts take the remaining stages
// of all the head's ranges from one counter, so a part that started late or
// streams slowly is helped by the others.  Pool item j = stage c of part p's
// tail (j = p * cpp + c), tiles [p*tpp + ns + c*kCW, ...) within the part's
// range.  s_tile / s_nt: per-stage tile base and count, handed by the
// producer to the consumers through the full barrier (-1: no more stages).
struct StreamPool {
    int *ctr;
    int tpp, ns, tiles, cpp, npool;
    int *s_tile, *s_nt;
};

// Phase 1 of both score kernels, for the tiles [tile0, tile1) of head bh:
// one producer warp (warp kCW) keeps the TMA bulk-copy pipeline full, the
// kCW consumer warps score one 32-row tile per stage (lane = row), store the
// keys (L2 evict-last) and the candidate mask, and histogram the keys: the
// sampled coarse histogram without a hint (s_hist), the exact window around
// the hint otherwise (s_win, plus the rows above the window in *s_above).
//
// it0: stages the producer already issued before pdl_wait (score_prefetch_stages).
//
// PF (the fused kernel): rows whose key reaches kpf -- the previous step's
// k-th largest key, so mostly this step's winners -- have their K and V rows
// (pf_k, pf_v) and their proxy row prefetched into L2 (evict-last) while the
// stream still runs, so the attention gathers after the selection hit L2.
//
// DYN: [tile0, tile1) is the part's own share; the pool (sp) follows it.
template <typename T, int NPK, bool PF = false, bool DYN = false>
LRQK_DEV void score_stream(const lrqk_layer_t &L, int bh, int tile0, int tile1, int n, int lite_start, int stride,
                           bool win, uint32_t klo, uint32_t kc, uint8_t *tsm, uint64_t *full, uint64_t *empty,
                           int *s_hist, int *s_win, int *s_above, int it0 = 0, const T *pf_k = nullptr,
                           const T *pf_v = nullptr, uint32_t kpf = 0xFFFFFFFFu, StreamPool sp = {}) {
    using SS = ScoreStages<NPK>;
    constexpr int N = Pack<T>::N;
    constexpr int R = NPK * N;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n_stage_iters = (tile1 - tile0 + kCW - 1) / kCW;
    uint32_t *cmask = L.cmask + (size_t)bh * ((L.t_max + 31) >> 5);
    const uint8_t *src = reinterpret_cast<const uint8_t *>(reinterpret_cast<const T *>(L.proxy) +
                                                           (size_t)bh * L.t_max * R);
    uint32_t *keys = L.keys + (size_t)bh * L.t_max;
    const uint64_t pol_stream = l2_policy_evict_first(), pol_keys = l2_policy_evict_last();
    if (warp == kCW) {
        // ---------------- producer ----------------
        if (lane == 0) {
            for (int it = it0; it < n_stage_iters; ++it) {  // stages before it0: score_prefetch_stages
                const int s2 = it % SS::kStages;
                if (it >= SS::kStages) {
                    mbar_wait(empty + s2, ((it / SS::kStages) - 1) & 1);
                    // the consumers' generic-proxy reads of this stage, observed through
                    // the empty barrier, before the async-proxy (TMA) overwrite
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                const int nt = min(kCW, tile1 - tile0 - it * kCW);
                const uint32_t bytes = (uint32_t)nt * SS::kTileBytes;
                mbar_expect_tx(full + s2, bytes);
                // the proxy store is streamed once per step: evict it first, so the
                // keys (read again by the selection) stay in L2
                bulk_g2s_hint(tsm + s2 * SS::kStageBytes, src + (size_t)(tile0 + it * kCW) * SS::kTileBytes, bytes,
                              full + s2, pol_stream);
            }
            if constexpr (DYN) {
                int it = n_stage_iters > it0 ? n_stage_iters : it0;
                int j = atomicAdd(sp.ctr, 1);
                for (;; ++it) {
                    int ta = -1, te = 0;
                    while (j < sp.npool) {
                        const int p = j / sp.cpp, c = j - p * sp.cpp;
                        ta = p * sp.tpp + sp.ns + c * kCW;
                        te = min(sp.tiles, (p + 1) * sp.tpp);
                        if (ta < te) break;
                        ta = -1;
                        j = atomicAdd(sp.ctr, 1);
                    }
                    const int s2 = it % SS::kStages;
                    if (it >= SS::kStages) {
                        mbar_wait(empty + s2, ((it / SS::kStages) - 1) & 1);
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    }
                    if (ta < 0) {  // pool drained: release the consumers
                        sp.s_tile[s2] = -1;
                        mbar_arrive(full + s2);
                        break;
                    }
                    const int nt = min(kCW, te - ta);
                    sp.s_tile[s2] = ta;
                    sp.s_nt[s2] = nt;
                    const int jn = atomicAdd(sp.ctr, 1);  // the next grab, in flight during this copy
                    const uint32_t bytes = (uint32_t)nt * SS::kTileBytes;
                    mbar_expect_tx(full + s2, bytes);
                    bulk_g2s_hint(tsm + s2 * SS::kStageBytes, src + (size_t)ta * SS::kTileBytes, bytes, full + s2,
                                  pol_stream);
                    j = jn;
                }
            }
        }
    } else {
        // ---------------- consumers ----------------
        float qv[R];
        const float *qh = L.q_hat + (size_t)bh * L.rank_stride;
#pragma unroll
        for (int e = 0; e < R; ++e) qv[e] = qh[e];
        int above = 0;
        for (int it = 0;; ++it) {
            if (!DYN && it >= n_stage_iters) break;
            const int s2 = it % SS::kStages;
            mbar_wait(full + s2, (it / SS::kStages) & 1);
            int ta = tile0 + it * kCW, ntl = min(kCW, tile1 - ta);
            if (DYN && it >= n_stage_iters) {
                ta = sp.s_tile[s2];
                if (ta < 0) break;
                ntl = sp.s_nt[s2];
            }
            const int tile = ta + warp;
            if (warp < ntl) {
                const uint4 *p4 = reinterpret_cast<const uint4 *>(tsm + s2 * SS::kStageBytes + warp * SS::kTileBytes) + lane;
                float s0 = 0.f, s1 = 0.f;
#pragma unroll
                for (int pk = 0; pk < NPK; ++pk) {
                    float f[N];
                    unpack16<T>(p4[pk * 32], f);
#pragma unroll
                    for (int e = 0; e < N; e += 2) {
                        s0 = fmaf(f[e], qv[pk * N + e], s0);
                        s1 = fmaf(f[e + 1], qv[pk * N + e + 1], s1);
                    }
                }
                const int row = tile * 32 + lane;
                const uint32_t key = score_key(s0 + s1);
                if (row < n) st_hint_u32(keys + row, key, pol_keys);
                if constexpr (PF) {
                    if (row < lite_start && key >= kpf) {
                        const int dd = L.dim_stride;
                        bulk_prefetch_l2_hint(pf_k + (size_t)row * dd, dd * (uint32_t)sizeof(T), pol_keys);
                        bulk_prefetch_l2_hint(pf_v + (size_t)row * dd, dd * (uint32_t)sizeof(T), pol_keys);
#pragma unroll
                        for (int pk = 0; pk < NPK; ++pk)
                            prefetch_l2_last(src + ((size_t)(tile * NPK + pk) * 32 + lane) * 16);
                    }
                }
                {   // candidate bit per row (the fused selection's shortlist)
                    const uint32_t cm = __ballot_sync(0xffffffffu, win && row < lite_start && key >= kc);
                    if (lane == 0) st_hint_u32(cmask + tile, cm, pol_keys);
                }
                if (row < lite_start) {
                    // the sampled coarse histogram only serves the no-hint path
                    if (!win && (tile % stride) == 0) atomicAdd(&s_hist[key >> (32 - kHistBits)], 1);
                    if (win && key >= klo) {
                        const uint32_t dk = key - klo;
                        if (dk < kWinKeys) atomicAdd(&s_win[dk >> kWinShift], 1);
                        else ++above;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s2);
        }
        above = __reduce_add_sync(0xffffffffu, above);
        if (lane == 0 && above) atomicAdd(s_above, above);
    }
}

// After the stream: add this part's histograms to the head's (global
// atomics) and, with a hint, store the part's suffix counts (mode 5):
// ph[i] = rows of the part with a key in window bin >= i or above the
// window; ph[kHistBins] = above.  Whole block.
LRQK_DEV void score_flush(const lrqk_layer_t &L, int bh, int P, int part, bool win, const int *s_hist,
                          const int *s_win, int s_above, int *s_scan, bool part_hist = true) {
    const int tid = threadIdx.x;
    int *meta = L.sel_meta + (size_t)bh * kMetaInts;
    uint32_t *ghist = L.hist + (size_t)bh * kHistLevels * kHistBins;
    uint32_t *gwin = ghist + 2 * kHistBins;
    for (int i = tid; i < kHistBins; i += blockDim.x) {
        if (s_hist[i]) atomicAdd(ghist + i, (uint32_t)s_hist[i]);
        if (s_win[i]) atomicAdd(gwin + i, (uint32_t)s_win[i]);
    }
    if (tid == 0 && s_above) atomicAdd(meta + M_ABOVE, s_above);
    if (win && part_hist) {
        uint32_t *ph = reinterpret_cast<uint32_t *>(L.fcand) + ((size_t)bh * P + part) * kPartHist;
        constexpr int CB = kHistBins / 256;  // bins per thread (threads 0..255)
        int loc = 0;
        if (tid < 256)
#pragma unroll
            for (int j = 0; j < CB; ++j) loc += s_win[tid * CB + j];
        int tot;
        const int ex = block_exclusive_scan(loc, s_scan, &tot);
        if (tid < 256) {
            int suf = s_above + tot - ex;  // rows in bins >= tid*CB, plus above
#pragma unroll
            for (int j = 0; j < CB; ++j) {
                ph[tid * CB + j] = (uint32_t)suf;
                suf -= s_win[tid * CB + j];
            }
        }
        if (tid == 0) ph[kHistBins] = (uint32_t)s_above;
    }
}

// The last block of a head (after every part flushed its histograms) turns
// the merged histograms into this step's selection mode and its parameters:
// mode 1 (everything fits), mode 5/3 (the k-th largest key lies in the hint
// window: exact bin D, with per-part winner offsets for mode 5), or mode 0
// (sampled coarse band, or the exact path when the window missed).
template <int Dummy = 0>
__device__ __forceinline__ void score_last_block(const lrqk_layer_t &L, int bh, int P, bool win, uint32_t klo, uint32_t kc,
                                              int lite_start, int stride, int *s_hist, int *s_win, int *s_scan,
                                              int *s_out, bool allow5 = true) {
    const int tid = threadIdx.x;
    int *meta = L.sel_meta + (size_t)bh * kMetaInts;
    uint32_t *ghist = L.hist + (size_t)bh * kHistLevels * kHistBins;
    uint32_t *gwin = ghist + 2 * kHistBins;
    // ---- last block of this head: candidate bins ----------------------------
    const int k_eff = min(L.k_budget, lite_start);
    if (lite_start == 0 || k_eff >= lite_start) {
        if (tid == 0) {
            meta[M_MODE] = 1; meta[M_K_EFF] = k_eff; meta[M_LITE] = lite_start;
            meta[M_SURE] = 0; meta[M_CAND] = 0; meta[M_ABOVE] = 0;
        }
        return;
    }
    if (win) {
        // mode 3 if the k-th largest key falls inside the hint window: the
        // window histogram is exact, so bin D and the count above it are exact
        const int above_win = __ldcg(meta + M_ABOVE);
        for (int i = tid; i < kHistBins; i += blockDim.x) s_win[i] = (int)__ldcg(gwin + i);
        __syncthreads();
        int D = -1;
        if (above_win < k_eff) {
            find_crossing(s_win, kHistBins, k_eff - above_win, s_scan, s_out);
            D = s_out[0];
        }
        if (D >= 0) {
            const int nabove = above_win + s_out[1];
            int mode = 3;
            if (L.policy == LRQK_SLOW_HBM && allow5) {
                // mode 5: certain winners per part -> exclusive offsets (fcnt)
                mode = 5;
                const uint32_t *ph0 = reinterpret_cast<const uint32_t *>(L.fcand) + (size_t)bh * P * kPartHist;
                const int c = tid < P ? (int)__ldcg(ph0 + (size_t)tid * kPartHist + D + 1) : 0;
                int tot;
                const int off = block_exclusive_scan(c, s_scan, &tot);
                if (tid < P) L.fcnt[(size_t)bh * P + tid] = off;
                // inconsistent counts, or a threshold bin too large to sort: scan path
                if (tot != nabove || s_win[D] > kFCrit) mode = 3;
            }
            if (tid == 0) {
                meta[M_KLO] = (int)klo;
                meta[M_KC] = (int)kc;
                meta[M_FBIN] = D;
                meta[M_NABOVE] = nabove;
                meta[M_SPARTS] = P;
                meta[M_K_EFF] = k_eff;
                meta[M_LITE] = lite_start;
                meta[M_SURE] = 0;
                meta[M_CAND] = 0;
                meta[M_ABOVE] = 0;
                meta[M_MODE] = mode;
            }
            trace(43);
            return;
        }
        __syncthreads();
    }
    if (win) {  // the hint window missed and no coarse histogram was taken: exact path
        if (tid == 0) {
            meta[M_B_HI] = kHistBins - 1;
            meta[M_B_LO] = 0;
            meta[M_STRIDE] = 1;
            meta[M_S2] = 0;
            meta[M_K_EFF] = k_eff;
            meta[M_LITE] = lite_start;
            meta[M_SURE] = 0;
            meta[M_CAND] = 0;
            meta[M_ABOVE] = 0;
            meta[M_MODE] = 0;
        }
        return;
    }
    for (int i = tid; i < kHistBins; i += blockDim.x) s_hist[i] = (int)__ldcg(ghist + i);
    __syncthreads();
    int b_hi, b_lo;
    if (stride == 1) {
        find_crossing(s_hist, kHistBins, k_eff, s_scan, s_out);
        b_hi = b_lo = s_out[0];
    } else {
        const int m_hi = max(1, (int)(0.8f * k_eff / stride));
        find_crossing(s_hist, kHistBins, m_hi, s_scan, s_out);
        b_hi = s_out[0] < 0 ? kHistBins - 1 : s_out[0];
        const int m_lo = (int)ceilf(1.25f * k_eff / stride) + 8;
        find_crossing(s_hist, kHistBins, m_lo, s_scan, s_out);
        b_lo = s_out[0] < 0 ? 0 : s_out[0];
    }
    if (tid == 0) {
        meta[M_B_HI] = b_hi;
        meta[M_B_LO] = b_lo;
        meta[M_STRIDE] = stride;
        int s2 = 0;
        while (s2 < 32 - kHistBits && ((b_hi - b_lo + 1) << (s2 + 1)) <= kHistBins) ++s2;
        meta[M_S2] = s2;
        meta[M_K_EFF] = k_eff;
        meta[M_LITE] = lite_start;
        meta[M_SURE] = 0;
        meta[M_CAND] = 0;
        meta[M_ABOVE] = 0;
        meta[M_MODE] = 0;
    }
    trace(43);
}

}  // namespace lrqk
