// K3 + K4 + K6 in one kernel (selection mode 6, HBM policy): proxy scores,
// top-k + lite-window selection and exact attention over the winners.
// ref: cache.py:141-146 (proxy_scores), cache.py:149-171 (select_active),
// linalg.py:96-110 (topk_indices), attention.py:23-34 (exact_attention),
// session.py:98-102.
//
// The score kernel + select_attend pair (select.cu, select_attend.cu) hands
// the selection from one kernel to the next: every head waits for the whole
// score grid, then for its own last block, then for select_attend's last
// block and for attention_kernel's merge.  Here the P blocks of a head stay
// resident and meet at two per-head barriers instead, so each head moves on
// as soon as its own parts have streamed their rows, while other heads are
// still streaming:
//
//   stream   each block streams its part of A_K through the TMA pipeline
//            (score_common.cuh): keys, candidate mask, and the exact
//            histogram of the keys in the hint window.
//   B1       per-head barrier: every part's histogram is in the head's.
//            Every block finds the threshold bin D (the window bin that
//            holds the k-th largest key) and its part's output offset from
//            the per-part suffix counts -- no last-block hand-off.
//   classify the block's certain winners (bins above D) go straight to
//            res_idx[offset + rank], ascending; its bin-D rows go to the
//            head's candidate list.
//   B2       per-head barrier: the bin-D list is complete.  Every block
//            ranks it (reference tie rule: ties -> lower index) and keeps
//            the bin-D winners inside its own rows; the last part adds the
//            lite window.
//   attend   the block gathers its winners' K, V (and proxy rows, for the
//            next step's Y = A^T K, G = A^T A) and writes one online-softmax
//            partial; the last block to finish publishes the step's
//            selection metadata.  attention_kernel merges the head's P
//            partials into the output (and folds the Y|G slots) next.
//
// The barriers need the head's P blocks co-resident: the launcher only takes
// this path when the whole grid fits on the GPU at once (occupancy check) and
// blocks are dispatched in index order, head by head; a bounded spin sets
// LRQK_ST_BARRIER instead of hanging if that ever fails.  Heads that are not
// on the hint-window path this step (the first step after a prompt, a window
// miss, a threshold bin too large to rank here) leave the selection to
// select_kernel / attention_kernel exactly as the score kernel would.
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "select_common.cuh"
#include "score_common.cuh"
#include "mma_common.cuh"
#include "attend_common.cuh"

namespace lrqk {

int yg_slots(const lrqk_layer_t &L);
int score_tma_parts(const lrqk_layer_t &L);
int num_sms();

constexpr int kSAThreads = 32 * (kCW + 1);  // 8 consumer warps + the TMA producer warp

struct SAArgs {
    lrqk_layer_t L;
    const void *q;
    float *out;
    int parts;
    int yg_slots;
    int union_bytes;  // shared bytes shared by the stream stages + histograms and the attention chunks
    int pool_pct;     // share of each part's tiles streamed from the head's shared pool (StreamPool)
};

LRQK_DEV int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Arrive on the head's counter and wait until `target` arrivals are in.
// Bounded: a wait that outlives any real step sets LRQK_ST_BARRIER.
LRQK_DEV void head_barrier(int *counter, int target, uint32_t *status) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1);
        unsigned ns = 32;
        for (int spins = 0; ld_acquire(counter) < target; ++spins) {
            if (spins > (1 << 22)) {
                set_status(status, LRQK_ST_BARRIER);
                break;
            }
            __nanosleep(ns);
            if (ns < 256) ns <<= 1;
        }
    }
    __syncthreads();
}

// Final arrival: adds `add`; true in the one block that completes `total`,
// which re-arms the counter for the next step.
LRQK_DEV bool final_arrival(int *counter, int add, int total, int *s_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int prev = atomicAdd(counter, add);
        const bool last = prev + add == total;
        if (last) {
            atomicExch(counter, 0);
            __threadfence();
        }
        *s_flag = last;
    }
    __syncthreads();
    return *s_flag != 0;
}

template <typename T, int NPK, int LPR, int PPL, int YGM, int CR, int NS>
__global__ void __maxnreg__(96)  // 2 blocks x 9 warps: 5 warps on one SM sub-partition x 96 regs fit its 16K registers
score_attend_kernel(const SAArgs a) {
    using SS = ScoreStages<NPK>;
    const lrqk_layer_t &L = a.L;
    constexpr int N = Pack<T>::N;
    extern __shared__ __align__(128) uint8_t sa_smem[];
    // [0, union_bytes): stream stages, s_win, s_hist  |  later the attention
    // chunks and phase scratch; then the mbarriers; then s_rows[s_cap]
    uint8_t *stage = sa_smem;
    int *s_win = reinterpret_cast<int *>(sa_smem + SS::kStages * SS::kStageBytes);
    int *s_hist = s_win + kHistBins;
    uint64_t *full = reinterpret_cast<uint64_t *>(sa_smem + a.union_bytes);
    uint64_t *empty = full + SS::kStages;
    int *s_rows = reinterpret_cast<int *>(full + 2 * SS::kStages);
    __shared__ float s_m[kSAThreads / 32], s_l[kSAThreads / 32];
    __shared__ int s_scan[32];
    __shared__ int s_flag, s_above, s_ncrit, s_cbase, s_nmine;
    __shared__ int s_out[2];
    __shared__ int s_off[2];
    __shared__ int s_pt[16];  // StreamPool stage tiles | counts
    __shared__ uint32_t s_hint;
    __shared__ uint64_t s_crit[kFCrit];
    trace(40);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int P = a.parts;
    const int bh = blockIdx.x / P, part = blockIdx.x - bh * P;
    const int b = bh / L.n_q_heads, h = bh - b * L.n_q_heads;
    const int G = L.n_q_heads / L.n_kv_heads, g = h / G;
    const int d = L.dim_stride, R = L.rank_stride;
    const int sub = lane / LPR, sl = lane - sub * LPR;
    const int t = L.ctx_len[b];
    if (t >= L.t_max) return;
    const int n = t + 1;
    const int lite_start = max(0, n - L.lite_budget);
    const int tiles = (n + 31) >> 5;
    const int tpp = (tiles + P - 1) / P;
    const int tile0 = min(tiles, part * tpp), tile1 = min(tiles, tile0 + tpp);
    // the part streams the first ns tiles of its range itself; the rest of
    // every range is the head's shared pool (classification and attention
    // keep the static ranges [tile0, tile1))
    const int ns = min(tpp, (tpp * (100 - a.pool_pct) / 100) / kCW * kCW);
    const int s_end = min(tile1, tile0 + ns);
    const int cpp = (tpp - ns + kCW - 1) / kCW;
    int *cnt = L.counters + (size_t)bh * kCounterInts + C_SCORE;
    int *pool_ctr = L.counters + (size_t)bh * kCounterInts + C_POOL;
    const StreamPool sp{pool_ctr, tpp, ns, tiles, cpp, P * cpp, s_pt, s_pt + 8};
    const int stride = sample_stride(lite_start);
    int *meta = L.sel_meta + (size_t)bh * kMetaInts;
    // hint window (persistent meta written by the previous step's selection)
    const bool win = meta[M_HINT_OK] != 0;
    uint32_t klo = 0, kc = 0xFFFFFFFFu;  // set after pdl_wait (the hint scales with this step's q_hat)
    for (int i = tid; i < kHistBins; i += blockDim.x) { s_hist[i] = 0; s_win[i] = 0; }
    if (tid == 0) {
        s_above = 0;
        s_ncrit = 0;
        for (int s2 = 0; s2 < SS::kStages; ++s2) {
            mbar_init(full + s2, 1);
            mbar_init(empty + s2, kCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int it0 = 0;  // stages in flight before the wait (producer lane)
    if (warp == kCW && lane == 0) it0 = score_prefetch_stages<T, NPK>(L, bh, tile0, s_end, t, stage, full);
    pdl_wait();  // q_hat, the appended proxy row and ctx_len come from compress
    pdl_trigger();
    if (win) hint_window(scaled_hint(meta, qhat_norm(L, bh)), klo, kc);

    // ---- stream ------------------------------------------------------------
    score_stream<T, NPK, false, true>(L, bh, tile0, s_end, n, lite_start, stride, win, klo, kc, stage, full, empty,
                                      s_hist, s_win, &s_above, it0, nullptr, nullptr, 0xFFFFFFFFu, sp);
    trace(41);
    __syncthreads();
    // merged histograms only: a part's rows were not all streamed by the part
    score_flush(L, bh, P, part, win, s_hist, s_win, s_above, s_scan, false);
    const int k_eff = min(L.k_budget, lite_start);
    if (!win || lite_start == 0 || k_eff >= lite_start) {
        // no hint (the first step after a prompt) or everything fits: the
        // score kernel's hand-off to select_kernel
        if (!last_arrival(cnt, P, &s_flag)) return;
        if (tid == 0) atomicExch(pool_ctr, 0);  // every part has left the stream
        score_last_block(L, bh, P, win, klo, kc, lite_start, stride, s_hist, s_win, s_scan, s_out, false);
        return;
    }

    // ---- this part's rows and candidate mask ----------------------------------------
    const int row0 = min(lite_start, tile0 * 32), row1 = min(lite_start, tile1 * 32);
    const int w0 = row0 >> 5, w1 = (row1 + 31) >> 5, nwrd = w1 - w0;
    const int wpt = (nwrd + blockDim.x - 1) / blockDim.x;  // contiguous mask words per thread
    const size_t kv_rows = ((size_t)b * L.n_kv_heads + g) * L.t_max;
    const T *kb = reinterpret_cast<const T *>(L.slow_k) + kv_rows * d;
    const T *vb = reinterpret_cast<const T *>(L.slow_v) + kv_rows * d;
    const T *proxy = reinterpret_cast<const T *>(L.proxy) + (size_t)bh * L.t_max * R;
    const T *arows = L.proxy_rowmajor ? reinterpret_cast<const T *>(L.proxy_rowmajor) + (size_t)bh * L.t_max * R
                                      : nullptr;

    // ---- B1: the head's window histogram (and every row's key) is complete ---------
    head_barrier(cnt, P, L.status);
    trace(42);
    if (part == 0 && tid == 0) atomicExch(pool_ctr, 0);  // every part has left the stream
    uint32_t wv[4];  // this part's candidate mask words (streamed by any part)
    {
        const uint32_t *cmw = L.cmask + (size_t)bh * ((L.t_max + 31) >> 5) + w0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int wi = tid * wpt + u;
            wv[u] = (u < wpt && wi < nwrd) ? __ldcg(cmw + wi) : 0u;
        }
    }
    const uint32_t *gwin = L.hist + (size_t)bh * kHistLevels * kHistBins + 2 * kHistBins;
    const int above_win = __ldcg(meta + M_ABOVE);
    for (int i = tid; i < kHistBins; i += blockDim.x) s_win[i] = (int)__ldcg(gwin + i);
    __syncthreads();
    trace(46);
    int D = -1, nabove = 0;
    if (above_win < k_eff) {
        find_crossing(s_win, kHistBins, k_eff - above_win, s_scan, s_out);
        D = s_out[0];
        nabove = above_win + s_out[1];
    }
    trace(47);
    if (D < 0 || s_win[D] > kFCrit) {
        // window miss, or a threshold bin too large to rank here: the last
        // block to get here hands the head to select_kernel (mode 3 / 0)
        if (final_arrival(cnt, 2, 3 * P, &s_flag))
            score_last_block(L, bh, P, win, klo, kc, lite_start, stride, s_hist, s_win, s_scan, s_out, false);
        return;
    }

    // ---- classify this part's keys ---------------------------------------------
    const uint32_t *keys = L.keys + (size_t)bh * L.t_max;
    int *dst = L.res_idx + (size_t)bh * L.s_cap;
    uint64_t *cand = L.cand + (size_t)bh * L.cand_cap;
    int nloc = 0;
    // shortlist: this step's threshold bin lies above the candidate bound,
    // so only the rows marked in cmask can win
    bool shortlist = kc != 0xFFFFFFFFu && klo + ((uint32_t)D << kWinShift) >= kc && wpt <= 4;
    if (shortlist) {
        // the part's candidates, listed ascending in shared memory (thread t
        // owns rows of words [t*wpt, (t+1)*wpt)), then classified blockDim at
        // a time; an exclusive scan per round keeps the winners ascending
        int cnt_c = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) cnt_c += __popc(wv[u]);
        int tot_c;
        int off = block_exclusive_scan(cnt_c, s_scan, &tot_c);
        int *s_cl = reinterpret_cast<int *>(stage);
        shortlist = tot_c <= a.union_bytes / 4;  // same in every thread
        if (shortlist) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                uint32_t rem = wv[u];
                while (rem) {
                    s_cl[off++] = (w0 + tid * wpt + u) * 32 + __ffs(rem) - 1;
                    rem &= rem - 1u;
                }
            }
            __syncthreads();
            trace(49);
            // thread t classifies the contiguous candidates [t*per, (t+1)*per)
            // (their keys loaded together), then one scan places the winners:
            // ascending when per <= kCl (rounds of kCl keep the registers
            // bounded; past that the order is still deterministic)
            constexpr int kCl = 8;
            const int per = (tot_c + blockDim.x - 1) / blockDim.x;
            for (int c0 = 0; c0 < per; c0 += kCl) {
                const int j0 = tid * per + c0, j1 = min(tid * per + min(per, c0 + kCl), tot_c);
                uint32_t kk[kCl];
#pragma unroll
                for (int u = 0; u < kCl; ++u) kk[u] = j0 + u < j1 ? __ldcg(keys + s_cl[j0 + u]) : 0u;
                uint32_t wmask = 0;
#pragma unroll
                for (int u = 0; u < kCl; ++u) {
                    if (j0 + u >= j1 || kk[u] < klo) continue;
                    const uint32_t dk = kk[u] - klo;
                    if (dk >= kWinKeys || (int)(dk >> kWinShift) > D) {
                        wmask |= 1u << u;
                    } else if ((int)(dk >> kWinShift) == D) {
                        const int q = atomicAdd(&s_ncrit, 1);
                        if (q < kFCrit) s_crit[q] = make_comp(kk[u], s_cl[j0 + u]);
                    }
                }
                int tot2;
                int o = nloc + block_exclusive_scan(__popc(wmask), s_scan, &tot2);
                while (wmask) {
                    const int x = s_cl[j0 + __ffs(wmask) - 1];
                    wmask &= wmask - 1u;
                    if (o < L.s_cap) s_rows[o] = x;
                    ++o;
                }
                nloc += tot2;
            }
            trace(58);
        }
    }
    for (int base = row0; base < row1 && !shortlist; base += (int)blockDim.x * 32) {
        uint4 kv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = base + tid * 32 + u * 4;
            kv[u] = i < row1 ? __ldcg(reinterpret_cast<const uint4 *>(keys + i)) : make_uint4(0, 0, 0, 0);
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
                    } else if ((int)(dk >> kWinShift) == D) {
                        const int q = atomicAdd(&s_ncrit, 1);
                        if (q < kFCrit) s_crit[q] = make_comp(kk[e], i);
                    }
                }
            }
        }
        int tot2;
        int o = nloc + block_exclusive_scan(__popc(smask), s_scan, &tot2);
        while (smask) {  // thread-contiguous keys: ascending order is (thread, bit)
            const int bpos = __ffs(smask) - 1;
            smask &= smask - 1u;
            const int x = base + tid * 32 + bpos;
            if (o < L.s_cap) s_rows[o] = x;
            ++o;
        }
        nloc += tot2;
    }
    __syncthreads();
    {   // this part's threshold-bin rows -> the head's list (one reservation)
        const int nc = min(s_ncrit, kFCrit);
        if (tid == 0) s_cbase = nc ? atomicAdd(meta + M_CAND, nc) : 0;
        __syncthreads();
        for (int j = tid; j < nc; j += blockDim.x)
            if (s_cbase + j < L.cand_cap) cand[s_cbase + j] = s_crit[j];
        if (tid == 0) L.fcnt[(size_t)bh * P + part] = nloc;  // certain winners: the parts' offsets after B2
    }
    trace(44);

    // ---- B2: the head's threshold-bin list is complete --------------------------
    head_barrier(cnt, 2 * P, L.status);
    trace(45);
    {   // every block has read the head's histograms: ready them for the next step
        uint32_t *ghist = L.hist + (size_t)bh * kHistLevels * kHistBins;
        for (int i = part * blockDim.x + tid; i < kHistLevels * kHistBins; i += P * blockDim.x) ghist[i] = 0u;
    }
    const int need2 = k_eff - nabove;
    // the list's first 32 entries travel with its length (one round trip)
    const uint64_t v0 = warp == 0 ? __ldcg(cand + lane) : 0ull;
    const int n_crit = __ldcg(meta + M_CAND);
    if (warp == 1) {  // the parts' certain-winner counts: this part's output offset, and the total
        int o = 0, tt = 0;
        for (int q0 = 0; q0 < P; q0 += 32) {
            const int q = q0 + lane;
            const int c = q < P ? __ldcg(L.fcnt + (size_t)bh * P + q) : 0;
            tt += c;
            o += q < part ? c : 0;
        }
        tt = __reduce_add_sync(0xffffffffu, tt);
        o = __reduce_add_sync(0xffffffffu, o);
        if (lane == 0) { s_off[0] = o; s_off[1] = tt; }
    }
    bool ok = need2 >= 0 && need2 <= n_crit && n_crit <= L.cand_cap && n_crit <= kFCrit;
    // bin-D winners, ascending, in the (now free) stage area
    int *s_list = reinterpret_cast<int *>(stage);
    uint64_t *crit = reinterpret_cast<uint64_t *>(stage + kFCrit * 4);
    if (tid == 0) {
        s_hint = klo + ((uint32_t)(D + 1) << kWinShift);
        s_nmine = 0;
    }
    if (!ok) {
        if (tid == 0) set_status(L.status, LRQK_ST_INDEX_RANGE);  // inconsistent selection state (never expected)
    } else if (n_crit <= 32) {
        // one warp: bitonic sort of the composites (descending), then of the
        // winners' indices (ascending), through shuffles
        if (warp == 0) {
            uint64_t v = lane < n_crit ? v0 : 0ull;
#pragma unroll
            for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
                for (int j = kk >> 1; j > 0; j >>= 1) {
                    const uint64_t o = __shfl_xor_sync(0xffffffffu, v, j);
                    const bool hi = ((lane & kk) == 0) == ((lane & j) == 0);  // keep the larger one
                    v = hi ? (v > o ? v : o) : (v < o ? v : o);
                }
            const uint64_t last = __shfl_sync(0xffffffffu, v, max(need2 - 1, 0));
            if (need2 > 0 && lane == 0) s_hint = (uint32_t)(last >> kIdxBits);
            uint32_t ix = lane < need2 ? (uint32_t)comp_index(v) : 0xFFFFFFFFu;
#pragma unroll
            for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
                for (int j = kk >> 1; j > 0; j >>= 1) {
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, ix, j);
                    const bool lo = ((lane & kk) == 0) == ((lane & j) == 0);  // keep the smaller one
                    ix = lo ? min(ix, o) : max(ix, o);
                }
            if (lane < need2) s_list[lane] = (int)ix;
        }
    } else {
        int M = 1;
        while (M < n_crit) M <<= 1;
        for (int i = tid; i < M; i += blockDim.x) crit[i] = i < n_crit ? __ldcg(cand + i) : 0ull;
        __syncthreads();
        block_bitonic(crit, M, true);  // descending composites: ties -> lower index first
        if (need2 > 0 && tid == 0) s_hint = (uint32_t)(crit[need2 - 1] >> kIdxBits);
        int M2 = 1;
        while (M2 < need2) M2 <<= 1;
        for (int i = tid; i < M2; i += blockDim.x) crit[i] = i < need2 ? (uint64_t)comp_index(crit[i]) : ~0ull;
        __syncthreads();
        block_bitonic(crit, M2, false);  // winners by ascending index
        for (int i = tid; i < need2; i += blockDim.x) s_list[i] = (int)crit[i];
    }
    __syncthreads();
    trace(48);
    const int out = s_off[0];
    if (ok && s_off[1] != nabove) {  // the certain winners disagree with the histogram (never expected)
        ok = false;
        if (tid == 0) set_status(L.status, LRQK_ST_INDEX_RANGE);
    }
    if (ok)
        for (int i = tid; i < min(nloc, L.s_cap); i += blockDim.x)
            if (out + i < k_eff) dst[out + i] = s_rows[i];
    const int nwin = ok ? need2 : 0;
    // part 0 writes the bin-D winners; every block attends those in its rows
    if (part == 0)
        for (int i = tid; i < nwin; i += blockDim.x) dst[nabove + i] = s_list[i];
    if (warp == 0) {
        int base = min(nloc, L.s_cap);
        for (int i0 = 0; i0 < nwin; i0 += 32) {
            const int x = i0 + lane < nwin ? s_list[i0 + lane] : -1;
            const bool mine = x >= row0 && x < row1;
            const uint32_t bal = __ballot_sync(0xffffffffu, mine);
            const int pos = base + __popc(bal & ((1u << lane) - 1u));
            if (mine && pos < L.s_cap) s_rows[pos] = x;
            base += __popc(bal);
        }
        if (lane == 0) s_nmine = base - min(nloc, L.s_cap);
    }
    __syncthreads();
    nloc = min(nloc, L.s_cap) + s_nmine;
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

    // ---- attend this block's rows (+ Y|G) ----------------------------------------
    const float c = 1.4426950408889634f * rsqrtf((float)L.head_dim);  // log2(e) / sqrt(d)
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
    constexpr bool YG = YGM > 0;
    constexpr int MT = YGM > 0 ? YGM : 1;
    float yacc[MT][2][4], gacc[4][4];
#pragma unroll
    for (int i = 0; i < MT * 8; ++i) yacc[i / 8][(i / 4) & 1][i & 3] = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) gacc[i / 4][i & 3] = 0.f;
    if (ok) attend_reduce_list<T, LPR, PPL, YGM, CR, NS>(L, kb, vb, proxy, arows, s_rows, min(nloc, L.s_cap), qv, c, m, l, acc,
                                                      stage, yacc, gacc);
    trace(52);
    const size_t PF = yg_part_floats(R, d);
    if constexpr (YG) {
        if (warp < 8) mma_write_partial<MT, 2>(yacc, gacc, R, d, L.red_scratch + ((size_t)bh * a.yg_slots + part) * PF);
    }
    float *s_acc = reinterpret_cast<float *>(stage);  // [nwarps][d]
    float *parts = L.attn_scratch + (size_t)bh * attn_slots_dev(L, P) * (size_t)(d + 2);
    block_partial<T, LPR, PPL>(m, l, acc, d, s_m, s_l, s_acc, parts + (size_t)part * (d + 2));
    trace(57);

    // ---- the last block of the head: publish (attention_kernel merges the
    // P partials into the output, beside its Y|G fold) ----------------------------
    if (!final_arrival(cnt, 1, 3 * P, &s_flag)) return;
    trace(53);
    if (tid == 0) {
        L.res_cnt[bh] = k_eff + nl;
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
        meta[M_HINT] = (int)s_hint;
        meta[M_HINT_OK] = ok ? 1 : 0;
        meta[M_HINT_QN] = __float_as_int(qhat_norm(L, bh));
        meta[M_YG] = YG ? P : 0;  // Y|G partial slots (the finish kernel sums them)
        meta[M_YG_ADD] = 0;
        meta[M_ATT_PARTS] = P;
        meta[M_MODE] = 6;
        meta[M_STAT + 5] += 1;
    }
    trace(54);
}

// ---------------------------------------------------------------------------
// launcher
// ---------------------------------------------------------------------------
template <int NPK> constexpr int sa_stream_bytes() {
    return ScoreStages<NPK>::kStages * ScoreStages<NPK>::kStageBytes + 2 * kHistBins * 4;
}

template <typename T, int NPK, int LPR, int PPL, int YGM, int CR, int NS>
static int launch_sa(const SAArgs &a0, cudaStream_t st) {
    const lrqk_layer_t &L = a0.L;
    SAArgs a = a0;
    const int ldk = L.dim_stride * (int)sizeof(T) + 16, lda = L.rank_stride * 2 + 16;
    const int chunks = NS * (2 * CR * ldk + (YGM > 0 ? CR * lda : 0));
    const int part_scratch = kFCrit * 4 + kFCrit * 8;  // bin-D list + its sort buffer
    const int cand_scratch = kSAThreads * 16 * 4;      // shortlist candidates
    const int acc_scratch = kSAThreads / 32 * L.dim_stride * 4;
    int u = sa_stream_bytes<NPK>();
    u = u > chunks ? u : chunks;
    u = u > part_scratch ? u : part_scratch;
    u = u > cand_scratch ? u : cand_scratch;
    u = u > acc_scratch ? u : acc_scratch;
    a.union_bytes = (u + 127) & ~127;
    const size_t smem = (size_t)a.union_bytes + 2 * ScoreStages<NPK>::kStages * 8 + (size_t)L.s_cap * 4;
    auto fn = score_attend_kernel<T, NPK, LPR, PPL, YGM, CR, NS>;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        if (getenv("LRQK_DEBUG")) fprintf(stderr, "score_attend: smem %zu: %s\n", smem, cudaGetErrorString(cudaGetLastError()));
        cudaGetLastError();
        return LRQK_EUNSUPPORTED;
    }
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    // every block of the grid must be resident at once (per-head barriers)
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSAThreads, smem) != cudaSuccess) {
        cudaGetLastError();
        return LRQK_EUNSUPPORTED;
    }
    const int grid = L.batch * L.n_q_heads * a.parts;
    if (getenv("LRQK_DEBUG")) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, fn);
        fprintf(stderr, "score_attend: grid %d, %d blocks/SM x %d SMs, smem %zu (+%zu static), union %d, %d regs\n",
                grid, per_sm, num_sms(), smem, fa.sharedSizeBytes, a.union_bytes, fa.numRegs);
        for (int kb : {0, 32, 48, 64, 72, 80, 88, 96}) {
            int o = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, kSAThreads, (size_t)kb * 1024);
            int o2 = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, fn, 256, (size_t)kb * 1024);
            fprintf(stderr, "  smem %d KB: %d blocks/SM (288 thr), %d (256 thr)\n", kb, o, o2);
        }
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        fprintf(stderr, "  max smem/SM %d\n", v);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
        fprintf(stderr, "  max regs/SM %d\n", v);
    }
    if (a.parts > 1 && per_sm * num_sms() < grid) return LRQK_EUNSUPPORTED;
    launch_kernel(fn, grid, kSAThreads, smem, st, true, a);
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

// The fused path covers the d = 128 layouts: bf16 with the Y|G reduction
// (rank 16, 32, 64) and f32.  LRQK_EUNSUPPORTED -> the caller runs
// lrqk_score + lrqk_select_attend instead.
int launch_score_attend(const lrqk_layer_t &L, const void *q, float *out, cudaStream_t st) {
    if (L.policy != LRQK_SLOW_HBM || L.dim_stride != 128) return LRQK_EUNSUPPORTED;
    static const int pool_pct = [] {
        const char *e = getenv("LRQK_SA_POOL");  // percent of each part's tiles in the shared pool
        const int v = e ? atoi(e) : 10;
        return v < 0 ? 0 : (v > 100 ? 100 : v);
    }();
    SAArgs a{L, q, out, score_tma_parts(L), yg_slots(L), 0, pool_pct};
    if (L.dtype == LRQK_BF16) {
        switch (L.rank_stride) {
            case 16: return launch_sa<__nv_bfloat16, 2, 16, 1, 1, 64, 2>(a, st);
            case 32: return launch_sa<__nv_bfloat16, 4, 16, 1, 2, 64, 2>(a, st);
            case 64: return launch_sa<__nv_bfloat16, 8, 16, 1, 4, 48, 2>(a, st);
            default: return LRQK_EUNSUPPORTED;
        }
    }
    switch (L.rank_stride) {
        case 8: return launch_sa<float, 2, 32, 1, 0, 32, 2>(a, st);
        case 16: return launch_sa<float, 4, 32, 1, 0, 32, 2>(a, st);
        case 32: return launch_sa<float, 8, 32, 1, 0, 32, 2>(a, st);
        case 64: return launch_sa<float, 16, 32, 1, 0, 32, 2>(a, st);
        default: return LRQK_EUNSUPPORTED;
    }
}

}  // namespace lrqk
