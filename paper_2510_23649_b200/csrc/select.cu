// K3: proxy scores fused with the (sampled) radix histogram (cache.py:141-146)
// K4: top-k + lite-window selection (cache.py:149-171, linalg.py:96-110)
// K5: hit/miss accounting and slot replacement (cache.py:174-196, 63-74)
//
// Selection is exact, including the reference's tie rule: the k largest
// scores win, equal scores prefer the lower index, the result is ascending.
// Scores become order-preserving uint32 keys (-0.0 == +0.0) and every token
// gets the unique 53-bit composite
//     comp = key(32) || (2^21 - 1 - index)(21)
// which orders exactly like (score desc, index asc).
//
//   score_kernel   streams the proxy store once (lane = row, tiles of 32 rows
//                  interleaved so every load is a 512-byte run), writes keys,
//                  and histograms the top 11 key bits of every s-th tile
//                  (s = 1, i.e. exact, up to 16K candidate rows).  The last
//                  block of a head turns the histogram into two bins:
//                  tokens above b_hi are certainly in the top k, tokens in
//                  [b_lo, b_hi] are candidates, everything below is out.
//   select_kernel  re-reads the keys, appends the certain winners and the
//                  candidates; the last block of a head then verifies
//                  |sure| <= k <= |sure| + |cand| (the sampled bounds are only
//                  a hint), bitonic-sorts the candidates' composites, builds
//                  omega_k ascending through a shared bitmap, appends omega_l,
//                  and does the cache update.  If the verification fails the
//                  block falls back to an exact radix select over all keys.
#include "common.cuh"
#include "select_common.cuh"
#include "score_common.cuh"

namespace lrqk {

constexpr int kScoreThreads = 256;
constexpr int kSelThreads = 512;
// Direct selection (mode 5, HBM policy): the score kernel also keeps each
// part's window histogram (fcand, reinterpreted as [parts][kHistBins + 1]
// uint32: bins, then the count above the window), so its last block knows
// how many certain winners every part holds -> each select block writes its
// winners straight to their final positions in res_idx.


// fine (level-2) bin of a key inside the candidate band [b_lo, b_hi]
LRQK_DEV int fine_bin(uint32_t key, int b_lo, int s2) {
    return (int)(key >> (32 - kHistBits - s2)) - (b_lo << s2);
}



// ---------------------------------------------------------------------------
// K3: score kernel.  NPK = 16-byte packs per proxy row (rank_stride*e/16).
// ---------------------------------------------------------------------------
template <typename T, int NPK>
__global__ void __launch_bounds__(kScoreThreads)
score_kernel(const ScoreArgs a) {
    const lrqk_layer_t &L = a.L;
    constexpr int N = Pack<T>::N;
    constexpr int R = NPK * N;
    constexpr int U = NPK <= 4 ? 4 : (NPK <= 8 ? 2 : 1);  // tiles in flight per warp
    constexpr int NW = kScoreThreads / 32;
    __shared__ int s_hist[kHistBins];
    __shared__ int s_scan[32];
    __shared__ int s_flag;
    __shared__ int s_out[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int BH = L.batch * L.n_q_heads;
    const int P = a.parts;

    for (int item = blockIdx.x; item < BH * P; item += gridDim.x) {
        const int bh = item / P, part = item - bh * P;
        const int b = bh / L.n_q_heads;
        const int t = L.ctx_len[b];
        if (t >= L.t_max) continue;
        const int n = t + 1;  // scores over tokens 0..t
        const int lite_start = max(0, n - L.lite_budget);
        const int tiles = (n + 31) >> 5;
        const int tpp = (tiles + P - 1) / P;
        const int tile0 = part * tpp, tile1 = min(tiles, tile0 + tpp);
        const int stride = sample_stride(lite_start);
        for (int i = tid; i < kHistBins; i += blockDim.x) s_hist[i] = 0;
        __syncthreads();
        uint32_t *keys = L.keys + (size_t)bh * L.t_max;
        if (a.ext_scores == nullptr) {
            float qv[R];
            const float *qh = L.q_hat + (size_t)bh * L.rank_stride;
#pragma unroll
            for (int e = 0; e < R; ++e) qv[e] = qh[e];
            const uint4 *base = reinterpret_cast<const uint4 *>(reinterpret_cast<const T *>(L.proxy) +
                                                                 (size_t)bh * L.t_max * R);
            for (int tb = tile0 + warp; tb < tile1; tb += NW * U) {
                uint4 x[U][NPK];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int tile = tb + u * NW;
                    if (tile < tile1) {
                        const uint4 *p = base + (size_t)tile * NPK * 32 + lane;
#pragma unroll
                        for (int pk = 0; pk < NPK; ++pk) {
                            uint4 v;
                            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + pk * 32));
                            x[u][pk] = v;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int tile = tb + u * NW;
                    if (tile >= tile1) break;
                    float s0 = 0.f, s1 = 0.f;
#pragma unroll
                    for (int pk = 0; pk < NPK; ++pk) {
                        float f[N];
                        unpack16<T>(x[u][pk], f);
#pragma unroll
                        for (int e = 0; e < N; e += 2) {
                            s0 = fmaf(f[e], qv[pk * N + e], s0);
                            s1 = fmaf(f[e + 1], qv[pk * N + e + 1], s1);
                        }
                    }
                    const int row = tile * 32 + lane;
                    const uint32_t key = score_key(s0 + s1);
                    if (row < n) keys[row] = key;
                    if (row < lite_start && (tile % stride) == 0)
                        atomicAdd(&s_hist[key >> (32 - kHistBits)], 1);
                }
            }
        } else {
            const float *sc = a.ext_scores + (size_t)bh * n;
            for (int row = tile0 * 32 + tid; row < min(n, tile1 * 32); row += blockDim.x) {
                const uint32_t key = score_key(sc[row]);
                keys[row] = key;
                if (row < lite_start && ((row >> 5) % stride) == 0) atomicAdd(&s_hist[key >> (32 - kHistBits)], 1);
            }
        }
        __syncthreads();
        uint32_t *ghist = L.hist + (size_t)bh * kHistLevels * kHistBins;
        for (int i = tid; i < kHistBins; i += blockDim.x)
            if (s_hist[i]) atomicAdd(ghist + i, (uint32_t)s_hist[i]);
        int *cnt = L.counters + (size_t)bh * kCounterInts + C_SCORE;
        if (!last_arrival(cnt, P, &s_flag)) continue;
        // ---- last block of this head: candidate bins ------------------------
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
        __syncthreads();
        int b_hi, b_lo;
        if (stride == 1) {  // exact histogram: the threshold bin itself
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
            meta[M_MODE] = 0;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// K3 (main path): the proxy store streamed through a TMA bulk-copy pipeline.
// One producer warp keeps kStages 1-D bulk copies (cp.async.bulk, completion
// on an mbarrier) in flight; eight consumer warps each score one 32-row tile
// per stage straight out of shared memory (lane = row).  Every byte of the
// proxy store is read exactly once, with no register staging.
// ---------------------------------------------------------------------------
template <typename T, int NPK>
__global__ void __launch_bounds__(32 * (kCW + 1))
score_tma_kernel(const ScoreArgs a) {
    using SS = ScoreStages<NPK>;
    const lrqk_layer_t &L = a.L;
    extern __shared__ __align__(128) uint8_t tsm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(tsm + SS::kStages * SS::kStageBytes);
    uint64_t *empty = full + SS::kStages;
    __shared__ int s_hist[kHistBins];
    __shared__ int s_win[kHistBins];
    __shared__ int s_scan[32];
    __shared__ int s_flag;
    __shared__ int s_out[2];
    __shared__ int s_above;
    trace(40);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int P = a.parts;
    const int bh = blockIdx.x / P, part = blockIdx.x - bh * P;
    const int b = bh / L.n_q_heads;
    const int t = L.ctx_len[b];
    if (t >= L.t_max) return;
    const int n = t + 1;
    const int lite_start = max(0, n - L.lite_budget);
    const int tiles = (n + 31) >> 5;
    const int tpp = (tiles + P - 1) / P;
    const int tile0 = min(tiles, part * tpp), tile1 = min(tiles, tile0 + tpp);
    const int stride = sample_stride(lite_start);
    int *meta = L.sel_meta + (size_t)bh * kMetaInts;
    // hint window (persistent meta written by the previous step's select)
    const bool win = meta[M_HINT_OK] != 0;
    uint32_t klo = 0, kc = 0xFFFFFFFFu;  // set after pdl_wait (the hint scales with this step's q_hat)
    for (int i = tid; i < kHistBins; i += blockDim.x) { s_hist[i] = 0; s_win[i] = 0; }
    if (tid == 0) {
        s_above = 0;
        for (int s2 = 0; s2 < SS::kStages; ++s2) {
            mbar_init(full + s2, 1);
            mbar_init(empty + s2, kCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int it0 = 0;  // stages in flight before the wait (producer lane)
    if (warp == kCW && lane == 0) it0 = score_prefetch_stages<T, NPK>(L, bh, tile0, tile1, t, tsm, full);
    pdl_wait();  // q_hat, the appended proxy row and ctx_len come from compress
    pdl_trigger();
    if (win) hint_window(scaled_hint(meta, qhat_norm(L, bh)), klo, kc);
    score_stream<T, NPK>(L, bh, tile0, tile1, n, lite_start, stride, win, klo, kc, tsm, full, empty, s_hist, s_win,
                         &s_above, it0);
    trace(41);
    __syncthreads();
    score_flush(L, bh, P, part, win, s_hist, s_win, s_above, s_scan);
    int *cnt = L.counters + (size_t)bh * kCounterInts + C_SCORE;
    if (!last_arrival(cnt, P, &s_flag)) return;
    trace(42);
    score_last_block(L, bh, P, win, klo, kc, lite_start, stride, s_hist, s_win, s_scan, s_out);
}

// Radix select over unique composites (exact fallback): returns thr such that
// exactly m elements have comp >= thr.
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
        find_crossing(s_hist, nb, m, s_scan, s_out);
        const int D = s_out[0];
        m -= s_out[1];
        prefix |= (uint64_t)D << shift;
        __syncthreads();
    }
    return prefix;
}


// Exclusive block scan of four 16-bit counters packed in a uint64.
LRQK_DEV uint64_t block_exclusive_scan_u64(uint64_t v, uint64_t *s_warp, uint64_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint64_t w = lane < nw ? s_warp[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nw) s_warp[lane] = w;
    }
    __syncthreads();
    const uint64_t before = warp > 0 ? s_warp[warp - 1] : 0ull;
    *total = s_warp[nw - 1];
    __syncthreads();
    return before + x - v;
}

// ---------------------------------------------------------------------------
// K4 + K5: sure/candidate split with an exact fine histogram of the
// candidate band, then (last block per head) the exact top-k, ascending
// omega, and the cache update.
// ---------------------------------------------------------------------------
constexpr int kLocSure = 1024;  // block-local append buffers (spill to global beyond)
constexpr int kLocCand = 2048;

__global__ void __launch_bounds__(kSelThreads, 2)
select_kernel(const lrqk_layer_t L, int parts) {
    extern __shared__ __align__(16) uint32_t fsm[];
    __shared__ int s_hist[kHistBins];
    __shared__ int s_scan[32];
    __shared__ int s_out[2];
    __shared__ int s_flag;
    __shared__ int s_cnt[4];
    __shared__ uint32_t s_hint_key;
    __shared__ int s_hint_ok;
    const int tid = threadIdx.x, lane = tid & 31, nt = blockDim.x;
    const int BH = L.batch * L.n_q_heads;
    const bool host = L.policy == LRQK_SLOW_HOST;
    pdl_wait();
    pdl_trigger();

    for (int item = blockIdx.x; item < BH * parts; item += gridDim.x) {
        const int bh = item / parts, part = item - bh * parts;
        trace(20);
        const int b = bh / L.n_q_heads;
        const int t = L.ctx_len[b];
        if (t >= L.t_max) continue;
        int *meta = L.sel_meta + (size_t)bh * kMetaInts;
        const int mode0 = meta[M_MODE];
        if (mode0 >= 5) continue;  // select_attend_kernel / score_attend_kernel handled this head
        const int lite_start = meta[M_LITE];
        const int k_eff = meta[M_K_EFF];
        const uint32_t *keys = L.keys + (size_t)bh * L.t_max;
        uint32_t *hist2 = L.hist + (size_t)bh * kHistLevels * kHistBins + kHistBins;
        int *sure = L.sure_idx + (size_t)bh * parts * L.k_budget;  // = this head's part-0 region (mode 3)
        uint64_t *cand = L.cand + (size_t)bh * L.cand_cap;
        // ---- scan part: certain winners, candidates, fine histogram ----------
        if (mode0 == 0) {
            const int b_hi = meta[M_B_HI], b_lo = meta[M_B_LO], s2 = meta[M_S2];
            const int per = ((lite_start + parts - 1) / parts + 3) & ~3;  // 16-byte aligned parts
            const int row0 = min(lite_start, part * per), row1 = min(lite_start, row0 + per);
            int *loc_sure = reinterpret_cast<int *>(fsm);
            uint64_t *loc_cand = reinterpret_cast<uint64_t *>(fsm + kLocSure);
            for (int i = tid; i < kHistBins; i += nt) s_hist[i] = 0;
            if (tid < 4) s_cnt[tid] = 0;
            __syncthreads();
            constexpr int U = 4;  // 16-byte key loads in flight per thread
            for (int base = row0; base < row1; base += nt * 4 * U) {
                uint4 kv4[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = base + (u * nt + tid) * 4;
                    kv4[u] = i < row1 ? __ldcg(reinterpret_cast<const uint4 *>(keys + i)) : make_uint4(0, 0, 0, 0);
                }
                // classify, count, one warp scan per list
                uint32_t sure_m = 0, cand_m = 0;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t kk[4] = {kv4[u].x, kv4[u].y, kv4[u].z, kv4[u].w};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int i = base + (u * nt + tid) * 4 + c;
                        const int bin = (int)(kk[c] >> (32 - kHistBits));
                        if (i < row1 && bin > b_hi) sure_m |= 1u << (u * 4 + c);
                        else if (i < row1 && bin >= b_lo) cand_m |= 1u << (u * 4 + c);
                    }
                }
                if (!__any_sync(0xffffffffu, (sure_m | cand_m) != 0)) continue;
                const int ns_t = __popc(sure_m), nc_t = __popc(cand_m);
                int xs = ns_t, xc = nc_t;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int ys = __shfl_up_sync(0xffffffffu, xs, o), yc = __shfl_up_sync(0xffffffffu, xc, o);
                    if (lane >= o) { xs += ys; xc += yc; }
                }
                int bs = 0, bc = 0;
                if (lane == 31) {
                    bs = xs ? atomicAdd(&s_cnt[0], xs) : 0;
                    bc = xc ? atomicAdd(&s_cnt[1], xc) : 0;
                }
                bs = __shfl_sync(0xffffffffu, bs, 31) + xs - ns_t;
                bc = __shfl_sync(0xffffffffu, bc, 31) + xc - nc_t;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t kk[4] = {kv4[u].x, kv4[u].y, kv4[u].z, kv4[u].w};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int bit = u * 4 + c;
                        const int i = base + (u * nt + tid) * 4 + c;
                        if (sure_m & (1u << bit)) {
                            if (bs < kLocSure) loc_sure[bs] = i;
                            else {  // rare spill: straight to the global list
                                const int g = atomicAdd(meta + M_SURE, 1);
                                if (g < L.k_budget) sure[g] = i;
                            }
                            ++bs;
                        } else if (cand_m & (1u << bit)) {
                            atomicAdd(&s_hist[fine_bin(kk[c], b_lo, s2)], 1);
                            if (bc < kLocCand) loc_cand[bc] = make_comp(kk[c], i);
                            else {
                                const int g = atomicAdd(meta + M_CAND, 1);
                                if (g < L.cand_cap) cand[g] = make_comp(kk[c], i);
                            }
                            ++bc;
                        }
                    }
                }
            }
            __syncthreads();
            const int ns = min(s_cnt[0], kLocSure), nc = min(s_cnt[1], kLocCand);
            if (tid == 0) {
                s_cnt[2] = ns ? atomicAdd(meta + M_SURE, ns) : 0;
                s_cnt[3] = nc ? atomicAdd(meta + M_CAND, nc) : 0;
            }
            __syncthreads();
            for (int j = tid; j < ns; j += nt)
                if (s_cnt[2] + j < L.k_budget) sure[s_cnt[2] + j] = loc_sure[j];
            for (int j = tid; j < nc; j += nt)
                if (s_cnt[3] + j < L.cand_cap) cand[s_cnt[3] + j] = loc_cand[j];
            for (int i = tid; i < kHistBins; i += nt)
                if (s_hist[i]) atomicAdd(hist2 + i, (uint32_t)s_hist[i]);
        }
        if (mode0 == 3) {
            // ---- hint-window path: rows above the critical window bin are
            // certain winners, written per part in ascending order; rows in
            // the critical bin are collected (few) -------------------------
            const uint32_t klo = (uint32_t)meta[M_KLO];
            const int D = meta[M_FBIN];
            const int per = ((lite_start + parts - 1) / parts + 3) & ~3;  // 16-byte aligned parts
            const int row0 = min(lite_start, part * per), row1 = min(lite_start, row0 + per);
            int *psure = L.sure_idx + ((size_t)bh * parts + part) * L.k_budget;
            int out = 0;  // block-uniform running count
            constexpr int U = 4;
            for (int base = row0; base < row1; base += nt * 4 * U) {
                uint4 kv4[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = base + (u * nt + tid) * 4;
                    kv4[u] = i < row1 ? __ldcg(reinterpret_cast<const uint4 *>(keys + i)) : make_uint4(0, 0, 0, 0);
                }
                uint32_t smask = 0;
                uint64_t packed = 0;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t kk[4] = {kv4[u].x, kv4[u].y, kv4[u].z, kv4[u].w};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int i = base + (u * nt + tid) * 4 + c;
                        if (i < row1 && kk[c] >= klo) {
                            const uint32_t dk = kk[c] - klo;
                            if (dk >= kWinKeys || (int)(dk >> kWinShift) > D) {
                                smask |= 1u << (u * 4 + c);
                            } else if ((int)(dk >> kWinShift) == D) {
                                const int g = atomicAdd(meta + M_CAND, 1);
                                if (g < L.cand_cap) cand[g] = make_comp(kk[c], i);
                            }
                        }
                    }
                    packed |= (uint64_t)__popc((smask >> (u * 4)) & 0xFu) << (16 * u);
                }
                uint64_t tot;
                const uint64_t ex = block_exclusive_scan_u64(packed, reinterpret_cast<uint64_t *>(fsm), &tot);
                int off_u = out;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    int o = off_u + (int)((ex >> (16 * u)) & 0xFFFFu);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        if (smask & (1u << (u * 4 + c))) {
                            if (o < L.k_budget) psure[o] = base + (u * nt + tid) * 4 + c;
                            ++o;
                        }
                    }
                    off_u += (int)((tot >> (16 * u)) & 0xFFFFu);
                }
                out = off_u;
            }
            if (tid == 0) hist2[part] = (uint32_t)out;
        }
        trace(21);
        if (!last_arrival(L.counters + (size_t)bh * kCounterInts + C_SELECT, parts, &s_flag)) continue;
        trace(22);

        // ================= finalize (one block per head) =====================
        const int n_words = (lite_start + 31) >> 5;
        const int S = k_eff + (t + 1 - lite_start);  // |omega_k| + |omega_l|
        uint32_t *bitmap = fsm;
        int *newl = reinterpret_cast<int *>(bitmap + ((((L.t_max + 31) >> 5) + 3) & ~3));
        int *prevl = newl + L.s_cap;
        int *prevs = prevl + L.s_cap;
        int *news = prevs + L.s_cap;
        uint32_t *slot_used = reinterpret_cast<uint32_t *>(news + L.s_cap);
        const int slot_words = (L.n_slots + 31) >> 5;
        uint64_t *crit = reinterpret_cast<uint64_t *>(slot_used + ((slot_words + 3) & ~3));
        int *s_sure = reinterpret_cast<int *>(crit + kCritCap);  // [k_budget] mode 3
        int *s_poff = s_sure + L.k_budget;                        // [parts]   mode 3
        // prefetch in one round trip: Omega_{t-1} (+ slots), the fine
        // histogram, the list lengths; clear the bitmap meanwhile
        const int n_prev = L.res_cnt[bh];
        int *res_idx = L.res_idx + (size_t)bh * L.s_cap;
        int *res_slot = L.res_slot + (size_t)bh * L.s_cap;
        for (int i = tid; i < n_prev; i += nt) {
            prevl[i] = __ldcg(res_idx + i);
            if (host) prevs[i] = __ldcg(res_slot + i);
        }
        if (mode0 == 0)
            for (int i = tid; i < kHistBins; i += nt) s_hist[i] = (int)__ldcg(hist2 + i);
        if (tid == 0) { s_hint_key = 0u; s_hint_ok = 0; }
        bool exact_fb = false;  // exact radix fallback over all keys
        bool use_bitmap = false;  // newl comes from the bitmap compaction
        if (mode0 == 1) {
            for (int i = tid; i < k_eff; i += nt) newl[i] = i;  // everything fits
        } else if (mode0 == 3) {
            // ---- hint-window path: sorted per-part sure lists + the critical bin
            trace(26);
            const int nabove = meta[M_NABOVE];
            const int need2 = k_eff - nabove;
            const int n_crit = __ldcg(meta + M_CAND);
            const int pc = tid < parts ? (int)__ldcg(hist2 + tid) : 0;
            int ns_total;
            const int poff = block_exclusive_scan(pc, s_scan, &ns_total);
            if (tid < parts) s_poff[tid] = poff;
            const bool ok = ns_total == nabove && need2 >= 0 && need2 <= n_crit && n_crit <= kCritCap &&
                            n_crit <= L.cand_cap;
            int M = 1;
            while (M < n_crit) M <<= 1;
            __syncthreads();
            if (ok) {
                for (int j = tid; j < ns_total; j += nt) {  // parts are ascending row ranges
                    int lo = 0, hi = parts - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (s_poff[mid] <= j) lo = mid; else hi = mid - 1;
                    }
                    s_sure[j] = __ldcg(L.sure_idx + ((size_t)bh * parts + lo) * L.k_budget + (j - s_poff[lo]));
                }
                for (int i = tid; i < M; i += nt) crit[i] = i < n_crit ? __ldcg(cand + i) : 0ull;
                __syncthreads();
                trace(27);
                block_bitonic(crit, M, true);  // descending composites
                trace(28);
                if (tid == 0) {
                    s_hint_ok = 1;
                    s_hint_key = need2 > 0 ? (uint32_t)(crit[need2 - 1] >> kIdxBits)
                                           : (uint32_t)meta[M_KLO] + ((uint32_t)(meta[M_FBIN] + 1) << kWinShift);
                }
                __syncthreads();
                int M2 = 1;
                while (M2 < need2) M2 <<= 1;
                for (int i = tid; i < M2; i += nt) crit[i] = i < need2 ? (uint64_t)comp_index(crit[i]) : ~0ull;
                __syncthreads();
                block_bitonic(crit, M2, false);  // winners by ascending index
                trace(29);
                // merge the ascending sure list and the ascending winners
                for (int j = tid; j < ns_total; j += nt) {
                    const int x = s_sure[j];
                    int lo = 0, hi = need2;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if ((int)crit[mid] < x) lo = mid + 1; else hi = mid;
                    }
                    newl[j + lo] = x;
                }
                for (int i = tid; i < need2; i += nt) {
                    const int w = (int)crit[i];
                    int lo = 0, hi = ns_total;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (s_sure[mid] < w) lo = mid + 1; else hi = mid;
                    }
                    newl[i + lo] = w;
                }
            } else {
                exact_fb = true;
            }
        } else {
            use_bitmap = true;
            for (int w = tid; w < n_words; w += nt) bitmap[w] = 0u;
            const int n_sure = __ldcg(meta + M_SURE);
            const int n_cand = __ldcg(meta + M_CAND);
            const int need = k_eff - n_sure;
            bool ok = n_sure <= L.k_budget && need >= 0 && need <= n_cand && n_cand <= L.cand_cap;
            if (tid == 0) s_cnt[0] = 0;
            __syncthreads();
            if (ok) {
                for (int i = tid; i < n_sure; i += nt) {
                    const int x = __ldcg(sure + i);
                    atomicOr(&bitmap[x >> 5], 1u << (x & 31));
                }
                if (need > 0) {
                    const int b_lo = meta[M_B_LO], s2 = meta[M_S2];
                    find_crossing(s_hist, kHistBins, need, s_scan, s_out);
                    const int fstar = s_out[0];
                    const int need2 = need - s_out[1];
                    const int n_crit = fstar >= 0 ? s_hist[fstar] : 0;
                    int M = 1;
                    while (M < n_crit) M <<= 1;
                    if (fstar < 0 || M > kCritCap) ok = false;  // uniform
                    if (ok) {
                        for (int i = tid; i < n_cand; i += nt) {
                            const uint64_t c = __ldcg(cand + i);
                            const int f = fine_bin((uint32_t)(c >> kIdxBits), b_lo, s2);
                            if (f > fstar) {
                                const int x = comp_index(c);
                                atomicOr(&bitmap[x >> 5], 1u << (x & 31));
                            } else if (f == fstar) {
                                crit[atomicAdd(&s_cnt[0], 1)] = c;
                            }
                        }
                        __syncthreads();
                        for (int i = n_crit + tid; i < M; i += nt) crit[i] = 0ull;
                        __syncthreads();
                        block_bitonic(crit, M, true);  // descending
                        for (int i = tid; i < need2; i += nt) {
                            const int x = comp_index(crit[i]);
                            atomicOr(&bitmap[x >> 5], 1u << (x & 31));
                        }
                        if (tid == 0 && need2 > 0) {
                            s_hint_ok = 1;
                            s_hint_key = (uint32_t)(crit[need2 - 1] >> kIdxBits);
                        }
                    }
                } else if (tid == 0) {
                    const int b_hi = meta[M_B_HI];
                    s_hint_ok = 1;
                    s_hint_key = b_hi >= kHistBins - 1 ? 0xFFFFFFFFu : (uint32_t)(b_hi + 1) << (32 - kHistBits);
                }
            }
            if (!ok) exact_fb = true;
        }
        if (exact_fb) {
            // exact fallback over the whole key array
            use_bitmap = true;
            __syncthreads();
            for (int w = tid; w < n_words; w += nt) bitmap[w] = 0u;
            if (tid == 0) set_status(L.status, LRQK_ST_FALLBACK);
            auto get = [&](int i) { return make_comp(__ldcg(keys + i), i); };
            const uint64_t thr = radix_top_m(get, lite_start, k_eff, 32 + kIdxBits, s_hist, s_scan, s_out);
            for (int i = tid; i < lite_start; i += nt)
                if (make_comp(__ldcg(keys + i), i) >= thr) atomicOr(&bitmap[i >> 5], 1u << (i & 31));
            if (tid == 0) {
                s_hint_ok = 1;
                s_hint_key = (uint32_t)(thr >> kIdxBits);
            }
        }
        trace(23);
        __syncthreads();
        if (use_bitmap) {
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
        for (int i = tid; i < t + 1 - lite_start; i += nt) newl[k_eff + i] = lite_start + i;  // omega_l

        trace(24);
        // ---- K5: hit/miss against Omega_{t-1} U {t} ---------------------------
        if (host) for (int w = tid; w < slot_words; w += nt) slot_used[w] = 0u;
        __syncthreads();
        const int spare = host ? L.spare_slot[bh] : 0;
        int hits_local = 0;
        if (!host) {
            // |Omega_t ∩ (Omega_{t-1} ∪ {t})| = 1 + #{x in Omega_{t-1} : x in Omega_t}, with
            // membership read straight off the selection bitmap (t is never in Omega_{t-1})
            if (tid == 0) hits_local = 1;
            for (int i = tid; i < n_prev; i += nt) {
                const int x = prevl[i];
                bool in_new = mode0 == 1 || x >= lite_start;
                if (!in_new) {
                    if (use_bitmap) {
                        in_new = (bitmap[x >> 5] >> (x & 31)) & 1u;
                    } else {  // newl[0, k_eff) is ascending
                        int lo = 0, hi = k_eff;
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            if (newl[mid] < x) lo = mid + 1; else hi = mid;
                        }
                        in_new = lo < k_eff && newl[lo] == x;
                    }
                }
                hits_local += in_new ? 1 : 0;
            }
        } else
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
            hits_local += ((x == t) || pos >= 0) ? 1 : 0;
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
            const int per = (S + nt - 1) / nt;
            const int i0 = tid * per;
            int mloc = 0;
            for (int i = i0; i < min(S, i0 + per); ++i) mloc += news[i] < 0;
            int mtot;
            int moff = block_exclusive_scan(mloc, s_scan, &mtot);
            const int fper = (slot_words + nt - 1) / nt;
            const int f0 = tid * fper;
            int floc = 0;
            for (int w = f0; w < min(slot_words, f0 + fper); ++w) {
                uint32_t freew = ~slot_used[w];
                if (w == slot_words - 1 && (L.n_slots & 31)) freew &= (1u << (L.n_slots & 31)) - 1u;
                floc += __popc(freew);
            }
            int ftot;
            int foff = block_exclusive_scan(floc, s_scan, &ftot);
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
                news[i] = s | kSlotMiss;  // fetched by attention_kernel (or lrqk_gather_misses)
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
            if (host) {  // HBM policy: counted by compress_prepare from the residency bitmap
                L.c_miss[bh] += miss;
                L.c_total[bh] += S;
                L.step_miss[bh] = miss;
                L.step_total[bh] = S;
            }
            meta[M_SURE] = 0;
            meta[M_CAND] = 0;
            meta[M_PCRIT] = 0;
            meta[M_HITS] = 0;
            meta[M_HINT] = (int)s_hint_key;
            meta[M_HINT_OK] = s_hint_ok;
            meta[M_HINT_QN] = __float_as_int(qhat_norm(L, bh));
            meta[M_STAT + min(max(mode0, 0), 5)] += 1;
            if (exact_fb) meta[M_STAT + 6] += 1;
        }
        trace(25);
        uint32_t *ghist = L.hist + (size_t)bh * kHistLevels * kHistBins;  // both levels, ready for the next step
        for (int i = tid; i < kHistLevels * kHistBins; i += nt) ghist[i] = 0u;
        __syncthreads();
    }
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

static int score_parts(const lrqk_layer_t &L) {
    const int BH = L.batch * L.n_q_heads;
    const int tiles = (L.t_max + 31) / 32;
    const int want = (num_sms() * 4 + BH - 1) / BH;
    return max(1, min(want, max(1, tiles / 8)));
}

template <typename T>
static int launch_score_t(const ScoreArgs &a, cudaStream_t st) {
    const lrqk_layer_t &L = a.L;
    const int BH = L.batch * L.n_q_heads;
    const int grid = max(1, min(BH * a.parts, num_sms() * 4));
    const int npk = L.rank_stride * (int)sizeof(T) / 16;
    switch (npk) {
        case 1: score_kernel<T, 1><<<grid, kScoreThreads, 0, st>>>(a); break;
        case 2: score_kernel<T, 2><<<grid, kScoreThreads, 0, st>>>(a); break;
        case 4: score_kernel<T, 4><<<grid, kScoreThreads, 0, st>>>(a); break;
        case 8: score_kernel<T, 8><<<grid, kScoreThreads, 0, st>>>(a); break;
        case 16: score_kernel<T, 16><<<grid, kScoreThreads, 0, st>>>(a); break;
        default: return LRQK_EUNSUPPORTED;
    }
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

template <typename T, int NPK>
static void launch_score_tma_t(const ScoreArgs &a, int grid, cudaStream_t st) {
    using SS = ScoreStages<NPK>;
    auto fn = score_tma_kernel<T, NPK>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SS::kSmem);
    launch_kernel(fn, grid, 32 * (kCW + 1), SS::kSmem, st, true, a);
}

// parts (blocks) per head of the TMA score kernel; each owns a contiguous
// tile range and one fcand region
int score_tma_parts(const lrqk_layer_t &L) {
    const int BH = L.batch * L.n_q_heads;
    const int tiles = L.t_max / 32;
    return max(1, min((2 * num_sms()) / BH, max(1, tiles / 64)));
}
int score_part_rows(const lrqk_layer_t &L) { return L.batch * L.n_q_heads * score_tma_parts(L); }

template <typename T>
static int launch_score_tma(const lrqk_layer_t &L, cudaStream_t st) {
    const int BH = L.batch * L.n_q_heads;
    const int P = score_tma_parts(L);
    ScoreArgs a{L, nullptr, P};
    const int grid = BH * P;
    const int npk = L.rank_stride * (int)sizeof(T) / 16;
    switch (npk) {
        case 1: launch_score_tma_t<T, 1>(a, grid, st); break;
        case 2: launch_score_tma_t<T, 2>(a, grid, st); break;
        case 4: launch_score_tma_t<T, 4>(a, grid, st); break;
        case 8: launch_score_tma_t<T, 8>(a, grid, st); break;
        case 16: launch_score_tma_t<T, 16>(a, grid, st); break;
        default: return LRQK_EUNSUPPORTED;
    }
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

int launch_score(const lrqk_layer_t &L, const float *ext_scores, cudaStream_t st) {
    if (ext_scores == nullptr)
        return L.dtype == LRQK_BF16 ? launch_score_tma<__nv_bfloat16>(L, st) : launch_score_tma<float>(L, st);
    ScoreArgs a{L, ext_scores, score_parts(L)};
    return L.dtype == LRQK_BF16 ? launch_score_t<__nv_bfloat16>(a, st) : launch_score_t<float>(a, st);
}

size_t finalize_smem_bytes(const lrqk_layer_t &L) {
    const size_t n_words = ((size_t)L.t_max + 31) / 32;
    const size_t slot_words = ((size_t)L.n_slots + 31) / 32;
    const size_t cand_pow2 = kCritCap;
    const size_t fin = ((n_words + 3) & ~(size_t)3) * 4 + 4 * (size_t)L.s_cap * 4 +
                       ((slot_words + 3) & ~(size_t)3) * 4 + cand_pow2 * 8;
    const size_t mode3 = ((size_t)L.k_budget + 512) * 4;
    const size_t scan = (size_t)kLocSure * 4 + (size_t)kLocCand * 8;
    return fin + mode3 > scan ? fin + mode3 : scan;
}

// select parts per head (one block each); the mode-3 sure lists need one
// k_budget-row region per (head, part)
int score_tma_parts(const lrqk_layer_t &L);
int select_parts(const lrqk_layer_t &L) { return score_tma_parts(L); }  // mode 5 reuses the score partition
int select_sure_rows(const lrqk_layer_t &L) { return L.batch * L.n_q_heads * select_parts(L); }

int launch_select(const lrqk_layer_t &L, cudaStream_t st) {
    const int BH = L.batch * L.n_q_heads;
    const int parts = select_parts(L);
    const int grid = max(1, min(BH * parts, num_sms() * 2));
    const size_t smem = finalize_smem_bytes(L);
    cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_kernel(select_kernel, grid, kSelThreads, smem, st, true, L, parts);
    return cudaGetLastError() == cudaSuccess ? LRQK_OK : LRQK_ECUDA;
}

}  // namespace lrqk
