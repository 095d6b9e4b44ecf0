// Selection helpers shared by select.cu (K3/K4) and select_attend.cu (K4+K6).
#pragma once
#include "common.cuh"

namespace lrqk {

// Scores become order-preserving uint32 keys (-0.0 == +0.0); every row gets
// the unique composite  comp = key(32) || (2^21 - 1 - index)(21), which
// orders exactly like (score desc, index asc) -- the reference tie rule
// (linalg.py:96-110).
constexpr int kIdxBits = 21;        // tokens per head < 2^21
constexpr uint32_t kIdxMax = (1u << kIdxBits) - 1u;

// Hint window (modes 3 and 5): an exact histogram of the keys in
// [klo, klo + kWinKeys), centred on the previous step's k-th largest key.
// kWinKeys = 2^25 keys = two octaves of |score| either side; 2048 bins of
// 2^14 keys (1/512 octave), so the bin holding this step's k-th largest
// usually has a handful of rows and no second level is needed.
constexpr uint32_t kWinKeys = 1u << 25;
constexpr int kWinShift = 14;
constexpr int kCritCap = 4096;  // critical bin sorted in shared memory (larger -> exact fallback)
constexpr int kFCrit = 256;     // threshold-bin rows of the fused path (more -> the general select path)
// Candidate bound of the fused path: the score kernel marks (cmask) every
// row whose key is at least hint - kCandBelow (half an octave of |score|
// under the previous threshold); when this step's threshold bin starts at
// or above that bound, the selection only needs the marked rows' keys.
constexpr uint32_t kCandBelow = 1u << 22;

LRQK_DEV uint64_t make_comp(uint32_t key, int idx) {
    return ((uint64_t)key << kIdxBits) | (uint64_t)(kIdxMax - (uint32_t)idx);
}
LRQK_DEV int comp_index(uint64_t c) { return (int)(kIdxMax - (uint32_t)(c & kIdxMax)); }

// |q_hat| of head bh this step (the hint's scale reference), as compress
// left it in sel_meta; 0 when no compress ran (standalone selection)
LRQK_DEV float qhat_norm(const lrqk_layer_t &L, int bh) {
    if (L.q_hat == nullptr) return 0.f;
    return __int_as_float(L.sel_meta[(size_t)bh * kMetaInts + M_QN]);
}

// This step's threshold hint: the previous step's k-th largest score, scaled
// by |q_hat_t| / |q_hat_{t-1}| (every proxy score is linear in q_hat, so a
// change of its norm moves all scores, and the threshold, by that factor),
// as a key.  The hint window is centred on it; without a stored norm the
// previous key is used as is.
LRQK_DEV uint32_t scaled_hint(const int *meta, float qn_now) {
    const uint32_t hk = (uint32_t)meta[M_HINT];
    const float qn0 = __int_as_float(meta[M_HINT_QN]);
    if (!(qn0 > 0.f) || !(qn_now > 0.f) || !isfinite(qn0) || !isfinite(qn_now)) return hk;
    const float sc = key_score(hk) * (qn_now / qn0);
    return isfinite(sc) ? score_key(sc) : hk;
}

// klo (hint window start) and kc (candidate bound) around the hint key
LRQK_DEV void hint_window(uint32_t hk, uint32_t &klo, uint32_t &kc) {
    klo = hk > kWinKeys / 2 ? hk - kWinKeys / 2 : 0u;
    if (klo > 0xFFFFFFFFu - (kWinKeys - 1)) klo = 0xFFFFFFFFu - (kWinKeys - 1);
    kc = max(klo, hk > kCandBelow ? hk - kCandBelow : 0u);
}

LRQK_DEV int n_words_of(int rows) { return (rows + 31) >> 5; }

// Bitonic sort of a[0, M) in shared memory (M a power of two), whole block.
static __device__ __noinline__ void block_bitonic(uint64_t *a, int M, bool descending) {
    for (int kk = 2; kk <= M; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < M; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t x = a[i], y = a[ixj];
                    const bool first_big = ((i & kk) == 0) == descending;
                    if (first_big ? (x < y) : (x > y)) { a[i] = y; a[ixj] = x; }
                }
            }
            __syncthreads();
        }
    }
}

}  // namespace lrqk
