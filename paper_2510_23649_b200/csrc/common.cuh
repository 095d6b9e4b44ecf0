// Shared device helpers for the LRQK sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/lrqk_b200.h"

#define LRQK_DEV __device__ __forceinline__

namespace lrqk {

constexpr int kHistBits = 11;
constexpr int kHistBins = 1 << kHistBits;  // 2048 bins on the top 11 key bits
constexpr int kMetaInts = 48;
constexpr int kPartHist = 2048 + 1 + 1;  // per score part: window histogram + count above (+pad)
constexpr int kCandPart = kPartHist / 2;  // fcand uint64 entries per score part
constexpr int kHistLevels = 3;   // per head: coarse | band fine (mode 0) or part counts (mode 3) | hint window
constexpr int kCounterInts = 8;
constexpr int kRedRows = 384;      // resident rows per compression partial
constexpr int kAttnRows = 128;     // selected rows per attention split

// sel_meta layout, per (b, h)
enum Meta : int {
    M_THR_BIN = 0,     // radix bin holding the k-th largest candidate
    M_N_ABOVE = 1,     // candidates in bins above it
    M_N_BIN = 2,       // candidates in that bin
    M_K_EFF = 3,       // min(k_budget, lite_start)
    M_LITE = 4,        // lite_start
    M_SURE = 5,        // sure list length (atomic)
    M_CAND = 6,        // candidate list length (atomic)
    M_MODE = 7,        // 0 sampled radix path, 1 everything fits, 3 hint window + scan, 5 hint window, direct writes
    // 8..11: mode-0 band (select.cu MetaExt)
    M_HINT = 16,       // persistent: key of the previous step's k-th largest score
    M_HINT_OK = 17,    // persistent: M_HINT is valid
    M_KLO = 18,        // this step's hint window start (key)
    M_FBIN = 19,       // mode 3: window bin holding the k-th largest
    M_NABOVE = 20,     // mode 3: rows strictly above that bin (all sure)
    M_ABOVE = 21,      // rows above the hint window (atomic, score kernel)
    M_SPARTS = 22,     // mode 5: score parts of this head
    M_HITS = 23,       // mode 5: hits among Omega_{t-1} outside the threshold bin
    M_PCRIT = 24,      // mode 5: Omega_{t-1} rows inside the threshold bin (atomic count)
    M_PCRIT_LIST = 25, // mode 5: ... their indices (kPrevCrit)
    M_STAT = 33,       // persistent: head-steps finalized per mode (33 + mode, modes 0..5; 39: exact fallbacks)
    M_BITS_FRESH = 40, // res_bits already holds res_idx (set by seed; prepare then skips the hit count)
    M_YG = 41,         // Y|G partial slots written by select_attend this step (0: cluster reduce does it)
    M_YG_ADD = 42,     // bin-D winners (res_idx[M_NABOVE, +n)) whose Y|G the finish kernel adds
    M_ATT_PARTS = 43,  // softmax partials select_attend left for attention_kernel to merge (parts + 1)
    M_KC = 44,         // this step's candidate bound (key) of cmask; 0xFFFFFFFF: no mask
    M_YG_FOLD = 45,    // attention_kernel already summed the M_YG slots into slot 0
    M_HINT_QN = 46,    // persistent: |q_hat| (f32 bits) of the step that set M_HINT
    M_QN = 47,         // |q_hat| (f32 bits) of this step, written by compress
};
constexpr int kPrevCrit = 8;
// Host policy: select_kernel marks the fast-tier slots of this step's misses
// in res_slot with this bit; the attention kernel reads those rows straight
// from the pinned host tier (zero-copy), stores them into their slots and
// clears the bit (lrqk_gather_misses does the same copy as a separate pass).
constexpr int kSlotMiss = 1 << 30;

// attention partial slots per head (attention splits, or select_attend parts)
// attention partial slots per head: attention splits, or select_attend's
// parts plus its last block
LRQK_DEV int attn_slots_dev(const lrqk_layer_t &L, int parts) {
    const int splits = (L.s_cap + kAttnRows - 1) / kAttnRows;
    return splits > parts + 1 ? splits : parts + 1;
}

// compress_prepare reductions, per head: `yg_slots` partials of
// [Y = A_res^T K_res (R x d) | G = A_res^T A_res (R x R)], summed by the
// finish kernel.  select_attend writes one per score part plus one for the
// threshold-bin winners (meta M_YG = slots used); otherwise the cluster
// reduce writes slot 0.  yg_slots is computed on the host (capi.cu).
__host__ __device__ inline size_t yg_part_floats(int R, int d) { return (size_t)R * d + (size_t)R * R; }

enum Counter : int { C_COMPRESS = 0, C_SCORE = 1, C_ATTN = 2, C_SELECT = 3, C_PREPARE = 4, C_FUSED = 5, C_POOL = 6 };

// ---------------------------------------------------------------------------
// vector loads: 16 bytes of storage -> float lanes
// ---------------------------------------------------------------------------
template <typename T> struct Pack;
template <> struct Pack<float> {
    static constexpr int N = 4;
    LRQK_DEV static void load(const float *p, float (&o)[4]) {
        float4 v = *reinterpret_cast<const float4 *>(p);
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
    LRQK_DEV static void load_nc(const float *p, float (&o)[4]) {
        float4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
    LRQK_DEV static void store(float *p, const float (&o)[4]) {
        *reinterpret_cast<float4 *>(p) = make_float4(o[0], o[1], o[2], o[3]);
    }
    LRQK_DEV static float cvt(float x) { return x; }
    LRQK_DEV static float to_f(float x) { return x; }
};
template <> struct Pack<__nv_bfloat16> {
    static constexpr int N = 8;
    LRQK_DEV static void unpack(uint4 v, float (&o)[8]) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            o[2 * i] = __uint_as_float(w[i] << 16);
            o[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
        }
    }
    LRQK_DEV static void load(const __nv_bfloat16 *p, float (&o)[8]) {
        unpack(*reinterpret_cast<const uint4 *>(p), o);
    }
    LRQK_DEV static void load_nc(const __nv_bfloat16 *p, float (&o)[8]) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
        unpack(v, o);
    }
    LRQK_DEV static void store(__nv_bfloat16 *p, const float (&o)[8]) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            __nv_bfloat162 h = __floats2bfloat162_rn(o[2 * i], o[2 * i + 1]);
            w[i] = *reinterpret_cast<uint32_t *>(&h);
        }
        *reinterpret_cast<uint4 *>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    LRQK_DEV static __nv_bfloat16 cvt(float x) { return __float2bfloat16_rn(x); }
    LRQK_DEV static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
};

template <typename T> LRQK_DEV void unpack16(uint4 v, float (&o)[Pack<T>::N]);
template <> LRQK_DEV void unpack16<float>(uint4 v, float (&o)[4]) {
    o[0] = __uint_as_float(v.x); o[1] = __uint_as_float(v.y);
    o[2] = __uint_as_float(v.z); o[3] = __uint_as_float(v.w);
}
template <> LRQK_DEV void unpack16<__nv_bfloat16>(uint4 v, float (&o)[8]) { Pack<__nv_bfloat16>::unpack(v, o); }

// Proxy-store layout: rows are interleaved in tiles of 32, so that the 16-byte
// pack p of rows 32*i .. 32*i+31 is one contiguous 512-byte run:
//     pack index(row, p) = ((row / 32) * packs_per_row + p) * 32 + row % 32
// The proxy-score GEMV then has lane = row and every warp load fully
// coalesced; a single row (gathered by index) is packs_per_row 16-byte pieces.
LRQK_DEV size_t proxy_pack_offset(int row, int p, int packs_per_row) {
    return ((size_t)(row >> 5) * packs_per_row + p) * 32 + (row & 31);
}

template <typename T> LRQK_DEV T from_float(float x);
template <> LRQK_DEV float from_float<float>(float x) { return x; }
template <> LRQK_DEV __nv_bfloat16 from_float<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <typename T> LRQK_DEV float to_float(T x);
template <> LRQK_DEV float to_float<float>(float x) { return x; }
template <> LRQK_DEV float to_float<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

// ---------------------------------------------------------------------------
// order-preserving float -> uint32 key; -0.0 is canonicalised to +0.0 so that
// the two compare equal, as numpy's argsort sees them.
// ---------------------------------------------------------------------------
LRQK_DEV uint32_t score_key(float x) {
    uint32_t u = __float_as_uint(x);
    if (u == 0x80000000u) u = 0u;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
LRQK_DEV float key_score(uint32_t k) {
    uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    return __uint_as_float(u);
}

LRQK_DEV float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
LRQK_DEV float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <int W> LRQK_DEV float group_sum(float v) {
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

LRQK_DEV void set_status(uint32_t *st, uint32_t bits) {
    if (st) atomicOr(st, bits);
}

// Block-wide exclusive scan of one int per thread (blockDim.x <= 1024).
// `warp_tot` must hold 32 ints of shared memory.  Returns the exclusive
// prefix; *total receives the block sum.
LRQK_DEV int block_exclusive_scan(int v, int *warp_tot, int *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int w = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nw) warp_tot[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    int base = wid ? warp_tot[wid - 1] : 0;
    int res = base + x - v;
    int tot = warp_tot[nw - 1];
    __syncthreads();
    if (total) *total = tot;
    return res;
}

// "last block to arrive" detection for per-head multi-CTA reductions.
// All threads of the block must call it; returns true in exactly one block
// per group once `expected` blocks have arrived, and re-arms the counter.
LRQK_DEV bool last_arrival(int *counter, int expected, int *s_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        int prev = atomicAdd(counter, 1);
        int last = (prev == expected - 1);
        if (last) {
            atomicExch(counter, 0);
            __threadfence();
        }
        *s_flag = last;
    }
    __syncthreads();
    return *s_flag != 0;
}

}  // namespace lrqk

// ---------------------------------------------------------------------------
// Programmatic dependent launch.  The decode chain (compress -> score ->
// select -> attention, layer after layer) is launched with programmatic
// stream serialization: a kernel's blocks may start while its predecessor
// is still running, do work that only depends on older kernels, then
// pdl_wait() until the predecessor has completed and its writes are
// visible.  Every kernel calls pdl_trigger() only after its own pdl_wait(),
// so when a kernel's prologue runs, everything before its predecessor has
// completed.  Both are no-ops for kernels launched without the attribute.
// ---------------------------------------------------------------------------
namespace lrqk {
LRQK_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
LRQK_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();  // capi.cu: on unless LRQK_PDL=0

template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
}  // namespace lrqk

// ---------------------------------------------------------------------------
// mbarrier + 1-D TMA bulk copy (cp.async.bulk) helpers
// ---------------------------------------------------------------------------
namespace lrqk {
LRQK_DEV uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
LRQK_DEV void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
LRQK_DEV void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
LRQK_DEV void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
LRQK_DEV void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
    } while (!ok);
}
LRQK_DEV void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// same, with an L2 eviction policy (createpolicy)
LRQK_DEV void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t policy) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
LRQK_DEV uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
LRQK_DEV uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// L2 prefetches that survive an evict-first stream: a bulk range with a cache
// policy, and one line with evict-last priority
LRQK_DEV void bulk_prefetch_l2_hint(const void *p, uint32_t bytes, uint64_t policy) {
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(policy)
                 : "memory");
}
LRQK_DEV void prefetch_l2_last(const void *p) {
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}
LRQK_DEV void st_hint_u32(uint32_t *p, uint32_t v, uint64_t policy) {
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(policy) : "memory");
}
}  // namespace lrqk

// ---------------------------------------------------------------------------
// Development tracing: when g_lrqk_trace_on is set (lrqk_trace_enable),
// thread 0 of a block stores (tag, block, %globaltimer) into a fixed slot
// per (block, tag) -- a plain store, so tracing adds no round trip to the
// critical path.  Off by default.
// ---------------------------------------------------------------------------
namespace lrqk {
constexpr int kTraceCap = 1 << 16;
extern __device__ int g_lrqk_trace_on;
extern __device__ unsigned long long g_lrqk_trace[kTraceCap][2];
LRQK_DEV void trace(int tag) {
#ifdef LRQK_NO_TRACE
    (void)tag;
    return;
#endif
    if (threadIdx.x == 0 && g_lrqk_trace_on) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        const unsigned blk = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        const unsigned i = ((blk & 1023u) << 6) | (unsigned)(tag & 63);
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_lrqk_trace[i][0] = ((unsigned long long)tag << 48) | ((unsigned long long)(smid & 0xFFFFu) << 32) | blk;
        g_lrqk_trace[i][1] = t;
    }
}
}  // namespace lrqk
