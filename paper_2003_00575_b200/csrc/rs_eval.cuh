// rs_eval.cuh — instance-scoring support on the GPU: the
// (ground-truth instance, predicted cluster) contingency table behind
// evaluation.match_instances (/root/reference/pkg/src/rangeseg/evaluation.py:65-129)
// for a batch of frames.
//
// The reference counts pairs with np.unique over packed (gt, pred) integers
// (:91-99) and gets the instance / cluster sizes from np.unique as well
// (:83-89).  Here one CTA counts one frame in a shared-memory hash table of
// (gt, pred) keys: a warp first merges equal keys among its lanes
// (__match_any_sync: neighbouring points mostly share their instance and
// cluster), then one lane adds the group's count (linear probing,
// atomicCAS-claimed slots).  Keys that find no slot within kEvalProbe probes
// spill to a per-frame hash table in global memory.  The frame's distinct keys
// are then compacted and sorted (bitonic, in shared memory; in global memory
// for a frame with more distinct pairs than the table holds), a second kernel
// scans the per-frame counts and a third moves every frame's sorted table to
// its place in the output.  Every point with gt > 0 or pred > 0 counts under
// the key (frame << 44 | gt << 22 | pred), so both size tables follow by
// summing rows and columns; the points with gt == pred == 0 are one extra key
// (kEvalNone) at the end.  The per-instance matching over that small table is
// host code in paper_2003_00575_b200/evaluation.py.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace rs {

constexpr int kEvalThreads = 1024;
constexpr int kEvalLabelBits = 22;    // gt ids and cluster labels < 2^22
constexpr int kEvalFrameBits = 19;    // frames < 2^19 (key < 2^63)
constexpr long long kEvalNone = 0x7fffffffffffffffLL;   // points with gt == pred == 0
constexpr unsigned long long kEvalEmpty = ~0ull;         // empty hash slot (sorts last)
constexpr int kEvalTable = 8192;      // shared-memory slots per frame (8 + 4 B each)
constexpr int kEvalProbe = 64;        // probes before a key spills to global memory
constexpr size_t kEvalSmem = (size_t)kEvalTable * 12;

__device__ __forceinline__ uint32_t eval_hash(unsigned long long k) {
    k ^= k >> 29;
    k *= 0xbf58476d1ce4e5b9ull;
    k ^= k >> 32;
    return (uint32_t)k;
}

__device__ __forceinline__ size_t pow2_at_least(size_t n) {
    size_t p = 1;
    while (p < n) p <<= 1;
    return p;
}

// Per-frame scratch of the workspace: a spill hash table and a sort buffer of
// `slots` = pow2_at_least(n_f + 1) entries each, keys in one array (u64) and
// counts in another (u32).  Frame b's scratch starts at entry 4 (offsets[b] + b):
// 2 slots < 4 (n_f + 1) entries fit before the next frame's.
struct EvalScratch {
    unsigned long long *key;   // spill keys [slots], then sorted keys [slots]
    uint32_t *cnt;             // their counts
    size_t slots;
};

__device__ __forceinline__ EvalScratch eval_scratch(unsigned long long *K, uint32_t *C, const int64_t *offsets,
                                                    int b) {
    EvalScratch s;
    const int64_t n = offsets[b + 1] - offsets[b];
    s.slots = pow2_at_least((size_t)n + 1);
    const size_t base = 4 * ((size_t)(offsets[b] - offsets[0]) + (size_t)b);
    s.key = K + base;
    s.cnt = C + base;
    return s;
}

// Bitonic sort of n (a power of two) (key, count) pairs by key; K / C may be
// shared or global memory; called by every thread of the CTA.
template <class KeyT, class CntT>
__device__ __forceinline__ void bitonic_pairs(KeyT *K, CntT *C, size_t n) {
    for (size_t size = 2; size <= n; size <<= 1)
        for (size_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (size_t i = threadIdx.x; i < n / 2; i += blockDim.x) {
                const size_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long a = K[lo], b = K[hi];
                if ((a > b) == up) {
                    K[lo] = b;
                    K[hi] = a;
                    const auto t = C[lo];
                    C[lo] = C[hi];
                    C[hi] = t;
                }
            }
            __syncthreads();
        }
}

// Kernel 1: one CTA per frame.  Writes the frame's sorted distinct keys to the
// start of its sort buffer, their number to frame_n[b], the none count to
// frame_none[b], and ORs 1 into *bad for an out-of-range label.
__global__ void __launch_bounds__(kEvalThreads, 1)
    rs_cont_count_kernel(const int32_t *gt, const int32_t *pred, const int64_t *offsets, unsigned long long *K,
                         uint32_t *C, unsigned long long *frame_n, unsigned long long *frame_none, int *bad) {
    extern __shared__ __align__(16) unsigned char eval_sm[];
    unsigned long long *tk = reinterpret_cast<unsigned long long *>(eval_sm);
    uint32_t *tc = reinterpret_cast<uint32_t *>(tk + kEvalTable);
    __shared__ unsigned long long n_none;
    __shared__ uint32_t n_sm, spilled, n_out;
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    const int64_t p0 = offsets[b], p1 = offsets[b + 1];
    EvalScratch sc = eval_scratch(K, C, offsets, b);
    for (int i = tid; i < kEvalTable; i += blockDim.x) { tk[i] = kEvalEmpty; tc[i] = 0; }
    if (tid == 0) { n_none = 0; n_sm = 0; spilled = 0; n_out = 0; }
    __syncthreads();
    // ---- count
    unsigned long long my_none = 0;
    bool my_bad = false;
    for (int64_t base = p0; base < p1; base += blockDim.x) {
        const int64_t i = base + tid;
        const bool act = i < p1;
        int g = 0, p = 0;
        if (act) {
            g = gt[i];
            p = pred[i];
            my_bad |= g < 0 || p < 0 || g >= (1 << kEvalLabelBits) || p >= (1 << kEvalLabelBits);
        }
        const bool has = act && (g != 0 || p != 0);
        my_none += (act && !has) ? 1u : 0u;
        const unsigned long long key =
            has ? ((unsigned long long)(g & ((1 << kEvalLabelBits) - 1)) << kEvalLabelBits) |
                      (unsigned long long)(p & ((1 << kEvalLabelBits) - 1))
                : kEvalEmpty;
        const uint32_t grp = __match_any_sync(0xffffffffu, key);
        if (!has || lane != __ffs(grp) - 1) continue;
        const uint32_t add = __popc(grp);
        uint32_t h = eval_hash(key) & (kEvalTable - 1);
        bool done = false;
        for (int pr = 0; pr < kEvalProbe && !done; ++pr, h = (h + 1) & (kEvalTable - 1)) {
            unsigned long long k = tk[h];
            if (k == kEvalEmpty) k = atomicCAS(&tk[h], kEvalEmpty, key);
            if (k == kEvalEmpty || k == key) {
                atomicAdd(&tc[h], add);
                done = true;
            }
        }
        if (!done) spilled = 1;   // counted by the spill pass below
    }
    if (__any_sync(0xffffffffu, my_bad) && lane == 0) atomicOr(bad, 1);
    for (int off = 16; off; off >>= 1) my_none += __shfl_xor_sync(0xffffffffu, my_none, off);
    if (lane == 0 && my_none) atomicAdd(&n_none, my_none);
    __syncthreads();
    if (spilled) {
        // rare: a key found neither itself nor a free slot within kEvalProbe
        // probes.  The shared table is frozen now (every key in it is fully
        // counted: any occurrence probes past its slot); the points are read
        // again and the keys missing from it are counted in the frame's global
        // table.
        for (size_t i = tid; i < sc.slots; i += blockDim.x) { sc.key[i] = kEvalEmpty; sc.cnt[i] = 0; }
        __syncthreads();
        for (int64_t base = p0; base < p1; base += blockDim.x) {
            const int64_t i = base + tid;
            const bool act = i < p1;
            const int g = act ? gt[i] : 0, p = act ? pred[i] : 0;
            const bool has = act && (g != 0 || p != 0);
            const unsigned long long key =
                has ? ((unsigned long long)(g & ((1 << kEvalLabelBits) - 1)) << kEvalLabelBits) |
                          (unsigned long long)(p & ((1 << kEvalLabelBits) - 1))
                    : kEvalEmpty;
            const uint32_t grp = __match_any_sync(0xffffffffu, key);
            if (!has || lane != __ffs(grp) - 1) continue;
            uint32_t h = eval_hash(key) & (kEvalTable - 1);
            bool in_table = false;
            for (int pr = 0; pr < kEvalProbe; ++pr, h = (h + 1) & (kEvalTable - 1)) {
                const unsigned long long k = tk[h];
                if (k == key) { in_table = true; break; }
                if (k == kEvalEmpty) break;
            }
            if (in_table) continue;
            size_t sl = eval_hash(key) & (sc.slots - 1);
            while (true) {
                unsigned long long k = sc.key[sl];
                if (k == kEvalEmpty) k = atomicCAS(&sc.key[sl], kEvalEmpty, key);
                if (k == kEvalEmpty || k == key) {
                    atomicAdd(&sc.cnt[sl], (uint32_t)__popc(grp));
                    break;
                }
                sl = (sl + 1) & (sc.slots - 1);
            }
        }
        __syncthreads();
    }
    // ---- compact the shared table's keys to its front (slot order is free: it is sorted next)
    // every thread first reads its slots, then writes after the barrier
    const unsigned long long fb = (unsigned long long)b << (2 * kEvalLabelBits);
    constexpr int kPer = kEvalTable / kEvalThreads;
    unsigned long long mk[kPer];
    uint32_t mc[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        mk[j] = tk[tid * kPer + j];
        mc[j] = tc[tid * kPer + j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPer; ++j)
        if (mk[j] != kEvalEmpty) {
            const uint32_t at = atomicAdd(&n_sm, 1u);
            tk[at] = fb | mk[j];
            tc[at] = mc[j];
        }
    __syncthreads();
    const uint32_t m_sm = n_sm;
    if (!spilled) {
        // common case: sort in shared memory, write the sorted keys to the sort buffer
        size_t n2 = 1;
        while (n2 < m_sm) n2 <<= 1;
        for (size_t i = m_sm + tid; i < n2; i += blockDim.x) { tk[i] = kEvalEmpty; tc[i] = 0; }
        __syncthreads();
        if (m_sm > 1) bitonic_pairs(tk, tc, n2);
        unsigned long long *ok = sc.key + sc.slots;
        uint32_t *oc = sc.cnt + sc.slots;
        for (uint32_t i = tid; i < m_sm; i += blockDim.x) { ok[i] = tk[i]; oc[i] = tc[i]; }
        if (tid == 0) { frame_n[b] = m_sm; frame_none[b] = n_none; }
        return;
    }
    // rare: shared and spilled keys together in the global sort buffer
    unsigned long long *ok = sc.key + sc.slots;
    uint32_t *oc = sc.cnt + sc.slots;
    for (uint32_t i = tid; i < m_sm; i += blockDim.x) { ok[i] = tk[i]; oc[i] = tc[i]; }
    if (tid == 0) n_out = m_sm;
    __syncthreads();
    for (size_t i = tid; i < sc.slots; i += blockDim.x) {
        const unsigned long long k = sc.key[i];
        if (k != kEvalEmpty) {
            const uint32_t at = atomicAdd(&n_out, 1u);
            ok[at] = fb | k;
            oc[at] = sc.cnt[i];
        }
    }
    __syncthreads();
    const uint32_t m = n_out;
    size_t n2 = 1;
    while (n2 < m) n2 <<= 1;   // <= slots: m <= n_f < slots
    for (size_t i = m + tid; i < n2; i += blockDim.x) { ok[i] = kEvalEmpty; oc[i] = 0; }
    __syncthreads();
    bitonic_pairs(ok, oc, n2);
    if (tid == 0) { frame_n[b] = m; frame_none[b] = n_none; }
}

// Kernel 2: one CTA.  Exclusive scan of the per-frame key counts into
// frame_off, the status words and the none key at the end.
__global__ void __launch_bounds__(1024)
    rs_cont_scan_kernel(int B, const unsigned long long *frame_n, const unsigned long long *frame_none,
                        unsigned long long *frame_off, int64_t *pairs, int64_t *counts, int64_t *status,
                        const int *bad) {
    __shared__ unsigned long long carry;
    __shared__ unsigned long long wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry = 0;
    unsigned long long none = 0;
    __syncthreads();
    for (int base = 0; base < B; base += blockDim.x) {
        const int i = base + tid;
        const unsigned long long v = i < B ? frame_n[i] : 0;
        none += i < B ? frame_none[i] : 0;
        unsigned long long inc = v;
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, off);
            if (lane >= off) inc += t;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            unsigned long long s = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
            for (int off = 1; off < 32; off <<= 1) {
                const unsigned long long t = __shfl_up_sync(0xffffffffu, s, off);
                if (lane >= off) s += t;
            }
            wsum[lane] = s;   // inclusive over warps
        }
        __syncthreads();
        const unsigned long long before = carry + (warp ? wsum[warp - 1] : 0) + inc - v;
        if (i < B) frame_off[i] = before;
        __syncthreads();
        if (tid == blockDim.x - 1) carry = before + v;
        __syncthreads();
    }
    for (int off = 16; off; off >>= 1) none += __shfl_xor_sync(0xffffffffu, none, off);
    if (lane == 0) wsum[warp] = none;
    __syncthreads();
    if (tid == 0) {
        unsigned long long tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += wsum[w];
        unsigned long long n = carry;
        if (tot) {
            pairs[n] = kEvalNone;
            counts[n] = (int64_t)tot;
            ++n;
        }
        status[0] = (int64_t)n;
        status[1] = *bad ? 1 : 0;
    }
}

// Kernel 3: frame b's sorted keys to their place in the output.
__global__ void __launch_bounds__(256)
    rs_cont_move_kernel(const int64_t *offsets, const unsigned long long *K, const uint32_t *C,
                        const unsigned long long *frame_n, const unsigned long long *frame_off, int64_t *pairs,
                        int64_t *counts) {
    const int b = blockIdx.x;
    const EvalScratch sc = eval_scratch(const_cast<unsigned long long *>(K), const_cast<uint32_t *>(C), offsets, b);
    const unsigned long long *ok = sc.key + sc.slots;
    const uint32_t *oc = sc.cnt + sc.slots;
    const unsigned long long s = frame_off[b], m = frame_n[b];
    for (unsigned long long i = threadIdx.x; i < m; i += blockDim.x) {
        pairs[s + i] = (int64_t)ok[i];
        counts[s + i] = (int64_t)oc[i];
    }
}

}  // namespace rs
