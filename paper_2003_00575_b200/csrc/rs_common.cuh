// rs_common.cuh — shared device code: kernel arguments, the float32 decision
// rules of the reference, bit helpers, TMA/mbarrier wrappers, phase markers.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "../../include/rangeseg_b200.h"

namespace cg = cooperative_groups;

namespace rs {

constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kFlag = 0x80000000u;

struct KArgs {
    const float *ranges;
    const float *tables;
    int32_t *labels;
    int32_t *ncl;
    int64_t *sizes;
    int64_t sizes_stride;
    int H, W, R, C, SH, WPR;      // WPR = 32-bit words per row (rows are word-aligned)
    int n_off;
    int dy[RS_MAX_OFFSETS];
    int dx[RS_MAX_OFFSETS];
    int min_points, ground;
    float dmax2, mount, keep_above, tch;
    unsigned long long magicWPR;  // ceil(2^40 / WPR): exact w / WPR for w*WPR < 2^40
    int nwords;                   // R * WPR
    // shared-memory layout (32-bit words); meaning depends on the kernel
    int o_P, o_L, o_U, o_SB, o_RS, o_Ph, o_Lh, o_MC, o_TL, o_LR, o_K, o_E, o_SZ;
    int NC, SHN;                  // fast kernel: run-node capacity per band, id bits
    int use_tma;                  // dense kernel: stage rows with TMA bulk copies
    int stop_after;               // experiments only (RS_EXPERIMENTS builds): leave the fast kernel after phase N
    uint32_t *planes;             // debug export (rs_fast_planes): the fast kernel's bit planes after step B, or NULL
    int udyn;                     // fast kernel: dynamic edge grabbing in the local unions (clusters of >= 2 bands)
    int ring;                     // fast kernel (RS_TMA_RING builds): slots of each warp's TMA row ring in step A, 0 = off
};

// ------------------------------------------------------------ phase markers
constexpr int kProfSlots = 24;   // clock64 marks 0-15 and 19-23, [16] start / [17] end globaltimer, [18] SM id
constexpr int kProfCtas = 8192;
#ifdef RS_PHASE_PROF
__device__ long long g_prof[kProfCtas * kProfSlots];
#define RS_MARK(i)                                                             \
    do {                                                                       \
        if (threadIdx.x == 0 && blockIdx.x < kProfCtas) {                      \
            ::rs::g_prof[blockIdx.x * kProfSlots + (i)] = clock64();           \
            if ((i) == 0 || (i) == 15) {                                       \
                unsigned long long gt;                                         \
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));         \
                ::rs::g_prof[blockIdx.x * kProfSlots + 16 + ((i) == 15)] = gt; \
            }                                                                  \
            if ((i) == 0) {                                                    \
                unsigned smid;                                                 \
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));              \
                ::rs::g_prof[blockIdx.x * kProfSlots + 18] = smid;             \
            }                                                                  \
        }                                                                      \
    } while (0)
#else
#define RS_MARK(i) \
    do {           \
    } while (0)
#endif

// ------------------------------------------------------------ bounds checks
// RS_CHECKED builds (scripts/gpu_checked.sh) trap on any out-of-range index
// into shared memory, DSMEM or the outputs — the substitute for
// compute-sanitizer memcheck, which this GPU pool does not allow.
#ifdef RS_CHECKED
#include <cstdio>
#define RS_CHECK(cond, what)                                                                                 \
    do {                                                                                                   \
        if (!(cond)) {                                                                                     \
            printf("RS_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, blockIdx.x, \
                   threadIdx.x);                                                                           \
            __trap();                                                                                      \
        }                                                                                                  \
    } while (0)
#else
#define RS_CHECK(cond, what) \
    do {                     \
    } while (0)
#endif

// ---------------------------------------------------------------- arithmetic

// pair_distance_sq (connectivity.py:54) compared with d_max_sq: five separately
// rounded float32 ops.  The >=0 clamp (:55) cannot change the decision.
__device__ __forceinline__ bool pair_pass(float d1, float d2, float c, float thr) {
    const float a = __fmul_rn(d1, d1);
    const float b = __fmul_rn(d2, d2);
    const float s = __fadd_rn(a, b);
    const float p = __fmul_rn(d1, d2);
    const float q = __fmul_rn(c, p);
    return __fsub_rn(s, q) <= thr;
}

// Row constants of the ground rule for cell row r (pair kk = max(r,1)-1).
struct GroundRow {
    float sa, ca, lo, hi, sc;
};

__device__ __forceinline__ GroundRow ground_row(const KArgs &a, int r) {
    const float *t = a.tables;
    const int H = a.H;
    const int kk = (r >= 1 ? r : 1) - 1;
    GroundRow g;
    g.sa = __ldg(t + H + kk);
    g.ca = __ldg(t + 2 * H - 1 + kk);
    g.lo = __ldg(t + 3 * H - 2 + kk);
    g.hi = __ldg(t + 4 * H - 3 + kk);
    g.sc = __ldg(t + r);
    return g;
}

// Ground decision of a valid cell with range v (ground.py:112-140,
// range_image.py:125-127): d1/d2 are the upper/lower ranges of the row's
// pair.  The tangent bounds are multiplied through by the denominator (never
// divided), with the interval flipped when it is negative.
__device__ __forceinline__ bool ground_rule(const KArgs &a, const GroundRow &g, float d1, float d2, float v) {
    const float num = __fmul_rn(d2, g.sa);
    const float den = __fsub_rn(d1, __fmul_rn(d2, g.ca));
    const float L = __fmul_rn(g.lo, den);
    const float U = __fmul_rn(g.hi, den);
    const bool okp = num >= L && num <= U;
    const bool okn = num <= L && num >= U;
    const bool ok = (den > 0.f ? okp : okn) && den != 0.f && d1 > 0.f && d2 > 0.f;
    const float z = __fadd_rn(__fmul_rn(v, g.sc), a.mount);
    return ok && z <= a.keep_above;
}

// The height test z = v*sc + mount <= keep_above (two rounded ops) as one
// product against a per-row threshold: both rounded ops are monotone in v, so
// the cells passing are {v <= T} (sc > 0), {v >= T} (sc < 0) or all / none
// (sc == 0, or no finite v at the boundary).  cond(v) == (v * zs <= zt) with
// zs in {1, -1, 0}; T is found by bisection over float bit patterns with the
// reference's exact ops.  Valid for finite v >= 0 (the range contract).
__device__ __forceinline__ bool z_pass(float v, float sc, float mount, float keep) {
    return __fadd_rn(__fmul_rn(v, sc), mount) <= keep;
}

__device__ inline void z_threshold(float sc, float mount, float keep, float &zs, float &zt) {
    const float vmax = __int_as_float(0x7f7fffff);
    const bool at0 = z_pass(0.f, sc, mount, keep), atmax = z_pass(vmax, sc, mount, keep);
    if (!(sc > 0.f || sc < 0.f) || at0 == atmax) {   // constant over [0, FLT_MAX]
        zs = 0.f;
        zt = at0 ? 0.f : -1.f;
        return;
    }
    // The boundary is within a few ulps of (keep - mount) / sc: bracket it
    // by walking ulps from that estimate (bit patterns of non-negative floats
    // are ordered), then bisect whatever bracket remains.  Invariant:
    // f(lo) == at0, f(hi) == atmax.
    int lo = 0, hi = 0x7f7fffff;
    {
        const double est = ((double)keep - (double)mount) / (double)sc;
        int t = est <= 0.0 ? 0 : est >= 3.0e38 ? 0x7f7fffff : __float_as_int((float)est);
        t = max(0, min(t, 0x7f7fffff));
        for (int i = 0; i < 8; ++i) {
            const int a = max(0, t - 1), b = min(0x7f7fffff, t + 1);
            if (z_pass(__int_as_float(a), sc, mount, keep) == at0) lo = max(lo, a); else { hi = min(hi, a); t = a - 1; continue; }
            if (z_pass(__int_as_float(b), sc, mount, keep) != at0) { hi = min(hi, b); break; }
            lo = max(lo, b);
            t = b + 1;
        }
    }
    while (hi - lo > 1) {
        const int mid = lo + (hi - lo) / 2;
        if (z_pass(__int_as_float(mid), sc, mount, keep) == at0) lo = mid; else hi = mid;
    }
    if (at0) { zs = 1.f; zt = __int_as_float(lo); }     // passes for v <= lo
    else { zs = -1.f; zt = -__int_as_float(hi); }       // passes for v >= hi
}

// Ground decision for BitsStrip with the row constants in registers:
//  * window: [L, U] = [lo, hi] * den is ordered for den > 0 and reversed for
//    den < 0 (the reference's two branches); with |den| the bounds are
//    |L|, |U| exactly (round-to-nearest is sign-symmetric) and the test is
//    lo*|den| <= num*sign(den) <= hi*|den|; den == 0 fails either way;
//  * only the partner range `other` needs the > 0 test: the cell's own range
//    v > 0 is part of the presence predicate this result is combined with;
//  * the height test is z_threshold's single product.
__device__ __forceinline__ bool ground_fast(float sa, float ca, float lo, float hi, float zs, float zt, float d1,
                                            float d2, float v, float other) {
    const float num = __fmul_rn(d2, sa);
    const float den = __fsub_rn(d1, __fmul_rn(d2, ca));
    const float ad = fabsf(den);
    const float L = __fmul_rn(lo, ad);
    const float U = __fmul_rn(hi, ad);
    const float ns = __int_as_float(__float_as_int(num) ^ (__float_as_int(den) & 0x80000000));
    return (L <= ns) & (ns <= U) & (den != 0.f) & (other > 0.f) & (__fmul_rn(v, zs) <= zt);
}

// Presence = valid && !ground for cell (r, c); `get(row, col)` returns the range.
template <class Get>
__device__ __forceinline__ bool present_at(const KArgs &a, int r, int c, Get get) {
    const float v = get(r, c);
    if (!(v > 0.f)) return false;
    if (!a.ground) return true;
    const int kk = (r >= 1 ? r : 1) - 1;
    return !ground_rule(a, ground_row(a, r), get(kk, c), get(kk + 1, c), v);
}

// Input contract of from_ranges (range_image.py:47-54): finite and >= 0
// (-0.0 passes: it is not < 0).
__device__ __forceinline__ bool range_ok(float v) { return v >= 0.f && v <= 3.4028234663852886e38f; }

// Fast screen for the contract: the unsigned maximum of the raw bits of the
// ranges seen exceeds FLT_MAX's bits iff some value is +inf, NaN or has its
// sign bit set (a violation, or -0.0, which passes: range_ok re-checks).
constexpr uint32_t kMaxFiniteBits = 0x7f7fffffu;

__device__ __forceinline__ int divWPR(const KArgs &a, int w) {
    return (int)(((unsigned long long)(unsigned)w * a.magicWPR) >> 40);
}

__device__ __forceinline__ uint32_t lanemask_le(int lane) {
    return lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
}

// Run id of cell bit b of word w (fast kernel): runs started at or before the
// cell in this word, plus the runs started before the word.
__device__ __forceinline__ uint32_t run_of(const uint32_t *SB, const uint32_t *NB, int w, int b) {
    RS_CHECK(w >= 0 && b >= 0 && b < 32, "run_of word/bit");
    return NB[w] + __popc(SB[w] & lanemask_le(b)) - 1u;
}

// ------------------------------------------------------------- TMA staging

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// ordered against the mbarrier waits of the TMA row ring (never hoisted or merged)
__device__ __forceinline__ uint32_t lds_u32v(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(x), "r"(y), "r"(z), "r"(w)
                 : "memory");
}

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(phase)
            : "memory");
    }
}

__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

}  // namespace rs
