// rangeseg_b200.cu — fused range-image segmentation for sm_100a.
//
// One thread-block CLUSTER per frame, one CTA per band of R rows spanning the
// full azimuth width (so the 360-degree seam is CTA-local).  Per CTA:
//
//   1. TMA 1-D bulk copy (cp.async.bulk + mbarrier) of rows [r0-2, r0+R) of
//      the frame into shared memory (the halo rows feed the ground test and
//      the up edges).
//   2. Presence bits P = valid & !ground for the band and the halo row above
//      (ground.py:95-141, range_image.py:118-127), packed with __ballot_sync.
//   3. Edge bits: LEFT (horizontal, connectivity.py:80-84), seam, UP
//      (vertical, :86-90) and one bit per Map Connection offset
//      (map_connections.py:151-170), all in float32 with one rounding per op
//      (__fmul_rn/__fadd_rn/__fsub_rn: FMA contraction would flip decisions,
//      SURVEY.md finding 3).
//   4. Union-find over the band in shared memory: run starts from the LEFT
//      bits (ballot/clz), then atomicMin hooking for the remaining edges with
//      redundant-edge skipping, then a local flatten.
//   5. Cross-band unions over distributed shared memory (DSMEM) of the
//      cluster: atomicMin hooking with path halving across CTAs.
//   6. Roots are the minimum pixel index of each component (hooks always point
//      to the smaller index).  Sizes by warp-aggregated DSMEM atomicAdd, the
//      min_points filter, and a cluster-wide ordered scan of kept roots give
//      label = 1 + rank of the component's smallest pixel among kept
//      components — bit-identical to the reference's first-encounter flood
//      fill + _renumber_roots + filter_small (ccl.py:83-170,
//      map_connections.py:113-129; SURVEY.md finding 2).
//   7. Labels streamed out with coalesced stores.
//
// HBM traffic per pixel: 4 B range in + 4 B label out (+ L2-resident halo
// re-reads).  All union-find state lives in shared memory.
//
// Entry points are the C ABI in include/rangeseg_b200.h.

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/rangeseg_b200.h"

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kFlag = 0x80000000u;
constexpr int kMaxCluster = 16;
constexpr int kMaxRowsPerCta = 31;          // seam bits of R+1 rows fit one word
constexpr size_t kSmemLimit = 227 * 1024;   // per-CTA opt-in maximum on sm_100

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

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
    // shared-memory layout, in 32-bit words
    int o_P, o_L, o_U, o_SB, o_RS, o_Ph, o_Lh, o_seam, o_MC, o_TL;
    int nwords;                   // R * WPR
    int use_tma;
};

constexpr uint32_t kFull = 0xffffffffu;

// Optional per-phase timestamps (build with -DRS_PHASE_PROF; read back with
// rs_phase_profile).  Compiled out otherwise.
constexpr int kProfSlots = 16;
constexpr int kProfCtas = 8192;
#ifdef RS_PHASE_PROF
__device__ long long g_prof[kProfCtas * kProfSlots];
#define RS_MARK(i)                                                                  \
    do {                                                                            \
        if (threadIdx.x == 0 && blockIdx.x < kProfCtas)                             \
            g_prof[blockIdx.x * kProfSlots + (i)] = clock64();                      \
    } while (0)
#else
#define RS_MARK(i) \
    do {           \
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

// Ground decision of a valid cell with range v in row r (ground.py:112-140 and
// range_image.py:125-127): pair kk = max(r,1)-1 spans d1 (upper) and d2
// (lower); row 0 reuses pair 0 with its own height.  Slope bounds are
// multiplied through by the denominator, never divided.
__device__ __forceinline__ bool is_ground(const KArgs &a, float d1, float d2, float v, int kk, int r) {
    const float *t = a.tables;
    const int H = a.H;
    const float sa = __ldg(t + H + kk);
    const float ca = __ldg(t + 2 * H - 1 + kk);
    const float lo = __ldg(t + 3 * H - 2 + kk);
    const float hi = __ldg(t + 4 * H - 3 + kk);
    const float num = __fmul_rn(d2, sa);
    const float den = __fsub_rn(d1, __fmul_rn(d2, ca));
    const float L = __fmul_rn(lo, den);
    const float U = __fmul_rn(hi, den);
    bool ok = den > 0.f ? (num >= L && num <= U) : (num <= L && num >= U);
    ok = ok && den != 0.f && d1 > 0.f && d2 > 0.f;
    const float z = __fadd_rn(__fmul_rn(v, __ldg(t + r)), a.mount);
    return ok && z <= a.keep_above;
}

// Presence = valid && !ground for cell (r, c); `get(row, col)` returns the range.
template <class Get>
__device__ __forceinline__ bool present_at(const KArgs &a, int r, int c, Get get) {
    const float v = get(r, c);
    if (!(v > 0.f)) return false;
    if (!a.ground) return true;
    const int kk = (r >= 1 ? r : 1) - 1;
    return !is_ground(a, get(kk, c), get(kk + 1, c), v, kk, r);
}

__device__ __forceinline__ int divWPR(const KArgs &a, int w) {
    return (int)(((unsigned long long)(unsigned)w * a.magicWPR) >> 40);
}

__device__ __forceinline__ uint32_t lanemask_le(int lane) {
    return lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
}

// ------------------------------------------------------------- TMA staging

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
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

// ---------------------------------------------------------------- union-find
//
// Nodes are horizontal runs of linked cells inside a band, identified by the
// local index of their first cell.  Entries hold cluster-encoded indices
// e = (band << SH) | local, which order exactly like frame-linear indices.
// Invariant: E[x] <= x (hooks point to the smaller root), so every tree's
// root is its minimum cell.  Once roots are marked, a root's entry carries
// kFlag | value (its size, later its label); finds treat kFlag as "root".


// Node (local cell index) of cell bit b of word w: the last run start at or
// before the cell, else the run node carried into the word.
__device__ __forceinline__ uint32_t node_of(const uint32_t *SB, const uint32_t *RS, int w, int q, int cw,
                                            int W, int b) {
    const uint32_t s = SB[w] & lanemask_le(b);
    return s ? (uint32_t)(q * W + cw * 32 + 31 - __clz(s)) : RS[w];
}

struct UF {
    uint32_t *E;
    cg::cluster_group cl;
    uint32_t mask;
    int SH;
    int rank;

    __device__ __forceinline__ uint32_t *slot(uint32_t e) const {
        const int owner = (int)(e >> SH);
        uint32_t *base = owner == rank ? E : cl.map_shared_rank(E, owner);
        return base + (e & mask);
    }
    __device__ __forceinline__ uint32_t ld(uint32_t e) const {
        return *reinterpret_cast<volatile uint32_t *>(slot(e));
    }
    // find over the whole cluster (DSMEM), path halving, flag-aware
    __device__ uint32_t find(uint32_t e) const {
        while (true) {
            const uint32_t p = ld(e);
            if (p == e || (p & kFlag)) return e;
            const uint32_t gp = ld(p);
            if (gp == p || (gp & kFlag)) return p;
            *reinterpret_cast<volatile uint32_t *>(slot(e)) = gp;
            e = gp;
        }
    }
    // read-only find: used while owners overwrite their entries with final
    // roots, where a late path-halving store could replace a root with an
    // intermediate ancestor
    __device__ uint32_t find_nc(uint32_t e) const {
        while (true) {
            const uint32_t p = ld(e);
            if (p == e || (p & kFlag)) return e;
            e = p;
        }
    }
    __device__ void unite(uint32_t x, uint32_t y) const {
        while (true) {
            x = find(x);
            y = find(y);
            if (x == y) return;
            if (x > y) { const uint32_t t = x; x = y; y = t; }
            const uint32_t old = atomicMin(slot(y), x);
            if (old == y) return;
            y = old;
        }
    }
    // band-local versions (all entries owned by this CTA): plain shared memory
    __device__ uint32_t find_local(uint32_t e) const {
        volatile uint32_t *V = E;
        while (true) {
            const uint32_t p = V[e & mask];
            if (p == e) return e;
            const uint32_t gp = V[p & mask];
            if (gp == p) return p;
            V[e & mask] = gp;
            e = gp;
        }
    }
    __device__ void unite_local(uint32_t x, uint32_t y) const {
        while (true) {
            x = find_local(x);
            y = find_local(y);
            if (x == y) return;
            if (x > y) { const uint32_t t = x; x = y; y = t; }
            const uint32_t old = atomicMin(E + (y & mask), x);
            if (old == y) return;
            y = old;
        }
    }
};

// -------------------------------------------------------------- the kernel

__global__ void __launch_bounds__(kThreads, 2) rs_segment_kernel(const __grid_constant__ KArgs a) {
    extern __shared__ __align__(128) uint32_t sm[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t warp_tot[kWarps];
    __shared__ uint32_t cta_cnt, cta_sum, cta_prefix, seam;

    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int frame = blockIdx.x / a.C;
    const int H = a.H, W = a.W, R = a.R, WPR = a.WPR;
    const int r0 = k * R;
    const int rows = min(R, H - r0);
    const int nw = rows * WPR;          // own words
    const float *fr = a.ranges + (size_t)frame * H * W;
    const int lo_row = max(r0 - 2, 0);
    const int hi_row = min(max(r0 + rows - 1, 1), H - 1);
    const float thr = a.dmax2, tch = a.tch;
    const uint32_t band = (uint32_t)k << a.SH;

    float *stage = reinterpret_cast<float *>(sm);
    uint32_t *E = sm;   // aliases the staging area once the edge bits exist
    uint32_t *P = sm + a.o_P, *L = sm + a.o_L, *U = sm + a.o_U;
    uint32_t *SB = sm + a.o_SB, *RS = sm + a.o_RS;
    uint32_t *Ph = sm + a.o_Ph, *Lh = sm + a.o_Lh;
    uint32_t *MC = sm + a.o_MC, *TL = sm + a.o_TL;

    RS_MARK(0);
    // ---- 1. stage rows [lo_row, hi_row] (TMA bulk copies) ---------------------
    const int n_stage = (hi_row - lo_row + 1) * W;
    const float *src = fr + (size_t)lo_row * W;
    if (tid == 0) seam = 0;
    if (a.use_tma) {
        if (tid == 0) {
            mbar_init(&mbar, 1);
            mbar_expect_tx(&mbar, (uint32_t)n_stage * 4u);
            const uint32_t row_bytes = (uint32_t)W * 4u;
            for (int s = 0; s <= hi_row - lo_row; ++s)
                tma_load_1d(stage + (size_t)s * W, src + (size_t)s * W, row_bytes, &mbar);
        }
        __syncthreads();
        mbar_wait(&mbar, 0);
    } else {
        for (int i = tid; i < n_stage; i += kThreads) stage[i] = __ldg(src + i);
        __syncthreads();
    }
    RS_MARK(1);
    auto S = [&](int r, int c) -> float { return stage[(r - lo_row) * W + c]; };
    auto G = [&](int r, int c) -> float { return __ldg(fr + (size_t)r * W + c); };

    // ---- 2. presence, left and up edge bits -----------------------------------
    // A warp walks a 32-column strip down the band, carrying the row above in
    // registers; rows r0-1 (halo) .. r0+rows-1.  LEFT bit 0 of each word and
    // the seam are completed in step 3.
    {
        const float *tcv = a.tables + 5 * H - 4;
        const int rstart = r0 > 0 ? r0 - 1 : 0;
        for (int cw = warp; cw < WPR; cw += kWarps) {
            const int c = cw * 32 + lane;
            const bool inb = c < W;
            float vprev = (inb && rstart >= 1) ? S(rstart - 1, c) : 0.f;
            bool pprev = false;
            for (int r = rstart; r < r0 + rows; ++r) {
                const float v = inb ? S(r, c) : 0.f;
                bool p = v > 0.f;
                if (a.ground && p) {
                    const float d1 = r >= 1 ? vprev : v;
                    const float d2 = r >= 1 ? v : S(1, c);
                    p = !is_ground(a, d1, d2, v, r >= 1 ? r - 1 : 0, r);
                }
                const float vl = __shfl_up_sync(kFull, v, 1);
                const bool pl = __shfl_up_sync(kFull, p, 1);
                const bool left = lane > 0 && p && pl && pair_pass(vl, v, tch, thr);
                const bool up = r > rstart && p && pprev && pair_pass(vprev, v, __ldg(tcv + r - 1), thr);
                const uint32_t mp = __ballot_sync(kFull, p);
                const uint32_t ml = __ballot_sync(kFull, left);
                const uint32_t mu = __ballot_sync(kFull, up);
                if (lane == 0) {
                    if (r < r0) {
                        Ph[cw] = mp;
                        Lh[cw] = ml;
                    } else {
                        const int w = (r - r0) * WPR + cw;
                        P[w] = mp;
                        L[w] = ml;
                        U[w] = mu;
                    }
                }
                vprev = v;
                pprev = p;
            }
        }
    }
    __syncthreads();

    RS_MARK(2);
    // ---- 3. word-boundary LEFT bits, the seam, Map Connection bits ------------
    for (int w = tid; w < nw + WPR; w += kThreads) {
        int cw, r;
        uint32_t *Lw, pw, pprev;
        if (w < nw) {
            const int q = divWPR(a, w);
            cw = w - q * WPR;
            r = r0 + q;
            if (cw == 0) continue;
            Lw = L + w; pw = P[w]; pprev = P[w - 1];
        } else {
            if (r0 == 0) break;
            cw = w - nw;
            r = r0 - 1;
            if (cw == 0) continue;
            Lw = Lh + cw; pw = Ph[cw]; pprev = Ph[cw - 1];
        }
        const int c = cw * 32;
        if ((pw & 1u) && (pprev >> 31) && pair_pass(S(r, c - 1), S(r, c), tch, thr)) *Lw |= 1u;
    }
    if (W > 1) {
        for (int q = tid; q < rows; q += kThreads) {
            const int r = r0 + q;
            const uint32_t pe = P[q * WPR + (W - 1) / 32] >> ((W - 1) & 31);
            if ((pe & 1u) && (P[q * WPR] & 1u) && pair_pass(S(r, W - 1), S(r, 0), tch, thr))
                atomicOr(&seam, 1u << q);
        }
    }
    if (a.n_off > 0) {
        // Pairs (r-dy, c-dx mod W) <-> (r, c), evaluated by the lower/right cell.
        // TL = LEFT edge of the partner (for the redundant-edge test in step 4).
        for (int w = warp; w < nw; w += kWarps) {
            const int q = divWPR(a, w);
            const int cw = w - q * WPR;
            const int c = cw * 32 + lane;
            const bool inb = c < W;
            const int r = r0 + q;
            const bool p = inb && ((P[w] >> lane) & 1u);
            const float v = inb ? S(r, c) : 0.f;
            for (int o = 0; o < a.n_off; ++o) {
                const int dy = a.dy[o], dx = a.dx[o];
                const int tr = r - dy;
                int tc = (c - dx) % W;
                if (tc < 0) tc += W;
                const bool has = inb && tr >= 0;
                auto part = [&](int col, bool &pt, float &vt) {
                    if (tr >= r0) {
                        pt = (P[(tr - r0) * WPR + col / 32] >> (col & 31)) & 1u;
                        vt = S(tr, col);
                    } else if (tr == r0 - 1) {
                        pt = (Ph[col / 32] >> (col & 31)) & 1u;
                        vt = S(tr, col);
                    } else {
                        vt = G(tr, col);
                        pt = present_at(a, tr, col, G);
                    }
                };
                bool pt = false;
                float vt = 0.f;
                if (has) part(tc, pt, vt);
                bool ptl = __shfl_up_sync(kFull, pt, 1);
                float vtl = __shfl_up_sync(kFull, vt, 1);
                if (has && tc > 0 && c > 0 && lane == 0) part(tc - 1, ptl, vtl);
                const float tco = __ldg(a.tables + 6 * H - 5 + o * H + max(tr, 0));
                const bool mc = has && p && pt && pair_pass(vt, v, tco, thr);
                const bool tl = has && c > 0 && tc > 0 && pt && ptl && pair_pass(vtl, vt, tch, thr);
                const uint32_t mm = __ballot_sync(kFull, mc);
                const uint32_t mt = __ballot_sync(kFull, tl);
                if (lane == 0) {
                    MC[o * a.nwords + w] = mm;
                    TL[o * a.nwords + w] = mt;
                }
            }
        }
    }
    __syncthreads();   // staging is dead from here on; E aliases it

    RS_MARK(3);
    UF uf{E, cl, (1u << a.SH) - 1u, a.SH, k};

    // ---- 4. runs: start bits, carried run node per word, node init ----------
    // Warp w owns the contiguous word range [wr0, wr1); a run continuing into
    // the range gets a pseudo start at its first cell (united in step 5).
    const int per = (nw + kWarps - 1) / kWarps;
    const int wr0 = min(warp * per, nw), wr1 = min(wr0 + per, nw);
    {
        int carry = -1;
        for (int cb = wr0; cb < wr1; cb += 32) {
            const int w = cb + lane;
            const bool act = w < wr1;
            uint32_t sb = 0;
            int base = 0;
            if (act) {
                const uint32_t pw = P[w], lw = L[w];
                sb = pw & ~lw;
                if (w == wr0 && (pw & lw & 1u)) sb |= 1u;
                const int q = divWPR(a, w);
                base = q * W + (w - q * WPR) * 32;
            }
            int inc = sb ? base + 31 - __clz(sb) : -1;
            for (int off = 1; off < 32; off <<= 1) {
                const int t = __shfl_up_sync(kFull, inc, off);
                if (lane >= off) inc = max(inc, t);
            }
            inc = max(inc, carry);
            int exc = __shfl_up_sync(kFull, inc, 1);
            if (lane == 0) exc = carry;
            if (act) {
                SB[w] = sb;
                RS[w] = (uint32_t)exc;
                for (uint32_t m = sb; m; m &= m - 1) {
                    const int s = base + __ffs(m) - 1;
                    E[s] = band | (uint32_t)s;
                }
            }
            carry = __shfl_sync(kFull, inc, 31);
        }
    }
    __syncthreads();

    RS_MARK(4);
    // ---- 5. band-local unions -----------------------------------------------
    // UP / Map Connection edges are skipped when the same pair of runs is
    // already joined through the edge one cell to the left (both cells linked
    // to their left neighbours and that neighbour pair has the same edge).
    for (int w = tid; w < nw; w += kThreads) {
        const int q = divWPR(a, w);
        const int cw = w - q * WPR;
        const uint32_t lw = L[w], sb = SB[w];
        if (sb & lw & 1u)   // pseudo start: join the run it continues
            uf.unite_local(band | node_of(SB, RS, w, q, cw, W, 0),
                           band | node_of(SB, RS, w - 1, q, cw - 1, W, 31));
        const uint32_t uw = U[w];
        if (q > 0 && uw) {
            const uint32_t uprev = (uw << 1) | (cw > 0 ? U[w - 1] >> 31 : 0u);
            uint32_t nr = uw & ~(uprev & lw & L[w - WPR]);
            for (; nr; nr &= nr - 1) {
                const int b = __ffs(nr) - 1;
                uf.unite_local(band | node_of(SB, RS, w, q, cw, W, b),
                               band | node_of(SB, RS, w - WPR, q - 1, cw, W, b));
            }
        }
        if (cw == 0 && ((seam >> q) & 1u))
            uf.unite_local(band | node_of(SB, RS, w, q, 0, W, 0),
                           band | node_of(SB, RS, q * WPR + (W - 1) / 32, q, (W - 1) / 32, W, (W - 1) & 31));
        for (int o = 0; o < a.n_off; ++o) {
            const int dy = a.dy[o];
            if (q < dy) continue;   // partner above the band: step 7
            const uint32_t *M = MC + o * a.nwords;
            const uint32_t m = M[w];
            if (!m) continue;
            const uint32_t mprev = (m << 1) | (cw > 0 ? M[w - 1] >> 31 : 0u);
            uint32_t nr = m & ~(mprev & lw & TL[o * a.nwords + w]);
            for (; nr; nr &= nr - 1) {
                const int b = __ffs(nr) - 1;
                int tc = (cw * 32 + b - a.dx[o]) % W;
                if (tc < 0) tc += W;
                const int tq = q - dy;
                uf.unite_local(band | node_of(SB, RS, w, q, cw, W, b),
                               band | node_of(SB, RS, tq * WPR + tc / 32, tq, tc / 32, W, tc & 31));
            }
        }
    }
    __syncthreads();
    RS_MARK(5);
    // local flatten: every node points at its band-local root
    for (int w = tid; w < nw; w += kThreads) {
        const int q = divWPR(a, w);
        const uint32_t base = (uint32_t)(q * W + (w - q * WPR) * 32);
        for (uint32_t m = SB[w]; m; m &= m - 1) {
            const uint32_t s = base + __ffs(m) - 1;
            E[s] = uf.find_local(band | s);
        }
    }
    cl.sync();   // #1: every band's runs are initialised and locally flat

    RS_MARK(6);
    // ---- 6. cross-band unions over DSMEM ----------------------------------
    if (r0 > 0) {
        const int ku = k - 1;
        const uint32_t *SBu = cl.map_shared_rank(SB, ku), *RSu = cl.map_shared_rank(RS, ku);
        const uint32_t bandu = (uint32_t)ku << a.SH;
        for (int cw = tid; cw < WPR; cw += kThreads) {
            const uint32_t uw = U[cw];
            if (!uw) continue;
            const uint32_t uprev = (uw << 1) | (cw > 0 ? U[cw - 1] >> 31 : 0u);
            uint32_t nr = uw & ~(uprev & L[cw] & Lh[cw]);
            const int wu = (R - 1) * WPR + cw;
            for (; nr; nr &= nr - 1) {
                const int b = __ffs(nr) - 1;
                uf.unite(band | node_of(SB, RS, cw, 0, cw, W, b),
                         bandu | node_of(SBu, RSu, wu, R - 1, cw, W, b));
            }
        }
        for (int o = 0; o < a.n_off; ++o) {
            const int dy = a.dy[o];
            const uint32_t *M = MC + o * a.nwords;
            const int lim = min(dy, rows) * WPR;
            for (int w = tid; w < lim; w += kThreads) {
                const uint32_t m = M[w];
                if (!m) continue;
                const int q = divWPR(a, w);
                const int cw = w - q * WPR;
                const uint32_t mprev = (m << 1) | (cw > 0 ? M[w - 1] >> 31 : 0u);
                uint32_t nr = m & ~(mprev & L[w] & TL[o * a.nwords + w]);
                const int tr = r0 + q - dy;
                if (tr < 0) continue;
                const int kt = tr / R, tq = tr - kt * R;
                const uint32_t *SBt = cl.map_shared_rank(SB, kt), *RSt = cl.map_shared_rank(RS, kt);
                for (; nr; nr &= nr - 1) {
                    const int b = __ffs(nr) - 1;
                    int tc = (cw * 32 + b - a.dx[o]) % W;
                    if (tc < 0) tc += W;
                    uf.unite(band | node_of(SB, RS, w, q, cw, W, b),
                             ((uint32_t)kt << a.SH) |
                                 node_of(SBt, RSt, tq * WPR + tc / 32, tq, tc / 32, W, tc & 31));
                }
            }
        }
    }
    cl.sync();   // #2: the forest is final

    RS_MARK(7);
    // ---- 7. resolve every node to its root; roots start a size counter ------
    for (int w = tid; w < nw; w += kThreads) {
        const int q = divWPR(a, w);
        const uint32_t base = (uint32_t)(q * W + (w - q * WPR) * 32);
        for (uint32_t m = SB[w]; m; m &= m - 1) {
            const uint32_t s = base + __ffs(m) - 1;
            const uint32_t g = uf.find_nc(band | s);
            E[s] = g == (band | s) ? kFlag : g;
        }
    }
    cl.sync();   // #3

    RS_MARK(8);
    // ---- 8. component sizes: one atomicAdd of the run length per run -------
    {
        int carry = INT_MAX;   // first run end after the current chunk
        const int nchunks = (wr1 - wr0 + 31) / 32;
        for (int ci = nchunks - 1; ci >= 0; --ci) {
            const int w = wr0 + ci * 32 + lane;
            const bool act = w < wr1;
            uint32_t eb = 0, sb = 0;
            int base = 0;
            if (act) {
                const int q = divWPR(a, w);
                const int cw = w - q * WPR;
                base = q * W + cw * 32;
                const uint32_t lnext = (w + 1 < wr1 && cw + 1 < WPR) ? (L[w + 1] & 1u) : 0u;
                eb = P[w] & ~((L[w] >> 1) | (lnext << 31));
                sb = SB[w];
            }
            int inc = eb ? base + __ffs(eb) - 1 : INT_MAX;
            for (int off = 1; off < 32; off <<= 1) {
                const int t = __shfl_down_sync(kFull, inc, off);
                if (lane + off < 32) inc = min(inc, t);
            }
            inc = min(inc, carry);
            int exc = __shfl_down_sync(kFull, inc, 1);
            if (lane == 31) exc = carry;
            for (uint32_t m = sb; m; m &= m - 1) {
                const int b = __ffs(m) - 1;
                const uint32_t after = eb & ~((1u << b) - 1u);
                const int end = after ? base + __ffs(after) - 1 : exc;
                const uint32_t s = (uint32_t)(base + b);
                const uint32_t v = E[s];
                const uint32_t root = (v & kFlag) ? (band | s) : v;
                atomicAdd(uf.slot(root), (uint32_t)(end - (int)s + 1));
            }
            carry = __shfl_sync(kFull, inc, 0);
        }
    }
    cl.sync();   // #4

    RS_MARK(9);
    // ---- 9. filter + ordered rank of kept roots ---------------------------
    uint32_t *K = U;    // U and L are dead after the unions and sizes
    uint32_t *WP = L;
    const uint32_t minp = a.min_points > 1 ? (uint32_t)a.min_points : 1u;
    if (tid == 0) cta_sum = 0;
    __syncthreads();
    for (int w = tid; w < nw; w += kThreads) {
        const int q = divWPR(a, w);
        const uint32_t base = (uint32_t)(q * W + (w - q * WPR) * 32);
        uint32_t kept = 0, s_sum = 0;
        for (uint32_t m = SB[w]; m; m &= m - 1) {
            const int b = __ffs(m) - 1;
            const uint32_t v = E[base + b];
            if ((v & kFlag) && (v & ~kFlag) >= minp) {
                kept |= 1u << b;
                s_sum += v & ~kFlag;
            }
        }
        K[w] = kept;
        if (s_sum) atomicAdd(&cta_sum, s_sum);
    }
    __syncthreads();
    {
        uint32_t run = 0;
        for (int cb = wr0; cb < wr1; cb += 32) {
            const int w = cb + lane;
            const uint32_t cnt = w < wr1 ? __popc(K[w]) : 0u;
            uint32_t inc = cnt;
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t t = __shfl_up_sync(kFull, inc, off);
                if (lane >= off) inc += t;
            }
            if (w < wr1) WP[w] = run + inc - cnt;
            run += __shfl_sync(kFull, inc, 31);
        }
        if (lane == 0) warp_tot[warp] = run;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int i = 0; i < kWarps; ++i) { const uint32_t x = warp_tot[i]; warp_tot[i] = t; t += x; }
        cta_cnt = t;
    }
    cl.sync();   // #5: every band's kept count and kept-size sum are published
    RS_MARK(10);
    if (tid == 0) {
        uint32_t pre = 0, tot = 0, sum = 0;
        for (int j = 0; j < a.C; ++j) {
            const uint32_t cj = *cl.map_shared_rank(&cta_cnt, j);
            if (j < k) pre += cj;
            tot += cj;
            sum += *cl.map_shared_rank(&cta_sum, j);
        }
        cta_prefix = pre;
        if (k == 0) {
            if (a.ncl) a.ncl[frame] = (int32_t)tot;
            if (a.sizes) a.sizes[(size_t)frame * a.sizes_stride] = (int64_t)H * W - (int64_t)sum;
        }
    }
    __syncthreads();
    {
        const uint32_t prefix = cta_prefix;
        for (int w = tid; w < nw; w += kThreads) {
            const int q = divWPR(a, w);
            const uint32_t base = (uint32_t)(q * W + (w - q * WPR) * 32);
            const uint32_t km = K[w];
            const uint32_t wbase = prefix + warp_tot[min(w / max(per, 1), kWarps - 1)] + WP[w];
            for (uint32_t m = SB[w]; m; m &= m - 1) {
                const int b = __ffs(m) - 1;
                const uint32_t s = base + b;
                const uint32_t v = E[s];
                if (!(v & kFlag)) continue;
                if ((km >> b) & 1u) {
                    const uint32_t label = wbase + __popc(km & ((1u << b) - 1u)) + 1u;
                    E[s] = kFlag | label;
                    if (a.sizes) a.sizes[(size_t)frame * a.sizes_stride + label] = (int64_t)(v & ~kFlag);
                } else {
                    E[s] = kFlag;   // dropped by filter_small
                }
            }
        }
    }
    cl.sync();   // #6

    RS_MARK(11);
    // ---- 10. every node takes its root's label -----------------------------
    for (int w = tid; w < nw; w += kThreads) {
        const int q = divWPR(a, w);
        const uint32_t base = (uint32_t)(q * W + (w - q * WPR) * 32);
        for (uint32_t m = SB[w]; m; m &= m - 1) {
            const uint32_t s = base + __ffs(m) - 1;
            const uint32_t v = E[s];
            if (!(v & kFlag)) E[s] = kFlag | (uf.ld(v) & ~kFlag);
        }
    }
    cl.sync();   // #7: no DSMEM access after this point

    RS_MARK(12);
    // ---- 11. per-cell labels, coalesced streaming stores -------------------
    int32_t *out = a.labels + (size_t)frame * H * W + (size_t)r0 * W;
    for (int w = warp; w < nw; w += kWarps) {
        const int q = divWPR(a, w);
        const int cw = w - q * WPR;
        const int c = cw * 32 + lane;
        if (c < W) {
            uint32_t lab = 0;
            if ((P[w] >> lane) & 1u) lab = E[node_of(SB, RS, w, q, cw, W, lane)] & ~kFlag;
            __stcs(out + q * W + c, (int32_t)lab);
        }
    }
    RS_MARK(13);
}

// Stage masks (parity/debug): ground, horizontal, vertical as bytes.
__global__ void rs_stage_kernel(const __grid_constant__ KArgs a, uint8_t *ground, uint8_t *horiz,
                                uint8_t *vert, long long total) {
    const int H = a.H, W = a.W;
    const long long HW = (long long)H * W;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long f = idx / HW;
        const int i = (int)(idx - f * HW);
        const int r = i / W, c = i - (i / W) * W;
        const float *fr = a.ranges + f * HW;
        auto G = [&](int rr, int cc) -> float { return __ldg(fr + (size_t)rr * W + cc); };
        const float v = G(r, c);
        const bool p = present_at(a, r, c, G);
        ground[idx] = (uint8_t)!p;
        bool h = false;
        if (W > 1) {
            const int c2 = c + 1 < W ? c + 1 : 0;
            h = p && present_at(a, r, c2, G) && pair_pass(v, G(r, c2), a.tch, a.dmax2);
        }
        horiz[idx] = (uint8_t)h;
        if (r < H - 1) {
            const bool vv = p && present_at(a, r + 1, c, G) &&
                            pair_pass(v, G(r + 1, c), __ldg(a.tables + 5 * H - 4 + r), a.dmax2);
            vert[f * (HW - W) + (long long)r * W + c] = (uint8_t)vv;
        }
    }
}

// ------------------------------------------------------------------ planning

struct Plan {
    int R, C, SH;
    size_t smem;
    KArgs k;
};

int validate(const rs_config *cfg) {
    if (!cfg) return fail(RS_EINVAL, "config is NULL");
    const int H = cfg->height, W = cfg->width;
    if (H < 2) return fail(RS_EINVAL, "need at least 2 rows (channels)");
    if (W < 1) return fail(RS_EINVAL, "width must be >= 1");
    if ((long long)H * W >= (1LL << 24)) return fail(RS_ETOOLARGE, "frame larger than 2^24 cells");
    if (cfg->n_offsets < 0 || cfg->n_offsets > RS_MAX_OFFSETS)
        return fail(RS_EINVAL, "n_offsets out of range [0, 32]");
    for (int o = 0; o < cfg->n_offsets; ++o) {
        const int dy = cfg->offsets[o][0], dx = cfg->offsets[o][1];
        if (dy < 0 || (dy == 0 && dx <= 0))
            return fail(RS_EINVAL, "offsets must be canonical: dy > 0, or dy == 0 and dx > 0");
        if (dy >= H || dx >= W || -dx >= W)
            return fail(RS_EINVAL, "offset (" + std::to_string(dy) + ", " + std::to_string(dx) +
                                       ") exceeds frame " + std::to_string(H) + "x" + std::to_string(W));
    }
    return RS_OK;
}

size_t smem_for(int R, int W, int n_off, int *o_words) {
    const int WPR = (W + 31) / 32;
    const int nwords = R * WPR;
    const int stage = std::max((R + 2) * W, R * W);
    int off = (stage + 31) & ~31;
    o_words[0] = off; off += nwords;               // P
    o_words[1] = off; off += nwords;               // L
    o_words[2] = off; off += nwords;               // U
    o_words[3] = off; off += nwords;               // SB (run starts)
    o_words[4] = off; off += nwords;               // RS (run node carried into a word)
    o_words[5] = off; off += WPR;                  // Ph (halo row)
    o_words[6] = off; off += WPR;                  // Lh
    o_words[7] = off; off += 0;                    // (seam lives in static smem)
    o_words[8] = off; off += n_off * nwords;       // MC
    o_words[9] = off; off += n_off * nwords;       // TL
    return (size_t)off * 4u;
}

int make_plan(const rs_config *cfg, Plan *pl) {
    int st = validate(cfg);
    if (st) return st;
    const int H = cfg->height, W = cfg->width, n_off = cfg->n_offsets;
    int o[10];
    int R = cfg->rows_per_cta;
    if (R <= 0) {
        // Prefer ~16K cells per CTA (two CTAs per SM) with a portable cluster.
        R = std::max(1, std::min(H, 16384 / std::max(W, 1)));
        R = std::min(R, kMaxRowsPerCta);
        while ((H + R - 1) / R > 8 && R < kMaxRowsPerCta && smem_for(R + 1, W, n_off, o) <= kSmemLimit) ++R;
        while ((H + R - 1) / R > kMaxCluster && R < kMaxRowsPerCta) ++R;
        while (smem_for(R, W, n_off, o) > kSmemLimit && R > 1 && (H + R - 2) / (R - 1) <= kMaxCluster) --R;
    }
    R = std::min(R, H);
    if (R > kMaxRowsPerCta) return fail(RS_EINVAL, "rows_per_cta must be <= 31");
    const int C = (H + R - 1) / R;
    if (C > kMaxCluster)
        return fail(RS_ETOOLARGE, "frame needs " + std::to_string(C) + " bands of " + std::to_string(R) +
                                      " rows; a cluster holds at most 16");
    const size_t smem = smem_for(R, W, n_off, o);
    if (smem > kSmemLimit)
        return fail(RS_ETOOLARGE, "band of " + std::to_string(R) + "x" + std::to_string(W) +
                                      " cells needs " + std::to_string(smem) + " B of shared memory");
    int SH = 0;
    while ((1 << SH) < R * W) ++SH;
    pl->R = R;
    pl->C = C;
    pl->SH = SH;
    pl->smem = smem;
    KArgs &k = pl->k;
    memset(&k, 0, sizeof(k));
    k.H = H; k.W = W; k.R = R; k.C = C; k.SH = SH;
    k.n_off = n_off;
    for (int i = 0; i < n_off; ++i) { k.dy[i] = cfg->offsets[i][0]; k.dx[i] = cfg->offsets[i][1]; }
    k.min_points = cfg->min_cluster_points;
    k.ground = cfg->ground_removal ? 1 : 0;
    k.dmax2 = cfg->d_max_sq;
    k.mount = cfg->mount_height;
    k.keep_above = cfg->keep_above;
    k.tch = cfg->two_cos_h;
    k.WPR = (W + 31) / 32;
    k.magicWPR = ((1ULL << 40) + (unsigned long long)k.WPR - 1) / (unsigned long long)k.WPR;
    k.o_P = o[0]; k.o_L = o[1]; k.o_U = o[2]; k.o_SB = o[3]; k.o_RS = o[4];
    k.o_Ph = o[5]; k.o_Lh = o[6]; k.o_seam = o[7]; k.o_MC = o[8]; k.o_TL = o[9];
    k.nwords = R * k.WPR;
    return RS_OK;
}

int cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return RS_OK;
    return fail(RS_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

std::mutex g_attr_mu;
size_t g_attr_smem = 0;
bool g_attr_nonportable = false;

int launch_segment(const Plan &pl, KArgs k, int B, cudaStream_t stream) {
    {
        std::lock_guard<std::mutex> g(g_attr_mu);
        if (pl.smem > g_attr_smem) {
            int st = cuda_check(cudaFuncSetAttribute(rs_segment_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)std::max(pl.smem, (size_t)48 * 1024)),
                                "cudaFuncSetAttribute(max dynamic smem)");
            if (st) return st;
            g_attr_smem = pl.smem;
        }
        if (pl.C > 8 && !g_attr_nonportable) {
            int st = cuda_check(cudaFuncSetAttribute(rs_segment_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                                "cudaFuncSetAttribute(non-portable cluster)");
            if (st) return st;
            g_attr_nonportable = true;
        }
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(B * pl.C), 1, 1);
    lc.blockDim = dim3(kThreads, 1, 1);
    lc.dynamicSmemBytes = pl.smem;
    lc.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)pl.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cuda_check(cudaLaunchKernelEx(&lc, rs_segment_kernel, k), "rs_segment_kernel launch");
}

}  // namespace

// =================================================================== C ABI

extern "C" {

size_t rs_tables_count(int32_t height, int32_t n_offsets) {
    if (height < 2 || n_offsets < 0) return 0;
    return (size_t)height + 5u * (size_t)(height - 1) + (size_t)n_offsets * height;
}

int rs_plan(const rs_config *cfg, int32_t *rows_per_cta, int32_t *ctas_per_frame, size_t *smem_bytes) {
    Plan pl;
    int st = make_plan(cfg, &pl);
    if (st) return st;
    if (rows_per_cta) *rows_per_cta = pl.R;
    if (ctas_per_frame) *ctas_per_frame = pl.C;
    if (smem_bytes) *smem_bytes = pl.smem;
    return RS_OK;
}

int rs_segment_batch(const rs_config *cfg, const float *d_tables, const float *d_ranges, int32_t batch,
                     int32_t *d_labels, int32_t *d_n_clusters, int64_t *d_cluster_sizes, int64_t sizes_stride,
                     void *stream) {
    Plan pl;
    int st = make_plan(cfg, &pl);
    if (st) return st;
    if (batch < 0) return fail(RS_EINVAL, "batch must be >= 0");
    if (batch == 0) return RS_OK;
    if (!d_tables || !d_ranges || !d_labels) return fail(RS_EINVAL, "tables, ranges and labels are required");
    const long long HW = (long long)cfg->height * cfg->width;
    if (d_cluster_sizes) {
        const long long need = HW / std::max(cfg->min_cluster_points, 1) + 1;
        if (sizes_stride < need)
            return fail(RS_EINVAL, "sizes_stride must be >= H*W/max(min_cluster_points,1)+1 = " +
                                       std::to_string(need));
    }
    if ((long long)batch * pl.C > 0x7fffffffLL) return fail(RS_EINVAL, "batch too large");
    KArgs k = pl.k;
    k.ranges = d_ranges;
    k.tables = d_tables;
    k.labels = d_labels;
    k.ncl = d_n_clusters;
    k.sizes = d_cluster_sizes;
    k.sizes_stride = sizes_stride;
    k.use_tma = (cfg->width % 4 == 0) && ((reinterpret_cast<uintptr_t>(d_ranges) & 15u) == 0);
    return launch_segment(pl, k, batch, static_cast<cudaStream_t>(stream));
}

int rs_stage_masks(const rs_config *cfg, const float *d_tables, const float *d_ranges, int32_t batch,
                   uint8_t *d_ground, uint8_t *d_horizontal, uint8_t *d_vertical, void *stream) {
    Plan pl;
    int st = make_plan(cfg, &pl);
    if (st) return st;
    if (batch <= 0) return batch == 0 ? RS_OK : fail(RS_EINVAL, "batch must be >= 0");
    if (!d_tables || !d_ranges || !d_ground || !d_horizontal || !d_vertical)
        return fail(RS_EINVAL, "all buffers are required");
    KArgs k = pl.k;
    k.ranges = d_ranges;
    k.tables = d_tables;
    const long long total = (long long)batch * cfg->height * cfg->width;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
    rs_stage_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(k, d_ground, d_horizontal,
                                                                          d_vertical, total);
    return cuda_check(cudaGetLastError(), "rs_stage_kernel launch");
}

// Host-buffer entry: chunks of frames are pipelined over two streams so the
// host->device copy of chunk j+1 overlaps the kernel of chunk j and the
// device->host copy of chunk j-1.
namespace {
struct HostCtx {
    std::mutex mu;
    float *d_ranges = nullptr, *d_tables = nullptr;
    int32_t *d_labels = nullptr, *d_ncl = nullptr;
    int64_t *d_sizes = nullptr;
    size_t cap_frames = 0, cap_tables = 0, cap_sizes = 0, frame_cells = 0;
    cudaStream_t s[2] = {nullptr, nullptr};
    int device = -1;
};
HostCtx g_host;

void host_free() {
    cudaFree(g_host.d_ranges);
    cudaFree(g_host.d_labels);
    cudaFree(g_host.d_ncl);
    cudaFree(g_host.d_sizes);
    g_host.d_ranges = nullptr;
    g_host.d_labels = nullptr;
    g_host.d_ncl = nullptr;
    g_host.d_sizes = nullptr;
    g_host.cap_frames = 0;
    g_host.cap_sizes = 0;
}
}  // namespace

int rs_segment_batch_host(const rs_config *cfg, const float *h_tables, const float *h_ranges, int32_t batch,
                          int32_t *h_labels, int32_t *h_n_clusters, int64_t *h_cluster_sizes,
                          int64_t sizes_stride) {
    Plan pl;
    int st = make_plan(cfg, &pl);
    if (st) return st;
    if (batch < 0) return fail(RS_EINVAL, "batch must be >= 0");
    if (batch == 0) return RS_OK;
    if (!h_tables || !h_ranges || !h_labels) return fail(RS_EINVAL, "tables, ranges and labels are required");
    std::lock_guard<std::mutex> g(g_host.mu);
    int dev = 0;
    if ((st = cuda_check(cudaGetDevice(&dev), "cudaGetDevice"))) return st;
    if (g_host.device != dev) {
        host_free();
        g_host.device = dev;
        for (auto &s : g_host.s) {
            s = nullptr;
            if ((st = cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate")))
                return st;
        }
        g_host.cap_tables = 0;
        cudaFree(g_host.d_tables);
        g_host.d_tables = nullptr;
    }
    const size_t HW = (size_t)cfg->height * cfg->width;
    const size_t nt = rs_tables_count(cfg->height, cfg->n_offsets);
    if (g_host.cap_frames < (size_t)batch || g_host.frame_cells != HW ||
        (h_cluster_sizes && g_host.cap_sizes < (size_t)batch * sizes_stride)) {
        host_free();
        g_host.frame_cells = HW;
        if ((st = cuda_check(cudaMalloc(&g_host.d_ranges, (size_t)batch * HW * 4), "cudaMalloc ranges")) ||
            (st = cuda_check(cudaMalloc(&g_host.d_labels, (size_t)batch * HW * 4), "cudaMalloc labels")) ||
            (st = cuda_check(cudaMalloc(&g_host.d_ncl, (size_t)batch * 4), "cudaMalloc n_clusters")))
            return st;
        if (h_cluster_sizes &&
            (st = cuda_check(cudaMalloc(&g_host.d_sizes, (size_t)batch * sizes_stride * 8), "cudaMalloc sizes")))
            return st;
        g_host.cap_frames = batch;
        g_host.cap_sizes = h_cluster_sizes ? (size_t)batch * sizes_stride : 0;
    }
    if (g_host.cap_tables < nt) {
        cudaFree(g_host.d_tables);
        if ((st = cuda_check(cudaMalloc(&g_host.d_tables, nt * 4), "cudaMalloc tables"))) return st;
        g_host.cap_tables = nt;
    }
    if ((st = cuda_check(cudaMemcpyAsync(g_host.d_tables, h_tables, nt * 4, cudaMemcpyHostToDevice, g_host.s[0]),
                         "copy tables")))
        return st;
    cudaEvent_t tables_ready;
    cudaEventCreateWithFlags(&tables_ready, cudaEventDisableTiming);
    cudaEventRecord(tables_ready, g_host.s[0]);
    cudaStreamWaitEvent(g_host.s[1], tables_ready, 0);
    const int chunk = std::max(1, std::min<int>(batch, std::max<int>(1, (int)((8u << 20) / (HW * 4)))));
    for (int b0 = 0, j = 0; b0 < batch; b0 += chunk, ++j) {
        const int nb = std::min(chunk, batch - b0);
        cudaStream_t s = g_host.s[j & 1];
        const size_t off = (size_t)b0 * HW;
        if ((st = cuda_check(cudaMemcpyAsync(g_host.d_ranges + off, h_ranges + off, nb * HW * 4,
                                             cudaMemcpyHostToDevice, s), "copy ranges")))
            break;
        st = rs_segment_batch(cfg, g_host.d_tables, g_host.d_ranges + off, nb, g_host.d_labels + off,
                              g_host.d_ncl + b0, h_cluster_sizes ? g_host.d_sizes + (size_t)b0 * sizes_stride : nullptr,
                              sizes_stride, s);
        if (st) break;
        if ((st = cuda_check(cudaMemcpyAsync(h_labels + off, g_host.d_labels + off, nb * HW * 4,
                                             cudaMemcpyDeviceToHost, s), "copy labels")))
            break;
        if (h_n_clusters &&
            (st = cuda_check(cudaMemcpyAsync(h_n_clusters + b0, g_host.d_ncl + b0, nb * 4, cudaMemcpyDeviceToHost, s),
                             "copy n_clusters")))
            break;
        if (h_cluster_sizes &&
            (st = cuda_check(cudaMemcpyAsync(h_cluster_sizes + (size_t)b0 * sizes_stride,
                                             g_host.d_sizes + (size_t)b0 * sizes_stride,
                                             (size_t)nb * sizes_stride * 8, cudaMemcpyDeviceToHost, s),
                             "copy sizes")))
            break;
    }
    const int st0 = cuda_check(cudaStreamSynchronize(g_host.s[0]), "stream sync");
    const int st1 = cuda_check(cudaStreamSynchronize(g_host.s[1]), "stream sync");
    cudaEventDestroy(tables_ready);
    return st ? st : (st0 ? st0 : st1);
}

int rs_phase_profile(int64_t *host_out, int32_t max_ctas) {
#ifdef RS_PHASE_PROF
    const int n = std::min<int>(max_ctas, kProfCtas);
    if (!host_out || n <= 0) return fail(RS_EINVAL, "bad profile buffer");
    return cuda_check(cudaMemcpyFromSymbol(host_out, g_prof, (size_t)n * kProfSlots * sizeof(long long)),
                      "read phase profile");
#else
    (void)host_out;
    (void)max_ctas;
    return fail(RS_EINVAL, "library built without RS_PHASE_PROF");
#endif
}

const char *rs_last_error(void) { return g_err.c_str(); }

int rs_version(void) { return 100; }

}  // extern "C"
