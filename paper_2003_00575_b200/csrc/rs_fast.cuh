// rs_fast.cuh — the fast kernel: union-find over compactly numbered runs.
//
// One thread-block cluster per frame, one 512-thread CTA per band of R rows
// (about 64K cells: two bands for a 64x2048 frame) spanning the full width,
// so the azimuth seam is CTA-local.  Shared memory holds only bit planes and
// per-run state, so two CTAs share an SM:
//
//   A  presence / left-pair / up-pair ballots straight from global memory:
//      each warp walks a 128-column chunk down the band, keeping the row above
//      in registers and prefetching two rows ahead (the reference's float32
//      rules, one rounding per op: ground.py:112-140, connectivity.py:47-92);
//      a chunk row without any return skips the rules (in the kernel without
//      Map Connections: in the other the extra test costs more than it saves).
//   B  presence masking of the edge words, chunk-boundary left bits, the
//      seam.
//   R  runs: start bits, and a block scan of their counts that numbers the
//      runs of the band 0..n-1 in cell order (run id order == cell order).
//   U  band-local union-find over run ids in shared memory: non-redundant
//      edges listed, every run hooked under its smallest listed neighbour,
//      then all edges united (path halving); local flatten; Map Connections
//      inside the band (rs_fast_kernel<true>, rs_mc.cuh); run lengths added
//      to local roots.
//   X  cross-band unions over DSMEM (boundary edges and cross-band Map
//      Connection pairs listed, then united).
//   Z  every band-local root resolves its global root and adds its size there.
//   K  kept roots (size >= min_points): kept bits and word prefixes per band,
//      band bases -> label = 1 + rank of the component's first cell among kept
//      components, the reference's first-encounter numbering after
//      _renumber_roots and filter_small (SURVEY.md finding 2).
//   L  run labels from the root's band (DSMEM), then per-cell labels with
//      16-byte streaming stores.
//
// A band with more runs than the node capacity NC marks the frame; after
// barrier #1 the whole cluster then labels it with a union-find over cells in
// global memory (rs_overflow.cuh), so no second launch is ever needed.
#pragma once

#include "rs_common.cuh"
#include "rs_mc.cuh"
#include "rs_overflow.cuh"

namespace rs {

#ifndef RS_FAST_OCC
#define RS_FAST_OCC 2
#endif
#ifndef RS_FAST_THREADS
#define RS_FAST_THREADS 512
#endif
#ifndef RS_SWEEP_UNROLL
#define RS_SWEEP_UNROLL 2   // cell-label sweep: iterations in flight per warp
#endif
#ifndef RS_UDYN_GRAB
#define RS_UDYN_GRAB 2   // dynamic local unions: contiguous edges per lane and grab (measured 1, 2, 4, 8)
#endif
#ifndef RS_PF_L2
#define RS_PF_L2 0   // step A: L2 prefetch this many rows beyond the register prefetch (0 = off)
#endif
#ifndef RS_STRIP_SETS
#define RS_STRIP_SETS 4   // step A register sets: 4 = two-row prefetch, 3 = one-row prefetch
#endif
#ifdef RS_EXPERIMENTS   // phase ablation (scripts/ablation.py): leave after phase N, labels wrong
#define RS_STOP(n)                \
    if (a.stop_after == (n)) {    \
        cl.sync();                \
        return;                   \
    }
#else
#define RS_STOP(n) \
    do {           \
    } while (0)
#endif
constexpr int kFastThreads = RS_FAST_THREADS;
constexpr int kSweepUnroll = RS_SWEEP_UNROLL;
constexpr int kFastOcc = RS_FAST_OCC;   // CTAs per SM the fast kernel is sized for
constexpr int kFastWarps = kFastThreads / 32;


struct RunUF {
    uint32_t *E;
    cg::cluster_group cl;
    uint32_t mask;
    int SHN;
    int rank;

    int nc;   // node capacity per band (RS_CHECKED)
    int C;    // bands in the cluster (RS_CHECKED)

    __device__ __forceinline__ uint32_t *slot(uint32_t *arr, uint32_t e) const {
        const int owner = (int)(e >> SHN);
        RS_CHECK(owner < C && (int)(e & mask) < nc, "union-find node out of range");
        return (owner == rank ? arr : cl.map_shared_rank(arr, owner)) + (e & mask);
    }
    __device__ __forceinline__ uint32_t ld(uint32_t e) const {
        return *reinterpret_cast<volatile uint32_t *>(slot(E, e));
    }
    __device__ uint32_t find(uint32_t e) const {
        while (true) {
            const uint32_t p = ld(e);
            if (p == e) return e;
            const uint32_t gp = ld(p);
            if (gp == p) return p;
            *reinterpret_cast<volatile uint32_t *>(slot(E, e)) = gp;   // path halving
            e = gp;
        }
    }
    __device__ uint32_t find_nc(uint32_t e) const {   // read-only
        while (true) {
            const uint32_t p = ld(e);
            if (p == e) return e;
            e = p;
        }
    }
    // cluster-wide union of two runs: one hop to their band-local roots
    // (flattened in step U), then finds with path halving among roots only, so
    // every other run keeps pointing at its band-local root (step L relies on it)
    __device__ void unite(uint32_t x, uint32_t y) const {
        x = ld(x);
        y = ld(y);
        while (true) {
            x = find(x);
            y = find(y);
            if (x == y) return;
            if (x > y) { const uint32_t t = x; x = y; y = t; }
            const uint32_t old = atomicMin(slot(E, y), x);   // larger root hooks under smaller
            if (old == y) return;
            y = old;
        }
    }
    // union of two entries that were roots recently (no hop from a run first)
    __device__ void unite_roots(uint32_t x, uint32_t y) const {
        while (true) {
            x = find(x);
            y = find(y);
            if (x == y) return;
            if (x > y) { const uint32_t t = x; x = y; y = t; }
            const uint32_t old = atomicMin(slot(E, y), x);
            if (old == y) return;
            y = old;
        }
    }
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
    // band-local find whose path-halving stores are atomicMin
    __device__ uint32_t find_local_min(uint32_t e) const {
        volatile uint32_t *V = E;
        while (true) {
            const uint32_t p = V[e & mask];
            if (p == e) return e;
            const uint32_t gp = V[p & mask];
            if (gp == p) return p;
            atomicMin(E + (e & mask), gp);
            e = gp;
        }
    }
    // cluster-wide find whose path-halving stores are atomicMin (DSMEM)
    __device__ uint32_t find_min(uint32_t e) const {
        while (true) {
            const uint32_t p = ld(e);
            if (p == e) return e;
            const uint32_t gp = ld(p);
            if (gp == p) return p;
            atomicMin(slot(E, e), gp);
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

// Step A for one 128-column chunk: lane l owns cells ch*128 + 32*j + l
// (j = 0..3), so a ballot of a per-cell predicate is directly the bit-plane
// word ch*4 + j and the left / up edge words are warp-uniform bit operations.
// The warp walks rows rfirst..rend-1 with the row above in registers and a
// two-row prefetch; four rotating register sets (unrolled by four) avoid
// register moves (RS_STRIP_SETS=3: one-row prefetch, three sets).  Row 0 (whose ground pair is rows 0/1) is done by a
// separate ROW0 step.  FULL: the chunk lies inside the row (no load guards,
// 16-byte stores of the four words by lane 0).  GROUND: ground removal on.
// Plane stores use 32-bit shared-memory byte addresses (sP/sL/sU: the chunk's
// words in the band's first row; sPh/sLh: the halo row).
template <bool FULL, bool GROUND, bool RING = false, bool SKIP = true>
struct BitsStrip {
    const KArgs &a;
    const float *col;
    const float *rowc;
    uint32_t sP, sL, sU, sPh, sLh;
    int ch, lane, r0, rstart, rend, cb;
    float thr, tch;
    int rfirst;   // first row walked (rstart, or a later row when rows are split between warps)
    int rowf;     // floats per row (W)
    int wpb;      // bytes per plane row (4 WPR)
    mutable uint32_t mx = 0;   // unsigned max of the raw bits of the rows walked (input-contract screen)

    mutable const float *np = nullptr;   // the row the next step prefetches (advanced by a row per step)

    __device__ __forceinline__ void ld4(int r, float (&x)[4], bool pred = true) const {
        ldp(col + r * rowf, x, pred);   // 32-bit offset: a frame has < 2^24 cells
    }
    __device__ __forceinline__ void ldp(const float *p, float (&x)[4], bool pred = true) const {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (pred && (FULL || cb + 32 * j < a.W)) {
                x[j] = __ldg(p + 32 * j);
            } else if (!FULL) {
                x[j] = 0.f;
            }
    }

    // va = row above, v = this row, vb = row below (read by ROW0 only); vn <-
    // row r + RS_STRIP_SETS - 2 (prefetch).
    // Stores the raw ballots: presence P, left pair test EH (in the L plane)
    // and up pair test EV (in the U plane); step B masks them with presence
    // one word per thread, 32x cheaper than warp-uniform ops here.
    template <bool ROW0, bool HALO = false>
    __device__ __forceinline__ void step(int r, const float (&va)[4], const float (&v)[4], const float (&vb)[4],
                                         float (&vn)[4]) const {
        if (!ROW0 && !RING) {   // prefetch row r + RS_STRIP_SETS - 2
            ldp(np, vn, r + RS_STRIP_SETS - 2 < rend);
#if RS_PF_L2 > 0
            // and pull the row RS_PF_L2 further down into L2 (the chunk's four
            // 128-byte lines, eight lanes each; the frame's rows only)
            if (r + RS_STRIP_SETS - 2 + RS_PF_L2 < a.H)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(np + RS_PF_L2 * rowf - lane + (lane & 3) * 32));
#endif
            np += rowf;
        }
        const bool halo = HALO;   // only the first row walked in a band > 0 (peeled in run())
        const int cw = ch * 4;
        const uint32_t off = halo ? 0u : (uint32_t)((r - r0) * wpb);
#ifndef RS_NO_EMPTY_SKIP
        if (SKIP) {
            // input-contract screen on the row being decided (every row of the
            // walk is the current row exactly once; its values are in registers
            // by now): the unsigned maximum of the raw bits (VIMNMX3) ...
            const uint32_t t = max(__vimax3_u32(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2])),
                                   __float_as_uint(v[3]));
            mx = max(mx, t);
            // ... which also tells when the chunk's 128 cells of this row are
            // all +0.0 (no return: sky, beyond the range cut): no cell is
            // present, so the row's three plane words are zero whatever the
            // pair tests say (step B masks them with presence), and the rules
            // are skipped
            if (!__any_sync(kFull, t != 0u)) {
                if (FULL) {
                    if (lane == 0) {
                        sts128((halo ? sPh : sP) + off, 0u, 0u, 0u, 0u);
                        sts128((halo ? sLh : sL) + off, 0u, 0u, 0u, 0u);
                        if (!halo) sts128(sU + off, 0u, 0u, 0u, 0u);
                    }
                } else if (lane < 4 && cw + lane < a.WPR) {
                    const uint32_t lo = off + 4u * (uint32_t)lane;
                    sts32((halo ? sPh : sP) + lo, 0u);
                    sts32((halo ? sLh : sL) + lo, 0u);
                    if (!halo) sts32(sU + lo, 0u);
                }
                return;
            }
        }
#endif
        const float4 c = *reinterpret_cast<const float4 *>(rowc + (r - rstart) * 8);
        const float4 c2 = *reinterpret_cast<const float4 *>(rowc + (r - rstart) * 8 + 4);
        const int srcl = (lane + 31) & 31;
        const bool last = lane == 31;
        uint32_t pw[4], lw[4], uw[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float d1 = ROW0 ? v[j] : va[j];
            const float d2 = ROW0 ? vb[j] : v[j];
            const bool gr = GROUND && ground_fast(c.x, c.y, c.z, c.w, c2.x, c2.z, d1, d2, v[j], ROW0 ? vb[j] : va[j]);
            pw[j] = __ballot_sync(kFull, (v[j] > 0.f) & !gr);
            // left neighbour: lane l-1's cell; lane 0 reads lane 31's cell of
            // word j-1 (word 0 of the chunk: bit 0 is redone in step B)
            const float src = (j > 0 && last) ? v[j > 0 ? j - 1 : 0] : v[j];
            const float vl = __shfl_sync(kFull, src, srcl);
            lw[j] = __ballot_sync(kFull, pair_pass(vl, v[j], tch, thr));
            uw[j] = ROW0 ? 0u : __ballot_sync(kFull, pair_pass(va[j], v[j], c2.y, thr));
        }
#ifdef RS_NO_EMPTY_SKIP
        constexpr bool kScreenHere = true;
#else
        constexpr bool kScreenHere = !SKIP;
#endif
        if (kScreenHere) {
            // input-contract screen on the row just decided (every row of the
            // walk is the current row exactly once; its values are in registers
            // by now): two 3-input unsigned max (VIMNMX3) for the lane's four cells
            mx = __vimax3_u32(mx, __float_as_uint(v[0]), __float_as_uint(v[1]));
            mx = __vimax3_u32(mx, __float_as_uint(v[2]), __float_as_uint(v[3]));
        }
        if (FULL) {
            if (lane == 0) {
                sts128((halo ? sPh : sP) + off, pw[0], pw[1], pw[2], pw[3]);
                sts128((halo ? sLh : sL) + off, lw[0], lw[1], lw[2], lw[3]);
                if (!halo) sts128(sU + off, uw[0], uw[1], uw[2], uw[3]);
            }
        } else if (lane < 4 && cw + lane < a.WPR) {
            const uint32_t xp = lane == 0 ? pw[0] : lane == 1 ? pw[1] : lane == 2 ? pw[2] : pw[3];
            const uint32_t xl = lane == 0 ? lw[0] : lane == 1 ? lw[1] : lane == 2 ? lw[2] : lw[3];
            const uint32_t xu = lane == 0 ? uw[0] : lane == 1 ? uw[1] : lane == 2 ? uw[2] : uw[3];
            const uint32_t lo = off + 4u * (uint32_t)lane;
            sts32((halo ? sPh : sP) + lo, xp);
            sts32((halo ? sLh : sL) + lo, xl);
            if (!halo) sts32(sU + lo, xu);
        }
    }

#ifdef RS_TMA_RING
    // ---- TMA row ring (RS_TMA_RING builds; FULL chunks only) -----------------
    // The warp's 512-byte row segments are staged by 1-D bulk copies
    // (cp.async.bulk, issued by lane 0, completion on a per-slot mbarrier)
    // into a private ring of `nst` slots in the idle union-find arrays, up to
    // nst rows ahead of the walk.  The step's ranges come from shared memory
    // (conflict-free 4-byte loads at 32 j + lane), so only the row above and
    // the current row live in registers (two sets instead of four).  A slot is
    // refilled by the warp itself after the step that consumed its row (the
    // ballots depend on the values, so the loads have completed): no
    // consumer-release barrier is needed.
    uint32_t ring = 0;      // shared-memory byte address of the warp's ring (+ 4 lane)
    uint32_t bars = 0;      // shared-memory byte address of the warp's mbarriers
    static constexpr int kSt = RS_TMA_RING;   // slots (a power of two)
    static_assert((kSt & (kSt - 1)) == 0 && kSt >= 2, "RS_TMA_RING must be a power of two");
    mutable uint32_t ci = 0;            // rows fetched so far: slot = ci % kSt, parity = (ci / kSt) & 1
    mutable int pnext = 0;              // next row to issue
    mutable const float *gsrc = nullptr;   // its chunk segment in global memory

    // lane 0: row pnext -> the slot of fetch number i (i % kSt)
    __device__ __forceinline__ void issue(uint32_t i) const {
        if (pnext < rend && lane == 0) {
            const uint32_t s = i & (kSt - 1);
            const uint32_t bar = bars + 8u * s, dst = ring + 512u * s;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 512;" ::"r"(bar) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(dst),
                         "l"(gsrc), "r"(bar)
                         : "memory");
        }
        ++pnext;
        gsrc += rowf;
    }
    // Rows are fetched strictly in order.  Before waiting for fetch ci the slot
    // of fetch ci - 1 is refilled: its values were consumed by the previous
    // step (or, for the very first rows, are refilled one fetch later).
    template <bool REFILL = true>
    __device__ __forceinline__ void get(float (&x)[4]) const {
        if (REFILL) issue(ci - 1u);
        const uint32_t s = ci & (kSt - 1);
        const uint32_t bar = bars + 8u * s;
        const uint32_t par = (ci / kSt) & 1u;
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(bar), "r"(par)
                : "memory");
        }
        const uint32_t src = ring + 512u * s + 4u * (uint32_t)lane;
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = __uint_as_float(lds_u32v(src + 128u * j));
        ++ci;
    }

    __device__ __forceinline__ void run_ring() const {
        float S0[4], S1[4];
        const int first = rfirst == 0 ? 0 : rfirst - 1;
        pnext = first;
        gsrc = col - lane + (size_t)first * rowf;
        ci = 0;
#pragma unroll 1
        for (uint32_t i = 0; i < (uint32_t)kSt; ++i) issue(i);
        int r;
        // the first two fetches are consumed by the first step: their slots are
        // refilled after it (fetch 0 by the next get, fetch 1 by the one after)
        get<false>(S0);
        if (rfirst == 0) {   // row 0: ground pair (0, 1), no up edges
            if (1 < rend) get<false>(S1);
            else {
#pragma unroll
                for (int j = 0; j < 4; ++j) S1[j] = 0.f;
            }
            if (r0 > 0) step<true, true>(0, S0, S0, S1, S0);
            else step<true>(0, S0, S0, S1, S0);
            if (1 >= rend) return;
            issue(0u);
            step<false>(1, S0, S1, S1, S0);
            r = 2;   // row above = S1
        } else {
            get<false>(S1);
            if (rfirst < r0) step<false, true>(rfirst, S0, S1, S1, S0);   // the halo row: P / L only
            else step<false>(rfirst, S0, S1, S1, S0);
            issue(0u);
            r = rfirst + 1;   // row above = S1
        }
        for (; r < rend; r += 2) {
            get(S0);
            step<false>(r, S1, S0, S0, S1);
            if (r + 1 >= rend) break;
            get(S1);
            step<false>(r + 1, S0, S1, S1, S0);
        }
    }
#endif

#if RS_STRIP_SETS == 3
    // three rotating sets: rows r-1, r and the target of the one-row prefetch
    __device__ __forceinline__ void run() const {
        float S0[4], S1[4], S2[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) S0[j] = S1[j] = S2[j] = 0.f;
        int rf = rfirst;
        if (rfirst == 0) {   // row 0: ground pair (0, 1), no up edges; band 1 of R = 1: the halo row
            ld4(0, S1);
            ld4(1, S2);
            if (r0 > 0) step<true, true>(0, S0, S1, S2, S0);
            else step<true>(0, S0, S1, S2, S0);
            rf = 1;
        }
        if (rf >= rend) return;
        ld4(rf - 1, S0);
        ld4(rf, S1);
        np = col + (rf + 1) * rowf;
        if (rf < r0) {
            // the halo row (first row walked in a band > 0): P / L only
            step<false, true>(rf, S0, S1, S1, S2);
            ++rf;
            if (rf >= rend) return;
#pragma unroll
            for (int j = 0; j < 4; ++j) {   // (S0, S1, S2) = (r-2, r-1, r) -> (r-1, r, r-2)
                const float t = S0[j];
                S0[j] = S1[j];
                S1[j] = S2[j];
                S2[j] = t;
            }
        }
        for (int r = rf; r < rend; r += 3) {
            step<false>(r, S0, S1, S1, S2);
            if (r + 1 >= rend) break;
            step<false>(r + 1, S1, S2, S2, S0);
            if (r + 2 >= rend) break;
            step<false>(r + 2, S2, S0, S0, S1);
        }
    }
#else
    // four rotating sets: rows r-1, r, r+1 (prefetched) and the target of
    // the two-row prefetch
    __device__ __forceinline__ void run() const {
        float S0[4], S1[4], S2[4], S3[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) S0[j] = S1[j] = S2[j] = S3[j] = 0.f;
        int rf = rfirst;
        if (rfirst == 0) {   // row 0: ground pair (0, 1), no up edges; band 1 of R = 1: the halo row
            ld4(0, S1);
            ld4(1, S2);
            if (r0 > 0) step<true, true>(0, S0, S1, S2, S3);
            else step<true>(0, S0, S1, S2, S3);
            rf = 1;
        }
        if (rf >= rend) return;
        ld4(rf - 1, S0);
        ld4(rf, S1);
        ld4(rf + 1, S2, rf + 1 < rend);
        np = col + (rf + 2) * rowf;
        if (rf < r0) {
            // the halo row (first row walked in a band > 0): P / L only
            step<false, true>(rf, S0, S1, S2, S3);
            ++rf;
            if (rf >= rend) return;
#pragma unroll
            for (int j = 0; j < 4; ++j) {   // (r-2, r-1, r, r+1) -> (r-1, r, r+1, r-2)
                const float t = S0[j];
                S0[j] = S1[j];
                S1[j] = S2[j];
                S2[j] = S3[j];
                S3[j] = t;
            }
        }
        for (int r = rf; r < rend; r += 4) {
            step<false>(r, S0, S1, S2, S3);
            if (r + 1 >= rend) break;
            step<false>(r + 1, S1, S2, S3, S0);
            if (r + 2 >= rend) break;
            step<false>(r + 2, S2, S3, S0, S1);
            if (r + 3 >= rend) break;
            step<false>(r + 3, S3, S0, S1, S2);
        }
    }
#endif
};

// MC: the frame has Map Connection offsets (a.n_off > 0).  A separate
// instantiation, so the code generation of the default kernel (whose speed is
// sensitive to register allocation) does not depend on the Map Connection code.
template <bool MC>
__global__ void __launch_bounds__(kFastThreads, kFastOcc) rs_fast_kernel(const __grid_constant__ KArgs a) {
    extern __shared__ __align__(128) uint32_t sm[];
    __shared__ uint32_t warp_tot[kFastWarps];
    __shared__ uint32_t cta_cnt, cta_sum, ovf, ovf_any, n_edges, n_xedges, ucur;
    __shared__ uint32_t cta_bad;       // a range of the band breaks the input contract (range_image.py:50-53)
    __shared__ uint32_t cta_pre[16];   // label base of every band of the cluster
    __shared__ uint32_t ovf_cnt[2];    // overflow path: kept roots and their cells in this band
    __shared__ uint32_t seam[2];   // seam edge per own row (R <= 64)
    __shared__ __align__(16) float rowc[(64 + 1) * 8];   // per-row constants of the band

    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int frame = blockIdx.x / a.C;
    const int H = a.H, W = a.W, R = a.R, WPR = a.WPR;
    const int r0 = k * R;
    const int rows = min(R, H - r0);
    const int nw = rows * WPR;
    const float *fr = a.ranges + (size_t)frame * H * W;
    const float thr = a.dmax2, tch = a.tch;
    const uint32_t band = (uint32_t)k << a.SHN;
    const uint32_t maskN = (1u << a.SHN) - 1u;

    uint32_t *P = sm + a.o_P, *L = sm + a.o_L, *U = sm + a.o_U;
    uint32_t *SB = sm + a.o_SB, *NB = sm + a.o_RS;
    uint32_t *Ph = sm + a.o_Ph, *Lh = sm + a.o_Lh;
    uint32_t *LR = sm + a.o_LR, *KB = sm + a.o_K;
    uint32_t *E = sm + a.o_E, *SZ = sm + a.o_SZ;
    auto G = [&](int r, int c) -> float { return __ldg(fr + (size_t)r * W + c); };

    RS_MARK(0);
    if (tid == 0) { seam[0] = seam[1] = 0; cta_sum = 0; n_edges = 0; n_xedges = 0; ucur = 0; cta_bad = 0; }

    // ---- A. presence, left and up bits --------------------------------------
    // Row constants of the band (ground pair, height sine, vertical 2cos)
    // are staged once; each lane then handles 4 consecutive cells of a
    // 128-column chunk and walks down the rows with the row above in
    // registers.  Nibbles are gathered into 32-bit words with a 3-step OR
    // butterfly over the 8 lanes of a word.
    const int rstart = r0 > 0 ? r0 - 1 : 0;
    const int rend = r0 + rows;
    for (int r = rstart + tid; r < rend; r += kFastThreads) {
        const GroundRow g = ground_row(a, r);
        float *rc = rowc + (r - rstart) * 8;
        rc[0] = g.sa; rc[1] = g.ca; rc[2] = g.lo; rc[3] = g.hi;
        z_threshold(g.sc, a.mount, a.keep_above, rc[4], rc[6]);
        rc[5] = r >= 1 ? __ldg(a.tables + 5 * H - 4 + r - 1) : 0.f;
    }
    __syncthreads();
    {
        uint32_t umx = 0;   // input-contract screen over every range this thread loads
        // narrow frames: split each chunk's rows between S warps so that no
        // warp idles (a part starts one row early for its row-above values)
        const int nchunk = (W + 127) / 128;
        const int nrow = rend - rstart;
        const int S = max(1, min(kFastWarps / nchunk, nrow / 8));
        const int per = (nrow + S - 1) / S;
#ifdef RS_TMA_RING
        // the warp's row ring (idle union-find arrays) and its mbarriers (idle LR / KB words)
        const uint32_t ring_base = smem_addr(sm + a.o_E) + 512u * (uint32_t)(warp * RS_TMA_RING);
        const uint32_t bars_base = smem_addr(sm + a.o_LR) + 8u * (uint32_t)(warp * RS_TMA_RING);
        if (a.ring) {
            if (lane == 0) {
                for (int i = 0; i < RS_TMA_RING; ++i)
                    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars_base + 8u * (uint32_t)i) : "memory");
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
            __syncwarp();
        }
#endif
        for (int t = warp; t < nchunk * S; t += kFastWarps) {
            const int ch = t % nchunk, part = t / nchunk;
            const int rlo = rstart + part * per, rhi = min(rend, rlo + per);
            const int cb = ch * 128 + lane;
            const uint32_t sb = smem_addr(sm) + 4u * (uint32_t)(ch * 4);
            const uint32_t sP = sb + 4u * a.o_P, sL = sb + 4u * a.o_L, sU = sb + 4u * a.o_U;
            const uint32_t sPh = sb + 4u * a.o_Ph, sLh = sb + 4u * a.o_Lh;
            const bool full = ch * 128 + 128 <= W && (WPR & 3) == 0;
#define RS_STRIP(F, G)                                                                                          \
    do {                                                                                                    \
        const BitsStrip<F, G, false, !MC> st{a, fr + cb, rowc, sP, sL, sU, sPh, sLh, ch, lane, r0, rstart, rhi, cb, \
                                             thr, tch, rlo, W, 4 * WPR};                                  \
        st.run();                                                                                           \
        umx = max(umx, st.mx);                                                                              \
    } while (0)
#ifdef RS_TMA_RING
#define RS_RING(G)                                                                                              \
    do {                                                                                                    \
        BitsStrip<true, G, true> st{a, fr + cb, rowc, sP, sL, sU, sPh, sLh, ch, lane, r0, rstart, rhi, cb, thr, \
                                    tch, rlo, W, 4 * WPR};                                                  \
        st.ring = ring_base;                                                                                \
        st.bars = bars_base;                                                                                \
        st.run_ring();                                                                                      \
        umx = max(umx, st.mx);                                                                              \
    } while (0)
            if (a.ring && full) {
                if (a.ground) RS_RING(true); else RS_RING(false);
                continue;
            }
#undef RS_RING
#endif
            if (a.ground) {
                if (full) RS_STRIP(true, true); else RS_STRIP(false, true);
            } else {
                if (full) RS_STRIP(true, false); else RS_STRIP(false, false);
            }
#undef RS_STRIP
        }
#ifdef RS_TMA_RING
        if (a.ring && lane == 0)
            for (int i = 0; i < RS_TMA_RING; ++i)
                asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bars_base + 8u * (uint32_t)i) : "memory");
#endif
        if (__any_sync(kFull, umx > kMaxFiniteBits) && lane == 0) cta_bad = 1u;
    }
    __syncthreads();
    if (cta_bad) {
        // rare (a contract violation, or a -0.0): exact re-check of the band's own rows
        bool b = false;
        const float *own = fr + (size_t)r0 * W;
        for (int i = tid; i < rows * W; i += kFastThreads) b |= !range_ok(__ldg(own + i));
        b = __syncthreads_or(b);
        if (tid == 0) cta_bad = b ? 1u : 0u;
    }
    RS_MARK(1);
    RS_STOP(1);

    // ---- B. edge words, seam, Map Connection bits ----------------------------
    // L = EH & P & (P shifted in from the left), U = EV & P & (P of the row
    // above); bit 0 of a chunk's first word (whose left cell step A did not
    // see) is tested here.  Word nw.. = the halo row (P / L only).
    for (int w = tid; w < nw + WPR; w += kFastThreads) {
        int cw, r;
        uint32_t *Lw, pw, pprev, pab = 0, *Uw = nullptr, ev = 0;
        if (w < nw) {
            const int q = divWPR(a, w);
            cw = w - q * WPR;
            r = r0 + q;
            Lw = L + w; Uw = U + w; pw = P[w]; ev = U[w];
            pab = q > 0 ? P[w - WPR] : (r0 > 0 ? Ph[cw] : 0u);
            pprev = cw > 0 ? P[w - 1] : 0u;
        } else {
            if (r0 == 0) break;
            cw = w - nw;
            r = r0 - 1;
            Lw = Lh + cw; pw = Ph[cw];
            pprev = cw > 0 ? Ph[cw - 1] : 0u;
        }
        uint32_t eh = *Lw;
        if ((cw & 3) == 0) {
            eh &= ~1u;
            const int c = cw * 32;
            if (cw > 0 && (pw & 1u) && (pprev >> 31) && pair_pass(G(r, c - 1), G(r, c), tch, thr)) eh |= 1u;
        }
        *Lw = eh & pw & ((pw << 1) | (pprev >> 31));
        if (Uw) *Uw = ev & pw & pab;
    }
    if (W > 1) {
        for (int q = tid; q < rows; q += kFastThreads) {
            const int r = r0 + q;
            const uint32_t pe = P[q * WPR + (W - 1) / 32] >> ((W - 1) & 31);
            if ((pe & 1u) && (P[q * WPR] & 1u) && pair_pass(G(r, W - 1), G(r, 0), tch, thr))
                atomicOr(&seam[q >> 5], 1u << (q & 31));
        }
    }
    __syncthreads();
    RS_MARK(2);
#ifndef RS_NO_PLANES
    if (a.planes) {
        // debug export (rs_fast_planes): P, L (bit 0 of a row = the seam edge)
        // and U of the band's own rows, final here (the Map Connection planes
        // are written by the Map Connection pass, mc_pass)
        const size_t fw = (size_t)H * WPR;
        uint32_t *out = a.planes + (size_t)frame * (3 + a.n_off) * fw + (size_t)r0 * WPR;
        for (int w = tid; w < nw; w += kFastThreads) {
            const int q = divWPR(a, w);
            const bool sm0 = (w - q * WPR) == 0 && ((seam[q >> 5] >> (q & 31)) & 1u);
            out[w] = P[w];
            out[fw + w] = L[w] | (sm0 ? 1u : 0u);
            out[2 * fw + w] = U[w];
        }
    }
#endif

    // ---- R. runs and their ids ------------------------------------------------
    // Warp `warp` owns words [wr0, wr1); a run continuing into the range gets a
    // pseudo start at its first cell (joined to its run in step U).
    const int per = (nw + kFastWarps - 1) / kFastWarps;
    const int wr0 = min(warp * per, nw), wr1 = min(wr0 + per, nw);
    {
        uint32_t run = 0;
        for (int cb = wr0; cb < wr1; cb += 32) {
            const int w = cb + lane;
            uint32_t sb = 0;
            if (w < wr1) {
                const uint32_t pw = P[w], lw = L[w];
                sb = (pw & ~lw) | ((w == wr0) ? (pw & lw & 1u) : 0u);
            }
            const uint32_t cnt = __popc(sb);
            uint32_t inc = cnt;
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t t = __shfl_up_sync(kFull, inc, off);
                if (lane >= off) inc += t;
            }
            if (w < wr1) {
                SB[w] = sb;
                NB[w] = run + inc - cnt;
            }
            run += __shfl_sync(kFull, inc, 31);
        }
        if (lane == 0) warp_tot[warp] = run;
    }
    __syncthreads();
    uint32_t n_runs = 0, my_off = 0;
    for (int i = 0; i < kFastWarps; ++i) {
        if (i < warp) my_off += warp_tot[i];
        n_runs += warp_tot[i];
    }
    if (tid == 0) ovf = n_runs > (uint32_t)a.NC;
    const bool overflow = n_runs > (uint32_t)a.NC;   // block-uniform
    RS_CHECK(overflow || n_runs <= (uint32_t)a.NC, "run count");
    if (!overflow) {
        for (int w = wr0 + lane; w < wr1; w += 32) NB[w] += my_off;
        for (uint32_t id = tid; id < n_runs; id += kFastThreads) {
            E[id] = band | id;
            SZ[id] = 0;
        }
    }
    __syncthreads();
    RS_MARK(3);
    RS_STOP(2);

    RunUF uf{E, cl, maskN, a.SHN, k, a.NC, a.C};
    if (!overflow) {
        // ---- U. band-local unions ----------------------------------------------
        // Edges are gathered into a list (the size array is the buffer; it is
        // zeroed again by the flatten below).  Then, with no finds at all,
        // every run hooks under its smallest neighbour (atomicMin on its own
        // entry: an acyclic forest since pointers go to smaller ids; about 9
        // in 10 edges are then inside one tree), and finally all listed edges
        // are united; path halving in those finds flattens the forest (a
        // separate flatten pass cost more than it saved).  A list that
        // overflowed is re-gathered with the unions done on the spot (the
        // union order never matters).
        uint32_t *EL = SZ;
        const uint32_t cap = (uint32_t)a.NC;
        auto gather = [&](const bool direct) {
            for (int wb = warp * 32; wb < nw; wb += kFastThreads) {
                const int w = wb + lane;
                const bool act = w < nw;
                const int q = act ? divWPR(a, w) : 0;
                const int cw = w - q * WPR;
                const uint32_t lw = act ? L[w] : 0u, sb = act ? SB[w] : 0u, uw = act ? U[w] : 0u;
                const bool pseudo = (sb & lw & 1u) != 0;
                uint32_t nru = 0;
                if (q > 0 && uw) {
                    const uint32_t uprev = (uw << 1) | (cw > 0 ? U[w - 1] >> 31 : 0u);
                    nru = uw & ~(uprev & lw & L[w - WPR]);
                }
                const bool sm_ = act && cw == 0 && ((seam[q >> 5] >> (q & 31)) & 1u);
                const uint32_t k = (uint32_t)pseudo + __popc(nru) + (uint32_t)sm_;
                uint32_t slot = 0;
                if (!direct && __any_sync(kFull, k != 0u)) {
                    // warp-aggregated reservation in the edge list
                    uint32_t inc = k;
                    for (int off = 1; off < 32; off <<= 1) {
                        const uint32_t t = __shfl_up_sync(kFull, inc, off);
                        if (lane >= off) inc += t;
                    }
                    uint32_t wbase = 0;
                    if (lane == 31 && inc) wbase = atomicAdd(&n_edges, inc);
                    wbase = __shfl_sync(kFull, wbase, 31);
                    slot = wbase + inc - k;
                }
                if (!k) continue;
                auto push = [&](uint32_t x, uint32_t y) {
                    RS_CHECK(x < n_runs && y < n_runs, "listed edge run ids");
                    if (direct) uf.unite_local(band | x, band | y);
                    else if (slot < cap) EL[slot] = (x << 16) | y;
                    ++slot;
                };
                // run ids from register copies: NB[w] counts the runs before
                // word w, so the run holding bit 31 of word w-1 is NB[w] - 1
                const uint32_t nbw = NB[w];
                const uint32_t x0 = nbw + (sb & 1u) - 1u;   // run of bit 0
                if (pseudo) push(nbw, nbw - 1u);
                if (nru) {
                    const uint32_t sbu = SB[w - WPR], nbu = NB[w - WPR] - 1u, nbm = nbw - 1u;
                    for (; nru; nru &= nru - 1) {
                        const uint32_t le = 0xffffffffu >> (31 - (__ffs(nru) - 1));
                        push(nbm + __popc(sb & le), nbu + __popc(sbu & le));
                    }
                }
                if (sm_) push(x0, run_of(SB, NB, q * WPR + (W - 1) / 32, (W - 1) & 31));
            }
        };
        gather(false);
        __syncthreads();
        RS_MARK(19);
        RS_STOP(9);
        const uint32_t ne = n_edges;   // block-uniform
        if (ne > cap) {
            gather(true);
        } else {
            // hook every run under its smallest listed neighbour
            for (uint32_t e = tid; e < ne; e += kFastThreads) {
                const uint32_t x = EL[e], u = x >> 16, v = x & 0xffffu;
                atomicMin(E + max(u, v), band | min(u, v));
            }
            __syncthreads();
            RS_MARK(20);
            if (a.udyn) {
                // bands of a multi-band frame (their loads differ, and the
                // cluster waits on the slowest): warps grab 64 edges at a
                // time, 2 contiguous per lane (config 1 -2.2%, config 2 -3.5%
                // against fixed contiguous slices)
                constexpr uint32_t kGrab = RS_UDYN_GRAB;
                while (true) {
                    uint32_t base = 0;
                    if (lane == 0) base = atomicAdd(&ucur, 32 * kGrab);
                    base = __shfl_sync(kFull, base, 0);
                    if (base >= ne) break;
                    const uint32_t e0 = min(base + lane * kGrab, ne), e1 = min(e0 + kGrab, ne);
                    for (uint32_t e = e0; e < e1; ++e) {
                        const uint32_t x = EL[e];
                        uf.unite_local(band | (x >> 16), band | (x & 0xffffu));
                    }
                }
            } else {
                // contiguous slices per thread: edges next to each other in
                // the list mostly join the same components
                const uint32_t per = (ne + kFastThreads - 1) / kFastThreads;
                const uint32_t e0 = min(tid * per, ne), e1 = min(e0 + per, ne);
                for (uint32_t e = e0; e < e1; ++e) {
                    const uint32_t x = EL[e];
                    uf.unite_local(band | (x >> 16), band | (x & 0xffffu));
                }
            }
        }
        __syncthreads();
        RS_MARK(4);
    RS_STOP(3);
        // local flatten; LR marks the band-local roots
        auto flatten = [&]() {
            for (uint32_t base = warp * 32; base < n_runs; base += kFastThreads) {
                const uint32_t id = base + lane;
                bool lr = false;
                if (id < n_runs) {
                    // most trees are at most two deep after the unions: two plain
                    // loads, then (rarely) path halving with atomicMin — entries only
                    // ever decrease, so a finished root pointer is never overwritten
                    const uint32_t p = E[id];
                    const uint32_t gp = E[p & maskN];
                    const uint32_t r = gp == p ? p : uf.find_local_min(gp);
                    E[id] = r;
                    SZ[id] = 0;   // it served as the edge list
                    lr = r == (band | id);
                }
                const uint32_t m = __ballot_sync(kFull, lr);
                if (lane == 0) LR[base >> 5] = m;
            }
        };
        flatten();
        if (MC && tid == 0) n_edges = ucur = 0;
        __syncthreads();
        RS_MARK(5);
        if (MC && a.n_off > 0 && !a.planes && (W & 31) == 0) {
            // ---- Map Connections inside the band (rs_mc.cuh: mc_axis_heads /
            // mc_chain_issue / mc_chain_finish), while nothing outside the CTA
            // touches its forest: chains of candidate pairs whose runs have
            // different local roots are listed (the size array is the
            // buffer), then tested and united by all threads, and the forest
            // is flattened again.  One round for the skip offsets (0, k) /
            // (k, 0) together (few candidates: only where the straight chain
            // of links is broken), one round for every other offset (every
            // present pair is a candidate; the re-flattened forest of the
            // earlier rounds rules most of them out).  Rows whose partner row
            // lies in another band are handled with the cross-band edges
            // (step X).
            const uint32_t lcap = (uint32_t)a.NC / 2u;   // two words per chain
            auto ul = [&](uint32_t x, uint32_t y) { uf.unite_local(band | x, band | y); };
            auto chain = [&](uint32_t e, uint32_t cells) {
                mc_chain_finish(a, SB, NB, fr, r0, e, cells, mc_chain_issue(a, fr, r0, e, cells), ul);
            };
            uint32_t *cnt = &n_edges, *cnt_next = &ucur;   // list counters of this / the next round (both zero)
            for (int o0 = 0; o0 < a.n_off;) {
                int o1 = o0 + 1;
                if (mc_axis_offset(a, o0))
                    while (o1 < a.n_off && mc_axis_offset(a, o1)) ++o1;   // consecutive skip offsets share a round
                mc_axis_heads(a, o0, o1, P, L, U, SB, NB, E, rows, tid, kFastThreads, SZ, lcap, cnt, chain);
                __syncthreads();
                RS_MARK(21);
                const uint32_t nl = min(*cnt, lcap);   // block-uniform
                for (uint32_t i = tid; i < nl; i += kFastThreads) {
                    const uint32_t e = SZ[2 * i], cells = SZ[2 * i + 1];
                    SZ[2 * i] = SZ[2 * i + 1] = 0;
                    chain(e, cells);
                }
                __syncthreads();
                RS_MARK(23);
                // every thread has read this round's counter: zero it for the round
                // after the next (nobody touches it during the next round)
                if (tid == 0) *cnt = 0;
                uint32_t *t = cnt; cnt = cnt_next; cnt_next = t;
                if (nl) {
                    // flatten again, in two steps: the roots of the last flatten
                    // (LR bits; every other run points at one of them) find
                    // their new root by pointer jumping (every such root repeats
                    // E[r] = E[E[r]] while the others do the same, so a chain of
                    // hooks of any depth — skips merge runs along a row one
                    // after the other — takes a logarithmic number of steps),
                    // then every run takes one hop
                    for (uint32_t w = warp; w < (n_runs + 31) / 32; w += kFastWarps) {
                        const uint32_t id = w * 32 + lane;
                        if (!((LR[w] >> lane) & 1u)) continue;
                        volatile uint32_t *V = E;
                        while (true) {
                            const uint32_t p = V[id];
                            const uint32_t gp = V[p & maskN];
                            if (gp == p) break;
                            V[id] = gp;
                        }
                    }
                    __syncthreads();
                    for (uint32_t base = warp * 32; base < n_runs; base += kFastThreads) {
                        const uint32_t id = base + lane;
                        bool lr = false;
                        if (id < n_runs) {
                            const uint32_t r = E[E[id] & maskN];
                            E[id] = r;
                            lr = r == (band | id);
                        }
                        const uint32_t m = __ballot_sync(kFull, lr);
                        if (lane == 0) LR[base >> 5] = m;
                    }
                    __syncthreads();
                }
                o0 = o1;
            }
            RS_MARK(22);
        }
        // local component sizes: each run adds its length to its local root
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
            // first run end at or after this word (inc) and after it (exc):
            // the first end of the next lane that has one (positions grow
            // with the lane), else the carry from the chunk after this one
            const int fe = eb ? base + __ffs(eb) - 1 : INT_MAX;
            const uint32_t he = __ballot_sync(kFull, eb != 0u);
            const uint32_t ge = he & ~((1u << lane) - 1u), gt = he & ~lanemask_le(lane);
            const int li = ge ? __ffs(ge) - 1 : 0, lx = gt ? __ffs(gt) - 1 : 0;
            const int fi = __shfl_sync(kFull, fe, li), fx = __shfl_sync(kFull, fe, lx);
            const int inc = ge ? fi : carry;
            const int exc = gt ? fx : carry;
            if (sb) {
                uint32_t id = NB[w];
                for (uint32_t m = sb; m; m &= m - 1, ++id) {
                    const int b = __ffs(m) - 1;
                    const uint32_t after = eb & ~((1u << b) - 1u);
                    const int end = after ? base + __ffs(after) - 1 : exc;
                    atomicAdd(SZ + (E[id] & maskN), (uint32_t)(end - (base + b) + 1));
                }
            }
            carry = __shfl_sync(kFull, inc, 0);
        }
    }
    RS_STOP(4);
    RS_MARK(6);
    cl.sync();   // #1: every band's runs are numbered, joined locally and sized

    if (tid == 0) {
        uint32_t any = 0;
        for (int j = 0; j < a.C; ++j) any |= *cl.map_shared_rank(&ovf, j);
        ovf_any = any;
    }
    __syncthreads();
    if (ovf_any) {   // cluster-uniform: union-find over cells in global memory (rs_overflow.cuh)
        overflow_frame(a, P, L, U, Lh, seam, ovf_cnt, warp_tot, frame, &cta_bad);
        return;
    }

    RS_MARK(7);
    // Map Connections were united inside the band before barrier #1 and are
    // finished with the cross-band edges below; step M is only needed for the
    // parity export and for widths that are not whole words
    const bool inband = MC && a.n_off > 0 && !a.planes && (W & 31) == 0;
    const bool mstep = MC && a.n_off > 0 && !inband;
    // ---- X. cross-band unions over DSMEM -----------------------------------
    // Boundary edges are listed first (rows 1.. of the U plane are free now and
    // serve as the buffer), then united by all threads in parallel.  The up
    // edges across a boundary are listed by both bands next to it: the lower
    // band takes the upper half of the words, the band above the lower half
    // (reading the lower band's row-0 planes over DSMEM), so the boundary work
    // is shared instead of falling on the lower band alone.
    if (a.C > 1) {
        uint32_t *XL = U + WPR;
        const uint32_t xcap = (uint32_t)((rows - 1) * WPR / 2);
        // warp-aggregated: every lane calls, `has` lanes push an edge
        auto xpush = [&](bool has, uint32_t x, uint32_t y) {
            const uint32_t m = __ballot_sync(kFull, has);
            if (!m) return;
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&n_xedges, (uint32_t)__popc(m));
            base = __shfl_sync(kFull, base, 0);
            if (!has) return;
            const uint32_t slot = base + __popc(m & ((1u << lane) - 1u));
            if (slot < xcap) {
                XL[2 * slot] = x;
                XL[2 * slot + 1] = y;
            } else {
                uf.unite(x, y);
            }
        };
        // up edges from row 0 of band bl to the last row of band bl - 1, words [wlo, whi)
        auto boundary = [&](int bl, int wlo, int whi) {
            const int bu = bl - 1;
            const bool lower = bl == k;
            const uint32_t *U0 = lower ? U : cl.map_shared_rank(U, bl);
            const uint32_t *L0 = lower ? L : cl.map_shared_rank(L, bl);
            const uint32_t *Lup = lower ? Lh : L + (R - 1) * WPR;   // left edges of the row above
            const uint32_t *SBl = lower ? SB : cl.map_shared_rank(SB, bl);
            const uint32_t *NBl = lower ? NB : cl.map_shared_rank(NB, bl);
            const uint32_t *SBu = lower ? cl.map_shared_rank(SB, bu) : SB;
            const uint32_t *NBu = lower ? cl.map_shared_rank(NB, bu) : NB;
            const uint32_t tagl = (uint32_t)bl << a.SHN, tagu = (uint32_t)bu << a.SHN;
            const int wu0 = (R - 1) * WPR;
            for (int cbase = (wlo + warp) * 32; cbase < whi * 32; cbase += kFastThreads) {
                const int c = cbase + lane;
                const int cw = c >> 5, b = c & 31;
                const uint32_t uw = U0[cw];
                const uint32_t upb = b > 0 ? (uw >> (b - 1)) & 1u : (cw > 0 ? U0[cw - 1] >> 31 : 0u);
                const bool has = ((uw >> b) & 1u) && !(upb && ((L0[cw] >> b) & 1u) && ((Lup[cw] >> b) & 1u));
                xpush(has, has ? tagl | run_of(SBl, NBl, cw, b) : 0u,
                      has ? tagu | run_of(SBu, NBu, wu0 + cw, b) : 0u);
            }
        };
        const int whalf = WPR / 2;
        if (r0 > 0) boundary(k, whalf, WPR);
        if (k + 1 < a.C) boundary(k + 1, 0, whalf);
        // Map Connection pairs whose partner row lies in a band above: a lane
        // per cell, passing pairs join the cross-band edge list; shared by the
        // two bands of a boundary like the up edges
        // The first such offset shares the list with the up edges; after that
        // the list is united and reused per offset, and the unions so far
        // rule out most of the later offsets' pairs (roots compared per chain).
        auto flush = [&]() {
            __syncthreads();
            const uint32_t nx = min(n_xedges, xcap);
            for (uint32_t e = tid; e < nx; e += kFastThreads) uf.unite(XL[2 * e], XL[2 * e + 1]);
        };
        if (inband) {
            auto xroot = [&](uint32_t e) { return uf.find_nc(uf.ld(e)); };
            bool first = true;
            for (int o = 0; o < a.n_off; ++o) {
                if (a.dy[o] == 0) continue;
                if (!first) {
                    flush();
                    __syncthreads();
                    if (tid == 0) n_xedges = 0;
                    __syncthreads();
                }
                if (r0 > 0)
                    mc_axis_cross(a, cl, k, k, o, P, L, SB, NB, fr, lane, warp, kFastWarps, !first, xroot, xpush);
                if (k + 1 < a.C)
                    mc_axis_cross(a, cl, k, k + 1, o, P, L, SB, NB, fr, lane, warp, kFastWarps, !first, xroot, xpush);
                first = false;
            }
        }
        flush();
    }
    RS_STOP(5);
    RS_MARK(8);
    cl.sync();   // #2: the forest of the direct edges is final
    RS_MARK(9);
#ifndef RS_MC_NO_PASS
    if (mstep) {
        // ---- M. Map Connection edges (rs_mc.cuh).  Every run first points
        // straight at its root (a compression of the final direct-edge forest;
        // other bands may still be compressing, which only makes a root
        // comparison say "different" more often), then pairs whose chains
        // join different roots are tested; passing ones are listed in the U
        // plane (free: the cross-band list is consumed) and united by all
        // threads.  Step L then takes two hops (run -> old root -> final root).
        for (uint32_t id = tid; id < n_runs; id += kFastThreads) E[id] = uf.find_nc(band | id);
        if (tid == 0) n_edges = 0;
        __syncthreads();
        RS_MARK(21);
        uint32_t *ML = U;
        const uint32_t mcap = (uint32_t)(nw / 2);
        uint32_t *exp = a.planes ? a.planes + (size_t)frame * (3 + a.n_off) * H * WPR : nullptr;
        auto run_in = [&](int kt, int tw, int tb) {
            const uint32_t *SBt = kt == k ? SB : cl.map_shared_rank(SB, kt);
            const uint32_t *NBt = kt == k ? NB : cl.map_shared_rank(NB, kt);
            return ((uint32_t)kt << a.SHN) | run_of(SBt, NBt, tw, tb);
        };
        if (!exp)
            mc_runs(a, cl, k, P, L, SB, NB, fr, r0, rows, n_runs, tid, kFastThreads, ML, mcap, &ucur,
                    [&](int kt, uint32_t id) { return kt == k ? E[id] : *cl.map_shared_rank(E + id, kt); },
                    [&](int kt, uint32_t id) { return uf.find_nc(((uint32_t)kt << a.SHN) | id); },
                    [&](uint32_t x, uint32_t y) { uf.unite_roots(x, y); });
        else   // parity export: every present pair tested and its decision written
        mc_pass<true>(
            a, cl, k, P, L, fr, r0, rows, lane, warp, kFastWarps, exp,
            [&](int w, int b) { return E[run_of(SB, NB, w, b)]; },
            [&](int kt, int tw, int tb) { return uf.ld(run_in(kt, tw, tb)); },
            [&](bool has, int w, int b, int kt, int tw, int, int, int, int tc) {
                uint32_t x = 0, y = 0;
                if (has) {
                    x = band | run_of(SB, NB, w, b);
                    y = run_in(kt, tw, tc & 31);
                }
                const uint32_t m = __ballot_sync(kFull, has);
                if (!m) return;
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&n_edges, (uint32_t)__popc(m));
                base = __shfl_sync(kFull, base, 0);
                if (!has) return;
                const uint32_t slot = base + __popc(m & ((1u << lane) - 1u));
                if (slot < mcap) {
                    ML[2 * slot] = x;
                    ML[2 * slot + 1] = y;
                } else {
                    uf.unite(x, y);
                }
            });
        __syncthreads();
        RS_MARK(22);
        const uint32_t nm = min(n_edges, mcap);
        for (uint32_t e = tid; e < nm; e += kFastThreads) uf.unite(ML[2 * e], ML[2 * e + 1]);
        RS_MARK(23);
        cl.sync();   // #2b: Map Connection unions done
    }
#endif

    // ---- Z. resolve: local roots chase their global root and add their size ---
    // Only band-local roots move (E[lr] = global root); other runs keep their
    // local root and resolve through it when labelled.
    for (uint32_t id = tid; id < n_runs; id += kFastThreads) {
        if (!((LR[id >> 5] >> (id & 31)) & 1u)) continue;
        const uint32_t g = uf.find_min(band | id);
        if (g != (band | id)) {
            E[id] = g;
            atomicAdd(uf.slot(SZ, g), SZ[id]);
        }
    }
    RS_STOP(6);
    RS_MARK(10);
    cl.sync();   // #3: sizes are final at every root

    // ---- K. kept roots, ordered rank ------------------------------------------
    const uint32_t minp = a.min_points > 1 ? (uint32_t)a.min_points : 1u;
    const uint32_t nkw = (n_runs + 31) / 32;
    for (uint32_t base = warp * 32; base < nkw * 32; base += kFastThreads) {
        const uint32_t id = base + lane;
        bool kept = false;
        uint32_t s = 0;
        if (id < n_runs && E[id] == (band | id)) {
            s = SZ[id];
            kept = s >= minp;
        }
        const uint32_t m = __ballot_sync(kFull, kept);
        s = kept ? s : 0u;
        s = __reduce_add_sync(kFull, s);
        if (lane == 0) {
            KB[base >> 5] = m;
            if (s) atomicAdd(&cta_sum, s);
        }
    }
    __syncthreads();
    {
        // block exclusive scan of popc(KB[w]) in word order; WK reuses LR
        uint32_t *WK = LR;
        uint32_t run = 0;
        const uint32_t wper = (nkw + kFastWarps - 1) / kFastWarps;
        const uint32_t w0 = min(warp * wper, nkw), w1 = min(w0 + wper, nkw);
        for (uint32_t cb = w0; cb < w1; cb += 32) {
            const uint32_t w = cb + lane;
            const uint32_t cnt = w < w1 ? __popc(KB[w]) : 0u;
            uint32_t inc = cnt;
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t t = __shfl_up_sync(kFull, inc, off);
                if (lane >= off) inc += t;
            }
            if (w < w1) WK[w] = run + inc - cnt;
            run += __shfl_sync(kFull, inc, 31);
        }
        if (lane == 0) warp_tot[warp] = run;
        __syncthreads();
        if (tid == 0) {
            uint32_t t = 0;
            for (int i = 0; i < kFastWarps; ++i) { const uint32_t x = warp_tot[i]; warp_tot[i] = t; t += x; }
            cta_cnt = t;
        }
        __syncthreads();
        for (uint32_t w = tid; w < nkw; w += kFastThreads)
            WK[w] += warp_tot[min(w / max(wper, 1u), (uint32_t)kFastWarps - 1)];
    }
    RS_MARK(11);
    cl.sync();   // #4: every band's kept bits, word prefixes and counts are published
    if (tid < a.C) {
        // label base of each band: kept roots of the bands before it
        uint32_t pre = 0, tot = 0, sum = 0, bad = 0;
        for (int j = 0; j < a.C; ++j) {
            const uint32_t cj = *cl.map_shared_rank(&cta_cnt, j);
            if (j < tid) pre += cj;
            tot += cj;
            if (tid == 0) {
                sum += *cl.map_shared_rank(&cta_sum, j);
                bad |= *cl.map_shared_rank(&cta_bad, j);
            }
        }
        cta_pre[tid] = pre;
        if (tid == 0 && k == 0) {
            // RS_FRAME_INVALID marks a frame that breaks the input contract
            if (a.ncl) a.ncl[frame] = bad ? RS_FRAME_INVALID : (int32_t)tot;
            if (a.sizes) a.sizes[(size_t)frame * a.sizes_stride] = (int64_t)H * W - (int64_t)sum;
        }
    }
    __syncthreads();
    RS_STOP(7);
    RS_MARK(12);

    // ---- L. run labels straight from the root's band: label = band base +
    // kept roots before it (word prefix + bits below) + 1, or 0 if dropped.
    // Kept bits and prefixes are final after barrier #4 (plain DSMEM loads).
    {
        const uint32_t *WK = LR;
#pragma unroll 4
        for (uint32_t id = tid; id < n_runs; id += kFastThreads) {
            const uint32_t lr = E[id];
            // lr: the band-local root (E[lr] = the final root after Z), or
            // with Map Connections the root before step M (a local root of
            // its band: one hop, possibly over DSMEM, to the final root)
            const uint32_t g = ((lr >> a.SHN) == (uint32_t)k) ? E[lr & maskN] : (mstep ? uf.ld(lr) : lr);
            const int owner = (int)(g >> a.SHN);
            const uint32_t gi = g & maskN;
            uint32_t km, wk;
            if (owner == k) {
                km = KB[gi >> 5];
                wk = WK[gi >> 5];
            } else {
                km = *cl.map_shared_rank(KB + (gi >> 5), owner);
                wk = *cl.map_shared_rank(WK + (gi >> 5), owner);
            }
            const uint32_t b = gi & 31;
            uint32_t label = 0;
            if ((km >> b) & 1u) {
                label = cta_pre[owner] + wk + __popc(km & ((1u << b) - 1u)) + 1u;
                RS_CHECK(!a.sizes || (int64_t)label < a.sizes_stride, "cluster_sizes row");
                if (g == (band | id) && a.sizes) a.sizes[(size_t)frame * a.sizes_stride + label] = (int64_t)SZ[id];
            }
            SZ[id] = label;   // only this thread read SZ[id] (the root's size)
        }
    }
    RS_STOP(8);
    RS_MARK(13);
    // #5, split: arrive now (this CTA reads no other CTA's shared memory after
    // this point), wait just before exiting (no CTA may exit while another
    // still reads its shared memory), so the wait overlaps the cell sweep
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    __syncthreads();   // run labels (SZ) of this band are complete

    RS_MARK(14);
    int32_t *out = a.labels + (size_t)frame * H * W + (size_t)r0 * W;
    if ((WPR & 3) == 0 && (W & 31) == 0) {
        // rows are whole words, so cell index == 32 * word + bit: a linear
        // sweep, lane = 4 consecutive cells, 16-byte streaming stores; run
        // ids of the lane's cells are the first id plus the run starts after it
        const int b0 = (lane & 7) * 4;
        const uint32_t lem = lanemask_le(b0);
        // byte addresses in shared memory: one add per cell instead of an
        // index → address computation per load
        const uint32_t szb = smem_addr(SZ) - 4u;
        int4 *dst = reinterpret_cast<int4 *>(out) + warp * 32 + lane;
#pragma unroll kSweepUnroll
        for (int w0 = warp * 4; w0 < nw; w0 += kFastWarps * 4, dst += kFastWarps * 32) {
            const int w = w0 + (lane >> 3);
            const uint32_t pw = P[w] >> b0, sbw = SB[w];
            const uint32_t st = sbw >> b0;
            uint32_t ad = szb + 4u * (NB[w] + __popc(sbw & lem));
            int4 lab;
            lab.x = (pw & 1u) ? (int)lds_u32(ad) : 0;
            ad += (st << 1) & 4u;
            lab.y = (pw & 2u) ? (int)lds_u32(ad) : 0;
            ad += st & 4u;
            lab.z = (pw & 4u) ? (int)lds_u32(ad) : 0;
            ad += (st >> 1) & 4u;
            lab.w = (pw & 8u) ? (int)lds_u32(ad) : 0;
            __stcs(dst, lab);
        }
    } else {
        for (int w = warp; w < nw; w += kFastWarps) {
            const int q = divWPR(a, w);
            const int c = (w - q * WPR) * 32 + lane;
            if (c < W) {
                const int lab = ((P[w] >> lane) & 1u) ? (int)SZ[run_of(SB, NB, w, lane)] : 0;
                __stcs(out + q * W + c, lab);
            }
        }
    }
    RS_MARK(15);
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace rs
