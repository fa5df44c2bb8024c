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
    int H, W, R, C, SH;
    int n_off;
    int dy[RS_MAX_OFFSETS];
    int dx[RS_MAX_OFFSETS];
    int min_points, ground;
    float dmax2, mount, keep_above, tch;
    unsigned long long magicW;    // ceil(2^40 / W): exact i / W for i*W < 2^40
    // shared-memory layout, in 32-bit words
    int o_P, o_L, o_U, o_Ph, o_Lh, o_seam, o_MC, o_TL, o_misc;
    int nwords, hwords;
    int use_tma;
};

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

// Presence = valid && !ground for cell (r, c); `get(row, col)` returns the range.
// ground.py:112-140 (pair k = max(r,1)-1; row 0 reuses pair 0 with its own
// height) and range_image.py:125-127 (z = r*sin + mount, two roundings).
template <class Get>
__device__ __forceinline__ bool present_at(const KArgs &a, int r, int c, Get get) {
    const float v = get(r, c);
    const bool valid = v > 0.f;
    if (!a.ground || !valid) return valid;
    const int H = a.H;
    const int k = (r >= 1 ? r : 1) - 1;
    const float d1 = get(k, c);
    const float d2 = get(k + 1, c);
    const float *t = a.tables;
    const float sa = __ldg(t + H + k);
    const float ca = __ldg(t + 2 * H - 1 + k);
    const float lo = __ldg(t + 3 * H - 2 + k);
    const float hi = __ldg(t + 4 * H - 3 + k);
    const float num = __fmul_rn(d2, sa);
    const float den = __fsub_rn(d1, __fmul_rn(d2, ca));
    const float L = __fmul_rn(lo, den);
    const float U = __fmul_rn(hi, den);
    bool ok = den > 0.f ? (num >= L && num <= U) : (num <= L && num >= U);
    ok = ok && den != 0.f && d1 > 0.f && d2 > 0.f;
    const float z = __fadd_rn(__fmul_rn(v, __ldg(t + r)), a.mount);
    const bool low = z <= a.keep_above;
    return !(ok && low);
}

__device__ __forceinline__ unsigned divW(const KArgs &a, unsigned i) {
    return (unsigned)(((unsigned long long)i * a.magicW) >> 40);
}

__device__ __forceinline__ bool bit(const uint32_t *w, int i) {
    return (w[i >> 5] >> (i & 31)) & 1u;
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
// Entries are cluster-encoded pixel indices e = (band << SH) | local, which
// order exactly like frame-linear indices.  Invariant: E[e] <= e, so a root is
// the minimum index of its tree.

struct UF {
    uint32_t *E;          // this CTA's entries (shared)
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
    __device__ uint32_t find(uint32_t e) const {
        uint32_t p = ld(e);
        while (p != e) {
            const uint32_t gp = ld(p);
            if (gp == p) return p;
            *reinterpret_cast<volatile uint32_t *>(slot(e)) = gp;   // path halving
            e = gp;
            p = ld(e);
        }
        return e;
    }
    __device__ void unite(uint32_t x, uint32_t y) const {
        while (true) {
            x = find(x);
            y = find(y);
            if (x == y) return;
            if (x > y) { const uint32_t t = x; x = y; y = t; }
            const uint32_t old = atomicMin(slot(y), x);   // hook larger root under smaller
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
    __shared__ uint32_t cta_cnt, cta_sum, cta_prefix;

    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int frame = blockIdx.x / a.C;
    const int H = a.H, W = a.W, R = a.R;
    const int r0 = k * R;
    const int rows = min(R, H - r0);
    const int n_own = rows * W;
    const int n_pad = a.nwords * 32;
    const float *fr = a.ranges + (size_t)frame * H * W;
    const int lo_row = max(r0 - 2, 0);
    const int hi_row = min(max(r0 + rows - 1, 1), H - 1);
    const float thr = a.dmax2;
    const uint32_t band = (uint32_t)k << a.SH;

    float *stage = reinterpret_cast<float *>(sm);
    uint32_t *E = sm;   // aliases the staging area after the edge phase
    uint32_t *P = sm + a.o_P, *L = sm + a.o_L, *U = sm + a.o_U;
    uint32_t *Ph = sm + a.o_Ph, *Lh = sm + a.o_Lh, *seam = sm + a.o_seam;
    uint32_t *MC = sm + a.o_MC, *TL = sm + a.o_TL;

    // ---- 1. stage rows [lo_row, hi_row] -------------------------------------
    const int n_stage = (hi_row - lo_row + 1) * W;
    const float *src = fr + (size_t)lo_row * W;
    if (a.use_tma) {
        if (tid == 0) {
            mbar_init(&mbar, 1);
            const uint32_t bytes = (uint32_t)n_stage * 4u;
            mbar_expect_tx(&mbar, bytes);
            const uint32_t row_bytes = (uint32_t)W * 4u;
            for (int s = 0; s <= hi_row - lo_row; ++s)
                tma_load_1d(stage + (size_t)s * W, src + (size_t)s * W, row_bytes, &mbar);
        }
        if (tid < 32) seam[0] = 0;   // cleared while the copy is in flight
        for (int i = tid; i < a.hwords; i += kThreads) { Ph[i] = 0; Lh[i] = 0; }
        __syncthreads();
        mbar_wait(&mbar, 0);
    } else {
        for (int i = tid; i < n_stage; i += kThreads) stage[i] = __ldg(src + i);
        if (tid == 0) seam[0] = 0;
        for (int i = tid; i < a.hwords; i += kThreads) { Ph[i] = 0; Lh[i] = 0; }
        __syncthreads();
    }

    auto S = [&](int r, int c) -> float { return stage[(r - lo_row) * W + c]; };
    auto G = [&](int r, int c) -> float { return __ldg(fr + (size_t)r * W + c); };

    // ---- 2. presence bits: own rows, then the halo row r0-1 -----------------
    for (int base = warp * 32; base < n_pad; base += kWarps * 32) {
        const int i = base + lane;
        bool p = false;
        if (i < n_own) {
            const int q = (int)divW(a, (unsigned)i);
            p = present_at(a, r0 + q, i - q * W, S);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, p);
        if (lane == 0) P[base >> 5] = m;
    }
    if (r0 > 0) {
        for (int base = warp * 32; base < a.hwords * 32; base += kWarps * 32) {
            const int c = base + lane;
            const bool p = c < W && present_at(a, r0 - 1, c, S);
            const uint32_t m = __ballot_sync(0xffffffffu, p);
            if (lane == 0) Ph[base >> 5] = m;
        }
    }
    __syncthreads();

    // ---- 3. edge bits --------------------------------------------------------
    // Halo row LEFT bits (needed by the cross-band redundant-edge test).
    if (r0 > 0) {
        for (int base = warp * 32; base < a.hwords * 32; base += kWarps * 32) {
            const int c = base + lane;
            bool l = false;
            if (c > 0 && c < W && bit(Ph, c) && bit(Ph, c - 1))
                l = pair_pass(S(r0 - 1, c - 1), S(r0 - 1, c), a.tch, thr);
            const uint32_t m = __ballot_sync(0xffffffffu, l);
            if (lane == 0) Lh[base >> 5] = m;
        }
    }
    const float *tcv = a.tables + 5 * H - 4;
    for (int base = warp * 32; base < n_pad; base += kWarps * 32) {
        const int i = base + lane;
        const bool inb = i < n_own;
        int q = 0, c = 0, r = r0;
        if (inb) {
            q = (int)divW(a, (unsigned)i);
            c = i - q * W;
            r = r0 + q;
        }
        const bool p = inb && bit(P, i);
        const float v = inb ? S(r, c) : 0.f;
        bool left = false, up = false;
        if (p) {
            if (c > 0) {
                left = bit(P, i - 1) && pair_pass(S(r, c - 1), v, a.tch, thr);
            } else if (W > 1) {
                // seam edge (r, W-1) <-> (r, 0): horizontal[r, W-1] in the reference
                if (bit(P, i + W - 1) && pair_pass(S(r, W - 1), v, a.tch, thr))
                    atomicOr(seam, 1u << (q + 1));
            }
            if (r >= 1) {
                const bool pu = (q == 0) ? bit(Ph, c) : bit(P, i - W);
                up = pu && pair_pass(S(r - 1, c), v, __ldg(tcv + r - 1), thr);
            }
        }
        const uint32_t ml = __ballot_sync(0xffffffffu, left);
        const uint32_t mu = __ballot_sync(0xffffffffu, up);
        if (lane == 0) {
            L[base >> 5] = ml;
            U[base >> 5] = mu;
        }
        // Map Connections, evaluated by the lower (or right) cell of each pair:
        // partner t = (r - dy, (c - dx) mod W); TL = LEFT edge of t (for the
        // redundant-edge test).
        for (int o = 0; o < a.n_off; ++o) {
            const int dy = a.dy[o], dx = a.dx[o];
            const int tr = r - dy;
            int tc = (c - dx) % W;
            if (tc < 0) tc += W;
            bool pt = false;
            float vt = 0.f;
            const bool has = inb && tr >= 0;
            if (has) {
                if (tr >= r0) {
                    pt = bit(P, (tr - r0) * W + tc);
                    vt = S(tr, tc);
                } else if (tr == r0 - 1) {
                    pt = bit(Ph, tc);
                    vt = S(tr, tc);
                } else {
                    vt = G(tr, tc);
                    pt = present_at(a, tr, tc, G);
                }
            }
            // partner's left neighbour: lane-1's partner when (c > 0, tc > 0)
            bool ptl = __shfl_up_sync(0xffffffffu, pt, 1);
            float vtl = __shfl_up_sync(0xffffffffu, vt, 1);
            if (has && tc > 0 && c > 0 && lane == 0) {
                const int tl = tc - 1;
                if (tr >= r0) {
                    ptl = bit(P, (tr - r0) * W + tl);
                    vtl = S(tr, tl);
                } else if (tr == r0 - 1) {
                    ptl = bit(Ph, tl);
                    vtl = S(tr, tl);
                } else {
                    vtl = G(tr, tl);
                    ptl = present_at(a, tr, tl, G);
                }
            }
            const float tco = __ldg(a.tables + 6 * H - 5 + o * H + max(tr, 0));
            const bool mc = has && p && pt && pair_pass(vt, v, tco, thr);
            const bool tl = has && c > 0 && tc > 0 && pt && ptl && pair_pass(vtl, vt, a.tch, thr);
            const uint32_t mm = __ballot_sync(0xffffffffu, mc);
            const uint32_t mt = __ballot_sync(0xffffffffu, tl);
            if (lane == 0) {
                MC[o * a.nwords + (base >> 5)] = mm;
                TL[o * a.nwords + (base >> 5)] = mt;
            }
        }
    }
    __syncthreads();   // staging is dead from here on; E aliases it

    // ---- 4. local union-find ---------------------------------------------
    for (int base = warp * 32; base < n_pad; base += kWarps * 32) {
        const int i = base + lane;
        if (i < n_own) {
            const uint32_t pw = P[base >> 5];
            if (!((pw >> lane) & 1u)) {
                E[i] = kFlag;
            } else {
                const uint32_t notl = ~L[base >> 5] & lanemask_le(lane);
                const int j = notl ? 31 - __clz(notl) : 0;
                E[i] = band | (uint32_t)(base + j);
            }
        }
    }
    __syncthreads();

    UF uf{E, cl, (1u << a.SH) - 1u, a.SH, k};
    const uint32_t seamw = seam[0];
    for (int base = warp * 32; base < n_pad; base += kWarps * 32) {
        const int i = base + lane;
        if (i >= n_own) continue;
        const int q = (int)divW(a, (unsigned)i);
        const int c = i - q * W;
        const bool l = bit(L, i);
        if (lane == 0 && l) uf.unite(band | (uint32_t)(i - 1), band | (uint32_t)i);
        if (q > 0 && bit(U, i)) {
            const bool skip = c > 0 && l && bit(L, i - W) && bit(U, i - 1);
            if (!skip) uf.unite(band | (uint32_t)i, band | (uint32_t)(i - W));
        }
        if (c == 0 && ((seamw >> (q + 1)) & 1u))
            uf.unite(band | (uint32_t)(i + W - 1), band | (uint32_t)i);
        for (int o = 0; o < a.n_off; ++o) {
            const uint32_t *mcb = MC + o * a.nwords;
            if (!bit(mcb, i)) continue;
            const int tr = r0 + q - a.dy[o];
            if (tr < r0) continue;   // cross-band: phase 5
            const bool skip = c > 0 && l && bit(mcb, i - 1) && bit(TL + o * a.nwords, i);
            if (skip) continue;
            int tc = (c - a.dx[o]) % W;
            if (tc < 0) tc += W;
            uf.unite(band | (uint32_t)i, band | (uint32_t)((tr - r0) * W + tc));
        }
    }
    __syncthreads();
    for (int i = tid; i < n_own; i += kThreads) {
        const uint32_t e = E[i];
        if (!(e & kFlag)) E[i] = uf.find(e);
    }
    cl.sync();   // #1: every band's entries initialised and locally flat

    // ---- 5. cross-band unions (DSMEM) -------------------------------------
    if (r0 > 0) {
        const uint32_t up_band = (uint32_t)(k - 1) << a.SH;
        for (int c = tid; c < W; c += kThreads) {
            if (!bit(U, c)) continue;
            const bool skip = c > 0 && bit(L, c) && bit(Lh, c) && bit(U, c - 1);
            if (!skip) uf.unite(band | (uint32_t)c, up_band | (uint32_t)((R - 1) * W + c));
        }
        for (int o = 0; o < a.n_off; ++o) {
            const int dy = a.dy[o];
            const int lim = min(dy, rows) * W;   // rows q < dy have partners above r0
            const uint32_t *mcb = MC + o * a.nwords;
            for (int i = tid; i < lim; i += kThreads) {
                if (!bit(mcb, i)) continue;
                const int q = (int)divW(a, (unsigned)i);
                const int c = i - q * W;
                const int tr = r0 + q - dy;
                if (tr < 0) continue;
                const bool skip = c > 0 && bit(L, i) && bit(mcb, i - 1) && bit(TL + o * a.nwords, i);
                if (skip) continue;
                int tc = (c - a.dx[o]) % W;
                if (tc < 0) tc += W;
                const int tk = tr / R;
                uf.unite(band | (uint32_t)i, ((uint32_t)tk << a.SH) | (uint32_t)((tr - tk * R) * W + tc));
            }
        }
    }
    cl.sync();   // #2: the forest is final

    // ---- 6a. resolve every pixel to its root (warp-aggregated chase) -------
    for (int base = warp * 32; base < n_pad; base += kWarps * 32) {
        const int i = base + lane;
        const uint32_t e = i < n_own ? E[i] : kFlag;
        const uint32_t prev = __shfl_up_sync(0xffffffffu, e, 1);
        const bool head = (lane == 0) || (e != prev);
        uint32_t g = e;
        if (head && !(e & kFlag)) g = uf.find(e);
        const uint32_t heads = __ballot_sync(0xffffffffu, head);
        const int hl = 31 - __clz(heads & lanemask_le(lane));
        g = __shfl_sync(0xffffffffu, g, hl);
        if (i < n_own && !(e & kFlag)) E[i] = g;
    }
    cl.sync();   // #3

    // ---- 6b. mark roots (size counters start at 0) -------------------------
    for (int i = tid; i < n_own; i += kThreads)
        if (E[i] == (band | (uint32_t)i)) E[i] = kFlag;
    cl.sync();   // #4

    // ---- 6c. component sizes ----------------------------------------------
    for (int base = warp * 32; base < n_pad; base += kWarps * 32) {
        const int i = base + lane;
        const bool p = i < n_own && bit(P, i);
        uint32_t root = 0xffffffffu;
        if (p) {
            const uint32_t v = E[i];
            root = (v & kFlag) ? (band | (uint32_t)i) : v;
        }
        const uint32_t prev = __shfl_up_sync(0xffffffffu, root, 1);
        const bool head = (lane == 0) || (root != prev);
        const uint32_t heads = __ballot_sync(0xffffffffu, head);
        if (head && p) {
            const uint32_t after = heads & ~lanemask_le(lane);
            const int next = after ? __ffs(after) - 1 : 32;
            atomicAdd(uf.slot(root), (uint32_t)(next - lane));
        }
    }
    cl.sync();   // #5

    // ---- 6d. kept roots, ordered scan, labels for roots ---------------------
    uint32_t *K = U;    // reuse: U/L bits are dead after the unions
    uint32_t *WP = L;
    const uint32_t minp = a.min_points > 1 ? (uint32_t)a.min_points : 1u;
    if (tid == 0) { cta_cnt = 0; cta_sum = 0; }
    __syncthreads();
    for (int base = warp * 32; base < n_pad; base += kWarps * 32) {
        const int i = base + lane;
        bool kept = false;
        uint32_t sz = 0;
        if (i < n_own && bit(P, i)) {
            const uint32_t v = E[i];
            if (v & kFlag) {
                sz = v & ~kFlag;
                kept = sz >= minp;
            }
        }
        const uint32_t m = __ballot_sync(0xffffffffu, kept);
        uint32_t s = kept ? sz : 0u;
        for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) {
            K[base >> 5] = m;
            if (s) atomicAdd(&cta_sum, s);
        }
    }
    __syncthreads();
    // word-ordered exclusive scan: warp w owns words [w*per, (w+1)*per)
    const int per = (a.nwords + kWarps - 1) / kWarps;
    {
        uint32_t run = 0;
        const int w0 = warp * per, w1 = min(w0 + per, a.nwords);
        for (int cb = w0; cb < w1; cb += 32) {
            const int w = cb + lane;
            const uint32_t cnt = w < w1 ? __popc(K[w]) : 0u;
            uint32_t inc = cnt;
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, inc, off);
                if (lane >= off) inc += t;
            }
            if (w < w1) WP[w] = run + inc - cnt;
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) warp_tot[warp] = run;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kWarps; ++w) { const uint32_t x = warp_tot[w]; warp_tot[w] = t; t += x; }
        cta_cnt = t;
    }
    cl.sync();   // #6: every band's count and kept-size sum are published
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
    const uint32_t prefix = cta_prefix;
    for (int base = warp * 32; base < n_pad; base += kWarps * 32) {
        const int i = base + lane;
        if (i >= n_own || !bit(P, i)) continue;
        const uint32_t v = E[i];
        if (!(v & kFlag)) continue;
        const int w = base >> 5;
        const uint32_t km = K[w];
        if ((km >> lane) & 1u) {
            const uint32_t label = prefix + warp_tot[w / per] + WP[w] +
                                   __popc(km & (lanemask_le(lane) >> 1)) + 1u;
            E[i] = kFlag | label;
            if (a.sizes) a.sizes[(size_t)frame * a.sizes_stride + label] = (int64_t)(v & ~kFlag);
        } else {
            E[i] = kFlag;   // dropped by filter_small
        }
    }
    cl.sync();   // #7

    // ---- 7. labels --------------------------------------------------------
    int32_t *out = a.labels + (size_t)frame * H * W + (size_t)r0 * W;
    for (int base = warp * 32; base < n_pad; base += kWarps * 32) {
        const int i = base + lane;
        const uint32_t v = i < n_own ? E[i] : kFlag;
        const uint32_t prev = __shfl_up_sync(0xffffffffu, v, 1);
        const bool head = (lane == 0) || (v != prev);
        uint32_t lab = v & ~kFlag;
        if (head && !(v & kFlag)) lab = uf.ld(v) & ~kFlag;
        const uint32_t heads = __ballot_sync(0xffffffffu, head);
        const int hl = 31 - __clz(heads & lanemask_le(lane));
        lab = __shfl_sync(0xffffffffu, lab, hl);
        if (i < n_own) __stcs(out + i, (int32_t)lab);
    }
    cl.sync();   // #8: no CTA leaves while its shared memory may still be read
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
    const int nwords = (R * W + 31) / 32;
    const int hwords = (W + 31) / 32;
    const int stage = (R + 2) * W;
    int off = (stage + 31) & ~31;
    o_words[0] = off; off += nwords;               // P
    o_words[1] = off; off += nwords;               // L
    o_words[2] = off; off += nwords;               // U
    o_words[3] = off; off += hwords;               // Ph
    o_words[4] = off; off += hwords;               // Lh
    o_words[5] = off; off += 1;                    // seam
    o_words[6] = off; off += n_off * nwords;       // MC
    o_words[7] = off; off += n_off * nwords;       // TL
    o_words[8] = off;
    return (size_t)off * 4u;
}

int make_plan(const rs_config *cfg, Plan *pl) {
    int st = validate(cfg);
    if (st) return st;
    const int H = cfg->height, W = cfg->width, n_off = cfg->n_offsets;
    int o[9];
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
    k.magicW = ((1ULL << 40) + (unsigned long long)W - 1) / (unsigned long long)W;
    k.o_P = o[0]; k.o_L = o[1]; k.o_U = o[2]; k.o_Ph = o[3]; k.o_Lh = o[4]; k.o_seam = o[5];
    k.o_MC = o[6]; k.o_TL = o[7]; k.o_misc = o[8];
    k.nwords = (R * W + 31) / 32;
    k.hwords = (W + 31) / 32;
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

const char *rs_last_error(void) { return g_err.c_str(); }

int rs_version(void) { return 100; }

}  // extern "C"
