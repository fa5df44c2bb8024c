// rs_overflow.cuh — in-kernel fallback of rs_fast_kernel for a frame whose
// run count exceeds the shared-memory node capacity of some band.
//
// The cluster keeps its bit planes (presence P, left edges L, up edges U, seam
// bits: all final after step B) and runs a
// union-find over CELLS in global memory, with the frame's own label buffer
// as the parent array (no workspace).  It reproduces the same closed form as
// the fast path (SURVEY.md finding 2): the root of a component is its
// smallest cell (hooks always point to the smaller index), components are
// ranked by that cell in row-major order among those with at least
// min_points cells, label = 1 + rank, 0 = background / dropped.
//
// Entry encodings in the parent array during the passes:
//   absent cell          kAbsent (INT_MIN; F1-F6)
//   F1-F3 present cell   parent cell index (>= 0); a root points to itself
//   F4-F5 root           -(number of cells counted so far)
//   F6    root           -(label + 1)   (label 0 = dropped)
// and finally every cell holds its label.  Every present cell starts at the
// first cell of its run (F1), so left edges need no unions.
//
// Rare by construction (the planner sizes the node capacity above every
// BASELINE frame), so this path favours simplicity over speed: one relaxed
// global access per union-find step, a cluster barrier between passes.
#pragma once

#include "rs_common.cuh"
#include "rs_mc.cuh"

namespace rs {

constexpr int kAbsent = INT_MIN;

#ifndef RS_OVF_INLINE
#define RS_OVF_INLINE __forceinline__   // measured: inlined beats a call (config 1 -1%, config 3 -2%)
#endif

// Relaxed gpu-scope accesses: coherent with the atomics (no stale L1 line of
// an entry another CTA of the cluster updated), and never merged or hoisted
// by the compiler across the union-find loops.
__device__ __forceinline__ int ldg_relaxed(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void stg_relaxed(int *p, int v) {
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int ovf_find(int *par, int e) {
    while (true) {
        const int p = ldg_relaxed(par + e);
        if (p == e) return e;
        const int gp = ldg_relaxed(par + p);
        if (gp == p) return p;
        stg_relaxed(par + e, gp);   // path halving: e is not a root, gp is an ancestor
        e = gp;
    }
}

// read-only find (the forest is final): used to flatten, where a path-halving
// store could overwrite another thread's finished (root) entry with an
// intermediate ancestor
__device__ __forceinline__ int ovf_root(const int *par, int e) {
    while (true) {
        const int p = ldg_relaxed(par + e);
        if (p == e) return e;
        e = p;
    }
}

__device__ __forceinline__ void ovf_unite(int *par, int x, int y) {
    RS_CHECK(x >= 0 && y >= 0, "overflow union-find cell");
    while (true) {
        x = ovf_find(par, x);
        y = ovf_find(par, y);
        if (x == y) return;
        if (x > y) { const int t = x; x = y; y = t; }
        const int old = atomicMin(par + y, x);   // larger root hooks under the smaller
        if (old == y) return;
        y = old;
    }
}

// Called by every thread of every CTA of the cluster (cluster-uniform branch).
// P/L/U: this band's planes (shared memory); Lh: the halo row's left
// edges; seamw: this band's seam bits; cnt: two shared words of this CTA
// published to the cluster; wtot: one shared word per warp.
//
// Passes walk the band word by word, a warp per word and a lane per cell, so
// every global access of a warp is one coalesced 128-byte row segment.
__device__ RS_OVF_INLINE void overflow_frame(const KArgs &a, const uint32_t *P, const uint32_t *L, const uint32_t *U,
                                             const uint32_t *Lh, const uint32_t *seamw, uint32_t *cnt,
                                             uint32_t *wtot, int frame, const uint32_t *bad) {
    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarp = blockDim.x >> 5;
    const int H = a.H, W = a.W, WPR = a.WPR;
    const int r0 = k * a.R, rows = min(a.R, H - r0);
    const int g0 = r0 * W;   // first cell of the band
    int *par = a.labels + (size_t)frame * H * W;
    const uint32_t lt = (1u << lane) - 1u;

    // F1: every present cell points to the first cell of its run (runs are
    // the left-linked segments of a row); a warp walks one row's words
    for (int q = warp; q < rows; q += nwarp) {
        int carry = 0;   // first cell of the run entering the current word
        for (int cw = 0; cw < WPR; ++cw) {
            const int w = q * WPR + cw, c = cw * 32 + lane;
            const uint32_t pw = P[w], ts = pw & ~L[w];   // true run starts
            const uint32_t m = ts & (lt | (1u << lane));
            const int start = m ? cw * 32 + 31 - __clz(m) : carry;
            if (c < W) stg_relaxed(par + g0 + q * W + c, ((pw >> lane) & 1u) ? g0 + q * W + start : kAbsent);
            if (ts) carry = cw * 32 + 31 - __clz(ts);
        }
    }
    cl.sync();
    // F2: unite along the up edges that the left neighbour's up edge does not
    // already imply, the seam and the Map Connection edges (tested here from
    // the ranges, rs_mc.cuh)
    for (int w = warp; w < rows * WPR; w += nwarp) {
        const int q = w / WPR, cw = w - q * WPR, c = cw * 32 + lane;
        const int g = g0 + q * W + c, r = r0 + q;
        const uint32_t uw = U[w];
        if (uw) {
            const uint32_t lw = L[w], la = q > 0 ? L[w - WPR] : Lh[cw];
            const uint32_t uprev = (uw << 1) | (cw > 0 ? U[w - 1] >> 31 : 0u);
            if (((uw & ~(uprev & lw & la)) >> lane) & 1u) ovf_unite(par, g, g - W);
        }
        if (cw == 0 && lane == 0 && W > 1 && ((seamw[q >> 5] >> (q & 31)) & 1u)) ovf_unite(par, g, r * W + W - 1);
    }
    if (a.n_off > 0) {   // Map Connection edges (rs_mc.cuh)
        uint32_t *exp = a.planes ? a.planes + (size_t)frame * (3 + a.n_off) * H * WPR : nullptr;
        mc_pass<false>(a, cl, k, P, L, a.ranges + (size_t)frame * H * W, r0, rows, lane, warp, nwarp, exp,
                       [](int, int) { return 0u; }, [](int, int, int) { return 0u; },
                       [&](bool has, int, int, int, int, int r, int c, int tr, int tc) {
                           if (has) ovf_unite(par, r * W + c, tr * W + tc);
                       });
    }
    cl.sync();
    // F3: flatten.  Only run starts are ever roots or parents (every other
    // cell points to its run start from F1, and hooks and path halving only
    // ever target roots / ancestors), so first the starts take their root
    // (read-only finds: a path-halving store here could overwrite another
    // thread's finished entry), then every other cell its start's root.
    for (int w = warp; w < rows * WPR; w += nwarp) {
        const int q = w / WPR, cw = w - q * WPR, g = g0 + q * W + cw * 32 + lane;
        if (((P[w] & ~L[w]) >> lane) & 1u) stg_relaxed(par + g, ovf_root(par, g));
    }
    cl.sync();
    for (int w = warp; w < rows * WPR; w += nwarp) {
        const int q = w / WPR, cw = w - q * WPR, g = g0 + q * W + cw * 32 + lane;
        if (((P[w] & L[w]) >> lane) & 1u) stg_relaxed(par + g, ldg_relaxed(par + ldg_relaxed(par + g)));
    }
    cl.sync();
    // F4: roots start their count (themselves: -1) ...
    for (int w = warp; w < rows * WPR; w += nwarp) {
        const int q = w / WPR, cw = w - q * WPR, g = g0 + q * W + cw * 32 + lane;
        if (((P[w] >> lane) & 1u) && ldg_relaxed(par + g) == g) stg_relaxed(par + g, -1);
    }
    cl.sync();
    // F5: ... and every other present cell counts itself there, one atomic
    // per root and word (lanes grouped by root; a root's entry is < 0, every
    // other present entry is its root's index >= 0)
    for (int w = warp; w < rows * WPR; w += nwarp) {
        const int q = w / WPR, cw = w - q * WPR, g = g0 + q * W + cw * 32 + lane;
        const int v = ((P[w] >> lane) & 1u) ? ldg_relaxed(par + g) : -1;
        const bool member = v >= 0;
        const uint32_t grp = __match_any_sync(kFull, member ? v : -1);
        if (member && lane == __ffs(grp) - 1) atomicAdd(par + v, -__popc(grp));
    }
    cl.sync();
    // F6: kept roots ranked in cell order: warp w owns words [w*per, (w+1)*per)
    const uint32_t minp = a.min_points > 1 ? (uint32_t)a.min_points : 1u;
    const int nw = rows * WPR;
    const int per = (nw + nwarp - 1) / nwarp;
    const int w0 = min(warp * per, nw), w1 = min(w0 + per, nw);
    auto root_size = [&](int w, int &g) -> int {   // size of the root at this lane's cell, else 0
        const int q = w / WPR, cw = w - q * WPR;
        g = g0 + q * W + cw * 32 + lane;
        if (!((P[w] >> lane) & 1u)) return 0;
        const int v = ldg_relaxed(par + g);
        return v < 0 ? -v : 0;   // roots hold -(size); other cells their root (>= 0)
    };
    uint32_t wk = 0;
    unsigned long long wsum = 0;
    for (int w = w0; w < w1; ++w) {
        int g;
        const int sz = root_size(w, g);
        const bool kept = sz > 0 && (uint32_t)sz >= minp;
        wk += __popc(__ballot_sync(kFull, kept));
        unsigned long long sv = kept ? (unsigned long long)sz : 0ull;
        for (int off = 16; off; off >>= 1) sv += __shfl_xor_sync(kFull, sv, off);
        wsum += sv;
    }
    if (lane == 0) wtot[warp] = wk;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int j = 0; j < nwarp; ++j) { const uint32_t x = wtot[j]; wtot[j] = t; t += x; }
        cnt[0] = t;
        cnt[1] = 0;
    }
    __syncthreads();
    if (lane == 0 && wsum) atomicAdd(cnt + 1, (uint32_t)wsum);
    cl.sync();
    uint32_t base = 0, tot = 0, anybad = 0;
    unsigned long long sum = 0;
    for (int j = 0; j < a.C; ++j) {
        const uint32_t cj = *cl.map_shared_rank(cnt, j);
        if (j < k) base += cj;
        tot += cj;
        sum += *cl.map_shared_rank(cnt + 1, j);
        anybad |= *cl.map_shared_rank(bad, j);
    }
    if (k == 0 && tid == 0) {
        if (a.ncl) a.ncl[frame] = anybad ? RS_FRAME_INVALID : (int32_t)tot;
        if (a.sizes) a.sizes[(size_t)frame * a.sizes_stride] = (int64_t)H * W - (int64_t)sum;
    }
    // roots: entry -> -(label + 1), label 0 = dropped
    uint32_t run = base + wtot[warp];
    for (int w = w0; w < w1; ++w) {
        int g;
        const int sz = root_size(w, g);
        const bool kept = sz > 0 && (uint32_t)sz >= minp;
        const uint32_t m = __ballot_sync(kFull, kept);
        if (sz > 0) {
            uint32_t label = 0;
            if (kept) {
                label = run + __popc(m & lt) + 1u;
                if (a.sizes) a.sizes[(size_t)frame * a.sizes_stride + label] = (int64_t)sz;
            }
            stg_relaxed(par + g, -(int)label - 1);
        }
        run += __popc(m);
    }
    cl.sync();
    // F7: cells that are not roots take their root's label; absent cells 0
    for (int w = warp; w < rows * WPR; w += nwarp) {
        const int q = w / WPR, cw = w - q * WPR, c = cw * 32 + lane, g = g0 + q * W + c;
        if (c >= W) continue;
        if (!((P[w] >> lane) & 1u)) {
            stg_relaxed(par + g, 0);
        } else {
            const int p = ldg_relaxed(par + g);
            if (p >= 0) stg_relaxed(par + g, -ldg_relaxed(par + p) - 1);
        }
    }
    cl.sync();
    // F8: roots decode their own label
    for (int w = warp; w < rows * WPR; w += nwarp) {
        const int q = w / WPR, cw = w - q * WPR, g = g0 + q * W + cw * 32 + lane;
        if (!((P[w] >> lane) & 1u)) continue;
        const int p = ldg_relaxed(par + g);
        if (p < 0) stg_relaxed(par + g, -p - 1);
    }
}

}  // namespace rs
