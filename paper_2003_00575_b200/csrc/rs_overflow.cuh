// rs_overflow.cuh — in-kernel fallback of rs_fast_kernel for a frame whose
// run count exceeds the shared-memory node capacity of some band.
//
// The cluster keeps its bit planes (presence P, left edges L, up edges U, Map
// Connection edges MC, seam bits: all final after step B) and runs a
// union-find over CELLS in global memory, with the frame's own label buffer
// as the parent array (no workspace).  It reproduces the same closed form as
// the fast path (SURVEY.md finding 2): the root of a component is its
// smallest cell (hooks always point to the smaller index), components are
// ranked by that cell in row-major order among those with at least
// min_points cells, label = 1 + rank, 0 = background / dropped.
//
// Entry encodings in the parent array during the passes:
//   absent cell          kAbsent (INT_MIN)
//   F2-F3 present cell   parent cell index (>= 0); a root points to itself
//   F4-F5 root           -(number of cells counted so far)
//   F6    root           -(label + 1)   (label 0 = dropped)
// and finally every cell holds its label.
//
// Rare by construction (the planner sizes the node capacity above every
// BASELINE frame), so this path favours simplicity over speed: one relaxed
// global access per union-find step, a cluster barrier between passes.
#pragma once

#include "rs_common.cuh"

namespace rs {

constexpr int kAbsent = INT_MIN;

#ifndef RS_OVF_INLINE
#define RS_OVF_INLINE __forceinline__   // measured: inlined beats a call (config 1 -1%, config 3 -2%)
#endif

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
// P/L/U/MC: this band's planes (shared memory); seamw: this band's seam bits;
// cnt: two shared words of this CTA published to the cluster.
__device__ RS_OVF_INLINE void overflow_frame(const KArgs &a, const uint32_t *P, const uint32_t *L, const uint32_t *U,
                                            const uint32_t *MC, const uint32_t *seamw, uint32_t *cnt, uint32_t *wtot,
                                            int frame) {
    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthr = blockDim.x, nwarp = nthr >> 5;
    const int H = a.H, W = a.W, WPR = a.WPR;
    const int r0 = k * a.R, rows = min(a.R, H - r0);
    const int n = rows * W, g0 = r0 * W;   // band cells, first cell index
    int *par = a.labels + (size_t)frame * H * W;
    auto bit = [&](const uint32_t *pl, int i) -> bool {   // band cell i of a plane
        const int q = i / W, c = i - q * W;
        return (pl[q * WPR + (c >> 5)] >> (c & 31)) & 1u;
    };

    // F1: every present cell is its own root
    for (int i = tid; i < n; i += nthr) stg_relaxed(par + g0 + i, bit(P, i) ? g0 + i : kAbsent);
    cl.sync();
    // F2: unite along every edge (left, up, seam, Map Connections)
    for (int i = tid; i < n; i += nthr) {
        if (!bit(P, i)) continue;
        const int q = i / W, c = i - q * W, g = g0 + i, r = r0 + q;
        if (bit(L, i)) ovf_unite(par, g, g - 1);
        if (bit(U, i)) ovf_unite(par, g, g - W);
        if (c == 0 && W > 1 && ((seamw[q >> 5] >> (q & 31)) & 1u)) ovf_unite(par, g, r * W + W - 1);
        for (int o = 0; o < a.n_off; ++o) {
            if (!bit(MC + o * a.nwords, i)) continue;
            int tc = (c - a.dx[o]) % W;
            if (tc < 0) tc += W;
            ovf_unite(par, g, (r - a.dy[o]) * W + tc);
        }
    }
    cl.sync();
    // F3: flatten; every store writes a root, so a concurrent reader of an
    // entry sees its old parent or its root (both ancestors)
    for (int i = tid; i < n; i += nthr) {
        const int g = g0 + i;
        if (ldg_relaxed(par + g) != kAbsent) stg_relaxed(par + g, ovf_root(par, g));
    }
    cl.sync();
    // F4: roots start their count (themselves)
    for (int i = tid; i < n; i += nthr)
        if (ldg_relaxed(par + g0 + i) == g0 + i) stg_relaxed(par + g0 + i, -1);
    cl.sync();
    // F5: every other present cell counts itself at its root
    for (int i = tid; i < n; i += nthr) {
        const int p = ldg_relaxed(par + g0 + i);
        if (p >= 0) atomicAdd(par + p, -1);
    }
    cl.sync();
    // F6: kept roots ranked in cell order: warp w owns cells [w*per, (w+1)*per)
    const uint32_t minp = a.min_points > 1 ? (uint32_t)a.min_points : 1u;
    const int per = ((n + nwarp - 1) / nwarp + 31) & ~31;
    const int c0 = min(warp * per, n), c1 = min(c0 + per, n);
    uint32_t wk = 0;
    unsigned long long wsum = 0;
    for (int i = c0 + lane; i - lane < c1; i += 32) {
        const int v = i < c1 ? ldg_relaxed(par + g0 + i) : kAbsent;
        const bool kept = v != kAbsent && v < 0 && (uint32_t)(-v) >= minp;
        wk += __popc(__ballot_sync(kFull, kept));
        unsigned long long s = kept ? (unsigned long long)(-v) : 0ull;
        for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
        wsum += s;
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
    uint32_t base = 0, tot = 0;
    unsigned long long sum = 0;
    for (int j = 0; j < a.C; ++j) {
        const uint32_t cj = *cl.map_shared_rank(cnt, j);
        if (j < k) base += cj;
        tot += cj;
        sum += *cl.map_shared_rank(cnt + 1, j);
    }
    if (k == 0 && tid == 0) {
        if (a.ncl) a.ncl[frame] = (int32_t)tot;
        if (a.sizes) a.sizes[(size_t)frame * a.sizes_stride] = (int64_t)H * W - (int64_t)sum;
    }
    uint32_t run = base + wtot[warp];
    for (int i = c0 + lane; i - lane < c1; i += 32) {
        const int v = i < c1 ? ldg_relaxed(par + g0 + i) : kAbsent;
        const bool root = v != kAbsent && v < 0;
        const bool kept = root && (uint32_t)(-v) >= minp;
        const uint32_t m = __ballot_sync(kFull, kept);
        if (root) {
            uint32_t label = 0;
            if (kept) {
                label = run + __popc(m & ((1u << lane) - 1u)) + 1u;
                if (a.sizes) a.sizes[(size_t)frame * a.sizes_stride + label] = (int64_t)(-v);
            }
            stg_relaxed(par + g0 + i, -(int)label - 1);
        }
        run += __popc(m);
    }
    cl.sync();
    // F7: cells that are not roots take their root's label; absent cells 0
    for (int i = tid; i < n; i += nthr) {
        const int g = g0 + i, p = ldg_relaxed(par + g);
        if (p == kAbsent) stg_relaxed(par + g, 0);
        else if (p >= 0) stg_relaxed(par + g, -ldg_relaxed(par + p) - 1);
    }
    cl.sync();
    // F8: roots decode their own label
    for (int i = tid; i < n; i += nthr) {
        const int g = g0 + i, p = ldg_relaxed(par + g);
        if (p < 0) stg_relaxed(par + g, -p - 1);
    }
}

}  // namespace rs
