// rs_mc.cuh — Map Connections (map_connections.py:132-178) in the fused
// kernel, as extra edges of the component graph.
//
// The reference labels the frame first, then for every offset (dy, dx) tests
// the pairs (r, c) - (r + dy, (c + dx) mod W) whose labels are > 0 and differ
// (pair_distance_sq with the pair's upper-row constant, :155-169) and unions
// their clusters (ClusterUnion, :73-110); filter_small runs on the merged
// clusters.  The result is the connected components of the graph (present
// cells; direct edges plus every passing Map Connection pair).
//
// The fused kernel builds that graph in one forest.  Any passing pair may be
// united at any time (the unions commute), and a pair whose cells are already
// in one component need not be tested — the reference's "labels differ".
// Pairs come in chains: along a row, consecutive candidate pairs whose own
// cells and partner cells are left-linked join the same two runs, so the
// roots are compared once per chain (at its head) and the chain is united
// once, at its first passing cell.  Presence and left-link bits of the
// partner row are built a word at a time (a funnel shift of two plane words,
// local or over DSMEM).  No per-offset bit plane is kept in shared memory, so
// the band layout (and the two-CTAs-per-SM occupancy) is the same with any
// number of offsets.
//
//   * inside the band, before barrier #1 (production path, widths that are
//     whole words): mc_axis_heads lists the chains whose runs have different
//     band-local roots, mc_chain_issue / mc_chain_finish test and unite them,
//     spread evenly over the CTA; the caller re-flattens the forest;
//   * rows whose partner row lies in a band above: mc_axis_cross, a lane per
//     cell during the cross-band step, passing pairs join that step's list;
//   * after barrier #2 (mc_runs: other widths) / mc_pass (the parity export
//     rs_fast_planes and the overflow path, where every present pair is tested
//     and `out` receives the decision words as plane 3 + o of the frame).
#pragma once

#include "rs_common.cuh"

namespace rs {

#ifdef RS_MC_STATS
__device__ unsigned long long g_mcstats[8];
#define RS_MCSTAT(i, v) atomicAdd(&g_mcstats[i], (unsigned long long)(v))
#else
#define RS_MCSTAT(i, v) \
    do {                \
    } while (0)
#endif

// The 32 bits of plane row `row` (W cells, WPR words) starting at cell t0
// (wrapping at W; W % 32 == 0 for the funnel path).
__device__ __forceinline__ uint32_t row_bits(const uint32_t *row, int t0, int W, int WPR, int lane, bool funnel) {
    if (funnel) {
        const int a = t0 >> 5, sh = t0 & 31;
        const uint32_t lo = row[a], hi = row[a + 1 == WPR ? 0 : a + 1];
        return sh ? __funnelshift_r(lo, hi, sh) : lo;
    }
    const int t = (t0 + lane) % W;
    return __ballot_sync(kFull, (row[t >> 5] >> (t & 31)) & 1u);
}

// root_own(w, b) / root_partner(kt, tw, tb): root of the own cell (word w,
// bit b) / of the partner cell (band kt, word tw of that band, bit tb); only
// called when ROOTS.  edge(has, w, b, kt, tw, r, c, tr, tc) is called by
// EVERY lane of the warp (warp-synchronous; `has` marks a lane with an edge).
template <bool ROOTS, class RootOwn, class RootPartner, class Edge>
__device__ __forceinline__ void mc_pass(const KArgs &a, const cg::cluster_group &cl, int k, const uint32_t *P,
                                        const uint32_t *L, const float *fr, int r0, int rows, int lane, int warp,
                                        int nwarps, uint32_t *out, RootOwn root_own, RootPartner root_partner,
                                        Edge edge) {
    const int H = a.H, W = a.W, R = a.R, WPR = a.WPR;
    const size_t fw = (size_t)H * WPR;
    const float thr = a.dmax2;
    const bool filter = ROOTS && out == nullptr;
    const bool funnel = (W & 31) == 0;
    const uint32_t below = (1u << lane) - 1u;
    for (int q = warp; q < rows; q += nwarps) {
        const int r = r0 + q;
        for (int o = 0; o < a.n_off; ++o) {
            const int tr = r - a.dy[o];
            if (tr < 0) {
                if (out && lane == 0)
                    for (int cw = 0; cw < WPR; ++cw) out[(size_t)(3 + o) * fw + (size_t)r * WPR + cw] = 0u;
                continue;
            }
            const int dx = a.dx[o];
            const int kt = tr / R, tq = tr - kt * R;
            const uint32_t *Pt = (kt == k ? P : cl.map_shared_rank(P, kt)) + tq * WPR;
            const uint32_t *Lt = (kt == k ? L : cl.map_shared_rank(L, kt)) + tq * WPR;
            const float tco = __ldg(a.tables + 6 * H - 5 + o * H + tr);
            const float *trow = fr + (size_t)tr * W, *orow = fr + (size_t)r * W;
            int t0 = -dx % W;   // partner of column 0
            t0 = t0 < 0 ? t0 + W : t0;
            uint32_t ccand = 0, cdiff = 0, cm = 0;   // lane 31's candidate / chain verdict / decision, previous word
            for (int cw = 0; cw < WPR; ++cw, t0 = (t0 + 32 >= W ? t0 + 32 - W : t0 + 32)) {
                const int w = q * WPR + cw;
                const uint32_t pw = P[w];
                const uint32_t cand = pw ? pw & row_bits(Pt, t0, W, WPR, lane, funnel) : 0u;   // warp-uniform
                if (!cand) {
                    ccand = cdiff = cm = 0;
                    if (out && lane == 0) out[(size_t)(3 + o) * fw + (size_t)r * WPR + cw] = 0u;
                    continue;
                }
                const uint32_t lw = L[w], ltw = row_bits(Lt, t0, W, WPR, lane, funnel);
                // chain continuation: the left neighbours are a candidate pair and both cells are left-linked to them
                const uint32_t chain = cand & ((cand << 1) | ccand) & lw & ltw;
                const uint32_t heads = cand & ~chain;
                int tc = t0 + lane;
                tc = funnel ? (tc >= W ? tc - W : tc) : tc % W;
                const int tw = tq * WPR + (tc >> 5);
                const bool mine = (cand >> lane) & 1u;
                bool diff = mine;
                if (filter) {
                    bool hd = false;
                    if ((heads >> lane) & 1u) hd = root_own(w, lane) != root_partner(kt, tw, tc & 31);
                    const uint32_t D = __ballot_sync(kFull, hd);
                    const uint32_t hb = heads & (below | (1u << lane));   // heads at or below this lane
                    diff = mine && (hb ? (D >> (31 - __clz(hb))) & 1u : cdiff);
                }
                bool mc = false;
                if (__any_sync(kFull, diff) && diff)
                    mc = pair_pass(__ldg(trow + tc), __ldg(orow + min(cw * 32 + lane, W - 1)), tco, thr);
                const uint32_t m = __ballot_sync(kFull, mc);
                // the left neighbours' pair passed and links both cells to this pair's runs: nothing new
                const bool prev = lane > 0 ? (m >> (lane - 1)) & 1u : cm;
                const bool has = mc && !(prev && ((chain >> lane) & 1u));
                edge(has, w, lane, kt, tw, r, cw * 32 + lane, tr, tc);
                if (out && lane == 0) out[(size_t)(3 + o) * fw + (size_t)r * WPR + cw] = m;
                ccand = cand >> 31;
                cdiff = __shfl_sync(kFull, (uint32_t)diff, 31);
                cm = m >> 31;
            }
        }
    }
}

}  // namespace rs

namespace rs {


// Run end: the last cell of the run starting at bit b of word cw of a row
// (left links continuing after it).
__device__ __forceinline__ int run_end(const uint32_t *Lrow, int cw, int b, int WPR, int W) {
    const uint32_t y = b < 31 ? Lrow[cw] >> (b + 1) : 0u;
    const int n = __ffs(~y) - 1;   // consecutive links (<= 31 - b)
    int e;
    if (n < 31 - b) {
        e = cw * 32 + b + n;
    } else {
        e = cw * 32 + 31;
        for (int ww = cw + 1; ww < WPR; ++ww) {
            const uint32_t m = ~Lrow[ww];
            if (m) { e = ww * 32 + __ffs(m) - 2; break; }
            e = ww * 32 + 31;
        }
    }
    return min(e, W - 1);
}

// Is offset o an axis offset the band-local fast path (mc_axis) takes?
// (0, k): every row; (k, 0): the rows whose partner row lies in the band.
__device__ __forceinline__ bool mc_axis_offset(const KArgs &a, int o) {
    return (a.W & 31) == 0 && ((a.dy[o] == 0 && a.dx[o] > 0 && a.dx[o] < 32) || (a.dx[o] == 0 && a.dy[o] > 0));
}

// Axis-aligned Map Connections (BASELINE's skip offsets (0, k) and (k, 0)).
// They only ever join two runs that the direct edges have not joined already
// when the cells between them break the straight chain of links:
//   (0, k): the pair is inside one run unless a run starts in (c - k, c] (or
//           the pair crosses the seam, where runs end);
//   (k, 0): rows r - k .. r are linked at column c by k up-edges unless one
//           of the k U bits is clear.
// Those candidate bits are word operations on the P / L / U / SB planes.
//
// Inside the band (after the local flatten: E[run] = band-local root).
// mc_axis_heads: a thread per word; a chain of candidates along the row whose
// own and partner cells are left-linked joins one pair of runs, so the roots
// are compared once, at its head (bit 0 of a word is always a head), and the
// heads whose roots differ are LISTED (entry = word | bit << 16 | offset <<
// 21, and the chain's cell bits: two words, `cap` entries).  The caller then
// gives every listed head to a thread (mc_chain_issue / mc_chain_finish):
// the chain's cells are tested (ranges from global memory, four loads in
// flight) and the runs united on the first pass — the loads and unions are
// spread evenly over the CTA whatever the words look like, one union per
// chain.  A full list falls back to `now(entry)`.  (k, 0) rows whose partner
// row lies in another band: mc_axis_cross.
struct AxisWord {
    uint32_t cand, heads;
};

// candidate and chain-head bits of word w (row q of the band, word cw of the
// row) for axis offset o.  Besides the broken straight chain, a pair is ruled
// out when a detour of direct links one row (column) aside already joins its
// cells — the usual case around a dropped cell on a surface:
//   (0, k): both cells have an up edge and the row above is left-linked from
//           c - k to c (or the same through the row below);
//   (k, 0): both cells are left-linked to column c - 1 and that column has its
//           k up edges (or the same through column c + 1).
// (Bits that would need a neighbouring word are not ruled out.)
template <int KC>   // KC > 0: the offset's k as a compile-time constant (loops unrolled), 0: any k
__device__ __forceinline__ AxisWord mc_axis_word_k(const KArgs &a, const uint32_t *P, const uint32_t *L,
                                                   const uint32_t *U, const uint32_t *SB, int o, int w, int q, int cw,
                                                   int rows) {
    const int WPR = a.WPR;
    const int dy = KC ? (a.dy[o] ? KC : 0) : a.dy[o], k = KC ? KC : (a.dx[o] ? a.dx[o] : dy);
    const uint32_t pw = P[w];
    uint32_t cand = 0, ltw = 0;
    if (dy == 0) {
        const int wl = cw > 0 ? w - 1 : w + WPR - 1;   // word to the left (the seam wraps)
        const uint32_t pt = (pw << k) | (P[wl] >> (32 - k));
        ltw = (L[w] << k) | (L[wl] >> (32 - k));
        // a run start in (c - k, c]; across the seam runs always differ
        const uint32_t sb = SB[w], sbl = SB[wl];
        uint32_t diff = cw == 0 ? (1u << k) - 1u : 0u;
        for (int i = 0; i < k; ++i) diff |= (sb << i) | (i ? sbl >> (32 - i) : 0u);
        cand = pw & pt & diff;
#ifndef RS_MC_NO_DETOUR
        if (cand) {
            // detour through the row above / below (bits k.. of the word only)
            uint32_t det = 0;
            if (q > 0) {
                const uint32_t u = U[w], la = L[w - WPR];
                uint32_t d = u & (u << k);
                for (int i = 0; i < k; ++i) d &= la << i;
                det |= d;
            }
            if (q + 1 < rows) {
                const uint32_t u = U[w + WPR], lb = L[w + WPR];
                uint32_t d = u & (u << k);
                for (int i = 0; i < k; ++i) d &= lb << i;
                det |= d;
            }
            cand &= ~(det & (~0u << k));
        }
#endif
    } else if (a.dx[o] == 0) {
        const uint32_t lt = L[w - dy * WPR];
        ltw = lt;
        uint32_t chain = ~0u;
        for (int i = 0; i < dy; ++i) chain &= U[w - i * WPR];
        cand = pw & P[w - dy * WPR] & ~chain;
#ifndef RS_MC_NO_DETOUR
        // detour through column c - 1 (bits 1..) or c + 1 (bits ..30)
        const uint32_t both = L[w] & lt;
        cand &= ~((both & (chain << 1)) | (((both & chain) >> 1) & 0x7fffffffu));
#endif
    }
    return {cand, cand & ~((cand << 1) & L[w] & ltw)};
}

__device__ __forceinline__ AxisWord mc_axis_word(const KArgs &a, const uint32_t *P, const uint32_t *L,
                                                 const uint32_t *U, const uint32_t *SB, int o, int w, int q, int cw,
                                                 int rows) {
    // BASELINE's S = 1 is k = 2 on both axes: its loops unrolled
    const int k = a.dx[o] ? a.dx[o] : a.dy[o];
    return k == 2 ? mc_axis_word_k<2>(a, P, L, U, SB, o, w, q, cw, rows)
                  : mc_axis_word_k<0>(a, P, L, U, SB, o, w, q, cw, rows);
}

// the same for any other offset (no straight chain of links to rule pairs
// out): every present pair is a candidate; the partner row's bits are brought
// under the own columns with a funnel shift of two of its words
__device__ __forceinline__ AxisWord mc_any_word(const KArgs &a, const uint32_t *P, const uint32_t *L, int o, int w,
                                                int q, int cw) {
    const int WPR = a.WPR;
    int t0 = (cw * 32 - a.dx[o]) % a.W;   // partner column of the word's bit 0
    t0 = t0 < 0 ? t0 + a.W : t0;
    const int tqw = (q - a.dy[o]) * WPR;
    const uint32_t cand = P[w] & row_bits(P + tqw, t0, a.W, WPR, 0, true);
    const uint32_t ltw = row_bits(L + tqw, t0, a.W, WPR, 0, true);
    return {cand, cand & ~((cand << 1) & L[w] & ltw)};
}

// partner column of column c for offset dx (|dx| < W)
__device__ __forceinline__ int mc_partner_col(int c, int dx, int W) {
    const int t = c - dx;
    return t < 0 ? t + W : (t >= W ? t - W : t);
}

// offsets [o0, o1) of the pattern
template <class Now>
__device__ __forceinline__ void mc_axis_heads(const KArgs &a, int o0, int o1, const uint32_t *P, const uint32_t *L,
                                              const uint32_t *U, const uint32_t *SB, const uint32_t *NB,
                                              const uint32_t *E, int rows, int tid, int nthreads, uint32_t *list,
                                              uint32_t cap, uint32_t *count, Now now) {
    const int W = a.W, WPR = a.WPR;
    const int nw = rows * WPR;
    for (int o = o0; o < o1; ++o) {
        const int dy = a.dy[o], dx = a.dx[o];
        const bool axis = mc_axis_offset(a, o);
        for (int w = dy * WPR + tid; w < nw; w += nthreads) {   // rows q < dy: partner row in another band (or none)
            if (!P[w]) continue;
            const int q = divWPR(a, w), cw = w - q * WPR;
            const AxisWord aw = axis ? mc_axis_word(a, P, L, U, SB, o, w, q, cw, rows) : mc_any_word(a, P, L, o, w, q, cw);
            const uint32_t heads = aw.heads;
            RS_MCSTAT(0, 1);
            if (!heads) continue;
            RS_MCSTAT(1, __popc(heads));
            // heads whose two runs have different band-local roots (the words'
            // run counts stay in registers across the heads)
            const int tqw = (q - dy) * WPR;
            uint32_t live = 0;
            for (uint32_t m = heads; m; m &= m - 1) {
                const int b = __ffs(m) - 1;
                const int tc = mc_partner_col(cw * 32 + b, dx, W);
                if (E[run_of(SB, NB, w, b)] != E[run_of(SB, NB, tqw + (tc >> 5), tc & 31)]) live |= 1u << b;
            }
            if (!live) continue;
            RS_MCSTAT(2, __popc(live));
            uint32_t slot = atomicAdd(count, (uint32_t)__popc(live));
            for (uint32_t m = live; m; m &= m - 1, ++slot) {
                const int b = __ffs(m) - 1;
                const uint32_t e = (uint32_t)w | ((uint32_t)b << 16) | ((uint32_t)o << 21);
                // the chain: the candidates from b up to the next head of the word
                const uint32_t nxt = aw.heads & ~lanemask_le(b);
                const uint32_t upto = nxt ? ((1u << (__ffs(nxt) - 1)) - 1u) : ~0u;
                const uint32_t cells = aw.cand & upto & ~((1u << b) - 1u);
                if (slot < cap) {
                    list[2 * slot] = e;
                    list[2 * slot + 1] = cells;
                } else {
                    now(e, cells);
                }
            }
        }
    }
}

// One listed chain (head entry e, cell bits `live`; its runs had different
// roots), in two halves so that a thread can keep several chains' loads in
// flight: mc_chain_issue loads the ranges of the chain's first two cells,
// mc_chain_finish tests them, goes on through the rest of the chain (four
// loads in flight) while none passes, and calls `unite(x, y)` (run ids of the
// band) on the first pass.
struct ChainLoads {
    float vo[2], vt[2], tco;
};

__device__ __forceinline__ ChainLoads mc_chain_issue(const KArgs &a, const float *fr, int r0, uint32_t e,
                                                     uint32_t live) {
    const int W = a.W, WPR = a.WPR, H = a.H;
    const int w = (int)(e & 0xffffu), o = (int)(e >> 21);
    const int dy = a.dy[o], dx = a.dx[o];
    const int q = divWPR(a, w), cw = w - q * WPR;
    const int r = r0 + q, tr = r - dy;
    ChainLoads c;
    c.tco = __ldg(a.tables + 6 * H - 5 + o * H + tr);
    const float *orow = fr + (size_t)r * W + cw * 32, *trow = fr + (size_t)tr * W;
    uint32_t m = live;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        c.vo[j] = c.vt[j] = 0.f;
        if (m) {
            const int bb = __ffs(m) - 1;
            m &= m - 1;
            c.vo[j] = __ldg(orow + bb);
            c.vt[j] = __ldg(trow + mc_partner_col(cw * 32 + bb, dx, W));
        }
    }
    return c;
}

template <class Unite>
__device__ __forceinline__ void mc_chain_finish(const KArgs &a, const uint32_t *SB, const uint32_t *NB,
                                                const float *fr, int r0, uint32_t e, uint32_t live,
                                                const ChainLoads &c, Unite unite) {
    const int W = a.W, WPR = a.WPR;
    const int w = (int)(e & 0xffffu), b = (int)((e >> 16) & 31u), o = (int)(e >> 21);
    const int dy = a.dy[o], dx = a.dx[o];
    const int q = divWPR(a, w), cw = w - q * WPR;
    uint32_t m = live & (live - 1);   // the cells after the first
    const bool two = m != 0u;
    m &= m - 1;
    bool pass = pair_pass(c.vt[0], c.vo[0], c.tco, a.dmax2) || (two && pair_pass(c.vt[1], c.vo[1], c.tco, a.dmax2));
    if (!pass && m) {
        const int r = r0 + q, tr = r - dy;
        const float *orow = fr + (size_t)r * W + cw * 32, *trow = fr + (size_t)tr * W;
        while (m && !pass) {   // four cells per round: their loads overlap
            float vo[4], vt[4];
            bool on[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                on[j] = m != 0u;
                vo[j] = vt[j] = 0.f;
                if (m) {
                    const int bb = __ffs(m) - 1;
                    m &= m - 1;
                    vo[j] = __ldg(orow + bb);
                    vt[j] = __ldg(trow + mc_partner_col(cw * 32 + bb, dx, W));
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) pass |= on[j] && pair_pass(vt[j], vo[j], c.tco, a.dmax2);
        }
    }
    RS_MCSTAT(3, __popc(live));
    if (pass) {
        RS_MCSTAT(4, 1);
        const int tc = mc_partner_col(cw * 32 + b, dx, W);
        unite(run_of(SB, NB, w, b), run_of(SB, NB, (q - dy) * WPR + (tc >> 5), tc & 31));
    }
}

// Pairs of offsets with dy > 0 whose partner row lies in a band above (the
// first dy rows of band bl): a lane per cell.  Like the cross-band up edges
// the work is shared by the two bands of a boundary: band bl takes the upper
// half of the words, band bl - 1 the lower half of the pairs whose partner
// row is its own (a partner row further up — dy > R — stays with band bl).
// The other band's P / L / SB / NB planes are read over DSMEM (final since
// step R; its U plane is not — the band may already be listing cross-band
// edges in it — so every present pair is tested: any passing pair may be
// united at any time, the components are those of the graph of all passing
// edges).  Of consecutive passing pairs whose own and partner cells are
// left-linked only the first is pushed.  push(has, x, y) is called by every
// lane (band-tagged run ids).
template <class Root, class Push>
__device__ __forceinline__ void mc_axis_cross(const KArgs &a, const cg::cluster_group &cl, int kb, int bl, int o,
                                              const uint32_t *P, const uint32_t *L, const uint32_t *SB,
                                              const uint32_t *NB, const float *fr, int lane, int warp, int nwarps,
                                              bool filter, Root root, Push push) {
    const int W = a.W, WPR = a.WPR, R = a.R, H = a.H;
    const int r0 = bl * R, rows = min(R, H - r0);   // the lower band
    const bool lower = kb == bl;
    const int whalf = WPR / 2;
    auto plane = [&](const uint32_t *x, int band) { return band == kb ? x : cl.map_shared_rank(x, band); };
    const uint32_t *Pl = plane(P, bl), *Ll = plane(L, bl), *SBl = plane(SB, bl), *NBl = plane(NB, bl);
    const uint32_t low_tag = (uint32_t)bl << a.SHN;
    {
        const int dy = a.dy[o], dx = a.dx[o];
        if (dy == 0) return;
        const int nq = min(dy, rows);
        // a warp per word (W % 32 == 0), two words per round so that their
        // DSMEM and global loads overlap
        for (int wi0 = warp; wi0 < nq * WPR; wi0 += 2 * nwarps) {
            int w[2], twr[2], kt[2], tc[2];
            uint32_t both[2], ltw[2];
            float vo[2], vt[2], tco[2];
            bool diff[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int wi = wi0 + j * nwarps;
                both[j] = ltw[j] = 0;
                diff[j] = false;
                w[j] = twr[j] = kt[j] = tc[j] = 0;
                vo[j] = vt[j] = tco[j] = 0.f;
                if (wi >= nq * WPR) continue;   // warp-uniform
                const int q = divWPR(a, wi), cw = wi - q * WPR;
                const int r = r0 + q, tr = r - dy;
                if (tr < 0) continue;   // warp-uniform
                kt[j] = r0 - tr <= R ? bl - 1 : tr / R;   // (the band above, unless dy > R)
                // whose word is it?  shared pairs (partner row in band bl - 1) by halves
                const bool shared = kt[j] == bl - 1;
                if (lower ? (shared && cw < whalf) : !(shared && cw < whalf)) continue;
                w[j] = q * WPR + cw;
                twr[j] = (tr - kt[j] * R) * WPR;   // first word of the partner row in its band
                const int t0 = mc_partner_col(cw * 32, dx, W);
                both[j] = Pl[w[j]] & row_bits(plane(P, kt[j]) + twr[j], t0, W, WPR, 0, true);
                if (!both[j]) continue;   // warp-uniform
                ltw[j] = row_bits(plane(L, kt[j]) + twr[j], t0, W, WPR, 0, true);
                tc[j] = mc_partner_col(cw * 32 + lane, dx, W);
                // a chain of pairs (own and partner cells left-linked) joins one
                // pair of runs: their roots in the live forest are compared at
                // the chain's head (bit 0 of a word always is one) and only
                // chains that are still apart are tested
                // (`filter`: not before the first cross-band unions, when bands
                // are still apart anyway)
                diff[j] = (both[j] >> lane) & 1u;
                if (filter) {
                    const uint32_t heads = both[j] & ~((both[j] << 1) & Ll[w[j]] & ltw[j]);
                    bool hd = false;
                    if ((heads >> lane) & 1u)
                        hd = root(low_tag | run_of(SBl, NBl, w[j], lane)) !=
                             root(((uint32_t)kt[j] << a.SHN) |
                                  run_of(plane(SB, kt[j]), plane(NB, kt[j]), twr[j] + (tc[j] >> 5), tc[j] & 31));
                    const uint32_t D = __ballot_sync(kFull, hd);
                    const uint32_t hb = heads & lanemask_le(lane);
                    diff[j] = diff[j] && hb && ((D >> (31 - __clz(hb))) & 1u);
                }
                if (diff[j]) {
                    vt[j] = __ldg(fr + (size_t)tr * W + tc[j]);
                    vo[j] = __ldg(fr + (size_t)r * W + cw * 32 + lane);
                    tco[j] = __ldg(a.tables + 6 * H - 5 + o * H + tr);
                }
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (!both[j]) continue;   // warp-uniform
                const bool pass = diff[j] && pair_pass(vt[j], vo[j], tco[j], a.dmax2);
                const uint32_t m = __ballot_sync(kFull, pass);
                if (!m) continue;
                // the pair to the left passed and joins the same runs
                const uint32_t dup = (m << 1) & Ll[w[j]] & ltw[j];
                const bool has = pass && !((dup >> lane) & 1u);
                uint32_t x = 0, y = 0;
                if (has) {
                    x = low_tag | run_of(SBl, NBl, w[j], lane);
                    y = ((uint32_t)kt[j] << a.SHN) |
                        run_of(plane(SB, kt[j]), plane(NB, kt[j]), twr[j] + (tc[j] >> 5), tc[j] & 31);
                }
                push(has, x, y);
            }
        }
    }
}

// Map Connections over RUNS (the production path of the fast kernel; the
// cell-level mc_pass above serves the parity export and the overflow path).
// Called by every thread of the CTA (it synchronises the CTA).
//
// One round per offset.  Thread i takes runs i, i + nthreads, ... of the band
// (ids follow cell order: the word holding the j-th start is found by a
// binary search of the per-word run counts NB, the bit by __fns), so every
// lane has a run and the loop is uniform.  For the run [s, e] of row r the
// partner cells are the segment [s - dx, e - dx] (mod W) of row r - dy, and
// the partner runs overlapping it are a contiguous range of run ids.  Each is
// compared with the own run by root in the forest's compressed snapshot; a
// differing pair (the reference's "labels differ") is listed.  Then every
// thread takes a listed pair: if the live forest still has them apart (an
// earlier union may have joined them) the aligned cells are tested until one
// passes, and the runs are united.  Step R's pseudo starts (a run continuing
// into a warp's word range gets a second id there; both ids have one root) are
// skipped as own runs: the run is walked from its true start through them.
//
// Callbacks: root(kt, id) = snapshot root of run `id` of band kt (one load);
// live(kt, id) = its root in the live forest (a find); unite(x, y) joins two
// (possibly no longer) roots of the live forest.  list / cap / count: a buffer of 2 * cap
// words and a shared counter.
template <class Root, class Live, class Unite>
__device__ __forceinline__ void mc_runs(const KArgs &a, const cg::cluster_group &cl, int k, const uint32_t *P,
                                        const uint32_t *L, const uint32_t *SB, const uint32_t *NB, const float *fr,
                                        int r0, int rows, uint32_t n_runs, int tid, int nthreads, uint32_t *list,
                                        uint32_t cap, uint32_t *count, Root root, Live live,
                                        Unite unite) {
    const int H = a.H, W = a.W, R = a.R, WPR = a.WPR;
    const float thr = a.dmax2;
    const int nw = rows * WPR;
    // test the pair (own run starting at band cell sc, run j of band kt) and unite on a pass
    auto resolve = [&](int o, uint32_t own, int kt, uint32_t j, int sc, int part) {
#ifdef RS_MC_NOLIVE
        return;
#endif
        const uint32_t lx = live(k, own), ly = live(kt, j);
        if (lx == ly) return;
#ifdef RS_MC_NOSLOW
        return;
#endif
        const int q = sc / W, s = sc - q * W, r = r0 + q;
        const int e = run_end(L + q * WPR, s >> 5, s & 31, WPR, W);
        const int dy = a.dy[o], dx = a.dx[o], tr = r - dy;
        const int tq = tr - kt * R;
        const uint32_t *Pt = (kt == k ? P : cl.map_shared_rank(P, kt)) + tq * WPR;
        const uint32_t *SBt = kt == k ? SB : cl.map_shared_rank(SB, kt);
        const uint32_t *NBt = kt == k ? NB : cl.map_shared_rank(NB, kt);
        int t0 = (s - dx) % W;
        t0 = t0 < 0 ? t0 + W : t0;
        const int len = e - s;
        const int a0 = part ? 0 : t0, a1 = part ? t0 + len - W : min(t0 + len, W - 1);
        const float tco = __ldg(a.tables + 6 * H - 5 + o * H + tr);
        RS_MCSTAT(2, 1);
        for (int t = a0; t <= a1; ++t) {
            if (!((Pt[t >> 5] >> (t & 31)) & 1u) || run_of(SBt, NBt, tq * WPR + (t >> 5), t & 31) != j) continue;
            const int c = s + (t - a0) + (part ? (W - t0) : 0);
            RS_MCSTAT(3, 1);
            if (pair_pass(__ldg(fr + (size_t)tr * W + t), __ldg(fr + (size_t)r * W + c), tco, thr)) {
#ifndef RS_MC_NOUNITE
                unite(lx, ly);   // from the live roots: no finds from the runs again
#endif
                RS_MCSTAT(4, 1);
                return;
            }
        }
    };
    for (int o = 0; o < a.n_off; ++o) {
        const int dy = a.dy[o], dx = a.dx[o];
        // axis offsets done by mc_axis: none left for (0, k); for (k, 0) only
        // the runs of rows q < dy (run ids follow cell order: ids below the
        // first run of row dy)
        const uint32_t n_own = n_runs;
        if (tid == 0) *count = 0;
        __syncthreads();
        for (uint32_t own = tid; own < n_own; own += nthreads) {
            int lo = 0, hi = nw - 1;   // the word holding start `own`: the last w with NB[w] <= own
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (NB[mid] <= own) lo = mid; else hi = mid - 1;
            }
            const int w = lo;
            const int b = (int)__fns(SB[w], 0, (int)(own - NB[w]) + 1);
            if ((L[w] >> b) & 1u) continue;   // pseudo start: walked from the run's true start
            const int q = divWPR(a, w), cw = w - q * WPR, r = r0 + q;
            const int tr = r - dy;
            if (tr < 0) continue;
            const int s = cw * 32 + b;
            const int e = run_end(L + q * WPR, cw, b, WPR, W);
            const uint32_t rown = root(k, own);
            const int kt = tr / R, tq = tr - kt * R;
            const uint32_t *Pt = (kt == k ? P : cl.map_shared_rank(P, kt)) + tq * WPR;
            const uint32_t *SBt = kt == k ? SB : cl.map_shared_rank(SB, kt);
            const uint32_t *NBt = kt == k ? NB : cl.map_shared_rank(NB, kt);
            auto rid = [&](int t) { return run_of(SBt, NBt, tq * WPR + (t >> 5), t & 31); };
            RS_MCSTAT(0, 1);
            int t0 = (s - dx) % W;
            t0 = t0 < 0 ? t0 + W : t0;
            const int len = e - s;
            for (int part = 0; part < 2; ++part) {   // the partner segment, split at the seam
                if (part == 1 && t0 + len < W) break;
                const int a0 = part ? 0 : t0, a1 = part ? t0 + len - W : min(t0 + len, W - 1);
                const uint32_t j0 = rid(a0) + (((Pt[a0 >> 5] >> (a0 & 31)) & 1u) ? 0u : 1u);
                const uint32_t j1 = rid(a1);
                if (j1 + 1u == 0u || j0 > j1) continue;   // no partner run in the segment
                for (uint32_t j = j0; j <= j1; ++j) {
                    RS_MCSTAT(1, 1);
                    if (root(kt, j) == rown) continue;
                    // list slot: one shared atomic per group of lanes pushing together
                    const uint32_t am = __activemask();
                    const int leader = __ffs(am) - 1, lane = threadIdx.x & 31;
                    uint32_t base = 0;
                    if (lane == leader) base = atomicAdd(count, (uint32_t)__popc(am));
                    const uint32_t slot = __shfl_sync(am, base, leader) + __popc(am & ((1u << lane) - 1u));
                    if (slot < cap) {
                        list[2 * slot] = own | ((uint32_t)kt << 16) | ((uint32_t)part << 20);
                        list[2 * slot + 1] = j | ((uint32_t)(q * W + s) << 16);
                    } else {
                        resolve(o, own, kt, j, q * W + s, part);   // list full: at once
                    }
                }
            }
        }
        __syncthreads();
        const uint32_t n = min(*count, cap);
        for (uint32_t i = tid; i < n; i += nthreads) {
            const uint32_t x = list[2 * i], y = list[2 * i + 1];
            resolve(o, x & 0xffffu, (int)((x >> 16) & 15u), y & 0xffffu, (int)(y >> 16), (int)(x >> 20) & 1);
        }
        __syncthreads();
    }
}

}  // namespace rs
