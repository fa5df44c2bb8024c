// rs_dense.cuh — the dense kernel: one union-find slot per band cell.
//
// Rows [r0-2, r0+R) of the frame are staged in shared memory with TMA 1-D
// bulk copies; the union-find array aliases the staging area once the edge
// bits exist.  Used for frames whose run count exceeds the fast kernel's
// node capacity, and for geometries the fast kernel's plan cannot hold.
#pragma once

#include "rs_common.cuh"

namespace rs {

constexpr int kDenseThreads = 512;
constexpr int kDenseWarps = kDenseThreads / 32;

// Node (local cell index) of cell bit b of word w: the last run start at or
// before the cell, else the run node carried into the word.
__device__ __forceinline__ uint32_t dense_node_of(const uint32_t *SB, const uint32_t *RS, int w, int q, int cw,
                                                  int W, int b) {
    const uint32_t s = SB[w] & lanemask_le(b);
    return s ? (uint32_t)(q * W + cw * 32 + 31 - __clz(s)) : RS[w];
}

struct DenseUF {
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

struct DenseShared {
    uint32_t warp_tot[kDenseWarps];
    uint32_t cta_cnt, cta_sum, cta_prefix, seam;
    uint32_t bad;   // a range of the band breaks the input contract (range_image.py:50-53)
};

__device__ __forceinline__ void dense_frame(const KArgs &a, uint32_t *sm, DenseShared &sh, uint64_t *mbar,
                                            const int frame, const uint32_t parity) {
    uint32_t *warp_tot = sh.warp_tot;
    uint32_t &cta_cnt = sh.cta_cnt, &cta_sum = sh.cta_sum, &cta_prefix = sh.cta_prefix, &seam = sh.seam;
    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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
    if (tid == 0) {
        seam = 0;
        sh.bad = 0;
    }
    if (a.use_tma) {
        if (tid == 0) {
            mbar_expect_tx(mbar, (uint32_t)n_stage * 4u);
            const uint32_t row_bytes = (uint32_t)W * 4u;
            for (int s = 0; s <= hi_row - lo_row; ++s)
                tma_load_1d(stage + (size_t)s * W, src + (size_t)s * W, row_bytes, mbar);
        }
        __syncthreads();
        mbar_wait(mbar, parity);
    } else {
        for (int i = tid; i < n_stage; i += kDenseThreads) stage[i] = __ldg(src + i);
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
        bool bad = false;
        for (int cw = warp; cw < WPR; cw += kDenseWarps) {
            const int c = cw * 32 + lane;
            const bool inb = c < W;
            float vprev = (inb && rstart >= 1) ? S(rstart - 1, c) : 0.f;
            bool pprev = false;
            for (int r = rstart; r < r0 + rows; ++r) {
                const float v = inb ? S(r, c) : 0.f;
                bad |= !range_ok(v);
                bool p = v > 0.f;
                if (a.ground && p) {
                    const float d1 = r >= 1 ? vprev : v;
                    const float d2 = r >= 1 ? v : S(1, c);
                    p = !ground_rule(a, ground_row(a, r), d1, d2, v);
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
        if (__any_sync(kFull, bad) && lane == 0) sh.bad = 1u;
    }
    __syncthreads();

    RS_MARK(2);
    // ---- 3. word-boundary LEFT bits, the seam, Map Connection bits ------------
    for (int w = tid; w < nw + WPR; w += kDenseThreads) {
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
        for (int q = tid; q < rows; q += kDenseThreads) {
            const int r = r0 + q;
            const uint32_t pe = P[q * WPR + (W - 1) / 32] >> ((W - 1) & 31);
            if ((pe & 1u) && (P[q * WPR] & 1u) && pair_pass(S(r, W - 1), S(r, 0), tch, thr))
                atomicOr(&seam, 1u << q);
        }
    }
    if (a.n_off > 0) {
        // Pairs (r-dy, c-dx mod W) <-> (r, c), evaluated by the lower/right cell.
        // TL = LEFT edge of the partner (for the redundant-edge test in step 4).
        for (int w = warp; w < nw; w += kDenseWarps) {
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
    DenseUF uf{E, cl, (1u << a.SH) - 1u, a.SH, k};

    // ---- 4. runs: start bits, carried run node per word, node init ----------
    // Warp w owns the contiguous word range [wr0, wr1); a run continuing into
    // the range gets a pseudo start at its first cell (united in step 5).
    const int per = (nw + kDenseWarps - 1) / kDenseWarps;
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
    for (int w = tid; w < nw; w += kDenseThreads) {
        const int q = divWPR(a, w);
        const int cw = w - q * WPR;
        const uint32_t lw = L[w], sb = SB[w];
        if (sb & lw & 1u)   // pseudo start: join the run it continues
            uf.unite_local(band | dense_node_of(SB, RS, w, q, cw, W, 0),
                           band | dense_node_of(SB, RS, w - 1, q, cw - 1, W, 31));
        const uint32_t uw = U[w];
        if (q > 0 && uw) {
            const uint32_t uprev = (uw << 1) | (cw > 0 ? U[w - 1] >> 31 : 0u);
            uint32_t nr = uw & ~(uprev & lw & L[w - WPR]);
            for (; nr; nr &= nr - 1) {
                const int b = __ffs(nr) - 1;
                uf.unite_local(band | dense_node_of(SB, RS, w, q, cw, W, b),
                               band | dense_node_of(SB, RS, w - WPR, q - 1, cw, W, b));
            }
        }
        if (cw == 0 && ((seam >> q) & 1u))
            uf.unite_local(band | dense_node_of(SB, RS, w, q, 0, W, 0),
                           band | dense_node_of(SB, RS, q * WPR + (W - 1) / 32, q, (W - 1) / 32, W, (W - 1) & 31));
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
                uf.unite_local(band | dense_node_of(SB, RS, w, q, cw, W, b),
                               band | dense_node_of(SB, RS, tq * WPR + tc / 32, tq, tc / 32, W, tc & 31));
            }
        }
    }
    __syncthreads();
    RS_MARK(5);
    // local flatten: every node points at its band-local root
    for (int w = tid; w < nw; w += kDenseThreads) {
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
        for (int cw = tid; cw < WPR; cw += kDenseThreads) {
            const uint32_t uw = U[cw];
            if (!uw) continue;
            const uint32_t uprev = (uw << 1) | (cw > 0 ? U[cw - 1] >> 31 : 0u);
            uint32_t nr = uw & ~(uprev & L[cw] & Lh[cw]);
            const int wu = (R - 1) * WPR + cw;
            for (; nr; nr &= nr - 1) {
                const int b = __ffs(nr) - 1;
                uf.unite(band | dense_node_of(SB, RS, cw, 0, cw, W, b),
                         bandu | dense_node_of(SBu, RSu, wu, R - 1, cw, W, b));
            }
        }
        for (int o = 0; o < a.n_off; ++o) {
            const int dy = a.dy[o];
            const uint32_t *M = MC + o * a.nwords;
            const int lim = min(dy, rows) * WPR;
            for (int w = tid; w < lim; w += kDenseThreads) {
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
                    uf.unite(band | dense_node_of(SB, RS, w, q, cw, W, b),
                             ((uint32_t)kt << a.SH) |
                                 dense_node_of(SBt, RSt, tq * WPR + tc / 32, tq, tc / 32, W, tc & 31));
                }
            }
        }
    }
    cl.sync();   // #2: the forest is final

    RS_MARK(7);
    // ---- 7. resolve every node to its root; roots start a size counter ------
    for (int w = tid; w < nw; w += kDenseThreads) {
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
    for (int w = tid; w < nw; w += kDenseThreads) {
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
        for (int i = 0; i < kDenseWarps; ++i) { const uint32_t x = warp_tot[i]; warp_tot[i] = t; t += x; }
        cta_cnt = t;
    }
    cl.sync();   // #5: every band's kept count and kept-size sum are published
    RS_MARK(10);
    if (tid == 0) {
        uint32_t pre = 0, tot = 0, sum = 0, bad = 0;
        for (int j = 0; j < a.C; ++j) {
            const uint32_t cj = *cl.map_shared_rank(&cta_cnt, j);
            if (j < k) pre += cj;
            tot += cj;
            sum += *cl.map_shared_rank(&cta_sum, j);
            bad |= *cl.map_shared_rank(&sh.bad, j);
        }
        cta_prefix = pre;
        if (k == 0) {
            if (a.ncl) a.ncl[frame] = bad ? RS_FRAME_INVALID : (int32_t)tot;
            if (a.sizes) a.sizes[(size_t)frame * a.sizes_stride] = (int64_t)H * W - (int64_t)sum;
        }
    }
    __syncthreads();
    {
        const uint32_t prefix = cta_prefix;
        for (int w = tid; w < nw; w += kDenseThreads) {
            const int q = divWPR(a, w);
            const uint32_t base = (uint32_t)(q * W + (w - q * WPR) * 32);
            const uint32_t km = K[w];
            const uint32_t wbase = prefix + warp_tot[min(w / max(per, 1), kDenseWarps - 1)] + WP[w];
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
    for (int w = tid; w < nw; w += kDenseThreads) {
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
    for (int w = warp; w < nw; w += kDenseWarps) {
        const int q = divWPR(a, w);
        const int cw = w - q * WPR;
        const int c = cw * 32 + lane;
        if (c < W) {
            uint32_t lab = 0;
            if ((P[w] >> lane) & 1u) lab = E[dense_node_of(SB, RS, w, q, cw, W, lane)] & ~kFlag;
            __stcs(out + q * W + c, (int32_t)lab);
        }
    }
    RS_MARK(13);
    __syncthreads();   // the next frame of a list-mode loop reuses shared memory
}


// Dense kernel: every band cell owns a union-find slot (no capacity limit).
// Runs over a batch when the fast plan cannot hold the geometry.
__global__ void __launch_bounds__(kDenseThreads, 1) rs_dense_kernel(const __grid_constant__ KArgs a) {
    extern __shared__ __align__(128) uint32_t sm[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ DenseShared sh;
    if (threadIdx.x == 0 && a.use_tma) mbar_init(&mbar, 1);
    __syncthreads();
    dense_frame(a, sm, sh, &mbar, blockIdx.x / a.C, 0);
}

}  // namespace rs
