// rangeseg_b200.cu — host side of the B200 segmentation path: launch
// planning, the kernels' shared-memory layouts, and the C ABI declared in
// include/rangeseg_b200.h.
//
// Kernels (see the headers for the algorithms):
//   rs_fast_kernel   rs_fast.cuh   cluster per frame, compact run nodes, 4 CTAs/SM
//   rs_dense_kernel  rs_dense.cuh  cluster per frame, one slot per cell, TMA staging;
//                                  takes the frames the fast kernel's node
//                                  capacity cannot hold (overflow list)
//   rs_stage_kernel  rs_stage.cuh  per-cell ground / edge masks (parity checks)

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>

#include "../../include/rangeseg_b200.h"
#include "rs_common.cuh"
#include "rs_dense.cuh"
#include "rs_fast.cuh"
#include "rs_stage.cuh"
#include "rs_project.cuh"
#include "rs_eval.cuh"


using rs::KArgs;

namespace {

constexpr int kMaxCluster = 16;
constexpr int kMaxRowsPerCta = 31;            // dense kernel: seam bits of band + halo fit a word
constexpr int kMaxRowsFast = 64;              // fast kernel: two seam words
// per-CTA shared memory on sm_100 is at most 227 KB, static + dynamic: the
// dynamic part of each kernel is capped below that by its static use
// (fast kernel ~3.3 KB, dense kernel ~1.2 KB; rounded up)
constexpr size_t kSmemLimit = 227 * 1024 - 4096;
// kFastOcc fast CTAs per SM: 228 KB per SM, minus 1 KB reserved and the
// static shared memory of each CTA
constexpr size_t kFastSmemTarget = std::min<size_t>(228 * 1024 / rs::kFastOcc - 1024 - 2560, kSmemLimit);
constexpr int kMinNodeCap = 512;
constexpr long long kFillCtas = 148;          // one CTA per SM: below this a batch gets thinner bands
#ifndef RS_UDYN_MIN_C
#define RS_UDYN_MIN_C 2   // clusters of at least this many bands grab edges dynamically in the local unions
#endif

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return RS_OK;
    return fail(RS_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

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
    if (cfg->rows_per_cta < 0 || cfg->rows_per_cta > kMaxRowsFast)
        return fail(RS_EINVAL, "rows_per_cta must be in [0, 64]");
    if (cfg->reserved[0] < 0) return fail(RS_EINVAL, "reserved[0] (node capacity) must be >= 0");
#ifndef RS_EXPERIMENTS
    if (cfg->reserved[1] != 0 || cfg->reserved[2] != 0) return fail(RS_EINVAL, "reserved[1] and reserved[2] must be 0");
#endif
    return RS_OK;
}

void fill_common(const rs_config *cfg, int R, KArgs &k) {
    memset(&k, 0, sizeof(k));
    const int H = cfg->height, W = cfg->width;
    k.H = H;
    k.W = W;
    k.R = R;
    k.C = (H + R - 1) / R;
    k.n_off = cfg->n_offsets;
    for (int i = 0; i < k.n_off; ++i) {
        k.dy[i] = cfg->offsets[i][0];
        k.dx[i] = cfg->offsets[i][1];
    }
    k.min_points = cfg->min_cluster_points;
    k.ground = cfg->ground_removal ? 1 : 0;
    k.dmax2 = cfg->d_max_sq;
    k.mount = cfg->mount_height;
    k.keep_above = cfg->keep_above;
    k.tch = cfg->two_cos_h;
    k.WPR = (W + 31) / 32;
    k.magicWPR = ((1ULL << 40) + (unsigned long long)k.WPR - 1) / (unsigned long long)k.WPR;
    k.nwords = R * k.WPR;
}

// ---- dense kernel layout ------------------------------------------------------
size_t dense_layout(int R, int W, int n_off, KArgs *k) {
    const int WPR = (W + 31) / 32, nwords = R * WPR;
    int off = (((R + 2) * W) + 31) & ~31;   // staging (float), later the union-find array
    int o[9];
    o[0] = off; off += nwords;          // P
    o[1] = off; off += nwords;          // L
    o[2] = off; off += nwords;          // U
    o[3] = off; off += nwords;          // SB
    o[4] = off; off += nwords;          // RS
    o[5] = off; off += WPR;             // Ph
    o[6] = off; off += WPR;             // Lh
    o[7] = off; off += n_off * nwords;  // MC
    o[8] = off; off += n_off * nwords;  // TL
    if (k) {
        k->o_P = o[0]; k->o_L = o[1]; k->o_U = o[2]; k->o_SB = o[3]; k->o_RS = o[4];
        k->o_Ph = o[5]; k->o_Lh = o[6]; k->o_MC = o[7]; k->o_TL = o[8];
    }
    return (size_t)off * 4u;
}

// ---- fast kernel layout ---------------------------------------------------------
// No Map Connection planes: the offsets are tested after the band-local
// union-find, straight from the ranges (rs_mc.cuh), so the layout does not
// depend on the offsets.
size_t fast_layout(int R, int W, int NC, KArgs *k) {
    const int WPR = (W + 31) / 32, nwords = R * WPR;
    const int ncw = (NC + 31) / 32;
    int off = 0;
    int o[12];
    const int nw4 = (nwords + 3) & ~3, wpr4 = (WPR + 3) & ~3;   // 16-byte aligned planes
    o[0] = off; off += nw4;             // P
    o[1] = off; off += nw4;             // L
    o[2] = off; off += nw4;             // U
    o[3] = off; off += nw4;             // SB
    o[4] = off; off += nw4;             // NB (run ids before each word)
    o[5] = off; off += wpr4;            // Ph
    o[6] = off; off += wpr4;            // Lh
    o[7] = off;                         // (MC: none)
    o[8] = off;                         // (TL: none)
    o[9] = off; off += ncw;             // LR (band-local roots), later kept-word prefixes
    o[10] = off; off += ncw;            // KB (kept roots)
    off = (off + 3) & ~3;
    o[11] = off; off += NC;             // E (parents)
    const int o_sz = off; off += NC;    // SZ (sizes, then labels)
    if (k) {
        k->o_P = o[0]; k->o_L = o[1]; k->o_U = o[2]; k->o_SB = o[3]; k->o_RS = o[4];
        k->o_Ph = o[5]; k->o_Lh = o[6]; k->o_MC = o[7]; k->o_TL = o[8];
        k->o_LR = o[9]; k->o_K = o[10]; k->o_E = o[11]; k->o_SZ = o_sz;
    }
    return (size_t)off * 4u;
}

// Upper bound of runs in a band: every cell may start one (neighbours farther
// apart than d_max), plus one pseudo start per warp range.
int max_runs(int R, int W) { return R * W + rs::kFastWarps; }

struct Plan {
    bool fast;            // run rs_fast_kernel (else rs_dense_kernel directly)
    bool may_overflow;    // a band may exceed the node capacity (fast kernel's overflow path, rs_overflow.cuh)
    bool dense_ok;        // rs_dense_kernel can hold the geometry
    KArgs kf, kd;         // arguments of the fast / dense kernels
    size_t smem_f, smem_d;
    int stop_after;       // experiments (rs_config.reserved[1]); 0 in production
};

int pick_dense_rows(const rs_config *cfg) {
    const int H = cfg->height, W = cfg->width, n_off = cfg->n_offsets;
    int R = std::max(1, std::min(H, 16384 / std::max(W, 1)));
    R = std::min(R, kMaxRowsPerCta);
    while ((H + R - 1) / R > 8 && R < kMaxRowsPerCta && dense_layout(R + 1, W, n_off, nullptr) <= kSmemLimit) ++R;
    while ((H + R - 1) / R > kMaxCluster && R < kMaxRowsPerCta) ++R;
    while (dense_layout(R, W, n_off, nullptr) > kSmemLimit && R > 1 && (H + R - 2) / (R - 1) <= kMaxCluster) --R;
    return std::min(R, H);
}

int make_plan_uncached(const rs_config *cfg, Plan *pl, int32_t batch) {
    int st = validate(cfg);
    if (st) return st;
    const int H = cfg->height, W = cfg->width, n_off = cfg->n_offsets;
#ifdef RS_EXPERIMENTS
    pl->stop_after = cfg->reserved[1];
#else
    pl->stop_after = 0;
#endif

    // dense plan (geometries the fast plan cannot hold)
    int Rd = cfg->rows_per_cta > 0 ? std::min({cfg->rows_per_cta, H, kMaxRowsPerCta}) : pick_dense_rows(cfg);
    if (dense_layout(Rd, W, n_off, nullptr) > kSmemLimit) Rd = pick_dense_rows(cfg);
    const int Cd = (H + Rd - 1) / Rd;
    const size_t smem_d = dense_layout(Rd, W, n_off, nullptr);
    std::string dense_err;
    if (Cd > kMaxCluster)
        dense_err = "frame needs " + std::to_string(Cd) + " bands of " + std::to_string(Rd) +
                    " rows; a cluster holds at most 16";
    else if (smem_d > kSmemLimit)
        dense_err = "band of " + std::to_string(Rd) + "x" + std::to_string(W) + " cells needs " +
                    std::to_string(smem_d) + " B of shared memory";
    fill_common(cfg, Rd, pl->kd);
    dense_layout(Rd, W, n_off, &pl->kd);
    int SH = 0;
    while ((1 << SH) < Rd * W) ++SH;
    pl->kd.SH = SH;
    pl->smem_d = smem_d;
    pl->dense_ok = dense_err.empty();

    // fast plan: ~16K cells per band, node capacity from the shared-memory target
    // ~64K cells per band: fewer, larger bands mean fewer cross-band edges and
    // cheaper cluster barriers (measured: 2 bands of 32 rows beat 8 of 8 for
    // 64x2048 frames).  The band shrinks until the run capacity is at least
    // an eighth of its cells (observed: <= 10% for 32-row bands of the
    // BASELINE configs; more take the in-kernel overflow path).
    pl->fast = false;
    pl->may_overflow = false;
    pl->smem_f = 0;
    memset(&pl->kf, 0, sizeof(pl->kf));
    int Rf = cfg->rows_per_cta > 0 ? std::min(cfg->rows_per_cta, H)
                                   : std::min({H, kMaxRowsFast, std::max(1, 65536 / std::max(W, 1))});
    while (cfg->rows_per_cta <= 0 && (H + Rf - 1) / Rf > kMaxCluster && Rf < kMaxRowsFast) ++Rf;
    // Small batches (the reference's one frame per call): a batch that fills
    // fewer than kFillCtas CTA slots is latency-bound on one or two SMs per
    // frame, so its frames are split into more, thinner bands (up to a
    // 16-CTA cluster per frame).
    if (cfg->rows_per_cta <= 0 && batch > 0)
        while (Rf > 1 && (long long)batch * ((H + Rf - 1) / Rf) < kFillCtas &&
               (H + (Rf + 1) / 2 - 1) / ((Rf + 1) / 2) <= kMaxCluster)
            Rf = (Rf + 1) / 2;
    for (; Rf >= 1; Rf = cfg->rows_per_cta > 0 ? 0 : Rf / 2) {
        if ((H + Rf - 1) / Rf > kMaxCluster) break;
        const int cap_full = max_runs(Rf, W);
        long long lo = 0, hi = cap_full;   // largest capacity under the shared-memory target
        while (lo < hi) {
            const long long mid = (lo + hi + 1) / 2;
            if (fast_layout(Rf, W, (int)mid, nullptr) <= kFastSmemTarget) lo = mid; else hi = mid - 1;
        }
        long long NC = lo;
        if (cfg->reserved[0] > 0) NC = std::min<long long>(NC, cfg->reserved[0]);   // test hook
        if (NC < cap_full) NC &= ~31LL;
        const long long need = std::min<long long>(cap_full, std::max<long long>(kMinNodeCap, (long long)Rf * W / 8));
        if (NC < need && cfg->reserved[0] <= 0) continue;
        NC = std::max<long long>(NC, 32);
        const size_t smem_f = fast_layout(Rf, W, (int)NC, nullptr);
        if (smem_f > kSmemLimit) continue;
        fill_common(cfg, Rf, pl->kf);
        fast_layout(Rf, W, (int)NC, &pl->kf);
        pl->kf.NC = (int)NC;
        pl->kf.udyn = pl->kf.C >= RS_UDYN_MIN_C;
#ifdef RS_TMA_RING
        {
            // step A's TMA row ring: per warp up to RS_TMA_RING slots of 512 B in
            // the union-find arrays (2 NC words), one mbarrier each in LR / KB
            const long long by_ring = 2 * NC / (rs::kFastWarps * 128);
            const long long by_bars = 2 * ((NC + 31) / 32) / (rs::kFastWarps * 2);
            const int nst = (int)std::min<long long>({(long long)RS_TMA_RING, by_ring, by_bars});
            const bool ok = W % 128 == 0 && W <= 128 * rs::kFastWarps && nst == RS_TMA_RING;   // one chunk task per warp
            pl->kf.ring = ok ? nst : 0;
        }
#endif
        int SHN = 0;
        while ((1 << SHN) < NC) ++SHN;
        pl->kf.SHN = SHN;
        pl->smem_f = smem_f;
        pl->fast = true;
        pl->may_overflow = NC < cap_full;
        break;
    }
    if (!pl->fast && !pl->dense_ok) return fail(RS_ETOOLARGE, dense_err);
    return RS_OK;
}

// Plans are cached per thread: a Pipeline calls with the same config every
// time, and planning (a capacity search per band height) costs microseconds.
struct PlanCache {
    bool valid = false;
    int32_t batch = 0;
    rs_config cfg;
    Plan pl;
    int st = RS_OK;
    std::string err;
};
thread_local PlanCache g_plan_cache;

// batch 0: the plan of a large batch (what rs_plan reports)
int make_plan(const rs_config *cfg, Plan *pl, int32_t batch = 0) {
    if (!cfg) return fail(RS_EINVAL, "config is NULL");
    PlanCache &c = g_plan_cache;
    if (batch >= kFillCtas) batch = 0;   // every large batch has the same plan
    if (c.valid && c.batch == batch && memcmp(&c.cfg, cfg, sizeof(rs_config)) == 0) {
        if (c.st) return fail(c.st, c.err);
        *pl = c.pl;
        return RS_OK;
    }
    const int st = make_plan_uncached(cfg, pl, batch);
    c.batch = batch;
    c.cfg = *cfg;
    c.st = st;
    c.err = st ? g_err : std::string();
    if (!st) c.pl = *pl;
    c.valid = true;
    return st;
}

std::mutex g_attr_mu;
int g_attr_device = -1;
size_t g_attr_smem_f = 0, g_attr_smem_d = 0;

int set_attrs(const Plan &pl) {
    std::lock_guard<std::mutex> g(g_attr_mu);
    int dev = 0;
    int st = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (st) return st;
    if (dev != g_attr_device) {
        g_attr_device = dev;
        g_attr_smem_f = g_attr_smem_d = 0;
        if ((st = cuda_check(cudaFuncSetAttribute(rs::rs_fast_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                             "cudaFuncSetAttribute(fast, non-portable cluster)")) ||
            (st = cuda_check(cudaFuncSetAttribute(rs::rs_fast_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                             "cudaFuncSetAttribute(fast + Map Connections, non-portable cluster)")) ||
            (st = cuda_check(cudaFuncSetAttribute(rs::rs_dense_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                             "cudaFuncSetAttribute(dense, non-portable cluster)")))
            return st;
    }
    if (pl.fast && pl.smem_f > g_attr_smem_f) {
        if ((st = cuda_check(cudaFuncSetAttribute(rs::rs_fast_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)std::max(pl.smem_f, (size_t)48 * 1024)),
                             "cudaFuncSetAttribute(fast, smem)")) ||
            (st = cuda_check(cudaFuncSetAttribute(rs::rs_fast_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)std::max(pl.smem_f, (size_t)48 * 1024)),
                             "cudaFuncSetAttribute(fast + Map Connections, smem)")))
            return st;
        g_attr_smem_f = pl.smem_f;
    }
    if (pl.smem_d > g_attr_smem_d) {
        if ((st = cuda_check(cudaFuncSetAttribute(rs::rs_dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)std::max(pl.smem_d, (size_t)48 * 1024)),
                             "cudaFuncSetAttribute(dense, smem)")))
            return st;
        g_attr_smem_d = pl.smem_d;
    }
    return RS_OK;
}

template <class Kern>
int launch_cluster(Kern kern, const KArgs &k, int clusters, int threads, size_t smem, cudaStream_t stream,
                   const char *what) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(clusters * k.C), 1, 1);
    lc.blockDim = dim3((unsigned)threads, 1, 1);
    lc.dynamicSmemBytes = smem;
    lc.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)k.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    // the hardware may place the CTAs of a cluster where there is room instead
    // of spreading them (measured: config 1 163.1 vs 164.1 us, config 2 196.2 vs 197.3)
    at[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    at[1].val.clusterSchedulingPolicyPreference = cudaClusterSchedulingPolicyLoadBalancing;
    lc.numAttrs = 2;
    return cuda_check(cudaLaunchKernelEx(&lc, kern, k), what);
}

// One launch per batch: rs_fast_kernel (frames whose bands overflow the node
// capacity are finished by the same kernel, rs_overflow.cuh), or
// rs_dense_kernel when the fast plan cannot hold the geometry.
int segment_launch(const Plan &pl, const float *d_tables, const float *d_ranges, int32_t batch, int32_t *d_labels,
                   int32_t *d_n_clusters, int64_t *d_cluster_sizes, int64_t sizes_stride, cudaStream_t stream,
                   uint32_t *d_planes = nullptr) {
    int st = set_attrs(pl);
    if (st) return st;
    KArgs k = pl.fast ? pl.kf : pl.kd;
    k.ranges = d_ranges;
    k.tables = d_tables;
    k.labels = d_labels;
    k.ncl = d_n_clusters;
    k.sizes = d_cluster_sizes;
    k.sizes_stride = sizes_stride;
    if (!pl.fast) {
        k.use_tma = (pl.kd.W % 4 == 0) && ((reinterpret_cast<uintptr_t>(d_ranges) & 15u) == 0);
        return launch_cluster(rs::rs_dense_kernel, k, batch, rs::kDenseThreads, pl.smem_d, stream,
                              "rs_dense_kernel launch");
    }
    k.stop_after = pl.stop_after;
    k.planes = d_planes;
    if ((reinterpret_cast<uintptr_t>(d_ranges) & 15u) != 0) k.ring = 0;   // bulk copies need 16-byte aligned rows
    // two instantiations: frames without / with Map Connection offsets
    if (k.n_off > 0)
        return launch_cluster(rs::rs_fast_kernel<true>, k, batch, rs::kFastThreads, pl.smem_f, stream,
                              "rs_fast_kernel<MC> launch");
    return launch_cluster(rs::rs_fast_kernel<false>, k, batch, rs::kFastThreads, pl.smem_f, stream,
                          "rs_fast_kernel launch");
}

// Output checks shared by the device and host entries (before any allocation
// or launch): the sizes stride bounds the label values the kernels write.
int validate_outputs(const rs_config *cfg, int32_t batch, const void *labels, const void *sizes,
                     int64_t sizes_stride) {
    if (batch < 0) return fail(RS_EINVAL, "batch must be >= 0");
    if (batch > 0 && !labels) return fail(RS_EINVAL, "labels are required");
    if (sizes) {
        const long long need = (long long)cfg->height * cfg->width / std::max(cfg->min_cluster_points, 1) + 1;
        if (sizes_stride < need)
            return fail(RS_EINVAL, "sizes_stride must be >= H*W/max(min_cluster_points,1)+1 = " +
                                       std::to_string(need));
    }
    return RS_OK;
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
    const KArgs &k = pl.fast ? pl.kf : pl.kd;
    if (rows_per_cta) *rows_per_cta = k.R;
    if (ctas_per_frame) *ctas_per_frame = k.C;
    if (smem_bytes) *smem_bytes = pl.fast ? pl.smem_f : pl.smem_d;
    return RS_OK;
}

int rs_plan_detail(const rs_config *cfg, int32_t *out, int32_t n) { return rs_plan_batch(cfg, 0, out, n); }

int rs_plan_batch(const rs_config *cfg, int32_t batch, int32_t *out, int32_t n) {
    Plan pl;
    int st = make_plan(cfg, &pl, std::max(batch, 0));
    if (st) return st;
    const int32_t v[] = {pl.fast ? 1 : 0, pl.may_overflow ? 1 : 0, pl.kf.R, pl.kf.C, (int32_t)pl.smem_f, pl.kf.NC,
                         pl.kd.R, pl.kd.C, (int32_t)pl.smem_d};
    for (int i = 0; i < n && i < (int)(sizeof(v) / sizeof(v[0])); ++i) out[i] = v[i];
    return RS_OK;
}

int rs_segment_batch(const rs_config *cfg, const float *d_tables, const float *d_ranges, int32_t batch,
                     int32_t *d_labels, int32_t *d_n_clusters, int64_t *d_cluster_sizes, int64_t sizes_stride,
                     void *stream) {
    Plan pl;
    int st = make_plan(cfg, &pl, std::max(batch, 0));
    if (st) return st;
    if ((st = validate_outputs(cfg, batch, d_labels, d_cluster_sizes, sizes_stride))) return st;
    if (batch == 0) return RS_OK;
    if (!d_tables || !d_ranges) return fail(RS_EINVAL, "tables and ranges are required");
    if (reinterpret_cast<uintptr_t>(d_labels) & 15u) return fail(RS_EINVAL, "d_labels must be 16-byte aligned");
    if ((long long)batch * std::max(pl.kf.C, pl.kd.C) > 0x7fffffffLL) return fail(RS_EINVAL, "batch too large");
    return segment_launch(pl, d_tables, d_ranges, batch, d_labels, d_n_clusters, d_cluster_sizes, sizes_stride,
                          static_cast<cudaStream_t>(stream));
}

int rs_fast_planes(const rs_config *cfg, const float *d_tables, const float *d_ranges, int32_t batch,
                   uint32_t *d_planes, int32_t *d_labels, int32_t *d_n_clusters, void *stream) {
    Plan pl;
    int st = make_plan(cfg, &pl, std::max(batch, 0));
    if (st) return st;
    if ((st = validate_outputs(cfg, batch, d_labels, nullptr, 0))) return st;
    if (!pl.fast) return fail(RS_EINVAL, "the fast kernel does not run this geometry (no planes to export)");
    if (batch == 0) return RS_OK;
    if (!d_tables || !d_ranges || !d_planes) return fail(RS_EINVAL, "tables, ranges and planes are required");
    if (reinterpret_cast<uintptr_t>(d_labels) & 15u) return fail(RS_EINVAL, "d_labels must be 16-byte aligned");
    if ((long long)batch * pl.kf.C > 0x7fffffffLL) return fail(RS_EINVAL, "batch too large");
    return segment_launch(pl, d_tables, d_ranges, batch, d_labels, d_n_clusters, nullptr, 0,
                          static_cast<cudaStream_t>(stream), d_planes);
}

int rs_stage_masks(const rs_config *cfg, const float *d_tables, const float *d_ranges, int32_t batch,
                   uint8_t *d_ground, uint8_t *d_horizontal, uint8_t *d_vertical, void *stream) {
    int st = validate(cfg);
    if (st) return st;
    if (batch <= 0) return batch == 0 ? RS_OK : fail(RS_EINVAL, "batch must be >= 0");
    if (!d_tables || !d_ranges || !d_ground || !d_horizontal || !d_vertical)
        return fail(RS_EINVAL, "all buffers are required");
    KArgs k;
    fill_common(cfg, 1, k);
    k.ranges = d_ranges;
    k.tables = d_tables;
    const long long total = (long long)batch * cfg->height * cfg->width;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
    rs::rs_stage_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(k, d_ground, d_horizontal,
                                                                              d_vertical, total);
    return cuda_check(cudaGetLastError(), "rs_stage_kernel launch");
}

namespace {
int stage_launch_args(const rs_config *cfg, const float *d_tables, const float *d_ranges, int32_t batch, KArgs &k,
                      long long &total, int &blocks) {
    int st = validate(cfg);
    if (st) return st;
    if (batch < 0) return fail(RS_EINVAL, "batch must be >= 0");
    if (batch > 0 && (!d_tables || !d_ranges)) return fail(RS_EINVAL, "tables and ranges are required");
    fill_common(cfg, 1, k);
    k.ranges = d_ranges;
    k.tables = d_tables;
    total = (long long)batch * cfg->height * cfg->width;
    blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, 148LL * 16));
    return RS_OK;
}
}  // namespace

int rs_height_image(const rs_config *cfg, const float *d_tables, const float *d_ranges, int32_t batch,
                    float *d_height, void *stream) {
    KArgs k;
    long long total;
    int blocks, st;
    if ((st = stage_launch_args(cfg, d_tables, d_ranges, batch, k, total, blocks))) return st;
    if (!total) return RS_OK;
    if (!d_height) return fail(RS_EINVAL, "height buffer is required");
    rs::rs_height_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(k, d_height, total);
    return cuda_check(cudaGetLastError(), "rs_height_kernel launch");
}

int rs_ground_mask(const rs_config *cfg, const float *d_tables, const float *d_ranges, const float *d_height,
                   int32_t batch, uint8_t *d_mask, void *stream) {
    KArgs k;
    long long total;
    int blocks, st;
    if ((st = stage_launch_args(cfg, d_tables, d_ranges, batch, k, total, blocks))) return st;
    if (!total) return RS_OK;
    if (!d_height || !d_mask) return fail(RS_EINVAL, "height and mask buffers are required");
    rs::rs_ground_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(k, d_height, d_mask, total);
    return cuda_check(cudaGetLastError(), "rs_ground_kernel launch");
}

int rs_connectivity(const rs_config *cfg, const float *d_tables, const float *d_ranges, const uint8_t *d_mask,
                    int32_t batch, uint8_t *d_horizontal, uint8_t *d_vertical, void *stream) {
    KArgs k;
    long long total;
    int blocks, st;
    if ((st = stage_launch_args(cfg, d_tables, d_ranges, batch, k, total, blocks))) return st;
    if (!total) return RS_OK;
    if (!d_mask || !d_horizontal || !d_vertical) return fail(RS_EINVAL, "mask and edge buffers are required");
    rs::rs_connectivity_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(k, d_mask, d_horizontal,
                                                                                     d_vertical, total);
    return cuda_check(cudaGetLastError(), "rs_connectivity_kernel launch");
}

// Host-buffer entry: chunks of frames are pipelined over two streams so the
// host->device copy of chunk j+1 overlaps the kernel of chunk j and the
// device->host copy of chunk j-1.
namespace {
struct HostCtx {
    std::mutex mu;
    float *d_ranges = nullptr, *d_tables = nullptr;
    int32_t *d_labels = nullptr, *d_ncl = nullptr;
    int32_t *h_ncl = nullptr;   // pinned: cluster counts when the caller passes none (invalid-frame check)
    int64_t *d_sizes = nullptr;
    // kHostStreams streams round-robin over chunks, so the host->device copy
    // of chunk j+2 can run while chunk j is copied back (both copy engines busy)
    static constexpr int kHostStreams = 4;
    size_t cap_frames = 0, cap_tables = 0, cap_sizes = 0, frame_cells = 0;
    cudaStream_t s[kHostStreams] = {};
    int device = -1;
};
HostCtx g_host;

void host_free() {
    cudaFree(g_host.d_ranges);
    cudaFree(g_host.d_labels);
    cudaFree(g_host.d_ncl);
    cudaFree(g_host.d_sizes);
    cudaFreeHost(g_host.h_ncl);
    g_host.h_ncl = nullptr;
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
    int st = make_plan(cfg, &pl, std::max(batch, 0));
    if (st) return st;
    if ((st = validate_outputs(cfg, batch, h_labels, h_cluster_sizes, sizes_stride))) return st;
    if (batch == 0) return RS_OK;
    if (!h_tables || !h_ranges) return fail(RS_EINVAL, "tables and ranges are required");
    if ((long long)batch * std::max(pl.kf.C, pl.kd.C) > 0x7fffffffLL) return fail(RS_EINVAL, "batch too large");
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
            (st = cuda_check(cudaMalloc(&g_host.d_ncl, (size_t)batch * 4), "cudaMalloc n_clusters")) ||
            (st = cuda_check(cudaMallocHost(&g_host.h_ncl, (size_t)batch * 4), "cudaMallocHost n_clusters")))
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
    for (int i = 1; i < HostCtx::kHostStreams; ++i) cudaStreamWaitEvent(g_host.s[i], tables_ready, 0);
    // 16 MB of ranges per chunk (measured best of 2-64 MB on the headline batch)
    const int chunk = std::max(1, std::min<int>(batch, std::max<int>(1, (int)((16u << 20) / (HW * 4)))));
    for (int b0 = 0, j = 0; b0 < batch; b0 += chunk, ++j) {
        const int nb = std::min(chunk, batch - b0);
        cudaStream_t s = g_host.s[j % HostCtx::kHostStreams];
        const size_t off = (size_t)b0 * HW;
        if ((st = cuda_check(cudaMemcpyAsync(g_host.d_ranges + off, h_ranges + off, nb * HW * 4,
                                             cudaMemcpyHostToDevice, s), "copy ranges")))
            break;
        st = segment_launch(pl, g_host.d_tables, g_host.d_ranges + off, nb, g_host.d_labels + off, g_host.d_ncl + b0,
                            h_cluster_sizes ? g_host.d_sizes + (size_t)b0 * sizes_stride : nullptr, sizes_stride, s);
        if (st) break;
        if ((st = cuda_check(cudaMemcpyAsync(h_labels + off, g_host.d_labels + off, nb * HW * 4,
                                             cudaMemcpyDeviceToHost, s), "copy labels")))
            break;
        int32_t *ncl_dst = h_n_clusters ? h_n_clusters : g_host.h_ncl;
        if ((st = cuda_check(cudaMemcpyAsync(ncl_dst + b0, g_host.d_ncl + b0, nb * 4, cudaMemcpyDeviceToHost, s),
                             "copy n_clusters")))
            break;
        if (h_cluster_sizes &&
            (st = cuda_check(cudaMemcpyAsync(h_cluster_sizes + (size_t)b0 * sizes_stride,
                                             g_host.d_sizes + (size_t)b0 * sizes_stride,
                                             (size_t)nb * sizes_stride * 8, cudaMemcpyDeviceToHost, s),
                             "copy sizes")))
            break;
    }
    int sst = RS_OK;
    for (auto &hs : g_host.s) {
        const int e = cuda_check(cudaStreamSynchronize(hs), "stream sync");
        if (!sst) sst = e;
    }
    cudaEventDestroy(tables_ready);
    if (st || sst) return st ? st : sst;
    const int32_t *ncl = h_n_clusters ? h_n_clusters : g_host.h_ncl;
    for (int b = 0; b < batch; ++b)
        if (ncl[b] == RS_FRAME_INVALID)
            return fail(RS_EINVAL, "frame " + std::to_string(b) + ": ranges must be finite and >= 0");
    return RS_OK;
}

int rs_project(const rs_project_config *pc, const double *d_asc, const double *d_points, int32_t stride,
               const int64_t *d_offsets, int32_t n_clouds, int64_t n_points, float *d_ranges,
               int64_t *d_point_index, int64_t *d_counts, void *d_workspace, size_t workspace_size,
               void *stream) {
    if (!pc) return fail(RS_EINVAL, "config is NULL");
    if (workspace_size < rs_project_workspace_size(n_points) || (n_points > 0 && !d_workspace))
        return fail(RS_EINVAL, "workspace smaller than rs_project_workspace_size(n_points)");
    if (pc->height < 2 || pc->width < 1) return fail(RS_EINVAL, "need at least 2 channels and 1 column");
    if (!(pc->azimuth_step > 0)) return fail(RS_EINVAL, "azimuth step must be > 0");
    if (stride < 3) return fail(RS_EINVAL, "points need at least 3 columns");
    if (n_clouds < 0 || n_points < 0) return fail(RS_EINVAL, "negative sizes");
    if (n_points >= (1LL << 31)) return fail(RS_ETOOLARGE, "at most 2^31 - 1 points per call");
    if (n_clouds == 0) return RS_OK;
    if (!d_asc || !d_offsets || !d_ranges || !d_point_index || !d_counts || (n_points > 0 && !d_points))
        return fail(RS_EINVAL, "NULL buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t cells = (int64_t)n_clouds * pc->height * pc->width;
    rs::ProjArgs a{};
    a.pts = d_points;
    a.stride = stride;
    a.offsets = d_offsets;
    a.B = n_clouds;
    a.H = pc->height;
    a.W = pc->width;
    a.desc = pc->descending ? 1 : 0;
    a.step = pc->azimuth_step;
    a.gap_lo = pc->gap_lo;
    a.gap_hi = pc->gap_hi;
    a.two_pi = 2.0 * 3.141592653589793;   // 2.0 * np.pi (range_image.py:93)
    a.asc = d_asc;
    a.n_total = n_points;
    a.ranges = d_ranges;
    a.point_index = d_point_index;
    a.counts = d_counts;
    a.rbits = static_cast<unsigned long long *>(d_workspace);
    a.cell = reinterpret_cast<int32_t *>(a.rbits + n_points);
    int st;
    // scratch: +inf-like range bits (all ones) and index -1 (all ones)
    if ((st = cuda_check(cudaMemsetAsync(d_point_index, 0xff, (size_t)cells * 8, s), "memset point_index")) ||
        (st = cuda_check(cudaMemsetAsync(d_ranges, 0xff, (size_t)cells * 4, s), "memset ranges")) ||
        (st = cuda_check(cudaMemsetAsync(d_counts, 0, (size_t)n_clouds * 16, s), "memset counts")))
        return st;
    const unsigned tp = rs::kProjThreads;
    if (n_points > 0) {
        const unsigned gp = (unsigned)((n_points + tp - 1) / tp);
        rs::rs_project_min_kernel<<<gp, tp, 0, s>>>(a);
        rs::rs_project_index_kernel<<<gp, tp, 0, s>>>(a);
    }
    rs::rs_project_finish_kernel<<<(unsigned)((cells + tp - 1) / tp), tp, 0, s>>>(a);
    rs::rs_project_counts_kernel<<<(unsigned)((n_clouds + 127) / 128), 128, 0, s>>>(a);
    return cuda_check(cudaGetLastError(), "rs_project launch");
}

size_t rs_project_workspace_size(int64_t n_points) { return (size_t)std::max<int64_t>(n_points, 0) * 12u; }

int rs_labels_to_points(const int32_t *d_labels, const int64_t *d_point_index, const int64_t *d_offsets,
                        int32_t n_clouds, int32_t height, int32_t width, int64_t n_points,
                        int32_t *d_point_labels, void *stream) {
    if (n_clouds < 0 || n_points < 0 || height < 1 || width < 1) return fail(RS_EINVAL, "bad sizes");
    if (n_clouds == 0) return RS_OK;
    if (!d_labels || !d_point_index || !d_offsets || (n_points > 0 && !d_point_labels))
        return fail(RS_EINVAL, "NULL buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int st;
    if (n_points > 0 &&
        (st = cuda_check(cudaMemsetAsync(d_point_labels, 0, (size_t)n_points * 4, s), "memset point labels")))
        return st;
    const int64_t HW = (int64_t)height * width, cells = (int64_t)n_clouds * HW;
    rs::rs_labels_to_points_kernel<<<(unsigned)((cells + rs::kProjThreads - 1) / rs::kProjThreads),
                                     rs::kProjThreads, 0, s>>>(d_labels, d_point_index, d_offsets, n_clouds, HW,
                                                               d_point_labels);
    return cuda_check(cudaGetLastError(), "rs_labels_to_points launch");
}

// workspace of rs_contingency: per frame count / offset / none count (u64
// each), the invalid-label flag, then the per-frame scratch (rs_eval.cuh):
// 4 (n_points + B) keys (u64) and counts (u32).  B is bounded by n_points + 1
// for the size query (frames may be empty), so it is taken from the caller.
namespace {
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
struct ContLayout {
    size_t frames, flag, keys, cnts, total;
};
ContLayout cont_layout(int64_t n_points, int64_t n_frames) {
    ContLayout l;
    const size_t ent = 4 * ((size_t)std::max<int64_t>(n_points, 0) + (size_t)std::max<int64_t>(n_frames, 0));
    l.frames = 0;
    l.flag = align256(3 * 8 * (size_t)std::max<int64_t>(n_frames, 1));
    l.keys = l.flag + 256;
    l.cnts = l.keys + align256(ent * 8);
    l.total = l.cnts + align256(ent * 4);
    return l;
}
}  // namespace

size_t rs_contingency_workspace_size(int64_t n_points, int32_t n_frames) {
    if (n_points < 0 || n_points >= (1LL << 31) || n_frames < 0) return 0;
    return cont_layout(n_points, n_frames).total;
}

int rs_contingency(const int32_t *d_gt, const int32_t *d_pred, const int64_t *d_offsets, int32_t n_frames,
                   int64_t n_points, int64_t *d_pairs, int64_t *d_counts, int64_t *d_status, void *d_workspace,
                   size_t workspace_size, void *stream) {
    if (n_frames < 0 || n_points < 0) return fail(RS_EINVAL, "negative sizes");
    if (n_frames >= (1 << rs::kEvalFrameBits)) return fail(RS_ETOOLARGE, "at most 2^19 - 1 frames per call");
    if (n_points >= (1LL << 31)) return fail(RS_ETOOLARGE, "at most 2^31 - 1 points per call");
    if (workspace_size < rs_contingency_workspace_size(n_points, n_frames))
        return fail(RS_EINVAL, "workspace smaller than rs_contingency_workspace_size(n_points, n_frames)");
    if (!d_status || (n_points > 0 && (!d_gt || !d_pred || !d_offsets || !d_pairs || !d_counts || !d_workspace)))
        return fail(RS_EINVAL, "NULL buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int st;
    if ((st = cuda_check(cudaMemsetAsync(d_status, 0, 2 * sizeof(int64_t), s), "memset status"))) return st;
    if (n_points == 0 || n_frames == 0) return RS_OK;
    const ContLayout l = cont_layout(n_points, n_frames);
    char *w = static_cast<char *>(d_workspace);
    auto *frame_n = reinterpret_cast<unsigned long long *>(w);
    auto *frame_off = frame_n + n_frames;
    auto *frame_none = frame_off + n_frames;
    int *bad = reinterpret_cast<int *>(w + l.flag);
    auto *K = reinterpret_cast<unsigned long long *>(w + l.keys);
    auto *C = reinterpret_cast<uint32_t *>(w + l.cnts);
    static bool attr_set = false;   // per process; the attribute is per function, any device of one arch
    if (!attr_set) {
        if ((st = cuda_check(cudaFuncSetAttribute(rs::rs_cont_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)rs::kEvalSmem), "cudaFuncSetAttribute(contingency)")))
            return st;
        attr_set = true;
    }
    if ((st = cuda_check(cudaMemsetAsync(bad, 0, sizeof(int), s), "memset flag"))) return st;
    rs::rs_cont_count_kernel<<<n_frames, rs::kEvalThreads, rs::kEvalSmem, s>>>(d_gt, d_pred, d_offsets, K, C, frame_n,
                                                                              frame_none, bad);
    rs::rs_cont_scan_kernel<<<1, 1024, 0, s>>>(n_frames, frame_n, frame_none, frame_off, d_pairs, d_counts, d_status,
                                              bad);
    rs::rs_cont_move_kernel<<<n_frames, 256, 0, s>>>(d_offsets, K, C, frame_n, frame_off, d_pairs, d_counts);
    return cuda_check(cudaGetLastError(), "rs_contingency launch");
}

int rs_phase_profile(int64_t *host_out, int32_t max_ctas) {
#ifdef RS_PHASE_PROF
    const int n = std::min<int>(max_ctas, rs::kProfCtas);
    if (!host_out || n <= 0) return fail(RS_EINVAL, "bad profile buffer");
    return cuda_check(cudaMemcpyFromSymbol(host_out, rs::g_prof, (size_t)n * rs::kProfSlots * sizeof(long long)),
                      "read phase profile");
#else
    (void)host_out;
    (void)max_ctas;
    return fail(RS_EINVAL, "library built without RS_PHASE_PROF");
#endif
}

#ifdef RS_MC_STATS
int rs_mc_stats(int64_t *host_out, int32_t reset) {
    int st = cuda_check(cudaMemcpyFromSymbol(host_out, rs::g_mcstats, sizeof(rs::g_mcstats)), "read stats");
    if (!st && reset) {
        unsigned long long z[8] = {};
        st = cuda_check(cudaMemcpyToSymbol(rs::g_mcstats, z, sizeof(z)), "reset stats");
    }
    return st;
}
#endif

const char *rs_last_error(void) { return g_err.c_str(); }

int rs_version(void) { return 300; }

}  // extern "C"
