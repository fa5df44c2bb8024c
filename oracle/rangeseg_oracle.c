/*
 * rangeseg_oracle.c — CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or as the timed CPU baseline.  The product path
 * (paper_2003_00575_b200) never links or calls it.
 *
 * It restates, step by step and in the reference's own algorithmic order, the
 * per-frame path behind Pipeline.segment_range_image
 * (/root/reference/pkg/src/rangeseg/pipeline.py:85-131):
 *
 *   height_image            range_image.py:118-127
 *   extract_ground          ground.py:95-141
 *   build_connectivity      connectivity.py:64-92  (pair_distance_sq :47-55)
 *   _flood_fill             ccl.py:83-131   first-encounter labels, wrap seam
 *   label_components        ccl.py:134-151  bincount sizes
 *   apply_map_connections   map_connections.py:132-178 (ClusterUnion :73-110,
 *                           _renumber_roots :113-129)
 *   filter_small            ccl.py:154-170
 *
 * Arithmetic contract: every float op is IEEE binary32
 * with its own rounding, exactly like the numpy ufunc chain.  Build with
 * -ffp-contract=off and without -ffast-math (see oracle/Makefile).
 *
 * Pinned against the reference itself: the tests/golden fixtures are produced by
 * tests/golden/make_golden.py, which imports the Python reference in the
 * build container and records its outputs; tests/test_oracle_golden.py checks
 * this file bit-for-bit against them.
 *
 * Table layout (float32, built by the host from float64 exactly as
 * sensor.py:97-141 and ground.py:76-92 do, then cast):
 *   sin_ch[H] | sin_a[H-1] | cos_a[H-1] | lo[H-1] | hi[H-1] | two_cos_v[H-1]
 *   | two_cos_off[k][H]  (row = upper row of the pair; dy == 0 rows repeat)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int32_t height, width;
    int32_t n_offsets;
    const int32_t *offsets;     /* [n_offsets][2] canonical (dy, dx) */
    int32_t min_cluster_points;
    int32_t ground_removal;
    float d_max_sq, mount_height, keep_above, two_cos_h;
    const float *tables;
} oracle_cfg;

/* pair_distance_sq, connectivity.py:54: ((d1*d1 + d2*d2) - c*(d1*d2)), each
 * op rounded; the >=0 clamp (:55) never changes a `<= d_max_sq` decision
 * (NaN stays NaN under np.maximum and compares false either way). */
static inline int pair_ok(float d1, float d2, float c, float thr) {
    float a = d1 * d1;
    float b = d2 * d2;
    float s = a + b;
    float p = d1 * d2;
    float q = c * p;
    float d = s - q;
    return d <= thr;
}

/* ---- ground.py:95-141 + range_image.py:118-127 ------------------------- */
static void oracle_ground(const float *rg, const oracle_cfg *cfg, uint8_t *mask) {
    const int H = cfg->height, W = cfg->width;
    const float *sin_ch = cfg->tables;
    const float *sin_a = sin_ch + H, *cos_a = sin_a + (H - 1);
    const float *lo = cos_a + (H - 1), *hi = lo + (H - 1);
    if (!cfg->ground_removal) {
        for (int i = 0; i < H * W; ++i) mask[i] = !(rg[i] > 0.0f);
        return;
    }
    for (int r = 0; r < H; ++r) {
        int k = (r >= 1 ? r : 1) - 1;          /* slope_ok[0] = pair_ok[0] */
        for (int c = 0; c < W; ++c) {
            float d1 = rg[k * W + c], d2 = rg[(k + 1) * W + c];
            float num = d2 * sin_a[k];
            float t = d2 * cos_a[k];
            float den = d1 - t;
            float L = lo[k] * den;
            float U = hi[k] * den;
            int ok = (den > 0.0f) ? (num >= L && num <= U) : (num <= L && num >= U);
            ok = ok && (den != 0.0f) && (d1 > 0.0f) && (d2 > 0.0f);
            float rv = rg[r * W + c];
            int valid = rv > 0.0f;
            float z = rv * sin_ch[r];
            float zz = z + cfg->mount_height;
            int low = valid && (zz <= cfg->keep_above);   /* NaN height → false */
            mask[r * W + c] = (!valid) || (ok && low);
        }
    }
}

/* ---- connectivity.py:64-92 ---------------------------------------------- */
static void oracle_connectivity(const float *rg, const uint8_t *gmask,
                                const oracle_cfg *cfg, uint8_t *horiz, uint8_t *vert) {
    const int H = cfg->height, W = cfg->width;
    const float *tcv = cfg->tables + H + 4 * (H - 1);
    const float thr = cfg->d_max_sq;
#define PRESENT(i) (rg[(i)] > 0.0f && !gmask[(i)])
    for (int r = 0; r < H; ++r)
        for (int c = 0; c < W; ++c) {
            int i = r * W + c;
            if (W > 1) {
                int j = r * W + (c + 1 == W ? 0 : c + 1);   /* np.roll(-1) */
                horiz[i] = pair_ok(rg[i], rg[j], cfg->two_cos_h, thr) && PRESENT(i) && PRESENT(j);
            } else {
                horiz[i] = 0;
            }
            if (r < H - 1) {
                int j = i + W;
                vert[i] = pair_ok(rg[i], rg[j], tcv[r], thr) && PRESENT(i) && PRESENT(j);
            }
        }
#undef PRESENT
}

/* ---- ccl.py:83-131: stack flood fill on the (implicit) lattice ---------- */
static int32_t oracle_flood_fill(const uint8_t *present, const uint8_t *horiz,
                                 const uint8_t *vert, int H, int W,
                                 int32_t *labels, int64_t *stack) {
    int32_t next = 0;
    memset(labels, 0, sizeof(int32_t) * (size_t)H * W);
    for (int r0 = 0; r0 < H; ++r0)
        for (int c0 = 0; c0 < W; ++c0) {
            if (!present[r0 * W + c0] || labels[r0 * W + c0]) continue;
            ++next;
            labels[r0 * W + c0] = next;
            stack[0] = (int64_t)r0 * W + c0;
            int64_t top = 1;
            while (top > 0) {
                int64_t idx = stack[--top];
                int r = (int)(idx / W), c = (int)(idx - (int64_t)r * W);
                /* right: lattice (2r, 2c+1) */
                if (horiz[r * W + c]) {
                    int c2 = c + 1 < W ? c + 1 : 0;
                    if (!labels[r * W + c2]) { labels[r * W + c2] = next; stack[top++] = (int64_t)r * W + c2; }
                }
                /* left: lattice (2r, 2c-1) or the seam column 2W-1 */
                int lc = c > 0 ? c - 1 : W - 1;
                if (horiz[r * W + lc]) {
                    int c2 = lc;
                    if (!labels[r * W + c2]) { labels[r * W + c2] = next; stack[top++] = (int64_t)r * W + c2; }
                }
                if (r > 0 && vert[(r - 1) * W + c]) {
                    if (!labels[(r - 1) * W + c]) { labels[(r - 1) * W + c] = next; stack[top++] = (int64_t)(r - 1) * W + c; }
                }
                if (r < H - 1 && vert[r * W + c]) {
                    if (!labels[(r + 1) * W + c]) { labels[(r + 1) * W + c] = next; stack[top++] = (int64_t)(r + 1) * W + c; }
                }
            }
        }
    return next;
}

/* ---- map_connections.py:73-110 ClusterUnion ----------------------------- */
static int64_t cu_find(int64_t *parent, int64_t x) {
    int64_t root = x;
    while (parent[root] != root) root = parent[root];
    while (parent[x] != root) { int64_t nx = parent[x]; parent[x] = root; x = nx; }
    return root;
}
static int cu_union(int64_t *parent, int64_t *size, int64_t a, int64_t b) {
    int64_t ra = cu_find(parent, a), rb = cu_find(parent, b);
    if (ra == rb) return 0;
    if (size[ra] < size[rb]) { int64_t t = ra; ra = rb; rb = t; }
    parent[rb] = ra;
    size[ra] += size[rb];
    return 1;
}

/* ---- map_connections.py:132-178 + _renumber_roots :113-129 --------------
 * Union order differs from the reference's np.unique order, but the final
 * partition and the min-member ranking do not depend on it. */
static int32_t oracle_map_connections(const float *rg, const oracle_cfg *cfg,
                                      int32_t *labels, int64_t *sizes, int32_t K) {
    const int H = cfg->height, W = cfg->width;
    const float thr = cfg->d_max_sq;
    int64_t *parent = malloc(sizeof(int64_t) * (size_t)(K + 1));
    int64_t *usize = malloc(sizeof(int64_t) * (size_t)(K + 1));
    for (int64_t i = 0; i <= K; ++i) { parent[i] = i; usize[i] = 1; }
    int64_t merged = 0;
    for (int k = 0; k < cfg->n_offsets; ++k) {
        int dy = cfg->offsets[2 * k], dx = cfg->offsets[2 * k + 1];
        const float *tc = cfg->tables + H + 5 * (H - 1) + (size_t)k * H;
        for (int r = 0; r + dy < H; ++r)
            for (int c = 0; c < W; ++c) {
                int c2 = ((c + dx) % W + W) % W;         /* np.roll(-dx) */
                int i = r * W + c, j = (r + dy) * W + c2;
                int32_t la = labels[i], lb = labels[j];
                if (la <= 0 || lb <= 0 || la == lb) continue;
                if (pair_ok(rg[i], rg[j], tc[r], thr))
                    merged += cu_union(parent, usize, la, lb);
            }
    }
    if (merged == 0) { free(parent); free(usize); return K; }
    /* roots → rank by minimum member label (first-encounter order kept) */
    int64_t *root = malloc(sizeof(int64_t) * (size_t)(K + 1));
    int64_t *minm = malloc(sizeof(int64_t) * (size_t)(K + 1));
    int32_t *rank = calloc((size_t)(K + 1), sizeof(int32_t));
    for (int64_t i = 0; i <= K; ++i) { root[i] = cu_find(parent, i); minm[i] = INT64_MAX; }
    for (int64_t i = 1; i <= K; ++i) if (i < minm[root[i]]) minm[root[i]] = i;
    /* labels are ids 1..K; the smallest member of each root, scanned in label
     * order, is first seen exactly in ascending min-member order */
    int32_t next = 0;
    for (int64_t i = 1; i <= K; ++i)
        if (minm[root[i]] == i) rank[root[i]] = ++next;
    int64_t *ns = calloc((size_t)next + 1, sizeof(int64_t));
    for (int64_t i = 0; i <= K; ++i) ns[rank[root[i]]] += sizes[i];
    for (int i = 0; i < H * W; ++i) labels[i] = rank[root[labels[i]]];
    for (int32_t i = 0; i <= next; ++i) sizes[i] = ns[i];
    free(parent); free(usize); free(root); free(minm); free(rank); free(ns);
    return next;
}

/* ---- ccl.py:154-170 ------------------------------------------------------ */
static int32_t oracle_filter_small(int32_t *labels, int64_t *sizes, int32_t K,
                                   int HW, int32_t min_points) {
    if (min_points <= 1) return K;
    int32_t *lut = calloc((size_t)K + 1, sizeof(int32_t));
    int32_t kept = 0;
    int64_t sum = 0;
    for (int32_t i = 1; i <= K; ++i)
        if (sizes[i] >= min_points) { lut[i] = ++kept; sizes[kept] = sizes[i]; sum += sizes[i]; }
    for (int i = 0; i < HW; ++i) labels[i] = lut[labels[i]];
    sizes[0] = (int64_t)HW - sum;
    free(lut);
    return kept;
}

/* Stage outputs (optional, may be NULL): ground mask [H*W] (True = ground or
 * invalid), horizontal [H*W], vertical [(H-1)*W].
 * sizes must hold H*W+1 entries.  Returns the cluster count K (>= 0), or -1
 * on allocation failure. */
int32_t oracle_segment_frame(const float *ranges, const oracle_cfg *cfg,
                             int32_t *labels, int64_t *sizes,
                             uint8_t *ground_out, uint8_t *horiz_out, uint8_t *vert_out) {
    const int H = cfg->height, W = cfg->width, HW = H * W;
    uint8_t *gm = malloc((size_t)HW), *hz = malloc((size_t)HW), *vt = malloc((size_t)HW);
    uint8_t *pr = malloc((size_t)HW);
    int64_t *stack = malloc(sizeof(int64_t) * (size_t)HW);
    if (!gm || !hz || !vt || !pr || !stack) return -1;
    oracle_ground(ranges, cfg, gm);
    oracle_connectivity(ranges, gm, cfg, hz, vt);
    for (int i = 0; i < HW; ++i) pr[i] = ranges[i] > 0.0f && !gm[i];   /* pipeline.py:109 */
    int32_t K = oracle_flood_fill(pr, hz, vt, H, W, labels, stack);
    memset(sizes, 0, sizeof(int64_t) * ((size_t)K + 1));
    for (int i = 0; i < HW; ++i) sizes[labels[i]]++;                    /* np.bincount */
    if (cfg->n_offsets > 0) K = oracle_map_connections(ranges, cfg, labels, sizes, K);
    K = oracle_filter_small(labels, sizes, K, HW, cfg->min_cluster_points);
    if (ground_out) memcpy(ground_out, gm, (size_t)HW);
    if (horiz_out) memcpy(horiz_out, hz, (size_t)HW);
    if (vert_out) memcpy(vert_out, vt, (size_t)(H - 1) * W);
    free(gm); free(hz); free(vt); free(pr); free(stack);
    return K;
}

/* ---- batch over frames on host threads (the CPU baseline) --------------- */
typedef struct {
    const float *ranges; const oracle_cfg *cfg; int32_t *labels; int32_t *nclusters;
    int64_t *sizes; int64_t sizes_stride; int B, tid, nthreads; int failed;
} batch_job;

static void *batch_worker(void *arg) {
    batch_job *j = (batch_job *)arg;
    const size_t HW = (size_t)j->cfg->height * j->cfg->width;
    int64_t *sz = malloc(sizeof(int64_t) * (HW + 1));
    for (int f = j->tid; f < j->B; f += j->nthreads) {
        int32_t K = oracle_segment_frame(j->ranges + f * HW, j->cfg, j->labels + f * HW,
                                         sz, NULL, NULL, NULL);
        if (K < 0) { j->failed = 1; break; }
        if (j->nclusters) j->nclusters[f] = K;
        if (j->sizes) {
            int64_t n = (int64_t)K + 1 < j->sizes_stride ? (int64_t)K + 1 : j->sizes_stride;
            memcpy(j->sizes + (size_t)f * j->sizes_stride, sz, sizeof(int64_t) * (size_t)n);
        }
    }
    free(sz);
    return NULL;
}

int oracle_segment_batch(const float *ranges, int B, const oracle_cfg *cfg,
                         int32_t *labels, int32_t *nclusters, int64_t *sizes,
                         int64_t sizes_stride, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > B) nthreads = B > 0 ? B : 1;
    pthread_t th[256];
    batch_job jobs[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (batch_job){ranges, cfg, labels, nclusters, sizes, sizes_stride, B, t, nthreads, 0};
        if (nthreads == 1) batch_worker(&jobs[0]);
        else pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
    }
    int failed = 0;
    for (int t = 0; t < nthreads; ++t) {
        if (nthreads > 1) pthread_join(th[t], NULL);
        failed |= jobs[t].failed;
    }
    return failed ? -1 : 0;
}

/* ---- edge decisions as packed bit planes (parity of the fused kernel's own
 * planes, rs_fast_planes in include/rangeseg_b200.h) ----------------------
 * [3 + n_offsets][H][ceil(W/32)] uint32 per frame, bit c%32 of word c/32:
 *   0 presence = valid and not ground          (ground.py:132-140, pipeline.py:109)
 *   1 left edge (r,c-1 mod W)-(r,c) = horizontal[r][c-1 mod W]   (connectivity.py:80-84)
 *   2 up edge (r-1,c)-(r,c) = vertical[r-1][c]                   (connectivity.py:86-90)
 *   3+k Map Connection k: (r-dy, c-dx mod W)-(r,c) for r >= dy, both present and
 *     pair_distance_sq <= d_max_sq with the pair's upper-row constant
 *     (map_connections.py:155-169; the reference evaluates it only between
 *     different labels, the plane holds the decision for every present pair). */
static void oracle_frame_planes(const float *rg, const oracle_cfg *cfg, uint32_t *out,
                                uint8_t *gm, uint8_t *hz, uint8_t *vt) {
    const int H = cfg->height, W = cfg->width, WPR = (W + 31) / 32;
    const size_t fw = (size_t)H * WPR;
    oracle_ground(rg, cfg, gm);
    oracle_connectivity(rg, gm, cfg, hz, vt);
    memset(out, 0, sizeof(uint32_t) * fw * (size_t)(3 + cfg->n_offsets));
#define SETB(pl, r, c) out[(size_t)(pl) * fw + (size_t)(r) * WPR + ((c) >> 5)] |= 1u << ((c) & 31)
#define PRES(r, c) (rg[(r) * W + (c)] > 0.0f && !gm[(r) * W + (c)])
    for (int r = 0; r < H; ++r)
        for (int c = 0; c < W; ++c) {
            if (PRES(r, c)) SETB(0, r, c);
            if (W > 1 && hz[r * W + (c + W - 1) % W]) SETB(1, r, c);
            if (r >= 1 && vt[(r - 1) * W + c]) SETB(2, r, c);
        }
    for (int k = 0; k < cfg->n_offsets; ++k) {
        const int dy = cfg->offsets[2 * k], dx = cfg->offsets[2 * k + 1];
        const float *tc = cfg->tables + H + 5 * (H - 1) + (size_t)k * H;
        for (int r = dy; r < H; ++r)
            for (int c = 0; c < W; ++c) {
                const int ur = r - dy, uc = ((c - dx) % W + W) % W;
                if (PRES(r, c) && PRES(ur, uc) && pair_ok(rg[ur * W + uc], rg[r * W + c], tc[ur], cfg->d_max_sq))
                    SETB(3 + k, r, c);
            }
    }
#undef SETB
#undef PRES
}

typedef struct {
    const float *ranges; const oracle_cfg *cfg; uint32_t *planes; int B, tid, nthreads; int failed;
} planes_job;

static void *planes_worker(void *arg) {
    planes_job *j = (planes_job *)arg;
    const int H = j->cfg->height, W = j->cfg->width, WPR = (W + 31) / 32;
    const size_t HW = (size_t)H * W, pw = (size_t)(3 + j->cfg->n_offsets) * H * WPR;
    uint8_t *gm = malloc(HW), *hz = malloc(HW), *vt = malloc(HW);
    if (!gm || !hz || !vt) { j->failed = 1; free(gm); free(hz); free(vt); return NULL; }
    for (int f = j->tid; f < j->B; f += j->nthreads)
        oracle_frame_planes(j->ranges + f * HW, j->cfg, j->planes + f * pw, gm, hz, vt);
    free(gm); free(hz); free(vt);
    return NULL;
}

int oracle_planes_batch(const float *ranges, int B, const oracle_cfg *cfg, uint32_t *planes, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > B) nthreads = B > 0 ? B : 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    planes_job jobs[256];
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (planes_job){ranges, cfg, planes, B, t, nthreads, 0};
        if (nthreads == 1) planes_worker(&jobs[0]);
        else pthread_create(&th[t], NULL, planes_worker, &jobs[t]);
    }
    int failed = 0;
    for (int t = 0; t < nthreads; ++t) {
        if (nthreads > 1) pthread_join(th[t], NULL);
        failed |= jobs[t].failed;
    }
    return failed ? -1 : 0;
}
