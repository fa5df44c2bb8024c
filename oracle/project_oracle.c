/*
 * project_oracle.c — CPU restatement of the reference's point-cloud
 * projection and label back-projection.
 *
 * TEST INFRASTRUCTURE ONLY (same rules as rangeseg_oracle.c): only tests/,
 * __graft_entry__.smoke() and bench.py's baseline legs may load it; the
 * product path never does.
 *
 * Restated from /root/reference/pkg/src/rangeseg/range_image.py:
 *   project            :57-115  float64 throughout; nearest channel by
 *                               elevation (searchsorted + the <= tie rule),
 *                               half-gap FOV gate, floor azimuth bin, the
 *                               smallest range wins a cell and equal ranges go
 *                               to the highest point index (assignment in a
 *                               stable descending-range order, :98-104)
 *   labels_to_points   :130-141
 * numpy's float floor_divide (npy_divmod) is restated in py_floor_divide;
 * asin / atan2 come from the C library, as numpy's do.
 *
 * Pinned against the reference itself: tests/golden/make_golden_project.py
 * records the reference's outputs; tests/test_oracle_golden.py checks this
 * file bit for bit against them.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct {
    int32_t height, width;
    int32_t descending;        /* channel_angles[0] > channel_angles[-1] */
    double azimuth_step;       /* radians (sensor.py:83) */
    const double *asc;         /* channel angles in ascending order, radians, [height] */
} oracle_proj_cfg;

/* numpy float64 floor_divide: npy_divmod's quotient */
static double py_floor_divide(double a, double b) {
    double mod = fmod(a, b);
    if (b == 0.0) return a / b;
    double div = (a - mod) / b;
    if (mod != 0.0) {
        if ((b < 0) != (mod < 0)) div -= 1.0;
    }
    double fl;
    if (div != 0.0) {
        fl = floor(div);
        if (div - fl > 0.5) fl += 1.0;
    } else {
        fl = copysign(0.0, a / b);
    }
    return fl;
}

/* row / column / range of one point; returns 0 when the point is dropped */
static int cell_of(const double *p, const oracle_proj_cfg *c, int32_t *row, int32_t *col, double *rng) {
    const double x = p[0], y = p[1], z = p[2];
    const double r = sqrt((x * x + y * y) + z * z);
    *rng = r;
    const int ok = r > 0;
    double q = ok ? z / r : 0.0;
    if (q < -1.0) q = -1.0;
    if (q > 1.0) q = 1.0;
    const double elev = asin(q);
    const int H = c->height;
    const double *asc = c->asc;
    int pos = 0;                       /* searchsorted(asc, elev, side="left") */
    while (pos < H && asc[pos] < elev) ++pos;
    const int lo = pos - 1 < 0 ? 0 : (pos - 1 > H - 1 ? H - 1 : pos - 1);
    const int hi = pos < 0 ? 0 : (pos > H - 1 ? H - 1 : pos);
    const int nearest = fabs(elev - asc[lo]) <= fabs(asc[hi] - elev) ? lo : hi;
    const double gap_lo = (asc[1] - asc[0]) / 2.0, gap_hi = (asc[H - 1] - asc[H - 2]) / 2.0;
    const int in_fov = ok && (elev >= asc[0] - gap_lo) && (elev <= asc[H - 1] + gap_hi);
    if (!in_fov) return 0;
    *row = c->descending ? H - 1 - nearest : nearest;
    double az = atan2(y, x);
    if (az < 0) az += 2.0 * 3.141592653589793;
    int64_t cc = (int64_t)py_floor_divide(az, c->azimuth_step) % c->width;
    if (cc < 0) cc += c->width;
    *col = (int32_t)cc;
    return 1;
}

/* points: float64 [n][stride] (x, y, z first).  Outputs: ranges float32
 * [H*W], point_index int64 [H*W] (-1 empty), counts[0] = n_dropped,
 * counts[1] = n_overwritten. */
int oracle_project(const double *pts, int64_t n, int32_t stride, const oracle_proj_cfg *c,
                   float *ranges, int64_t *point_index, int64_t *counts) {
    const int64_t HW = (int64_t)c->height * c->width;
    double *best = malloc(sizeof(double) * (size_t)HW);
    if (!best) return -1;
    for (int64_t p = 0; p < HW; ++p) { point_index[p] = -1; ranges[p] = 0.0f; }
    int64_t n_in = 0;
    for (int64_t i = 0; i < n; ++i) {
        int32_t row, col;
        double r;
        if (!cell_of(pts + i * stride, c, &row, &col, &r)) continue;
        ++n_in;
        const int64_t p = (int64_t)row * c->width + col;
        if (point_index[p] < 0 || r < best[p] || (r == best[p] && i > point_index[p])) {
            best[p] = r;
            point_index[p] = i;
        }
    }
    int64_t filled = 0;
    for (int64_t p = 0; p < HW; ++p)
        if (point_index[p] >= 0) { ranges[p] = (float)best[p]; ++filled; }
    counts[0] = n - n_in;
    counts[1] = n_in - filled;
    free(best);
    return 0;
}

void oracle_labels_to_points(const int32_t *labels, const int64_t *point_index, int64_t hw, int64_t n,
                             int32_t *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = 0;
    for (int64_t p = 0; p < hw; ++p)
        if (point_index[p] >= 0) out[point_index[p]] = labels[p];
}
