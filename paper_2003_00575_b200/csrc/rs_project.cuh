// rs_project.cuh — point clouds <-> range images on the GPU:
// range_image.project (/root/reference/pkg/src/rangeseg/range_image.py:57-115)
// and labels_to_points (:130-141), for a batch of clouds concatenated in one
// float64 array with CSR offsets.
//
// Per point, in float64 with the reference's op order (no contraction):
// range, elevation = asin(clip(z / r)), nearest channel by binary search plus
// the reference's <= tie rule, the half-gap field-of-view gate, azimuth =
// atan2(y, x) (+2*pi when negative) and numpy's floor_divide bin.  A cell keeps
// the smallest range and, among equal ranges, the highest point index (the
// reference assigns in a stable descending-range order, :98-104):
//   1. atomicMin of the range's float64 bits per cell (positive doubles order
//      like their bit patterns),
//   2. atomicMax of the point index over the points that hit that minimum,
//   3. per cell: float32 range and int64 index, counts of filled cells.
// Scratch lives in the outputs themselves (the minimum in the point_index
// buffer, the index in the ranges buffer) until step 3 rewrites them.
//
// asin / atan2 are CUDA's double-precision functions; like numpy's vectorised
// float64 arcsin (which already differs from the C library's), they may differ
// in the last ulp, which changes a decision only for a point within ~1e-16
// relative of a channel midpoint, the field-of-view edge or a column edge
// (tests/golden.py unstable_cells).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/rangeseg_b200.h"

namespace rs {

constexpr int kProjThreads = 256;

struct ProjArgs {
    const double *pts;
    int32_t stride;
    const int64_t *offsets;   // [B + 1]
    int32_t B, H, W, desc;
    double step, gap_lo, gap_hi, two_pi;
    const double *asc;        // [H] ascending channel angles (radians)
    int64_t n_total;
    float *ranges;            // [B][H][W]; int32 point index scratch until step 3
    int64_t *point_index;     // [B][H][W]; float64 range bits scratch until step 3
    int64_t *counts;          // [B][2]
    int32_t *cell;            // [n_total] workspace: cell of each point from step 1, -1 = dropped
    unsigned long long *rbits;   // [n_total] workspace: float64 range bits of each point
};

// Adds `v` (0 or 1 per thread) to counts[2*b + slot]: one barrier-count and
// one global atomic per block when the whole block works on one cloud (the
// usual case; per-warp atomics on one hot counter serialise in L2), else per
// (warp, cloud).  Every thread of the block must call it.
__device__ __forceinline__ void count_add(int64_t *counts, int b, int slot, unsigned v) {
    __shared__ int sb_first, sb_last;
    if (threadIdx.x == 0) sb_first = b;
    if (threadIdx.x == blockDim.x - 1) sb_last = b;
    const int n = __syncthreads_count(v != 0u);   // also orders the two stores above
    if (sb_first == sb_last && sb_first >= 0) {
        if (threadIdx.x == 0 && n) atomicAdd(reinterpret_cast<unsigned long long *>(counts) + 2 * b + slot,
                                             (unsigned long long)n);
        return;
    }
    const unsigned lanes = __match_any_sync(0xffffffffu, b);
    const unsigned tot = __popc(__ballot_sync(0xffffffffu, v != 0u) & lanes);
    if (b >= 0 && (threadIdx.x & 31) == __ffs(lanes) - 1 && tot)
        atomicAdd(reinterpret_cast<unsigned long long *>(counts) + 2 * b + slot, (unsigned long long)tot);
}

// cloud of point i (offsets[b] <= i < offsets[b+1]) inside [lo, hi)
__device__ __forceinline__ int cloud_in(const int64_t *offsets, int64_t i, int lo, int hi) {
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(offsets + mid) <= i) lo = mid; else hi = mid;
    }
    return lo;
}

// Cloud of point i: the block's first and last points are located once (a
// block nearly always lies inside one cloud), every thread then searches only
// between them.  Every thread of the block must call it.
__device__ __forceinline__ int cloud_of_block(const ProjArgs &a, int64_t i) {
    __shared__ int s_lo, s_hi;
    const int64_t first = (int64_t)blockIdx.x * blockDim.x;
    if (threadIdx.x == 0) s_lo = cloud_in(a.offsets, first, 0, a.B);
    if (threadIdx.x == 32 % blockDim.x)
        s_hi = cloud_in(a.offsets, (first + blockDim.x < a.n_total ? first + blockDim.x : a.n_total) - 1, 0, a.B) + 1;
    __syncthreads();
    return cloud_in(a.offsets, i, s_lo, s_hi);
}

// numpy float64 floor_divide (npy_divmod's quotient) for a >= 0, b > 0: the
// integer k with x = k*y + fmod(x, y), i.e. the floor of the exact quotient.
// Fast path: t = x / y rounded is within an ulp of the exact quotient, so
// floor(t) is the answer unless t lies within 1e-9 of an integer; only those
// (a measure-zero set of azimuths at column edges) take numpy's exact steps.
__device__ __forceinline__ double py_floor_divide(double x, double y) {
    const double t = __ddiv_rn(x, y);
    const double ft = floor(t);
    if (__dsub_rn(t, ft) > 1e-9 && __dsub_rn(__dadd_rn(ft, 1.0), t) > 1e-9 && t < 4.0e6) return ft;
    const double mod = fmod(x, y);
    const double div = __ddiv_rn(__dsub_rn(x, mod), y);
    if (div == 0.0) return copysign(0.0, __ddiv_rn(x, y));
    double fl = floor(div);
    if (__dsub_rn(div, fl) > 0.5) fl = __dadd_rn(fl, 1.0);
    return fl;
}

// cell (index within the frame) of point i, or -1 when it is dropped; r = its range
__device__ __forceinline__ int64_t proj_cell(const ProjArgs &a, const double *p, double &r) {
    const double x = p[0], y = p[1], z = p[2];
    r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
    if (!(r > 0.0)) return -1;           // the origin, NaN coordinates: dropped (ok = r > 0)
    double q = __ddiv_rn(z, r);
    if (isnan(q)) return -1;             // np.clip keeps NaN, asin(NaN) fails the gate
    q = fmin(fmax(q, -1.0), 1.0);
    const double el = asin(q);
    const int H = a.H;
    int pos = 0, hi = H;            // searchsorted(asc, el, side="left")
    while (pos < hi) {
        const int mid = (pos + hi) >> 1;
        if (__ldg(a.asc + mid) < el) pos = mid + 1; else hi = mid;
    }
    const int lo_i = min(max(pos - 1, 0), H - 1), hi_i = min(max(pos, 0), H - 1);
    const double alo = __ldg(a.asc + lo_i), ahi = __ldg(a.asc + hi_i);
    const int nearest = fabs(__dsub_rn(el, alo)) <= fabs(__dsub_rn(ahi, el)) ? lo_i : hi_i;
    const double a0 = __ldg(a.asc), aH = __ldg(a.asc + H - 1);
    if (!(el >= __dsub_rn(a0, a.gap_lo) && el <= __dadd_rn(aH, a.gap_hi))) return -1;
    const int row = a.desc ? H - 1 - nearest : nearest;
    double az = atan2(y, x);
    if (az < 0.0) az = __dadd_rn(az, a.two_pi);
    long long c = (long long)py_floor_divide(az, a.step) % a.W;
    if (c < 0) c += a.W;
    return (int64_t)row * a.W + c;
}

__global__ void __launch_bounds__(kProjThreads) rs_project_min_kernel(const __grid_constant__ ProjArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int b = -1;
    int64_t cell = -1;
    const int bi = cloud_of_block(a, i);
    if (i < a.n_total) {
        b = bi;
        double r;
        cell = proj_cell(a, a.pts + i * a.stride, r);
        a.cell[i] = (int32_t)cell;
        a.rbits[i] = (unsigned long long)__double_as_longlong(r);
        if (cell >= 0)
            atomicMin(reinterpret_cast<unsigned long long *>(a.point_index) + (int64_t)b * a.H * a.W + cell,
                      (unsigned long long)__double_as_longlong(r));
    }
    count_add(a.counts, b, 0, cell >= 0 ? 1u : 0u);   // points in the field of view
}

__global__ void __launch_bounds__(kProjThreads) rs_project_index_kernel(const __grid_constant__ ProjArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int bi = cloud_of_block(a, i);
    if (i >= a.n_total) return;
    const int32_t cell = a.cell[i];
    if (cell < 0) return;
    const int b = bi;
    const int64_t q = (int64_t)b * a.H * a.W + cell;
    const unsigned long long m = reinterpret_cast<const unsigned long long *>(a.point_index)[q];
    if (m == a.rbits[i])
        atomicMax(reinterpret_cast<int *>(a.ranges) + q, (int)(i - __ldg(a.offsets + b)));
}

__global__ void __launch_bounds__(kProjThreads) rs_project_finish_kernel(const __grid_constant__ ProjArgs a) {
    const int64_t HW = (int64_t)a.H * a.W;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int b = -1;
    bool filled = false;
    if (p < (int64_t)a.B * HW) {
        b = (int)(p / HW);
        const int ix = reinterpret_cast<const int *>(a.ranges)[p];
        const unsigned long long m = reinterpret_cast<const unsigned long long *>(a.point_index)[p];
        filled = ix >= 0;
        a.ranges[p] = filled ? __double2float_rn(__longlong_as_double((long long)m)) : 0.f;
        a.point_index[p] = filled ? (int64_t)ix : (int64_t)-1;
    }
    count_add(a.counts, b, 1, filled ? 1u : 0u);
}

// counts[b] = (n_in, n_filled) -> (n_dropped, n_overwritten)
__global__ void rs_project_counts_kernel(const __grid_constant__ ProjArgs a) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= a.B) return;
    const int64_t n = __ldg(a.offsets + b + 1) - __ldg(a.offsets + b);
    const int64_t n_in = a.counts[2 * b], filled = a.counts[2 * b + 1];
    a.counts[2 * b] = n - n_in;
    a.counts[2 * b + 1] = n_in - filled;
}

__global__ void __launch_bounds__(kProjThreads)
    rs_labels_to_points_kernel(const int32_t *labels, const int64_t *point_index, const int64_t *offsets, int B,
                               int64_t HW, int32_t *out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= (int64_t)B * HW) return;
    const int64_t ix = point_index[p];
    if (ix >= 0) out[__ldg(offsets + p / HW) + ix] = labels[p];
}

}  // namespace rs
