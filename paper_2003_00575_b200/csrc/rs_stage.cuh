// rs_stage.cuh — per-cell ground mask and edge images (parity checks of the
// float32 decisions against extract_ground / build_connectivity).
#pragma once

#include "rs_common.cuh"

namespace rs {

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

// height_image (range_image.py:118-127): z = f32(r * sin_ch[row]) + f32(mount),
// NaN where there is no return.
__global__ void rs_height_kernel(const __grid_constant__ KArgs a, float *z, long long total) {
    const long long HW = (long long)a.H * a.W;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int r = (int)((idx % HW) / a.W);
        const float v = __ldg(a.ranges + idx);
        z[idx] = v > 0.f ? __fadd_rn(__fmul_rn(v, __ldg(a.tables + r)), a.mount) : __int_as_float(0x7fc00000);
    }
}

// extract_ground (ground.py:95-141) with the caller's height image: mask =
// no return, or slope within the window of pair (max(r,1)-1, max(r,1)) and
// height <= keep_above.  NaN heights compare false, like the reference.
__global__ void rs_ground_kernel(const __grid_constant__ KArgs a, const float *height, uint8_t *mask,
                                 long long total) {
    const int H = a.H, W = a.W;
    const long long HW = (long long)H * W;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long f = idx / HW;
        const int i = (int)(idx - f * HW);
        const int r = i / W, c = i - r * W;
        const float *fr = a.ranges + f * HW;
        const float v = __ldg(fr + i);
        bool g = !(v > 0.f);
        if (!g && a.ground) {
            const int kk = (r >= 1 ? r : 1) - 1;
            const GroundRow gr = ground_row(a, r);
            const float d1 = __ldg(fr + (size_t)kk * W + c), d2 = __ldg(fr + (size_t)(kk + 1) * W + c);
            const float num = __fmul_rn(d2, gr.sa);
            const float den = __fsub_rn(d1, __fmul_rn(d2, gr.ca));
            const float L = __fmul_rn(gr.lo, den), U = __fmul_rn(gr.hi, den);
            const bool ok = (den > 0.f ? (num >= L && num <= U) : (num <= L && num >= U)) && den != 0.f &&
                            d1 > 0.f && d2 > 0.f;
            g = ok && __ldg(height + idx) <= a.keep_above;
        }
        mask[idx] = (uint8_t)g;
    }
}

// build_connectivity (connectivity.py:64-92) with the caller's ground mask:
// present = r > 0 and not masked; horizontal to (c+1) mod W, vertical to r+1.
__global__ void rs_connectivity_kernel(const __grid_constant__ KArgs a, const uint8_t *mask, uint8_t *horiz,
                                       uint8_t *vert, long long total) {
    const int H = a.H, W = a.W;
    const long long HW = (long long)H * W;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long f = idx / HW;
        const int i = (int)(idx - f * HW);
        const int r = i / W, c = i - r * W;
        const float *fr = a.ranges + f * HW;
        const uint8_t *mf = mask + f * HW;
        auto present = [&](int j) { return __ldg(fr + j) > 0.f && !mf[j]; };
        const float v = __ldg(fr + i);
        const bool p = present(i);
        bool h = false;
        if (W > 1) {
            const int j = r * W + (c + 1 < W ? c + 1 : 0);
            h = p && present(j) && pair_pass(v, __ldg(fr + j), a.tch, a.dmax2);
        }
        horiz[idx] = (uint8_t)h;
        if (r < H - 1) {
            const int j = i + W;
            vert[f * (HW - W) + i] = (uint8_t)(p && present(j) &&
                                             pair_pass(v, __ldg(fr + j), __ldg(a.tables + 5 * H - 4 + r), a.dmax2));
        }
    }
}

}  // namespace rs
