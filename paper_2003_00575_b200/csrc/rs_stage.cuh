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

}  // namespace rs
