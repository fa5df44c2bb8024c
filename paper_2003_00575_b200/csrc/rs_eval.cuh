// rs_eval.cuh — instance-scoring support on the GPU: the
// (ground-truth instance, predicted cluster) contingency table behind
// evaluation.match_instances (/root/reference/pkg/src/rangeseg/evaluation.py:65-129)
// for a batch of frames.
//
// The reference counts pairs with np.unique over packed (gt, pred) integers
// (:91-99) and gets the instance / cluster sizes from np.unique as well
// (:83-89).  Here every point with gt > 0 or pred > 0 becomes one 64-bit key
// (frame | gt | pred), the keys are radix-sorted and run-length encoded (CUB),
// giving per frame the sorted (gt, pred) pairs with their point counts —
// including the gt = 0 and pred = 0 pairs, so both size tables follow by
// summing rows and columns.  The per-instance matching over that (small)
// table is host code in paper_2003_00575_b200/evaluation.py.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace rs {

constexpr int kEvalThreads = 256;
constexpr int kEvalLabelBits = 22;    // gt ids and cluster labels < 2^22
constexpr int kEvalFrameBits = 19;    // frames < 2^19 (key < 2^63)
constexpr long long kEvalNone = 0x7fffffffffffffffLL;   // points with gt == pred == 0

__global__ void __launch_bounds__(kEvalThreads)
    rs_contingency_keys_kernel(const int32_t *gt, const int32_t *pred, const int64_t *offsets, int B, int64_t n,
                               long long *keys, int *bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int lo = 0, hi = B;   // frame of point i: offsets[lo] <= i < offsets[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(offsets + mid) <= i) lo = mid; else hi = mid;
    }
    const int g = gt[i], p = pred[i];
    if (g < 0 || p < 0 || g >= (1 << kEvalLabelBits) || p >= (1 << kEvalLabelBits)) atomicOr(bad, 1);
    keys[i] = (g > 0 || p > 0) ? (((long long)lo << (2 * kEvalLabelBits)) | ((long long)(g & ((1 << kEvalLabelBits) - 1))
                                                                              << kEvalLabelBits) |
                                  (long long)(p & ((1 << kEvalLabelBits) - 1)))
                               : kEvalNone;
}

}  // namespace rs
