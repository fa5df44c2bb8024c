// torch_ext.cpp — the thin PyTorch C++ extension over the C ABI
// (include/rangeseg_b200.h): tensors in, the library's entry points called on
// the current CUDA stream with the GIL released.  It adds no kernels; the work
// is librangeseg_b200.so's (linked, found next to this module).
//
// rs_config stays a plain C struct: Python passes the address of its ctypes
// copy (paper_2003_00575_b200._native.RsConfig), so the extension and the
// ctypes binding share one definition of the ABI.
#include <torch/extension.h>

#include <ATen/cuda/CUDAContext.h>
#include <c10/cuda/CUDAGuard.h>

#include <string>

#include "rangeseg_b200.h"

namespace {

void check(int st, const char *what) {
    if (st == RS_OK) return;
    const std::string msg = std::string(what) + ": " + rs_last_error();
    if (st == RS_EINVAL || st == RS_ETOOLARGE) throw std::invalid_argument(msg);   // -> ValueError
    throw std::runtime_error(msg);
}

const rs_config *cfg_of(int64_t addr) { return reinterpret_cast<const rs_config *>(static_cast<uintptr_t>(addr)); }

// rs_segment_batch on tensors: ranges float32 [B, H, W]; labels int32 [B, H, W],
// n_clusters int32 [B], cluster_sizes int64 [B, stride] or an empty tensor.
void segment_batch(int64_t cfg_addr, const at::Tensor &tables, const at::Tensor &ranges, at::Tensor &labels,
                   at::Tensor &n_clusters, at::Tensor &cluster_sizes) {
    TORCH_CHECK(ranges.is_cuda() && ranges.scalar_type() == at::kFloat && ranges.dim() == 3 &&
                    ranges.is_contiguous(), "ranges must be a contiguous float32 CUDA tensor [B, H, W]");
    TORCH_CHECK(labels.scalar_type() == at::kInt && labels.is_contiguous() && labels.sizes() == ranges.sizes(),
                "labels must be a contiguous int32 tensor shaped like ranges");
    TORCH_CHECK(n_clusters.scalar_type() == at::kInt && n_clusters.numel() == ranges.size(0),
                "n_clusters must be int32 [B]");
    const bool sizes = cluster_sizes.numel() > 0;
    TORCH_CHECK(!sizes || (cluster_sizes.scalar_type() == at::kLong && cluster_sizes.dim() == 2 &&
                           cluster_sizes.is_contiguous() && cluster_sizes.size(0) == ranges.size(0)),
                "cluster_sizes must be int64 [B, stride]");
    TORCH_CHECK(tables.device() == ranges.device() && labels.device() == ranges.device() &&
                    n_clusters.device() == ranges.device() && (!sizes || cluster_sizes.device() == ranges.device()),
                "all tensors must be on the ranges' device");
    TORCH_CHECK(tables.scalar_type() == at::kFloat && tables.is_contiguous(), "tables must be contiguous float32");
    const c10::cuda::CUDAGuard guard(ranges.device());
    cudaStream_t stream = at::cuda::getCurrentCUDAStream(ranges.device().index()).stream();
    int st;
    {
        pybind11::gil_scoped_release nogil;
        st = rs_segment_batch(cfg_of(cfg_addr), tables.data_ptr<float>(), ranges.data_ptr<float>(),
                              (int32_t)ranges.size(0), labels.data_ptr<int32_t>(), n_clusters.data_ptr<int32_t>(),
                              sizes ? cluster_sizes.data_ptr<int64_t>() : nullptr,
                              sizes ? cluster_sizes.size(1) : 0, stream);
    }
    check(st, "rs_segment_batch");
}

int64_t abi_version() { return rs_version(); }

}  // namespace

PYBIND11_MODULE(TORCH_EXTENSION_NAME, m) {
    m.doc() = "thin PyTorch binding of librangeseg_b200 (C ABI: include/rangeseg_b200.h)";
    m.def("segment_batch", &segment_batch, "rs_segment_batch on the current CUDA stream (GIL released)");
    m.def("abi_version", &abi_version);
}
