// assemble_gpu.h -- device part of the offline assembly (assemble_kernels.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "sbd_internal.h"

namespace sbdgpu {

struct CloseMatrixInput {
    const double* src_xy = nullptr;
    uint64_t n_src = 0;
    const double* tgt_xy = nullptr;
    uint64_t n_tgt = 0;
    bool single = true;
    double radius = 0.0;
    const double* xi_xy = nullptr; // physical frequencies
    const double* w = nullptr;     // weights (complex)
    uint64_t n_xi = 0;
    double wsum_re = 0.0, wsum_im = 0.0;
    double nufft_tol = 1e-9;
    uint64_t direct_threshold = uint64_t(1) << 20;
    uint64_t max_grid_bytes = uint64_t(4) << 30;
    bool laplace = true; // device adds log r; otherwise the host adds G(r)
    int device = 0;
};

struct CloseMatrixOutput {
    std::vector<uint64_t> row_offsets;
    std::vector<uint32_t> cols;
    std::vector<double> values; // complex; = G - far if laplace_done else -far
    bool laplace_done = false;
};

void build_close_matrix_gpu(const CloseMatrixInput& in, CloseMatrixOutput& out);

// Exact cloud diameter (assemble.cpp).
double cloud_diameter(const double* xy, uint64_t n);

} // namespace sbdgpu
