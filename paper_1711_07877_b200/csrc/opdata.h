// opdata.h -- host mirror of the reference CompressedOperator::Impl state
// (/root/reference/proj/src/conv_operator.cpp:135-160), i.e. everything the
// SBDOPv1 file carries (conv_operator.cpp:357-447).
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/sbd_b200.h"

namespace sbdgpu {

// SBD record (conv_operator.cpp:383-395), carried through save/load.
struct SbdRecord {
    double a = 0.0;
    int32_t P = 0;
    double constant_offset = 0.0, achieved_error = 0.0, radial_scale = 1.0;
    int32_t bc = 0;
    double H = 0.0;
    std::vector<double> coeffs, roots, norm_constants;
};

// Host-side mirror of CompressedOperator::Impl's persistent state.
struct OpData {
    int32_t kind = 0;
    double k = 0.0;
    bool single = true;
    double eps = 0, alpha = 0, a = 0, dmin = 0, dmax = 0, nufft_tol = 0;
    std::vector<double> src, tgt; // xy
    double src_diam = 0.0, tgt_diam = 0.0;
    std::vector<double> freqs, weights; // xy, complex (file order)
    std::vector<int32_t> ring_offsets;
    double total_error_budget = 0.0;
    std::vector<uint64_t> row_offsets;
    std::vector<uint32_t> cols;
    std::vector<double> values; // complex
    SbdRecord sbd;
    uint64_t direct_threshold = uint64_t(1) << 20;
    uint64_t max_grid_bytes = uint64_t(4) << 30;

    uint64_t n_src() const { return src.size() / 2; }
    uint64_t n_tgt() const { return single ? n_src() : tgt.size() / 2; }
    uint64_t n_xi() const { return freqs.size() / 2; }
    uint64_t nnz() const { return cols.size(); }
};

// Offline assembly (assemble.cpp): fills an OpData from clouds + options,
// following CompressedOperator::assemble (conv_operator.cpp:244-294).
void assemble_opdata(int kind, double k, const double* src_xy, uint64_t n_src, const double* tgt_xy,
                     uint64_t n_tgt, const sbd_assemble_options& o, OpData& d);

} // namespace sbdgpu
