// pruned_dft.h -- band- and support-pruned DFT passes (pruned_dft.cu).
#pragma once

#include <cstdint>

#include "sbd_internal.h"

namespace sbdgpu {

// false when n is not supported (then the caller keeps the cuFFT path)
bool make_pruned_pass(int n, int lo, int L, int rows, PrunedPass& p);
DevBuf<double2> make_twiddles(int n, cudaStream_t st);  // e^{+2 pi i q / n}, q < n
void launch_pruned_dft(const PrunedPass& p, const double2* in, double2* out, const double2* w,
                       cudaStream_t st);

} // namespace sbdgpu
