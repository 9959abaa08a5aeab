// pruned_dft.h -- band- and support-pruned DFT passes (pruned_dft.cu).
#pragma once

#include <cstdint>

#include "sbd_internal.h"

namespace sbdgpu {

// false when n is not supported (then the caller keeps the cuFFT path)
// forced: the last radix R3 (N = 256 R3), 0 = automatic
bool make_pruned_pass(int n, int lo, int L, int rows, int forced, PrunedPass& p);
// e^{+2 pi i q / n} (q < n) followed by e^{+2 pi i q / N} (q < N)
DevBuf<double2> make_twiddles(const PrunedPass& p, cudaStream_t st);
void launch_pruned_dft(const PrunedPass& p, const double2* in, double2* out, const double2* w,
                       cudaStream_t st);

} // namespace sbdgpu
