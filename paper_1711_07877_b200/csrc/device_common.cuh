// device_common.cuh -- device helpers shared by the apply kernels
// (kernels.cu) and the offline assembly kernels (assemble_kernels.cu).
#pragma once

#include "sbd_internal.h"

namespace sbdgpu {
namespace dev {


__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// kb_window_hat (nufft.cpp:34-45), arguments formed without FMA contraction so
// they round exactly like the reference's host code.
__device__ __forceinline__ double kb_hat(double beta, double w) {
    const double s2 = __dsub_rn(__dmul_rn(beta, beta), __dmul_rn(w, w));
    if (s2 > 1e-12) {
        const double s = sqrt(s2);
        return __ddiv_rn(2.0 * sinh(s), s);
    }
    if (s2 < -1e-12) {
        const double s = sqrt(-s2);
        return __ddiv_rn(2.0 * sin(s), s);
    }
    return __dmul_rn(2.0, __dadd_rn(1.0, __ddiv_rn(s2, 6.0)));
}

// Window taps at sub-cell offset u in [0,1): w[i] = phi((u - w/2 + i)/(w/2)).
template <int W>
__device__ __forceinline__ void kb_taps(double u, const WindowPoly& P, double (&wt)[W]) {
    const double v = 2.0 * u - 1.0;
    const double v2 = v * v;
#pragma unroll
    for (int i = 0; i < W / 2; ++i) {
        double e = P.e[i][kHorner - 1], o = P.o[i][kHorner - 1];
#pragma unroll
        for (int h = kHorner - 2; h >= 0; --h) {
            e = fma(e, v2, P.e[i][h]);
            o = fma(o, v2, P.o[i][h]);
        }
        wt[i] = fma(v, o, e);
        wt[W - 1 - i] = fma(-v, o, e);
    }
    if (W & 1) {
        constexpr int m = W / 2;
        double e = P.e[m][kHorner - 1];
#pragma unroll
        for (int h = kHorner - 2; h >= 0; --h) e = fma(e, v2, P.e[m][h]);
        wt[m] = e;
    }
}

// Same taps as kb_taps, handed to a sink f(i, w_i) as they are produced (keeps
// the register footprint small when the taps go straight to shared memory).
template <int W, typename F>
__device__ __forceinline__ void kb_taps_each(double u, const WindowPoly& P, F&& f) {
    const double v = 2.0 * u - 1.0;
    const double v2 = v * v;
#pragma unroll
    for (int i = 0; i < W / 2; ++i) {
        double e = P.e[i][kHorner - 1], o = P.o[i][kHorner - 1];
#pragma unroll
        for (int h = kHorner - 2; h >= 0; --h) {
            e = fma(e, v2, P.e[i][h]);
            o = fma(o, v2, P.o[i][h]);
        }
        f(i, fma(v, o, e));
        f(W - 1 - i, fma(-v, o, e));
    }
    if (W & 1) {
        constexpr int m = W / 2;
        double e = P.e[m][kHorner - 1];
#pragma unroll
        for (int h = kHorner - 2; h >= 0; --h) e = fma(e, v2, P.e[m][h]);
        f(m, e);
    }
}

// i mod n for i in [-n, 2n) without an integer division.
__device__ __forceinline__ int wrap_near(int i, int n) {
    i = i < 0 ? i + n : i;
    return i >= n ? i - n : i;
}

__device__ __forceinline__ int wrap_base(int i, int n) {
    int r = i % n;
    return r < 0 ? r + n : r;
}

} // namespace dev
} // namespace sbdgpu
