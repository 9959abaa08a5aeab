// sbd_fit.h -- offline SBD fit (see sbd_fit.cpp).
#pragma once

#include <functional>
#include <vector>

namespace sbdgpu {

// Radial kernel on the unit annulus (kernels.hpp:17-25 RadialKernel).
struct FitKernel {
    std::function<double(double)> eval, deriv;
    double oscillation_freq = 0.0;
    bool laplace_rhs = false; // r G'(r) == 1: closed-form right-hand side
    // optional closed form of int_a^1 r G'(r) J1(rho r) dr (else adaptive GL)
    std::function<double(double rho, double a)> rhs_integral;
};

struct SbdFit {
    double a = 0.0;
    int P = 0;
    std::vector<double> coeffs, roots, norms;
    double constant_offset = 0.0, achieved_error = 0.0, radial_scale = 1.0;
    int bc = 0; // 0 Dirichlet, 1 Robin
    double H = 0.0;
};

SbdFit solve_sbd(const FitKernel& k, double a, double tol, int bc, double H, bool subtract_offset,
                 int device);

} // namespace sbdgpu
