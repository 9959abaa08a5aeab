// bessel_host.h -- host special functions used by the offline assembly.
#pragma once

#include <vector>

namespace sbdgpu {

double bessel_j0(double x);
double bessel_j1(double x);
double bessel_y0(double x); // x > 0
double bessel_y1(double x); // x > 0
std::vector<double> dirichlet_roots(int P);
std::vector<double> robin_roots(double H, int P);
double first_y0_root();
double y0_root_above(double k);

} // namespace sbdgpu
