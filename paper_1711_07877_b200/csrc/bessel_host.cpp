// bessel_host.cpp -- host special functions for the offline assembly (the
// SBD fit and the Helmholtz close-correction values).
//
// Textbook formulas (Abramowitz & Stegun 9.1.10-9.1.13 power series, 9.2.5-9.2.10
// Hankel asymptotics), evaluated the way the reference does
// (/root/reference/proj/src/bessel.cpp:1-215): power series in long double below
// x = 12 and in __float128 on [12, 16) where cancellation eats ~log10 I0(x)
// digits, asymptotic expansion truncated at its smallest term from 16 on.
// Roots follow bessel_roots.cpp (bracketed Newton). Offline only: none of this
// runs inside apply().

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

#include "bessel_host.h"

namespace sbdgpu {

namespace {

constexpr long double kPiL = 3.141592653589793238462643383279502884L;
constexpr long double kEulerL = 0.577215664901532860606512090082402431L;
constexpr double kSeamLD = 12.0, kSeamQ = 16.0;

template <typename T>
T tabs(T v) {
    return v < T(0) ? -v : v;
}

// sum_m (-q)^m / (m! (m+nu)!), q = x^2/4  (nu = 0, 1)
template <typename T>
T j_series(double x, int nu) {
    const T q = T(x) * T(x) / T(4);
    T term = nu ? T(x) / T(2) : T(1);
    T sum = term;
    for (int m = 1; m < 300; ++m) {
        term *= -q / (T(m) * T(m + nu));
        sum += term;
        if (tabs(term) < T(1e-40) * (tabs(sum) + T(1e-300)) && m > x) break;
    }
    return sum;
}

// Y0 series part: sum_{m>=1} (-1)^{m+1} H_m q^m/(m!)^2
template <typename T>
T y0_part(double x) {
    const T q = T(x) * T(x) / T(4);
    T fact = T(1), h = T(0), sum = T(0);
    for (int m = 1; m < 300; ++m) {
        fact *= q / (T(m) * T(m));
        h += T(1) / T(m);
        const T term = ((m & 1) ? T(1) : T(-1)) * h * fact;
        sum += term;
        if (tabs(term) < T(1e-40) * (tabs(sum) + T(1e-300)) && m > x) break;
    }
    return sum;
}

// Y1 series part: sum_{k>=0} (-1)^k (H_k + H_{k+1}) (x/2)^{2k+1} / (k! (k+1)!)
template <typename T>
T y1_part(double x) {
    const T q = T(x) * T(x) / T(4);
    T fact = T(x) / T(2), hk = T(0), hk1 = T(1);
    T sum = fact * (hk + hk1);
    for (int k = 1; k < 300; ++k) {
        fact *= q / (T(k) * T(k + 1));
        hk += T(1) / T(k);
        hk1 += T(1) / T(k + 1);
        const T term = ((k & 1) ? T(-1) : T(1)) * (hk + hk1) * fact;
        sum += term;
        if (tabs(term) < T(1e-40) * (tabs(sum) + T(1e-300)) && k > x) break;
    }
    return sum;
}

// Hankel asymptotic amplitude series P, Q for order nu, truncated at the
// smallest term.
void hankel(int nu, long double x, long double& P, long double& Q) {
    const long double mu = 4.0L * nu * nu;
    long double s = 1.0L, prev = 1.0L;
    P = 1.0L;
    Q = 0.0L;
    for (int k = 1; k < 60; ++k) {
        const long double odd = 2.0L * k - 1.0L;
        s *= (mu - odd * odd) / (8.0L * k * x);
        if (tabs(s) >= prev) break;
        prev = tabs(s);
        switch (k & 3) {
            case 0: P += s; break;
            case 1: Q += s; break;
            case 2: P -= s; break;
            case 3: Q -= s; break;
        }
        if (prev < 1e-22L) break;
    }
}

double hankel_j(int nu, double x) {
    long double P, Q;
    hankel(nu, x, P, Q);
    const long double chi = (long double)x - (0.5L * nu + 0.25L) * kPiL;
    return (double)(sqrtl(2.0L / (kPiL * x)) * (P * cosl(chi) - Q * sinl(chi)));
}

double hankel_y(int nu, double x) {
    long double P, Q;
    hankel(nu, x, P, Q);
    const long double chi = (long double)x - (0.5L * nu + 0.25L) * kPiL;
    return (double)(sqrtl(2.0L / (kPiL * x)) * (P * sinl(chi) + Q * cosl(chi)));
}

template <typename F, typename DF>
double bracketed_newton(F f, DF df, double lo, double hi) {
    double flo = f(lo), fhi = f(hi);
    if (flo == 0.0) return lo;
    if (fhi == 0.0) return hi;
    if ((flo > 0) == (fhi > 0)) throw std::runtime_error("bracketed_newton: no sign change");
    double x = 0.5 * (lo + hi);
    for (int it = 0; it < 100; ++it) {
        const double fx = f(x);
        if (fx == 0.0) return x;
        if ((fx > 0) == (flo > 0)) {
            lo = x;
            flo = fx;
        } else {
            hi = x;
        }
        double xn = x - fx / df(x);
        if (!(xn > lo && xn < hi)) xn = 0.5 * (lo + hi);
        if (std::fabs(xn - x) < 1e-16 * (1.0 + std::fabs(x))) return xn;
        x = xn;
    }
    return x;
}

} // namespace

double bessel_j0(double x) {
    x = std::fabs(x);
    if (x < kSeamLD) return (double)j_series<long double>(x, 0);
    if (x < kSeamQ) return (double)j_series<__float128>(x, 0);
    return hankel_j(0, x);
}

double bessel_j1(double x) {
    const double s = x < 0 ? -1.0 : 1.0;
    x = std::fabs(x);
    if (x < kSeamLD) return s * (double)j_series<long double>(x, 1);
    if (x < kSeamQ) return s * (double)j_series<__float128>(x, 1);
    return s * hankel_j(1, x);
}

double bessel_y0(double x) {
    if (!(x > 0.0)) throw std::domain_error("bessel_y0: argument must be positive");
    if (x >= kSeamQ) return hankel_y(0, x);
    const long double lg = logl((long double)x / 2.0L) + kEulerL;
    long double j0, s;
    if (x < kSeamLD) {
        j0 = j_series<long double>(x, 0);
        s = y0_part<long double>(x);
    } else {
        j0 = (long double)j_series<__float128>(x, 0);
        s = (long double)y0_part<__float128>(x);
    }
    return (double)((2.0L / kPiL) * (lg * j0 + s));
}

double bessel_y1(double x) {
    if (!(x > 0.0)) throw std::domain_error("bessel_y1: argument must be positive");
    if (x >= kSeamQ) return hankel_y(1, x);
    const long double lg = logl((long double)x / 2.0L) + kEulerL;
    long double j1, s;
    if (x < kSeamLD) {
        j1 = j_series<long double>(x, 1);
        s = y1_part<long double>(x);
    } else {
        j1 = (long double)j_series<__float128>(x, 1);
        s = (long double)y1_part<__float128>(x);
    }
    return (double)((2.0L / kPiL) * lg * j1 - 2.0L / (kPiL * (long double)x) - s / kPiL);
}

// First P positive roots of J0 (bessel_roots.cpp:58-75 bracket).
std::vector<double> dirichlet_roots(int P) {
    std::vector<double> r;
    r.reserve(P);
    for (int p = 1; p <= P; ++p) {
        double lo = M_PI * (p - 0.25), hi = M_PI * (p - 0.125);
        lo -= 1e-12 * lo;
        hi += 1e-12 * hi;
        r.push_back(bracketed_newton([](double x) { return bessel_j0(x); },
                                     [](double x) { return -bessel_j1(x); }, lo, hi));
    }
    return r;
}

// Roots of H J0(r) - r J1(r) = 0 (bessel_roots.cpp:77-106).
std::vector<double> robin_roots(double H, int P) {
    if (H < 0.0) throw std::domain_error("robin_roots: H must be nonnegative");
    const auto f = [H](double r) { return H * bessel_j0(r) - r * bessel_j1(r); };
    const auto df = [H](double r) { return -H * bessel_j1(r) - r * bessel_j0(r); };
    std::vector<double> roots;
    roots.reserve(P);
    const double step = M_PI / 16.0;
    double lo = step * 1e-6, flo = f(lo), r = lo + step;
    while ((int)roots.size() < P) {
        const double fr = f(r);
        if (fr == 0.0)
            roots.push_back(r);
        else if ((fr > 0) != (flo > 0))
            roots.push_back(bracketed_newton(f, df, lo, r));
        lo = r;
        flo = fr;
        r += step;
    }
    return roots;
}

double first_y0_root() {
    static const double root = bracketed_newton([](double x) { return bessel_y0(x); },
                                                [](double x) { return -bessel_y1(x); }, 0.5, 1.5);
    return root;
}

// bessel_roots.cpp:126-149
double y0_root_above(double k) {
    if (!(k > 0.0)) throw std::domain_error("y0_root_above: k must be positive");
    const auto f = [](double x) { return bessel_y0(x); };
    const auto df = [](double x) { return -bessel_y1(x); };
    const double first = first_y0_root();
    if (k <= first) return first;
    double lo = k, flo = f(lo);
    if (flo == 0.0) return lo;
    const double step = M_PI / 4.0;
    for (int it = 0; it < 10000; ++it) {
        const double hi = lo + step, fhi = f(hi);
        if (fhi == 0.0) return hi;
        if ((fhi > 0) != (flo > 0)) return std::max(bracketed_newton(f, df, lo, hi), k);
        lo = hi;
        flo = fhi;
    }
    throw std::runtime_error("y0_root_above: scan failed");
}

} // namespace sbdgpu
