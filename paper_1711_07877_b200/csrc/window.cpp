// window.cpp -- host-side construction of the Kaiser-Bessel window polynomials
// evaluated by the sm_100a spread/interp kernels, plus the scalar plan helpers
// restated from the reference NUFFT.
//
// The reference evaluates phi(z) = I0(beta sqrt(1-z^2)) with a ~50-term power
// series per tap (nufft.cpp:28-32, bessel.cpp:216-227), i.e. 2w series per
// point. Here each tap i is a degree-15 polynomial in v = 2u - 1, u = ix0 - t +
// w/2 in [0,1) (exact in fp64, see kernels.cu), fitted once per plan by
// Chebyshev interpolation in long double. Evenness of phi lets taps i and
// w-1-i share one even/odd split, so a point costs ~8 FMAs per tap.
#include <cmath>
#include <cstring>

#include "sbd_internal.h"

namespace sbdgpu {

namespace {

long double i0l(long double r) {
    const long double q = 0.25L * r * r;
    long double term = 1.0L, sum = 1.0L;
    for (int m = 1; m < 400; ++m) {
        term *= q / ((long double)m * (long double)m);
        sum += term;
        if (term < 1e-22L * sum) break;
    }
    return sum;
}

long double phil(long double beta, long double z) {
    const long double s = 1.0L - z * z;
    if (s <= 0.0L) return s == 0.0L ? 1.0L : 0.0L;
    return i0l(beta * sqrtl(s));
}

} // namespace

double kb_window_host(double beta, double z) { return (double)phil(beta, z); }

// nufft.cpp:34-45
double kb_window_hat_host(double beta, double w) {
    const double s2 = beta * beta - w * w;
    if (s2 > 1e-12) {
        const double s = std::sqrt(s2);
        return 2.0 * std::sinh(s) / s;
    }
    if (s2 < -1e-12) {
        const double s = std::sqrt(-s2);
        return 2.0 * std::sin(s) / s;
    }
    return 2.0 * (1.0 + s2 / 6.0);
}

// nufft.cpp:47-52
int width_for_tol(double tol) {
    const double digits = -std::log10(std::max(tol, 1e-15));
    const int w = (int)std::ceil(digits) + 2;
    return w < 4 ? 4 : (w > 17 ? 17 : w);
}

// nufft.cpp:55-63
int next_fast_even(int n) {
    n += n & 1;
    for (;; n += 2) {
        int m = n;
        for (int f : {2, 3, 5})
            while (m % f == 0) m /= f;
        if (m == 1) return n;
    }
}

WindowPoly fit_window(int w, double beta, double* max_rel_err) {
    constexpr int D = 2 * kHorner - 1; // degree 15
    constexpr int M = D + 1;           // Chebyshev nodes
    const long double half = 0.5L * w;
    const long double pi = 3.141592653589793238462643383279502884L;
    WindowPoly out;
    std::memset(&out, 0, sizeof(out));
    long double nodes[M];
    for (int k = 0; k < M; ++k) nodes[k] = cosl(pi * (k + 0.5L) / M);

    const int pairs = (w + 1) / 2;
    for (int i = 0; i < pairs; ++i) {
        long double f[M];
        for (int k = 0; k < M; ++k)
            f[k] = phil(beta, (0.5L * (nodes[k] + 1.0L) - half + i) / half);
        // Chebyshev coefficients a_j of the interpolant.
        long double a[M];
        for (int j = 0; j < M; ++j) {
            long double s = 0.0L;
            for (int k = 0; k < M; ++k) s += f[k] * cosl(pi * j * (k + 0.5L) / M);
            a[j] = s * 2.0L / M;
        }
        a[0] *= 0.5L;
        // Chebyshev -> monomial in v: T_{j+1} = 2 v T_j - T_{j-1}.
        long double c[M] = {0}, Tm[M] = {0}, T0[M] = {0}, T1[M] = {0};
        T0[0] = 1.0L;
        T1[1] = 1.0L;
        for (int k = 0; k < M; ++k) c[k] += a[0] * T0[k];
        for (int k = 0; k < M; ++k) c[k] += a[1] * T1[k];
        for (int j = 2; j < M; ++j) {
            for (int k = 0; k < M; ++k) Tm[k] = -T0[k] + (k > 0 ? 2.0L * T1[k - 1] : 0.0L);
            for (int k = 0; k < M; ++k) c[k] += a[j] * Tm[k];
            std::memcpy(T0, T1, sizeof(T0));
            std::memcpy(T1, Tm, sizeof(T1));
        }
        for (int k = 0; k < kHorner; ++k) {
            out.e[i][k] = (double)c[2 * k];
            out.o[i][k] = (w % 2 == 1 && i == w / 2) ? 0.0 : (double)c[2 * k + 1];
        }
    }

    if (max_rel_err) {
        // Sup-norm check over all taps against the exact window, relative to
        // its peak I0(beta).
        const long double peak = i0l(beta);
        long double worst = 0.0L;
        for (int i = 0; i < w; ++i) {
            const int pi_ = i < pairs ? i : w - 1 - i;
            const double sg = i < pairs ? 1.0 : -1.0;
            for (int k = 0; k <= 200; ++k) {
                const double v = -1.0 + 2.0 * k / 200.0;
                const double v2 = v * v;
                double e = out.e[pi_][kHorner - 1], o = out.o[pi_][kHorner - 1];
                for (int h = kHorner - 2; h >= 0; --h) {
                    e = e * v2 + out.e[pi_][h];
                    o = o * v2 + out.o[pi_][h];
                }
                const double p = e + sg * v * o;
                const long double ex = phil(beta, (0.5L * (v + 1.0L) - half + i) / half);
                const long double err = fabsl((long double)p - ex) / peak;
                if (err > worst) worst = err;
            }
        }
        *max_rel_err = (double)worst;
    }
    return out;
}

} // namespace sbdgpu
