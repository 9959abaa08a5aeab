// sbd_fit.cpp -- offline Sparse Bessel Decomposition fit (the radial Bessel
// series of the kernel on the annulus a < r < 1), following the reference's
// algorithm: closed-form Gram matrix of the normalised J0 basis
// (gram.cpp:25-67), right-hand side b_p = -2 pi C_p rho_p int_a^1 r G'(r)
// J1(rho_p r) dr (gram.cpp:69-84), Cholesky of the Gram at the search cap and
// leading-block solves for each probe, validation L-inf error on a 2048-point
// geometric grid (sbd.cpp:32-130), and the bracket-then-dichotomy search for
// the smallest order P meeting tol (sbd.cpp:148-204).
//
// B200-specific: the cap x cap Gram factorisation runs on the GPU
// (cusolverDnDpotrf, fp64); Bessel tables and integrals are OpenMP-parallel on
// the host. Offline only -- "reported but not optimised" (north_star).
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <functional>
#include <numeric>

#include "bessel_host.h"
#include "sbd_fit.h"
#include "sbd_internal.h"

namespace sbdgpu {

namespace {

constexpr double kPi = 3.14159265358979323846;

struct GL16 {
    double x[16], w[16];
    GL16() {
        const int n = 16;
        for (int i = 0; i < n; ++i) {
            double z = std::cos(kPi * (i + 0.75) / (n + 0.5)), pp = 0.0;
            for (int it = 0; it < 100; ++it) {
                double p0 = 1.0, p1 = z;
                for (int k = 2; k <= n; ++k) {
                    const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
                    p0 = p1;
                    p1 = p2;
                }
                pp = n * (z * p1 - p0) / (z * z - 1.0);
                const double dz = p1 / pp;
                z -= dz;
                if (std::fabs(dz) < 1e-16) break;
            }
            x[i] = z;
            w[i] = 2.0 / ((1.0 - z * z) * pp * pp);
        }
    }
};

const GL16& gl16() {
    static const GL16 g;
    return g;
}

double gl_panels(const std::function<double(double)>& f, double a, double b, int panels) {
    const GL16& g = gl16();
    const double h = (b - a) / panels;
    double total = 0.0;
    for (int p = 0; p < panels; ++p) {
        const double c = a + (p + 0.5) * h;
        double s = 0.0;
        for (int i = 0; i < 16; ++i) s += g.w[i] * f(c + 0.5 * h * g.x[i]);
        total += 0.5 * h * s;
    }
    return total;
}

// Panel-doubling Gauss-Legendre to relative rel_tol (quadrature.cpp:55-74).
double integrate(const std::function<double(double)>& f, double a, double b, double rel_tol,
                 int panels0) {
    int n = panels0;
    double prev = gl_panels(f, a, b, n);
    for (int it = 0; it < 14; ++it) {
        n *= 2;
        const double cur = gl_panels(f, a, b, n);
        const double scale = std::max({std::fabs(cur), std::fabs(prev), 1e-300});
        if (std::fabs(cur - prev) <= rel_tol * scale) return cur;
        prev = cur;
    }
    return prev;
}

struct Basis {
    std::vector<double> roots, norms;
};

// basis.cpp:21-52: Dirichlet C_p = 1/(sqrt(pi) rho |J1(rho)|); Robin from the
// mode energy pi[rho^2 (J0^2 + J1^2) - 2 rho J0 J1] + 2 pi H J0^2.
Basis make_basis(int bc, double H, int P) {
    Basis b;
    b.roots = bc == 0 ? dirichlet_roots(P) : robin_roots(H, P);
    b.norms.resize(P);
#pragma omp parallel for schedule(dynamic, 64)
    for (int p = 0; p < P; ++p) {
        const double rho = b.roots[p];
        if (bc == 0) {
            b.norms[p] = 1.0 / (std::sqrt(kPi) * rho * std::fabs(bessel_j1(rho)));
        } else {
            const double j0 = bessel_j0(rho), j1 = bessel_j1(rho);
            const double e = kPi * (rho * rho * (j0 * j0 + j1 * j1) - 2.0 * rho * j0 * j1) +
                             2.0 * kPi * H * j0 * j0;
            b.norms[p] = 1.0 / std::sqrt(e);
        }
    }
    return b;
}

// gram.cpp:25-67: A_ij = int_A grad e_i . grad e_j (+ H boundary term),
// closed form via Lommel's integral. Column-major P x P.
std::vector<double> assemble_gram(const Basis& b, double a, double H) {
    const int P = (int)b.roots.size();
    std::vector<double> j0a(P), j1a(P), j01(P), j11(P);
#pragma omp parallel for schedule(dynamic, 64)
    for (int i = 0; i < P; ++i) {
        const double r = b.roots[i];
        j0a[i] = bessel_j0(r * a);
        j1a[i] = bessel_j1(r * a);
        j01[i] = bessel_j0(r);
        j11[i] = bessel_j1(r);
    }
    auto diag_term = [](double rho, double r, double j0, double j1) {
        return 0.5 * rho * rho * r * r * (j0 * j0 + j1 * j1) - rho * r * j0 * j1;
    };
    std::vector<double> g((size_t)P * P);
#pragma omp parallel for schedule(dynamic, 16)
    for (int i = 0; i < P; ++i) {
        const double ri = b.roots[i], ci = b.norms[i];
        g[(size_t)i * P + i] =
            2.0 * kPi * ci * ci * (diag_term(ri, 1.0, j01[i], j11[i]) - diag_term(ri, a, j0a[i], j1a[i])) +
            2.0 * kPi * H * ci * ci * j01[i] * j01[i];
        for (int j = i + 1; j < P; ++j) {
            const double rj = b.roots[j], cj = b.norms[j];
            const double denom = ri * ri - rj * rj;
            const double fij1 = -ri * j01[i] * j11[j];
            const double fji1 = -rj * j01[j] * j11[i];
            const double fija = -ri * a * j0a[i] * j1a[j];
            const double fjia = -rj * a * j0a[j] * j1a[i];
            double v = 2.0 * kPi * ci * cj * ri * rj / denom * (fij1 - fji1 - fija + fjia);
            v += 2.0 * kPi * H * ci * cj * j01[i] * j01[j];
            g[(size_t)i * P + j] = v;
            g[(size_t)j * P + i] = v;
        }
    }
    return g;
}

// Lower Cholesky of the P x P column-major matrix on the GPU. Returns false
// when a pivot is not positive (the reference then falls back to LDLT).
bool gpu_cholesky(std::vector<double>& a, int P, int device) {
    cusolverDnHandle_t h = nullptr;
    if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) throw Error(4, "cusolverDnCreate failed");
    ck(cudaSetDevice(device), "cudaSetDevice");
    DevBuf<double> d((size_t)P * P);
    ck(cudaMemcpy(d.p, a.data(), a.size() * 8, cudaMemcpyHostToDevice), "gram H2D");
    int lwork = 0;
    cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, P, d.p, P, &lwork);
    DevBuf<double> work(std::max(lwork, 1));
    DevBuf<int> info(1);
    const cusolverStatus_t st =
        cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, P, d.p, P, work.p, lwork, info.p);
    int hinfo = 0;
    ck(cudaMemcpy(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost), "potrf info");
    ck(cudaMemcpy(a.data(), d.p, a.size() * 8, cudaMemcpyDeviceToHost), "L D2H");
    cusolverDnDestroy(h);
    if (st != CUSOLVER_STATUS_SUCCESS) throw Error(4, "cusolverDnDpotrf failed");
    return hinfo == 0;
}

// Dense LU with partial pivoting (fallback when the Gram loses definiteness).
std::vector<double> lu_solve(std::vector<double> A, int n, std::vector<double> b) {
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (std::fabs(A[(size_t)k * n + i]) > std::fabs(A[(size_t)k * n + p])) p = i;
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < n; ++j) std::swap(A[(size_t)j * n + k], A[(size_t)j * n + p]);
        std::swap(b[k], b[p]);
        const double d = A[(size_t)k * n + k];
        if (d == 0.0) throw Error(3, "solve_sbd: Gram factorization failed (conditioning)");
        for (int i = k + 1; i < n; ++i) A[(size_t)k * n + i] /= d;
        for (int j = k + 1; j < n; ++j) {
            const double akj = A[(size_t)j * n + k];
            if (akj == 0.0) continue;
            for (int i = k + 1; i < n; ++i) A[(size_t)j * n + i] -= A[(size_t)k * n + i] * akj;
        }
        for (int i = k + 1; i < n; ++i) b[i] -= A[(size_t)k * n + i] * b[k];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = b[i];
        for (int j = i + 1; j < n; ++j) s -= A[(size_t)j * n + i] * b[j];
        b[i] = s / A[(size_t)i * n + i];
    }
    return b;
}

class Workspace {
  public:
    Workspace(const FitKernel& k, double a, int bc, double H, bool subtract_offset, int device)
        : k_(k), a_(a), bc_(bc), H_(H), device_(device) {
        offset_ = subtract_offset ? k.eval(1.0) : 0.0;
        grid_.resize(kValidation);
        target_.resize(kValidation);
        for (int i = 0; i < kValidation; ++i) {
            grid_[i] = a * std::pow(1.0 / a, (double)i / (kValidation - 1));
            target_[i] = k.eval(grid_[i]) - offset_;
        }
    }

    void ensure(int P) {
        if (P <= cap_) return;
        const auto t0 = std::chrono::steady_clock::now();
        const int old = cap_;
        cap_ = P;
        basis_ = make_basis(bc_, H_, cap_);
        samples_.resize((size_t)kValidation * cap_);
#pragma omp parallel for schedule(dynamic, 8)
        for (int p = old; p < cap_; ++p)
            for (int i = 0; i < kValidation; ++i)
                samples_[(size_t)p * kValidation + i] = basis_.norms[p] * bessel_j0(basis_.roots[p] * grid_[i]);
        rhs_.resize(cap_);
#pragma omp parallel for schedule(dynamic, 4)
        for (int p = 0; p < cap_; ++p) rhs_[p] = rhs_entry(p);
        if (bc_ == 1) {
            const double bv = k_.eval(1.0) - offset_;
            if (bv != 0.0)
                for (int p = 0; p < cap_; ++p)
                    rhs_[p] += 2.0 * kPi * H_ * bv * basis_.norms[p] * bessel_j0(basis_.roots[p]);
        }
        gram_ = assemble_gram(basis_, a_, bc_ == 1 ? H_ : 0.0);
        chol_ = gram_;
        chol_ok_ = gpu_cholesky(chol_, cap_, device_);
        if (g_verbose)
            std::fprintf(stderr, "[sbd fit] ensure(P=%d) %.3f s\n", cap_,
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }

    // Solves the leading P x P system; returns the validation L-inf error.
    double solve_at(int P, std::vector<double>& alpha) const {
        if (chol_ok_) {
            alpha.assign(rhs_.begin(), rhs_.begin() + P);
            for (int i = 0; i < P; ++i) { // L y = b
                double s = alpha[i];
                for (int k = 0; k < i; ++k) s -= chol_[(size_t)k * cap_ + i] * alpha[k];
                alpha[i] = s / chol_[(size_t)i * cap_ + i];
            }
            for (int i = P - 1; i >= 0; --i) { // L^T x = y
                double s = alpha[i];
                const double* col = &chol_[(size_t)i * cap_];
                for (int k = i + 1; k < P; ++k) s -= col[k] * alpha[k];
                alpha[i] = s / col[i];
            }
        } else {
            std::vector<double> blk((size_t)P * P);
            for (int j = 0; j < P; ++j)
                for (int i = 0; i < P; ++i) blk[(size_t)j * P + i] = gram_[(size_t)j * cap_ + i];
            alpha = lu_solve(std::move(blk), P, std::vector<double>(rhs_.begin(), rhs_.begin() + P));
        }
        for (double v : alpha)
            if (!std::isfinite(v)) throw Error(3, "solve_sbd: Gram factorization failed (conditioning)");
        double err = 0.0;
#pragma omp parallel for reduction(max : err)
        for (int i = 0; i < kValidation; ++i) {
            double s = target_[i];
            for (int p = 0; p < P; ++p) s -= samples_[(size_t)p * kValidation + i] * alpha[p];
            err = std::max(err, std::fabs(s));
        }
        return err;
    }

    SbdFit pack(int P, const std::vector<double>& alpha, double err) const {
        SbdFit s;
        s.a = a_;
        s.P = P;
        s.coeffs.assign(alpha.begin(), alpha.begin() + P);
        s.roots.assign(basis_.roots.begin(), basis_.roots.begin() + P);
        s.norms.assign(basis_.norms.begin(), basis_.norms.begin() + P);
        s.constant_offset = offset_;
        s.achieved_error = err;
        s.bc = bc_;
        s.H = bc_ == 1 ? H_ : 0.0;
        return s;
    }

  private:
    static constexpr int kValidation = 2048; // sbd.hpp:44

    double rhs_entry(int p) const {
        const double rho = basis_.roots[p], c = basis_.norms[p];
        if (k_.laplace_rhs) {
            // r G'(r) = 1 for G = log(dmax r): the integral is (J0(rho a) - J0(rho)) / rho.
            return -2.0 * kPi * c * (bessel_j0(rho * a_) - bessel_j0(rho));
        }
        if (k_.rhs_integral) return -2.0 * kPi * c * rho * k_.rhs_integral(rho, a_);
        const int panels0 = std::max(4, (int)std::ceil((1.0 - a_) * rho * 10.0 / (2.0 * kPi * 16.0)));
        const double I = integrate([&](double r) { return r * k_.deriv(r) * bessel_j1(rho * r); }, a_, 1.0,
                                   1e-12, panels0);
        if (!std::isfinite(I)) throw Error(3, "assemble_rhs: integration failed");
        return -2.0 * kPi * c * rho * I;
    }

    const FitKernel& k_;
    double a_;
    int bc_;
    double H_;
    int device_;
    double offset_ = 0.0;
    int cap_ = 0;
    std::vector<double> grid_, target_, samples_, rhs_, gram_, chol_;
    Basis basis_;
    bool chol_ok_ = false;
};

} // namespace

// sbd.cpp:142-204 (solve_sbd_opts)
SbdFit solve_sbd(const FitKernel& k, double a, double tol, int bc, double H, bool subtract_offset,
                 int device) {
    if (!(a > 0.0 && a < 1.0)) throw Error(2, "solve_sbd: a must lie in (0, 1)");
    if (!(tol > 0.0)) throw Error(2, "solve_sbd: tol must be positive");
    const int P_max = (int)std::ceil(8.0 / a) + (int)std::ceil(k.oscillation_freq / kPi);
    Workspace ws(k, a, bc, H, subtract_offset, device);
    std::vector<double> alpha;
    const int P_lo = std::min((int)std::ceil(1.0 / a), P_max);
    ws.ensure(P_lo);
    double err_lo = ws.solve_at(P_lo, alpha);
    int lo, hi;
    double err_hi;
    if (err_lo <= tol) {
        if (P_lo == 1) return ws.pack(1, alpha, err_lo);
        lo = 0;
        hi = P_lo;
        err_hi = err_lo;
    } else {
        lo = hi = P_lo;
        err_hi = err_lo;
        double best = err_lo;
        while (err_hi > tol) {
            if (hi >= P_max)
                throw Error(5, "solve_sbd: tolerance not reached at P_max (best " + std::to_string(best) + ")");
            lo = hi;
            hi = std::min(P_max, std::max(hi * 2, hi + 8));
            ws.ensure(hi);
            err_hi = ws.solve_at(hi, alpha);
            best = std::min(best, err_hi);
        }
    }
    while (hi - lo > 1) {
        const int mid = lo + (hi - lo) / 2;
        const double e = ws.solve_at(mid, alpha);
        if (e <= tol) {
            hi = mid;
            err_hi = e;
        } else {
            lo = mid;
        }
    }
    err_hi = ws.solve_at(hi, alpha);
    return ws.pack(hi, alpha, err_hi);
}

} // namespace sbdgpu
