// assemble.cpp -- offline operator assembly on the host + device, following
// CompressedOperator::assemble (/root/reference/proj/src/conv_operator.cpp:244-294):
//
//   delta_max   exact cloud diameter (convex hull + rotating calipers,
//               point_cloud.cpp:13-72)
//   a           a_override, or the N-rule choose_parameters (:121-133), capped
//               for oscillatory kernels (kernel_a_cap, :53-77)
//   SBD fit     sbd_fit.cpp (Laplace: log(dmax r) on the unit annulus;
//               Helmholtz: Y0/4 in the root / rescaled / Robin regimes, :79-117)
//   spectrum    rings {rho_p * radial_scale, C_p alpha_p} (+ the exact J0 ring
//               -i/4 for Helmholtz) -> build_ring_quadrature
//               (ring_quadrature.cpp:14-69), xi /= dmax
//   nufft_tol   eps / (20 max(1, sum|w|))  (:287-289)
//   D           assemble_kernels.cu (neighbour search + far field on the GPU)
//
// Offline only: reported, not optimised (north_star).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "assemble_gpu.h"
#include "bessel_host.h"
#include "opdata.h"
#include "sbd_fit.h"
#include "sbd_internal.h"

namespace sbdgpu {

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kE = 2.71828182845904523536;
constexpr double kSbdToleranceShare = 0.375; // conv_operator.cpp:16
constexpr double kRingKSafe = 4.0;           // ring_quadrature.hpp:14

struct P2 {
    double x, y;
};

double cross(P2 o, P2 a, P2 b) { return (a.x - o.x) * (b.y - o.y) - (a.y - o.y) * (b.x - o.x); }

} // namespace

// Exact diameter: monotone-chain hull, then the farthest antipodal pair by
// rotating calipers (point_cloud.cpp:13-57).
double cloud_diameter(const double* xy, uint64_t n) {
    if (n < 2) return 0.0;
    std::vector<P2> p(n);
    for (uint64_t i = 0; i < n; ++i) p[i] = {xy[2 * i], xy[2 * i + 1]};
    std::sort(p.begin(), p.end(), [](const P2& a, const P2& b) { return a.x < b.x || (a.x == b.x && a.y < b.y); });
    p.erase(std::unique(p.begin(), p.end(), [](const P2& a, const P2& b) { return a.x == b.x && a.y == b.y; }),
            p.end());
    const int m0 = (int)p.size();
    if (m0 == 1) return 0.0;
    std::vector<P2> h(2 * m0);
    int k = 0;
    for (int i = 0; i < m0; ++i) {
        while (k >= 2 && cross(h[k - 2], h[k - 1], p[i]) <= 0) --k;
        h[k++] = p[i];
    }
    for (int i = m0 - 2, lo = k + 1; i >= 0; --i) {
        while (k >= lo && cross(h[k - 2], h[k - 1], p[i]) <= 0) --k;
        h[k++] = p[i];
    }
    h.resize(std::max(1, k - 1));
    const int m = (int)h.size();
    auto dist = [](P2 a, P2 b) { return std::hypot(a.x - b.x, a.y - b.y); };
    if (m == 1) return 0.0;
    if (m == 2) return dist(h[0], h[1]);
    double best = 0.0;
    int j = 1;
    for (int i = 0; i < m; ++i) {
        const P2 a = h[i], b = h[(i + 1) % m];
        auto area = [&](int q) { return std::fabs((b.x - a.x) * (h[q].y - a.y) - (b.y - a.y) * (h[q].x - a.x)); };
        while (area((j + 1) % m) > area(j)) j = (j + 1) % m;
        best = std::max({best, dist(h[j], a), dist(h[j], b)});
    }
    return best;
}

namespace {

// conv_operator.cpp:59-77
double oscillation_a_cap(double kappa, double eps) {
    if (kappa <= 0.0) return 1.0;
    const double gamma_tol = std::min(4.5, std::log(1.0 / std::max(kSbdToleranceShare * eps, 1e-14)) / 3.7 + 0.8);
    return std::clamp((6.2 - gamma_tol) * kPi / kappa, 0.005, 1.0);
}

// ring_quadrature.cpp:14-22
int ring_size(double rho, double tol) {
    const double extra = std::max(0.0, std::log(kRingKSafe / tol));
    int m = (int)std::ceil(0.5 * kE * rho + extra);
    m = std::max(m, 4);
    if (m & 1) ++m;
    return m;
}

struct Ring {
    double rho;
    std::complex<double> w;
};

// ring_quadrature.cpp:24-69
void build_ring_quadrature(const std::vector<Ring>& rings, double offset, double eps, OpData& d) {
    int active = 0;
    for (const Ring& r : rings)
        if (std::abs(r.w) > 0.0) ++active;
    std::vector<int> sizes;
    size_t total = offset != 0.0 ? 1 : 0;
    for (const Ring& r : rings) {
        if (std::abs(r.w) == 0.0) {
            sizes.push_back(0);
            continue;
        }
        sizes.push_back(ring_size(r.rho, eps / (2.0 * active * std::abs(r.w))));
        total += sizes.back();
    }
    d.freqs.clear();
    d.weights.clear();
    d.ring_offsets.clear();
    d.freqs.reserve(2 * total);
    d.weights.reserve(2 * total);
    if (offset != 0.0) {
        d.ring_offsets.push_back(0);
        d.freqs.insert(d.freqs.end(), {0.0, 0.0});
        d.weights.insert(d.weights.end(), {offset, 0.0});
    }
    for (size_t i = 0; i < rings.size(); ++i) {
        if (sizes[i] == 0) continue;
        d.ring_offsets.push_back((int32_t)(d.freqs.size() / 2));
        const int m = sizes[i];
        const std::complex<double> nw = rings[i].w / (double)m;
        for (int j = 0; j < m; ++j) {
            const double th = 2.0 * kPi * j / m;
            d.freqs.push_back(rings[i].rho * std::cos(th));
            d.freqs.push_back(rings[i].rho * std::sin(th));
            d.weights.push_back(nw.real());
            d.weights.push_back(nw.imag());
        }
    }
    d.ring_offsets.push_back((int32_t)(d.freqs.size() / 2));
    d.total_error_budget = eps;
}

} // namespace

namespace {
struct PhaseLog {
    bool on = g_verbose;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[sbd assemble] %-28s %8.3f s\n", what,
                     std::chrono::duration<double>(now - t).count());
        t = now;
    }
};
} // namespace

void assemble_opdata(int kind, double k, const double* src_xy, uint64_t n_src, const double* tgt_xy,
                     uint64_t n_tgt, const sbd_assemble_options& o, OpData& d) {
    PhaseLog plog;
    if (n_src == 0 || (tgt_xy && n_tgt == 0)) throw Error(SBD_ERR_INVALID_ARGUMENT, "assemble: clouds must be nonempty");
    if (kind != 0 && kind != 1) throw Error(SBD_ERR_INVALID_ARGUMENT, "assemble: unknown kernel kind");
    if (kind == 1 && !(k > 0.0)) throw Error(SBD_ERR_DOMAIN, "kernel_helmholtz: k must be positive");
    d.kind = kind;
    d.k = kind == 1 ? k : 0.0;
    d.single = tgt_xy == nullptr ||
               (n_tgt == n_src && std::memcmp(tgt_xy, src_xy, n_src * 16) == 0);
    d.src.assign(src_xy, src_xy + 2 * n_src);
    if (!d.single) d.tgt.assign(tgt_xy, tgt_xy + 2 * n_tgt);
    d.eps = o.eps;
    d.alpha = o.alpha;
    d.src_diam = cloud_diameter(src_xy, n_src);
    if (d.single) {
        d.dmax = d.src_diam;
    } else {
        d.tgt_diam = cloud_diameter(tgt_xy, n_tgt);
        std::vector<double> all(d.src);
        all.insert(all.end(), d.tgt.begin(), d.tgt.end());
        d.dmax = cloud_diameter(all.data(), all.size() / 2);
    }
    if (!(d.dmax > 0.0)) throw Error(SBD_ERR_INVALID_ARGUMENT, "assemble: degenerate cloud (zero diameter)");

    if (o.a_override > 0.0) {
        d.a = o.a_override;
        if (!(d.a < 1.0)) throw Error(SBD_ERR_DOMAIN, "assemble: a must lie in (0, 1)");
    } else {
        double a = 0.0;
        int ph = 0;
        if (sbd_choose_parameters(std::max(d.n_src(), d.n_tgt()), o.eps, o.alpha, &a, &ph) != SBD_OK)
            throw Error(SBD_ERR_DOMAIN, sbd_last_error());
        d.a = a;
    }
    if (kind == 1) d.a = std::min(d.a, oscillation_a_cap(k * d.dmax, o.eps));
    d.dmin = d.a * d.dmax;
    plog.mark("diameter + a");

    // ---- spectral model (conv_operator.cpp:79-117)
    const double tol = kSbdToleranceShare * o.eps;
    const double dmax = d.dmax;
    SbdFit fit;
    std::vector<Ring> rings;
    if (kind == 0) {
        FitKernel fk;
        fk.eval = [dmax](double r) { return std::log(dmax * r); };
        fk.deriv = [](double r) { return 1.0 / r; };
        fk.laplace_rhs = true;
        fit = solve_sbd(fk, d.a, tol, 0, 0.0, true, o.device);
    } else {
        const double kappa = k * dmax;
        auto quarter_y0 = [](double kap) {
            FitKernel fk;
            fk.eval = [kap](double r) { return 0.25 * bessel_y0(kap * r); };
            fk.deriv = [kap](double r) { return -0.25 * kap * bessel_y1(kap * r); };
            fk.oscillation_freq = kap;
            // Lommel: int r J1(rho r) Y1(kap r) dr = r [kap J1(rho r) Y0(kap r) - rho J0(rho r) Y1(kap r)]
            // / (rho^2 - kap^2); with G' = -kap Y1(kap r)/4. Exact where the reference's
            // relative-tolerance quadrature (gram.cpp:69-84) needs up to 2^14 panel doublings
            // for the nearly cancelling entries.
            fk.rhs_integral = [kap](double rho, double a) {
                auto F = [&](double r) {
                    return r * (kap * bessel_j1(rho * r) * bessel_y0(kap * r) -
                                rho * bessel_j0(rho * r) * bessel_y1(kap * r)) /
                           (rho * rho - kap * kap);
                };
                return -0.25 * kap * (F(1.0) - F(a));
            };
            return fk;
        };
        // kernels.cpp:53-66 regime selection
        if (std::fabs(bessel_y0(kappa)) < 1e-10) {
            fit = solve_sbd(quarter_y0(kappa), d.a, tol, 0, 0.0, true, o.device);
        } else if (kappa < o.small_k_factor * first_y0_root()) {
            const double H = -kappa * (-bessel_y1(kappa)) / bessel_y0(kappa);
            fit = solve_sbd(quarter_y0(kappa), d.a, tol, 1, H, false, o.device);
        } else {
            const double kp = y0_root_above(kappa);
            const double scale = kappa / kp;
            fit = solve_sbd(quarter_y0(kp), d.a * scale, tol, 0, 0.0, true, o.device);
            fit.radial_scale = scale;
            fit.a = d.a;
        }
        rings.push_back({kappa, std::complex<double>(0.0, -0.25)});
    }
    for (int p = 0; p < fit.P; ++p)
        rings.push_back({fit.roots[p] * fit.radial_scale, std::complex<double>(fit.coeffs[p] * fit.norms[p], 0.0)});
    plog.mark("SBD fit");
    build_ring_quadrature(rings, fit.constant_offset, o.eps, d);
    for (double& v : d.freqs) v /= dmax;
    plog.mark("ring quadrature");

    d.sbd.a = fit.a;
    d.sbd.P = fit.P;
    d.sbd.constant_offset = fit.constant_offset;
    d.sbd.achieved_error = fit.achieved_error;
    d.sbd.radial_scale = fit.radial_scale;
    d.sbd.bc = fit.bc;
    d.sbd.H = fit.H;
    d.sbd.coeffs = fit.coeffs;
    d.sbd.roots = fit.roots;
    d.sbd.norm_constants = fit.norms;

    double wabs = 0.0, wre = 0.0, wim = 0.0;
    for (size_t v = 0; v < d.weights.size() / 2; ++v) {
        wabs += std::hypot(d.weights[2 * v], d.weights[2 * v + 1]);
        wre += d.weights[2 * v];
        wim += d.weights[2 * v + 1];
    }
    d.nufft_tol = o.eps / (20.0 * std::max(1.0, wabs));

    // ---- close-correction matrix (conv_operator.cpp:172-237)
    CloseMatrixInput ci;
    ci.src_xy = d.src.data();
    ci.n_src = d.n_src();
    ci.tgt_xy = d.single ? d.src.data() : d.tgt.data();
    ci.n_tgt = d.n_tgt();
    ci.single = d.single;
    ci.radius = d.dmin;
    ci.xi_xy = d.freqs.data();
    ci.w = d.weights.data();
    ci.n_xi = d.n_xi();
    ci.wsum_re = wre;
    ci.wsum_im = wim;
    ci.nufft_tol = d.nufft_tol;
    ci.direct_threshold = o.nufft_direct_threshold;
    ci.max_grid_bytes = std::max<uint64_t>(o.max_grid_bytes, uint64_t(1) << 30);
    ci.laplace = kind == 0;
    ci.device = o.device;
    CloseMatrixOutput co;
    build_close_matrix_gpu(ci, co);
    plog.mark("close pairs + far field (GPU)");
    d.row_offsets = std::move(co.row_offsets);
    d.cols = std::move(co.cols);
    d.values = std::move(co.values);
    if (kind == 1) {
        // Helmholtz G(r) = Y0(kr)/4 - i J0(kr)/4 (kernels.cpp:73-75), host long-double series.
        const double* tg = ci.tgt_xy;
        const int64_t nt = (int64_t)d.n_tgt();
#pragma omp parallel for schedule(dynamic, 256)
        for (int64_t r = 0; r < nt; ++r) {
            for (uint64_t i = d.row_offsets[r]; i < d.row_offsets[r + 1]; ++i) {
                const uint32_t c = d.cols[i];
                if (d.single && c == (uint32_t)r) continue;
                const double rad = std::hypot(tg[2 * r] - d.src[2 * c], tg[2 * r + 1] - d.src[2 * c + 1]);
                d.values[2 * i] += 0.25 * bessel_y0(k * rad);
                d.values[2 * i + 1] += -0.25 * bessel_j0(k * rad);
            }
        }
        plog.mark("Helmholtz kernel values");
    }
}

} // namespace sbdgpu
