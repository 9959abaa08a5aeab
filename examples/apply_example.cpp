// examples/apply_example.cpp -- the reference's "assemble once, apply many"
// usage (proj/tools/sbdconv.cpp:45-102) on the B200 path through
// include/sbd_b200.hpp. Self-checking: compares apply() with the direct
// O(N^2) sum at a subset of targets (the reference's error contract,
// conv_operator.hpp:50-51) and the adjoint against <A f, u> = <f, A^H u>.
//
//   g++ -std=c++17 -I include examples/apply_example.cpp -L paper_1711_07877_b200 -lsbd_b200 \
//       -Wl,-rpath,$PWD/paper_1711_07877_b200 -o apply_example && ./apply_example [N]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "sbd_b200.hpp"

using sbd_b200::cplx;
using sbd_b200::Vec2;

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 20000;
    std::mt19937_64 rng(20260809);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::vector<Vec2> pts(n);
    for (auto& p : pts) {  // uniform in the disk of diameter 1
        const double r = 0.5 * std::sqrt(u(rng)), t = 2.0 * M_PI * u(rng);
        p = {r * std::cos(t), r * std::sin(t)};
    }
    sbd_b200::AssembleOptions o;
    o.eps = 1e-6;
    o.a_override = (2.74 / std::sqrt((double)n)) / sbd_b200::cloud_diameter(pts);
    auto t0 = std::chrono::steady_clock::now();
    auto op = sbd_b200::CompressedOperator::assemble(sbd_b200::kernel_laplace(), pts, o);
    const double offline = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<cplx> f(n);
    double fsum = 0.0;
    for (auto& v : f) {
        v = {gauss(rng), 0.0};
        fsum += std::abs(v);
    }
    auto q = op.apply(f);
    double best = 1e300;
    for (int rep = 0; rep < 3; ++rep) {  // best of 3, as sbdconv bench
        t0 = std::chrono::steady_clock::now();
        q = op.apply(f);
        best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    double worst = 0.0;
    for (int k = 0; k < n; k += std::max(1, n / 200)) {
        cplx acc = 0.0;
        for (int l = 0; l < n; ++l) {
            if (l == k) continue;
            acc += std::log(std::hypot(pts[k].x - pts[l].x, pts[k].y - pts[l].y)) * f[l];
        }
        worst = std::max(worst, std::abs(q[k] - acc));
    }
    std::vector<cplx> w(n);
    for (auto& v : w) v = {gauss(rng), gauss(rng)};
    const auto qa = op.apply_adjoint(w);
    cplx lhs = 0.0, rhs = 0.0;
    for (int i = 0; i < n; ++i) {
        lhs += std::conj(w[i]) * q[i];
        rhs += std::conj(qa[i]) * f[i];
    }
    const double ratio = worst / fsum;
    const double adj = std::abs(lhs - rhs) / std::abs(lhs);
    std::printf("N=%d offline=%.3fs online=%.6fs points/s=%.3e err/sum|f|=%.2e adjoint=%.2e P=%d n_xi=%llu nnz=%llu\n",
                n, offline, best, n / best, ratio, adj, op.info().P, (unsigned long long)op.info().n_xi,
                (unsigned long long)op.info().nnz);
    const bool ok = ratio <= o.eps && adj <= 1e-6;
    std::printf("%s\n", ok ? "PASS" : "FAIL");
    try {
        op.apply(std::vector<cplx>(3));
        return 1;
    } catch (const std::invalid_argument&) {
    }
    return ok ? 0 : 1;
}
