// Standalone check of one band-pruned DFT pass against a naive host DFT
// (links the built library's internal symbols).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1711_07877_b200/csrc/pruned_dft.h"
using namespace sbdgpu;
int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 2304;
    const int forced = argc > 2 ? atoi(argv[2]) : 0;
    const int lo = n / 4 - 7, L = n / 2 + 13, rows = argc > 3 ? atoi(argv[3]) : 3;
    PrunedPass p;
    if (!make_pruned_pass(n, lo, L, rows, forced, p)) { printf("unsupported\n"); return 1; }
    p.in_row = L; p.in_elem = 1; p.out_row = p.B; p.out_elem = 1;
    printf("n %d N %d D %d R3 %d\n", n, p.N, p.D, p.radix[2]);
    std::vector<double2> x((size_t)rows * L);
    srand(3);
    for (auto& v : x) v = make_double2(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
    DevBuf<double2> dx, dy;
    dx.upload(x.data(), x.size(), 0);
    dy.alloc((size_t)rows * p.B);
    cudaMemset(dy.p, 0, dy.bytes());
    DevBuf<double2> tw = make_twiddles(p, 0);
    launch_pruned_dft(p, dx.p, dy.p, tw.p, 0);
    printf("sync %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<double2> y((size_t)rows * p.B);
    cudaMemcpy(y.data(), dy.p, dy.bytes(), cudaMemcpyDeviceToHost);
    double err = 0, mag = 0;
    for (int r = 0; r < rows; r += (rows > 8 ? rows / 7 : 1))
        for (int j = -p.b; j <= p.b; j += 37) {
            long double re = 0, im = 0;
            for (int m = 0; m < L; ++m) {
                const long double a = 2.0L * M_PI * (long double)j * (lo + m) / n;
                const double2 v = x[(size_t)r * L + m];
                re += v.x * cosl(a) - v.y * sinl(a);
                im += v.x * sinl(a) + v.y * cosl(a);
            }
            const double2 g = y[(size_t)r * p.B + (j < 0 ? j + p.B : j)];
            err = fmax(err, hypot(g.x - (double)re, g.y - (double)im));
            mag = fmax(mag, hypot((double)re, (double)im));
            if (r == 0 && j == -p.b) printf("j=%d got %g %g want %g %g\n", j, g.x, g.y, (double)re, (double)im);
        }
    printf("max err %.3e (max |X| %.3e)\n", err, mag);
    int diff = 0;
    for (int it = 0; it < 5; ++it) {
        cudaMemset(dy.p, 0, dy.bytes());
        launch_pruned_dft(p, dx.p, dy.p, tw.p, 0);
        std::vector<double2> y2((size_t)rows * p.B);
        cudaMemcpy(y2.data(), dy.p, dy.bytes(), cudaMemcpyDeviceToHost);
        for (size_t i = 0; i < y.size(); ++i) diff += y2[i].x != y[i].x || y2[i].y != y[i].y;
    }
    printf("nondeterministic entries over 5 reruns: %d of %zu\n", diff, y.size());
}
