// pruned_dft.cu -- band-pruned, support-pruned 1D DFT passes for the forward
// NUFFT (replaces the full n1 x n2 FFTW_BACKWARD transform of
// /root/reference/proj/src/nufft.cpp:252 on the apply path).
//
// The spread grid of a type-III plan is nonzero only on its support window
// [lo, lo + L) of each axis (points live in [n/4, 3n/4] of the grid,
// nufft.cpp:166-169) and the interpolation only reads modes |j| <= b = n/4
// (nufft.cpp:194-205). One pass computes, for each of `rows` independent
// sequences x (support only),
//     X[j] = sum_{m in [lo, lo+L)} x[m] e^{+2 pi i j m / n},   |j| <= b,
// and stores X[j] at position (j mod B), B = 2b + 1 (the "band" layout).
//
// Method: decimate the output by D (n = D N'): for each residue e,
//     X[D k + e] = FFT_{N'}( y_e )[k mod N'],  y_e[p] = sum_{m = p mod N'} x[m] w_n^{e m},
// so one CTA folds the row into shared memory, runs an N'-point Stockham
// FFT there (radix 8/4/2/5/3 stages, ping-pong buffers), and writes the
// residue-e outputs; the D residues reuse the row from L1/L2. Every input
// element is read from HBM once and every band output written once.
#include <cmath>
#include <vector>

#include "pruned_dft.h"
#include "sbd_internal.h"

namespace sbdgpu {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul_i(double2 a) { return make_double2(-a.y, a.x); }   // * (+i)
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }  // * (-i)

// In-register DFT of length R with the e^{+2 pi i / R} convention.
template <int R>
__device__ __forceinline__ void dft_small(double2 (&v)[R]);

template <>
__device__ __forceinline__ void dft_small<2>(double2 (&v)[2]) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
}

template <>
__device__ __forceinline__ void dft_small<4>(double2 (&v)[4]) {
    const double2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
    const double2 s13 = cadd(v[1], v[3]), d13 = mul_i(csub(v[1], v[3]));
    v[0] = cadd(s02, s13);
    v[2] = csub(s02, s13);
    v[1] = cadd(d02, d13);
    v[3] = csub(d02, d13);
}

template <>
__device__ __forceinline__ void dft_small<8>(double2 (&v)[8]) {
    constexpr double h = 0.70710678118654752440;
    double2 e[4] = {v[0], v[2], v[4], v[6]};
    double2 o[4] = {v[1], v[3], v[5], v[7]};
    dft_small<4>(e);
    dft_small<4>(o);
    // twiddles w8^k = e^{+i pi k / 4}
    const double2 o1 = make_double2(h * (o[1].x - o[1].y), h * (o[1].x + o[1].y));
    const double2 o2 = mul_i(o[2]);
    const double2 o3 = make_double2(-h * (o[3].x + o[3].y), h * (o[3].x - o[3].y));
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], o1);
    v[5] = csub(e[1], o1);
    v[2] = cadd(e[2], o2);
    v[6] = csub(e[2], o2);
    v[3] = cadd(e[3], o3);
    v[7] = csub(e[3], o3);
}

template <>
__device__ __forceinline__ void dft_small<3>(double2 (&v)[3]) {
    constexpr double c = -0.5, s = 0.86602540378443864676;  // e^{+2 pi i/3}
    const double2 t = cadd(v[1], v[2]);
    const double2 d = csub(v[1], v[2]);
    const double2 m = make_double2(v[0].x + c * t.x, v[0].y + c * t.y);
    const double2 r = make_double2(-s * d.y, s * d.x);  // i s d
    v[0] = cadd(v[0], t);
    v[1] = cadd(m, r);
    v[2] = csub(m, r);
}

template <>
__device__ __forceinline__ void dft_small<5>(double2 (&v)[5]) {
    constexpr double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
    constexpr double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;
    const double2 t1 = cadd(v[1], v[4]), d1 = csub(v[1], v[4]);
    const double2 t2 = cadd(v[2], v[3]), d2 = csub(v[2], v[3]);
    const double2 a1 = make_double2(v[0].x + c1 * t1.x + c2 * t2.x, v[0].y + c1 * t1.y + c2 * t2.y);
    const double2 a2 = make_double2(v[0].x + c2 * t1.x + c1 * t2.x, v[0].y + c2 * t1.y + c1 * t2.y);
    // i (s1 d1 + s2 d2), i (s2 d1 - s1 d2)
    const double2 b1 = make_double2(-(s1 * d1.y + s2 * d2.y), s1 * d1.x + s2 * d2.x);
    const double2 b2 = make_double2(-(s2 * d1.y - s1 * d2.y), s2 * d1.x - s1 * d2.x);
    v[0] = cadd(v[0], cadd(t1, t2));
    v[1] = cadd(a1, b1);
    v[4] = csub(a1, b1);
    v[2] = cadd(a2, b2);
    v[3] = csub(a2, b2);
}

// One Stockham stage of radix R on N points in shared memory: X -> Y.
// Ns = product of the radices already applied; w = e^{+2 pi i q / n}, q in [0, n).
template <int R>
__device__ __forceinline__ void stockham_stage(const double2* __restrict__ X, double2* __restrict__ Y,
                                               int N, int Ns, int n, const double2* __restrict__ w) {
    const int nb = N / R;
    const int tstep = n / (Ns * R);  // w_{Ns R}^{q} = w_n^{q tstep}
    for (int j = threadIdx.x; j < nb; j += blockDim.x) {
        const int k = j % Ns;
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = X[j + r * nb];
        if (Ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(w + r * k * tstep));
        }
        dft_small<R>(v);
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) Y[base + r * Ns] = v[r];
    }
}

__global__ void __launch_bounds__(512) k_pruned_dft(PrunedPass p, const double2* __restrict__ in,
                                                    double2* __restrict__ out,
                                                    const double2* __restrict__ w) {
    extern __shared__ double2 sm[];
    const int N = p.N;
    double2* A = sm;
    double2* Bf = sm + N;
    const int row = blockIdx.x;
    const double2* x = in + (int64_t)row * p.in_row;
    double2* y = out + (int64_t)row * p.out_row;
    for (int e = 0; e < p.D; ++e) {
        // fold + twiddle: A[pp] = sum_{m = pp (mod N), m in [lo, lo+L)} x[m] w_n^{e m}
        for (int pp = threadIdx.x; pp < N; pp += blockDim.x) {
            int m = p.lo + ((pp - p.lo) % N + N) % N;
            double2 acc = make_double2(0.0, 0.0);
            for (; m < p.lo + p.L; m += N) {
                const double2 xv = x[(int64_t)(m - p.lo) * p.in_elem];
                if (e == 0) {
                    acc = cadd(acc, xv);
                } else {
                    const int q = (int)(((int64_t)e * m) % p.n);
                    acc = cadd(acc, cmul(xv, __ldg(w + q)));
                }
            }
            A[pp] = acc;
        }
        __syncthreads();
        double2* X = A;
        double2* Y = Bf;
        int Ns = 1;
        for (int s = 0; s < p.nstages; ++s) {
            const int R = p.radix[s];
            switch (R) {
                case 8: stockham_stage<8>(X, Y, N, Ns, p.n, w); break;
                case 4: stockham_stage<4>(X, Y, N, Ns, p.n, w); break;
                case 2: stockham_stage<2>(X, Y, N, Ns, p.n, w); break;
                case 5: stockham_stage<5>(X, Y, N, Ns, p.n, w); break;
                case 3: stockham_stage<3>(X, Y, N, Ns, p.n, w); break;
            }
            __syncthreads();
            Ns *= R;
            double2* t = X;
            X = Y;
            Y = t;
        }
        // outputs j = D k + e with |j| <= b, stored at (j mod B)
        const int kmin = -((p.b + e) / p.D);          // smallest k with D k + e >= -b
        const int kmax = (p.b - e) >= 0 ? (p.b - e) / p.D : -1;
        for (int k = kmin + threadIdx.x; k <= kmax; k += blockDim.x) {
            const int j = p.D * k + e;
            if (j < -p.b || j > p.b) continue;
            const int kk = k < 0 ? k + N : k;
            const int slot = j < 0 ? j + p.B : j;
            y[(int64_t)slot * p.out_elem] = X[kk];
        }
        __syncthreads();
    }
}

} // namespace

bool make_pruned_pass(int n, int lo, int L, int rows, PrunedPass& p) {
    p = PrunedPass{};
    p.n = n;
    p.lo = lo;
    p.L = L;
    p.rows = rows;
    p.b = n / 4;
    p.B = 2 * p.b + 1;
    if (lo < 0 || lo + L > n || L <= 0) return false;
    // smallest power-of-two decimation that fits two ping-pong buffers in smem
    const int max_smem_cells = (200 * 1024) / (2 * (int)sizeof(double2));
    for (int D = 1; D <= 64; D *= 2) {
        if (n % D) break;
        if (n / D <= max_smem_cells) {
            p.D = D;
            p.N = n / D;
            break;
        }
    }
    if (!p.D) return false;
    int m = p.N, s = 0;
    for (int r : {8, 4, 2, 5, 3}) {
        while (m % r == 0 && s < 32) {
            p.radix[s++] = r;
            m /= r;
        }
    }
    if (m != 1) return false;
    p.nstages = s;
    return true;
}

DevBuf<double2> make_twiddles(int n, cudaStream_t st) {
    std::vector<double2> h(n);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (int q = 0; q < n; ++q) {
        const long double a = two_pi * (long double)q / (long double)n;
        h[q] = make_double2((double)cosl(a), (double)sinl(a));
    }
    DevBuf<double2> d;
    d.upload(h.data(), n, st);
    ck(cudaStreamSynchronize(st), "twiddles");
    return d;
}

void launch_pruned_dft(const PrunedPass& p, const double2* in, double2* out, const double2* w,
                       cudaStream_t st) {
    if (p.rows <= 0) return;
    const size_t smem = (size_t)2 * p.N * sizeof(double2);
    static size_t attr = 0;
    if (smem > attr) {
        ck(cudaFuncSetAttribute(k_pruned_dft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
           "pruned dft smem");
        attr = smem;
    }
    k_pruned_dft<<<p.rows, 512, smem, st>>>(p, in, out, w);
    count_launch();
    ck(cudaGetLastError(), "k_pruned_dft");
}

} // namespace sbdgpu
