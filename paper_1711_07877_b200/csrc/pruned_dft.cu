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
// Method: decimate the output by D (n = D N, N = 256 R3): for each residue e,
//     X[D k + e] = FFT_N( y_e )[k mod N],  y_e[p] = w_n^{e p} sum_t x[p + t N] w_D^{e t},
// one CTA per (sequence, e): the fold operands stream through a bulk-copy
// ring (cp.async.bulk + mbarrier) into the stage-1 registers, then a
// 16 x 16 x R3 FFT runs through shared memory and writes only the residue-e
// band outputs. The D CTAs of a sequence share it through L2, so every input
// element is read from HBM once and every band output written once.
// Selected with SBD_FFT=dft (plan.cpp); on config 4 it matches the cuFFT
// row/column path, which stays the default.
#include <algorithm>
#include <cmath>
#include <cstdlib>
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

// e^{+2 pi i q / R} for R <= 18 (row R); literal, so every device image has it.
__constant__ double2 kW[19][18] = {
    {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {-1.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {-0.5, 0.8660254037844386}, {-0.5, -0.8660254037844386}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.0, 1.0}, {-1.0, 0.0}, {0.0, -1.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.30901699437494745, 0.9510565162951535}, {-0.8090169943749475, 0.5877852522924731}, {-0.8090169943749475, -0.5877852522924731}, {0.30901699437494745, -0.9510565162951535}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.5, 0.8660254037844386}, {-0.5, 0.8660254037844386}, {-1.0, 0.0}, {-0.5, -0.8660254037844386}, {0.5, -0.8660254037844386}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.6234898018587335, 0.7818314824680298}, {-0.2225209339563144, 0.9749279121818236}, {-0.9009688679024191, 0.4338837391175581}, {-0.9009688679024191, -0.4338837391175581}, {-0.2225209339563144, -0.9749279121818236}, {0.6234898018587335, -0.7818314824680298}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.7071067811865476, 0.7071067811865476}, {0.0, 1.0}, {-0.7071067811865476, 0.7071067811865476}, {-1.0, 0.0}, {-0.7071067811865476, -0.7071067811865476}, {0.0, -1.0}, {0.7071067811865476, -0.7071067811865476}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.766044443118978, 0.6427876096865394}, {0.17364817766693036, 0.984807753012208}, {-0.5, 0.8660254037844386}, {-0.9396926207859084, 0.3420201433256687}, {-0.9396926207859084, -0.3420201433256687}, {-0.5, -0.8660254037844386}, {0.17364817766693036, -0.984807753012208}, {0.766044443118978, -0.6427876096865394}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.8090169943749475, 0.5877852522924731}, {0.30901699437494745, 0.9510565162951535}, {-0.30901699437494745, 0.9510565162951535}, {-0.8090169943749475, 0.5877852522924731}, {-1.0, 0.0}, {-0.8090169943749475, -0.5877852522924731}, {-0.30901699437494745, -0.9510565162951535}, {0.30901699437494745, -0.9510565162951535}, {0.8090169943749475, -0.5877852522924731}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.8412535328311812, 0.5406408174555976}, {0.41541501300188644, 0.9096319953545183}, {-0.14231483827328514, 0.9898214418809327}, {-0.6548607339452851, 0.7557495743542583}, {-0.9594929736144974, 0.28173255684142967}, {-0.9594929736144974, -0.28173255684142967}, {-0.6548607339452851, -0.7557495743542583}, {-0.14231483827328514, -0.9898214418809327}, {0.41541501300188644, -0.9096319953545183}, {0.8412535328311812, -0.5406408174555976}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.8660254037844386, 0.5}, {0.5, 0.8660254037844386}, {0.0, 1.0}, {-0.5, 0.8660254037844386}, {-0.8660254037844386, 0.5}, {-1.0, 0.0}, {-0.8660254037844386, -0.5}, {-0.5, -0.8660254037844386}, {0.0, -1.0}, {0.5, -0.8660254037844386}, {0.8660254037844386, -0.5}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.8854560256532099, 0.46472317204376856}, {0.5680647467311558, 0.8229838658936564}, {0.12053668025532305, 0.992708874098054}, {-0.3546048870425356, 0.9350162426854148}, {-0.7485107481711011, 0.6631226582407952}, {-0.970941817426052, 0.23931566428755777}, {-0.970941817426052, -0.23931566428755777}, {-0.7485107481711011, -0.6631226582407952}, {-0.3546048870425356, -0.9350162426854148}, {0.12053668025532305, -0.992708874098054}, {0.5680647467311558, -0.8229838658936564}, {0.8854560256532099, -0.46472317204376856}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.9009688679024191, 0.4338837391175581}, {0.6234898018587335, 0.7818314824680298}, {0.2225209339563144, 0.9749279121818236}, {-0.2225209339563144, 0.9749279121818236}, {-0.6234898018587335, 0.7818314824680298}, {-0.9009688679024191, 0.4338837391175581}, {-1.0, 0.0}, {-0.9009688679024191, -0.4338837391175581}, {-0.6234898018587335, -0.7818314824680298}, {-0.2225209339563144, -0.9749279121818236}, {0.2225209339563144, -0.9749279121818236}, {0.6234898018587335, -0.7818314824680298}, {0.9009688679024191, -0.4338837391175581}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.9135454576426009, 0.4067366430758002}, {0.6691306063588582, 0.7431448254773942}, {0.30901699437494745, 0.9510565162951535}, {-0.10452846326765347, 0.9945218953682733}, {-0.5, 0.8660254037844386}, {-0.8090169943749475, 0.5877852522924731}, {-0.9781476007338057, 0.20791169081775934}, {-0.9781476007338057, -0.20791169081775934}, {-0.8090169943749475, -0.5877852522924731}, {-0.5, -0.8660254037844386}, {-0.10452846326765347, -0.9945218953682733}, {0.30901699437494745, -0.9510565162951535}, {0.6691306063588582, -0.7431448254773942}, {0.9135454576426009, -0.4067366430758002}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.9238795325112867, 0.3826834323650898}, {0.7071067811865476, 0.7071067811865476}, {0.3826834323650898, 0.9238795325112867}, {0.0, 1.0}, {-0.3826834323650898, 0.9238795325112867}, {-0.7071067811865476, 0.7071067811865476}, {-0.9238795325112867, 0.3826834323650898}, {-1.0, 0.0}, {-0.9238795325112867, -0.3826834323650898}, {-0.7071067811865476, -0.7071067811865476}, {-0.3826834323650898, -0.9238795325112867}, {0.0, -1.0}, {0.3826834323650898, -0.9238795325112867}, {0.7071067811865476, -0.7071067811865476}, {0.9238795325112867, -0.3826834323650898}, {0.0, 0.0}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.9324722294043558, 0.3612416661871529}, {0.7390089172206591, 0.6736956436465572}, {0.44573835577653825, 0.8951632913550623}, {0.092268359463302, 0.9957341762950345}, {-0.2736629900720829, 0.961825643172819}, {-0.6026346363792564, 0.7980172272802395}, {-0.8502171357296141, 0.5264321628773558}, {-0.9829730996839018, 0.18374951781657034}, {-0.9829730996839018, -0.18374951781657034}, {-0.8502171357296141, -0.5264321628773558}, {-0.6026346363792564, -0.7980172272802395}, {-0.2736629900720829, -0.961825643172819}, {0.092268359463302, -0.9957341762950345}, {0.44573835577653825, -0.8951632913550623}, {0.7390089172206591, -0.6736956436465572}, {0.9324722294043558, -0.3612416661871529}, {0.0, 0.0}},
    {{1.0, 0.0}, {0.9396926207859084, 0.3420201433256687}, {0.766044443118978, 0.6427876096865394}, {0.5, 0.8660254037844386}, {0.17364817766693036, 0.984807753012208}, {-0.17364817766693036, 0.984807753012208}, {-0.5, 0.8660254037844386}, {-0.766044443118978, 0.6427876096865394}, {-0.9396926207859084, 0.3420201433256687}, {-1.0, 0.0}, {-0.9396926207859084, -0.3420201433256687}, {-0.766044443118978, -0.6427876096865394}, {-0.5, -0.8660254037844386}, {-0.17364817766693036, -0.984807753012208}, {0.17364817766693036, -0.984807753012208}, {0.5, -0.8660254037844386}, {0.766044443118978, -0.6427876096865394}, {0.9396926207859084, -0.3420201433256687}},
};

// composite radices R = P Q (P first)
template <int R> struct Split;
template <> struct Split<6> { static constexpr int P = 2, Q = 3; };
template <> struct Split<9> { static constexpr int P = 3, Q = 3; };
template <> struct Split<10> { static constexpr int P = 2, Q = 5; };
template <> struct Split<12> { static constexpr int P = 4, Q = 3; };
template <> struct Split<15> { static constexpr int P = 3, Q = 5; };
template <> struct Split<16> { static constexpr int P = 4, Q = 4; };
template <> struct Split<18> { static constexpr int P = 2, Q = 9; };

// In-register DFT of any supported length R <= 16 (e^{+2 pi i / R}).
template <int R>
__device__ __forceinline__ void dft_reg(double2 (&v)[R]) {
    if constexpr (R == 2 || R == 3 || R == 4 || R == 5 || R == 8) {
        dft_small<R>(v);
    } else {
        // m = q + Q p, k = k1 + P k2: X[k] = sum_q w_Q^{q k2} w_R^{q k1} sum_p v[m] w_P^{p k1}
        constexpr int P = Split<R>::P, Q = Split<R>::Q;
        double2 t[Q][P];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
#pragma unroll
            for (int pp = 0; pp < P; ++pp) t[q][pp] = v[q + Q * pp];
            dft_reg<P>(t[q]);
#pragma unroll
            for (int k1 = 1; k1 < P; ++k1)
                if ((q * k1) % R) t[q][k1] = cmul(t[q][k1], kW[R][(q * k1) % R]);
        }
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) {
            double2 u[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) u[q] = t[q][k1];
            dft_reg<Q>(u);
#pragma unroll
            for (int k2 = 0; k2 < Q; ++k2) v[k1 + P * k2] = u[k2];
        }
    }
}

// shared-memory cell of element i: one pad cell per 16 keeps the stride-16
// stage-1 stores conflict-free
__device__ __forceinline__ int padx(int i) { return i + (i >> 4); }

// ---- bulk-copy ring (cp.async.bulk + mbarrier) for the fold operands
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred done;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
        "@!done bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
}

// One (sequence, residue e) per CTA: N = 16 * 16 * R3 = n / D.
//   fold   y[p] = w_n^{e p} sum_t x[p + t N] w_D^{e t}
//          operands arrive by bulk copy in chunks of NT elements (a ring of
//          kRing slots in the FFT buffer, two halves in flight) and are
//          accumulated into the stage-1 registers p = tid + NT r
//   FFT_N  radix 16 (registers -> smem), radix 16 (smem -> smem),
//          radix R3 (smem -> band outputs in global)
// The D CTAs of one sequence are adjacent in the grid, so the sequence is read
// from HBM once and from L2 D times. Sequences are contiguous (in_elem == 1).
constexpr int kRing = 8, kHalf = kRing / 2;

template <int R3, bool kBulk>
__global__ void __launch_bounds__(16 * R3) k_band_dft(PrunedPass p, const double2* __restrict__ in,
                                                      double2* __restrict__ out,
                                                      const double2* __restrict__ wn,
                                                      const double2* __restrict__ wN) {
    constexpr int N = 256 * R3, NT = 16 * R3;
    static_assert(kRing * NT <= N, "ring must fit in the FFT buffer");
    extern __shared__ __align__(128) double2 buf[];
    __shared__ double2 wDe[64];
    __shared__ __align__(8) uint64_t bar[kRing];
    const int tid = threadIdx.x;
    const int row = blockIdx.x / p.D, e = blockIdx.x - row * p.D;
    const double2* x = in + (int64_t)row * p.in_row;
    const int t0 = p.lo / N, t1 = (p.lo + p.L - 1) / N;
    const int nchunk = (t1 - t0 + 1) * 16;
    // chunk c covers support positions [(t0 + c/16) N - lo + NT (c%16), + NT)
    auto issue = [&](int c) {
        const int slot = c % kRing;
        const int m0 = (t0 + c / 16) * N - p.lo + NT * (c % 16);
        const int a = max(m0, 0), b = min(m0 + NT, p.L);
        if (b > a) {
            const uint32_t bytes = (uint32_t)(b - a) * (uint32_t)sizeof(double2);
            mbar_expect_tx(&bar[slot], bytes);
            bulk_g2s(buf + slot * NT + (a - m0), x + a, bytes, &bar[slot]);
        } else {
            mbar_arrive(&bar[slot]);
        }
    };
    double2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = make_double2(0.0, 0.0);
    if constexpr (kBulk) {
        if (tid == 0) {
            for (int i = 0; i < kRing; ++i) mbar_init(&bar[i], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        for (int t = tid; t < p.D; t += NT) wDe[t] = wn[((e * t) % p.D) * N];
        __syncthreads();
        if (tid == 0)
            for (int c = 0; c < min(kRing, nchunk); ++c) issue(c);

        for (int t = t0; t <= t1; ++t) {
            const double2 wt = wDe[t];
            const int cb = (t - t0) * 16;
    #pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int c = cb + r, slot = r % kRing;  // kRing divides 16
                mbar_wait(&bar[slot], (uint32_t)((c / kRing) & 1));
                const int m = t * N - p.lo + NT * r + tid;
                if ((unsigned)m < (unsigned)p.L) {
                    const double2 a = buf[slot * NT + tid];
                    v[r].x = fma(a.x, wt.x, fma(-a.y, wt.y, v[r].x));
                    v[r].y = fma(a.x, wt.y, fma(a.y, wt.x, v[r].y));
                }
                if ((r + 1) % kHalf == 0) {
                    // this half of the ring is consumed: refill it
                    __syncthreads();
                    if (tid == 0 && c + kRing - kHalf + 1 < nchunk) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        for (int i = 1; i <= kHalf; ++i)
                            if (c + kRing - kHalf + i < nchunk) issue(c + kRing - kHalf + i);
                    }
                }
            }
        }
    } else {
        for (int t = tid; t < p.D; t += NT) wDe[t] = wn[((e * t) % p.D) * N];
        __syncthreads();
        for (int t = t0; t <= t1; ++t) {
            const double2 wt = wDe[t];
            const int base = t * N - p.lo + tid;
            double2 a[16];  // all 16 loads in flight before the first use
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int m = base + NT * r;
                a[r] = (unsigned)m < (unsigned)p.L ? __ldg(x + m) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                v[r].x = fma(a[r].x, wt.x, fma(-a[r].y, wt.y, v[r].x));
                v[r].y = fma(a[r].x, wt.y, fma(a[r].y, wt.x, v[r].y));
            }
        }
    }
    __syncthreads();  // ring reads done before stage 1 reuses the buffer
    if (e) {
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = cmul(v[r], wn[e * (tid + NT * r)]);
    }

    // ---- stage 1: radix 16, Ns = 1
    dft_reg<16>(v);
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[padx(tid * 16 + r)] = v[r];
    __syncthreads();

    // ---- stage 2: radix 16, Ns = 16 (in place: read, sync, write)
    {
        const int j = tid, k = j & 15;
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = buf[padx(j + r * (N / 16))];
#pragma unroll
        for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], wN[r * k * R3]);
        dft_reg<16>(v);
        __syncthreads();
        const int o = (j - k) * 16 + k;
#pragma unroll
        for (int r = 0; r < 16; ++r) buf[padx(o + r * 16)] = v[r];
    }
    __syncthreads();

    // ---- stage 3: radix R3, Ns = 256; outputs k' = j + 256 r -> band
    double2* y = out + (int64_t)row * p.out_row;
    const int half = N / 2;
    for (int j = tid; j < 256; j += NT) {
        double2 u[R3];
#pragma unroll
        for (int r = 0; r < R3; ++r) u[r] = buf[padx(j + r * 256)];
#pragma unroll
        for (int r = 1; r < R3; ++r) u[r] = cmul(u[r], wN[r * j]);
        dft_reg<R3>(u);
#pragma unroll
        for (int r = 0; r < R3; ++r) {
            const int kp = j + 256 * r;
            const int f = p.D * (kp <= half ? kp : kp - N) + e;
            if (f >= -p.b && f <= p.b) y[(int64_t)(f < 0 ? f + p.B : f) * p.out_elem] = u[r];
        }
    }
}

} // namespace

bool make_pruned_pass(int n, int lo, int L, int rows, int forced, PrunedPass& p) {
    p = PrunedPass{};
    p.n = n;
    p.lo = lo;
    p.L = L;
    p.rows = rows;
    p.b = n / 4;
    p.B = 2 * p.b + 1;
    if (lo < 0 || lo + L > n || L <= 0) return false;
    static const int pref[] = {18, 16, 15, 12, 10, 9, 8, 6, 5, 4, 3, 2};
    for (int r3 : pref) {
        if (forced && r3 != forced) continue;
        const int N = 256 * r3;
        if (n % N == 0 && n / N <= 64) {
            p.N = N;
            p.D = n / N;
            p.nstages = 3;
            p.radix[0] = 16;
            p.radix[1] = 16;
            p.radix[2] = r3;
            return true;
        }
    }
    return false;
}

DevBuf<double2> make_twiddles(const PrunedPass& p, cudaStream_t st) {
    // [0, n): e^{+2 pi i q / n}; [n, n + N): e^{+2 pi i q / N}
    std::vector<double2> h((size_t)p.n + p.N);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    auto fill = [&](double2* t, int m) {
        for (int q = 0; q < m; ++q) {
            const long double a = two_pi * (long double)q / (long double)m;
            t[q] = make_double2((double)cosl(a), (double)sinl(a));
        }
    };
    fill(h.data(), p.n);
    fill(h.data() + p.n, p.N);
    DevBuf<double2> d;
    d.upload(h.data(), h.size(), st);
    ck(cudaStreamSynchronize(st), "twiddles");
    return d;
}

namespace {
template <int R3, bool kBulk>
void launch_r3(const PrunedPass& p, const double2* in, double2* out, const double2* w, cudaStream_t st) {
    constexpr int N = 256 * R3;
    const size_t smem = (size_t)(N + N / 16) * sizeof(double2);
    static bool attr = false;  // per instantiation
    if (!attr && smem > 48 * 1024) {
        ck(cudaFuncSetAttribute(k_band_dft<R3, kBulk>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
           "band dft smem");
    }
    attr = true;
    k_band_dft<R3, kBulk><<<(unsigned)((int64_t)p.rows * p.D), 16 * R3, smem, st>>>(p, in, out, w, w + p.n);
}
} // namespace

void launch_pruned_dft(const PrunedPass& p, const double2* in, double2* out, const double2* w,
                       cudaStream_t st) {
    if (p.rows <= 0) return;
    if (p.in_elem != 1) throw Error(3, "pruned dft: sequences must be contiguous");
    static const bool bulk = !(std::getenv("SBD_DFT_FOLD") && std::getenv("SBD_DFT_FOLD")[0] == 'r');
    switch (p.radix[2]) {
        case 2: bulk ? launch_r3<2, true>(p, in, out, w, st) : launch_r3<2, false>(p, in, out, w, st); break;
        case 3: bulk ? launch_r3<3, true>(p, in, out, w, st) : launch_r3<3, false>(p, in, out, w, st); break;
        case 4: bulk ? launch_r3<4, true>(p, in, out, w, st) : launch_r3<4, false>(p, in, out, w, st); break;
        case 5: bulk ? launch_r3<5, true>(p, in, out, w, st) : launch_r3<5, false>(p, in, out, w, st); break;
        case 6: bulk ? launch_r3<6, true>(p, in, out, w, st) : launch_r3<6, false>(p, in, out, w, st); break;
        case 8: bulk ? launch_r3<8, true>(p, in, out, w, st) : launch_r3<8, false>(p, in, out, w, st); break;
        case 9: bulk ? launch_r3<9, true>(p, in, out, w, st) : launch_r3<9, false>(p, in, out, w, st); break;
        case 10: bulk ? launch_r3<10, true>(p, in, out, w, st) : launch_r3<10, false>(p, in, out, w, st); break;
        case 12: bulk ? launch_r3<12, true>(p, in, out, w, st) : launch_r3<12, false>(p, in, out, w, st); break;
        case 15: bulk ? launch_r3<15, true>(p, in, out, w, st) : launch_r3<15, false>(p, in, out, w, st); break;
        case 16: bulk ? launch_r3<16, true>(p, in, out, w, st) : launch_r3<16, false>(p, in, out, w, st); break;
        case 18: bulk ? launch_r3<18, true>(p, in, out, w, st) : launch_r3<18, false>(p, in, out, w, st); break;
        default: throw Error(3, "pruned dft: unsupported radix");
    }
    count_launch();
    ck(cudaGetLastError(), "k_band_dft");
}

} // namespace sbdgpu
