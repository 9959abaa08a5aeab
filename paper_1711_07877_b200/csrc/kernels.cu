// kernels.cu -- sm_100a kernels of the SBD apply path (first correct version).
//
// Stage map (reference file:line -> kernel):
//   plan geometry per point/output  nufft.cpp:163-192     -> k_plan_points / k_plan_outputs
//   SPREAD                          nufft.cpp:229-250     -> k_spread<W>
//   DECONV + INTERP                 nufft.cpp:254-283     -> k_interp<W> (deconv folded into taps)
//   transpose spread/deconv/gather  nufft.cpp:308-361     -> k_spread<W>(deconv) / k_interp<W>
//   direct sum                      nufft.cpp:76-93       -> k_ndft
//   omega-hat multiply              conv_operator.cpp:305 -> fused into k_interp (mult)
//   CSR SpMV q += D f               point_cloud.cpp:116-123 -> k_spmv
//   adjoint q += D^H u              point_cloud.cpp:125-132 -> k_spmv_adjoint
#include <cub/cub.cuh>

#include <climits>
#include <cstring>
#include <type_traits>
#include <cstdlib>

#include "device_common.cuh"
#include "sbd_internal.h"

namespace sbdgpu {

namespace {

using namespace dev;
constexpr double kPi = 3.14159265358979323846;

// Per-point plan arrays (nufft.cpp:163-177), as device functions so the
// procedural xi-side kernels regenerate bitwise the values the plan was built
// from (explicitly rounded operations: no FMA contraction in either place).
__device__ __forceinline__ double2 plan_point_pos(double2 p, const Axis& ax, const Axis& ay) {
    const double px = __dsub_rn(p.x, ax.center);
    const double py = __dsub_rn(p.y, ay.center);
    const double ux = __ddiv_rn(px, ax.gamma);
    const double uy = __ddiv_rn(py, ay.gamma);
    const double two_pi = 2.0 * kPi;
    return make_double2(__ddiv_rn(__dmul_rn(__dadd_rn(ux, kPi), (double)ax.n), two_pi),
                        __ddiv_rn(__dmul_rn(__dadd_rn(uy, kPi), (double)ay.n), two_pi));
}

__device__ __forceinline__ double2 plan_point_pre(double2 p, const Axis& ax, const Axis& ay, double beta) {
    const double px = __dsub_rn(p.x, ax.center);
    const double py = __dsub_rn(p.y, ay.center);
    const double phase = __dadd_rn(__dmul_rn(px, ax.fcenter), __dmul_rn(py, ay.fcenter));
    const double dec = __dmul_rn(__dmul_rn(ax.alpha2, kb_hat(beta, __dmul_rn(ax.alpha2, px))),
                                 __dmul_rn(ay.alpha2, kb_hat(beta, __dmul_rn(ay.alpha2, py))));
    double sn, cs;
    sincos(phase, &sn, &cs);
    return make_double2(__ddiv_rn(cs, dec), __ddiv_rn(sn, dec));
}

__global__ void k_plan_points(const double2* __restrict__ pts, uint64_t n, Axis ax, Axis ay,
                              double beta, double2* __restrict__ t, double2* __restrict__ pre) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double2 p = pts[k];
    t[k] = plan_point_pos(p, ax, ay);
    pre[k] = plan_point_pre(p, ax, ay, beta);
}

// Per-output plan arrays (nufft.cpp:179-192). sgn = sign of the plan.
__device__ __forceinline__ double2 plan_output_pos(double2 f, const Axis& ax, const Axis& ay, double sgn) {
    const double fx = __dmul_rn(sgn, f.x), fy = __dmul_rn(sgn, f.y);
    return make_double2(__dmul_rn(ax.gamma, __dsub_rn(fx, ax.fcenter)),
                        __dmul_rn(ay.gamma, __dsub_rn(fy, ay.fcenter)));
}

__device__ __forceinline__ double2 plan_output_post(double2 f, const Axis& ax, const Axis& ay, double sgn,
                                                    double cxy) {
    const double fx = __dmul_rn(sgn, f.x), fy = __dmul_rn(sgn, f.y);
    const double phase = __dadd_rn(__dmul_rn(ax.center, fx), __dmul_rn(ay.center, fy));
    double sn, cs;
    sincos(phase, &sn, &cs);
    return make_double2(__dmul_rn(cs, cxy), __dmul_rn(sn, cxy));
}

__global__ void k_plan_outputs(const double2* __restrict__ frq, uint64_t n, Axis ax, Axis ay,
                               double sgn, double cxy, double2* __restrict__ s,
                               double2* __restrict__ post) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    const double2 f = frq[v];
    s[v] = plan_output_pos(f, ax, ay, sgn);
    post[v] = plan_output_post(f, ax, ay, sgn, cxy);
}

// Ring node `id` (ring_quadrature.cpp:58-63: rho (cos, sin)(2 pi j / m)); the
// angle is formed as pi * (j * (2 / m)) for sincospi, within 2 ulp of the
// reference's 2 pi j / m.
__device__ __forceinline__ double2 ring_node(uint32_t id, const RingRow* __restrict__ rings, double2* w = nullptr) {
    const RingRow r = rings[(id & ~kRingHalve) >> kRingJBits];
    const uint32_t j = id & ((1u << kRingJBits) - 1u);
    double sn, cs;
    sincospi(__dmul_rn((double)j, r.two_over_m), &sn, &cs);
    if (w) *w = make_double2(r.wre, r.wim);
    return make_double2(__dmul_rn(r.rho, cs), __dmul_rn(r.rho, sn));
}

__global__ void k_ring_nodes(const uint32_t* __restrict__ id, uint64_t n, const RingRow* __restrict__ rings,
                             double2* __restrict__ xi, double2* __restrict__ w) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    double2 wt;
    const double2 p = ring_node(id[k], rings, &wt);
    if (xi) xi[k] = p;
    if (w) w[k] = wt;
}

// max over nodes of |a - b| / max(|a|, tiny) as ordered uint64 bits
__global__ void k_node_deviation(const double2* __restrict__ a, const double2* __restrict__ b, uint64_t n,
                                 unsigned long long* __restrict__ worst) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    double d = 0.0;
    if (k < n) {
        const double2 p = a[k], q = b[k];
        const double mag = fmax(sqrt(p.x * p.x + p.y * p.y), 1e-300);
        d = sqrt((p.x - q.x) * (p.x - q.x) + (p.y - q.y) * (p.y - q.y)) / mag;
        if (!(d == d)) d = 1e300;
    }
    for (int o = 16; o; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    if ((threadIdx.x & 31) == 0 && d > 0.0) atomicMax(worst, (unsigned long long)__double_as_longlong(d));
}

// The materialised plan arrays of procedural nodes in one kernel order:
// grid coordinates + prephase (point side) or mode coordinates + postphase
// (output side), and kappa = omega-hat * prephase (halved nodes at 1/2 in kh).
__global__ void k_ring_point_arrays(NodeGen gen, uint64_t n, double2* __restrict__ t, double2* __restrict__ pre) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double2 p = ring_node(gen.id[k], gen.rings);
    if (t) t[k] = plan_point_pos(p, gen.px, gen.py);
    if (pre) pre[k] = plan_point_pre(p, gen.px, gen.py, gen.pbeta);
}

__global__ void k_ring_output_arrays(NodeGen gen, uint64_t n, double2* __restrict__ s, double2* __restrict__ post,
                                     double2* __restrict__ kappa, double2* __restrict__ kappa_h) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t id = gen.id[k];
    double2 w;
    const double2 p = ring_node(id, gen.rings, &w);
    if (s) s[k] = plan_output_pos(p, gen.ox, gen.oy, gen.osgn);
    if (post) post[k] = plan_output_post(p, gen.ox, gen.oy, gen.osgn, gen.ocxy);
    if (kappa || kappa_h) {
        const double2 kp = cmul(w, plan_point_pre(p, gen.px, gen.py, gen.pbeta));
        if (kappa) kappa[k] = kp;
        if (kappa_h) {
            const double h = (id & kRingHalve) ? 0.5 : 1.0;
            kappa_h[k] = make_double2(h * kp.x, h * kp.y);
        }
    }
}

__global__ void k_bin_keys(const double2* __restrict__ pos, uint64_t n, GridGeom g, int tile,
                           uint32_t* __restrict__ keys) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double2 p = pos[k];
    int ix = (int)ceil(p.x - g.half), iy = (int)ceil(p.y - g.half);
    ix = ((ix % g.n1) + g.n1) % g.n1;
    iy = ((iy % g.n2) + g.n2) % g.n2;
    const uint32_t ntx = (uint32_t)((g.n2 + tile - 1) / tile);
    keys[k] = (uint32_t)(ix / tile) * ntx + (uint32_t)(iy / tile);
}

__global__ void k_stencil_extent(const double2* __restrict__ pos, uint64_t n, double half,
                                 int* __restrict__ ext) {
    int a = INT_MAX, b = INT_MIN, c = INT_MAX, d = INT_MIN;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const double2 p = pos[k];
        const int ix = (int)ceil(p.x - half), iy = (int)ceil(p.y - half);
        a = min(a, ix);
        b = max(b, ix);
        c = min(c, iy);
        d = max(d, iy);
    }
    for (int o = 16; o; o >>= 1) {
        a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
        c = min(c, __shfl_xor_sync(0xffffffffu, c, o));
        d = max(d, __shfl_xor_sync(0xffffffffu, d, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(ext + 0, a);
        atomicMax(ext + 1, b);
        atomicMin(ext + 2, c);
        atomicMax(ext + 3, d);
    }
}

// key = tile index << 5 | 4x4 sub-tile index (kTileR = 16, kTileC = 32): points
// consecutive in the sorted order are within a few cells of each other, which
// is what makes 4-point MMA groups compact in the DMMA spread.
__global__ void k_tile_keys(const double2* __restrict__ pos, uint64_t n, double half, TileGeom tg,
                            uint32_t* __restrict__ keys, const uint8_t* __restrict__ tag) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double2 p = pos[k];
    const int rx = (int)ceil(p.x - half) - tg.rlo, ry = (int)ceil(p.y - half) - tg.clo;
    const int bx = rx / tg.tr, by = ry / kTileC;
    const int sub = (((rx % tg.tr) >> 2) * (kTileC >> 2) + ((ry % kTileC) >> 2)) & 31;
    keys[k] = (((uint32_t)bx * (uint32_t)tg.nby + (uint32_t)by) << 5) | (uint32_t)(sub & 31) |
              (tag && tag[k] ? 0x80000000u : 0u);
}

// Region lists of the CTA spread (k_spread_cta<.., LIST>): each point emits
// the 32 x 32 spread regions its stencil overlaps (at most 2 x 2 for W <= 32)
// as (region, entry) pairs, region count for unused slots; a stable sort by
// region then keeps the points of a region in sorted-point order.
__global__ void k_region_pairs(const double2* __restrict__ pos, uint64_t n, double half, int w,
                               TileGeom tg, int ncx, int ncy, uint32_t base, uint32_t tagbit,
                               uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double2 p = pos[k];
    const int rx = (int)ceil(p.x - half) - tg.rlo, ry = (int)ceil(p.y - half) - tg.clo;
    const int x0 = rx >> 5, x1 = (rx + w - 1) >> 5, y0 = ry >> 5, y1 = (ry + w - 1) >> 5;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int cx = x0 + (q >> 1), cy = y0 + (q & 1);
        const bool ok = cx <= x1 && cy <= y1 && cx >= 0 && cy >= 0 && cx < ncx && cy < ncy;
        keys[4 * k + q] = ok ? (uint32_t)cx * (uint32_t)ncy + (uint32_t)cy : (uint32_t)ncx * (uint32_t)ncy;
        vals[4 * k + q] = ((uint32_t)k + base) | tagbit;
    }
}

__global__ void k_shift_keys(uint32_t* __restrict__ keys, uint64_t n) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) keys[i] <<= 5;
}

// start[b] = first sorted position with key >= b, for b in [0, nbins]
__global__ void k_bin_bounds(const uint32_t* __restrict__ key, uint64_t n, uint32_t nbins,
                             uint32_t* __restrict__ start, uint32_t base, uint32_t mask) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    const int64_t prev = i > 0 ? (int64_t)((key[i - 1] & mask) >> 5) : -1;
    const int64_t cur = i < n ? (int64_t)((key[i] & mask) >> 5) : (int64_t)nbins;
    for (int64_t b = prev + 1; b <= cur; ++b) start[b] = base + (uint32_t)i;
}

__device__ __forceinline__ uint32_t spread_bits16(uint32_t v) {
    v &= 0xffffu;
    v = (v | (v << 8)) & 0x00ff00ffu;
    v = (v | (v << 4)) & 0x0f0f0f0fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}

// Morton (Z-order) key of the stencil-start cell, coordinates shifted by
// `shift` to be nonnegative: consecutive sorted outputs share small
// footprints (what the 8-output MMA groups of k_interp_mma rely on).
__global__ void k_morton_keys(const double2* __restrict__ pos, uint64_t n, double half, int shift,
                              uint32_t* __restrict__ keys, const uint8_t* __restrict__ tag) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double2 p = pos[k];
    const int cap = tag ? 32767 : 65535;
    const int ix = min(max((int)ceil(p.x - half) + shift, 0), cap);
    const int iy = min(max((int)ceil(p.y - half) + shift, 0), cap);
    keys[k] = (spread_bits16((uint32_t)ix) << 1) | spread_bits16((uint32_t)iy) |
              (tag && tag[k] ? 0x80000000u : 0u);
}

__global__ void k_iota(uint32_t* v, uint64_t n) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k < n) v[k] = (uint32_t)k;
}

template <typename T>
__global__ void k_gather(const T* __restrict__ src, const uint32_t* __restrict__ perm,
                         T* __restrict__ dst, uint64_t n) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k < n) dst[k] = src[perm[k]];
}

// Spread (nufft.cpp:229-250): one thread per point, fp64 reductions into the
// full grid. b = in * phase (* mult); taps optionally carry deconv factors
// (transpose path, nufft.cpp:328-335).
template <int W>
__global__ void __launch_bounds__(256) k_spread(WindowPoly P, GridGeom g, uint64_t n,
                                                const uint32_t* __restrict__ perm,
                                                const double2* __restrict__ in,
                                                const double2* __restrict__ pos,
                                                const double2* __restrict__ phase,
                                                const double2* __restrict__ mult,
                                                const double* __restrict__ dxt,
                                                const double* __restrict__ dyt,
                                                double2* __restrict__ grid, int conj_in) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    double2 c = in[perm ? perm[k] : k];
    if (conj_in) c.y = -c.y;
    double2 b = cmul(c, phase[k]);
    if (mult) b = cmul(b, mult[k]);
    if (b.x == 0.0 && b.y == 0.0) return;
    const double2 t = pos[k];
    const int ix0 = (int)ceil(t.x - g.half), iy0 = (int)ceil(t.y - g.half);
    double wx[W], wy[W];
    kb_taps<W>((ix0 - t.x) + g.half, P, wx);
    kb_taps<W>((iy0 - t.y) + g.half, P, wy);
    const int mx0 = wrap_base(ix0, g.n1), my0 = wrap_base(iy0, g.n2);
    if (dyt) {
#pragma unroll
        for (int j = 0; j < W; ++j) {
            int my = my0 + j;
            if (my >= g.n2) my -= g.n2;
            wy[j] *= dyt[my];
        }
    }
#pragma unroll
    for (int i = 0; i < W; ++i) {
        int mx = mx0 + i;
        if (mx >= g.n1) mx -= g.n1;
        double wxi = wx[i];
        if (dxt) wxi *= dxt[mx];
        const double bxr = b.x * wxi, bxi = b.y * wxi;
        double* row = reinterpret_cast<double*>(grid + (size_t)mx * g.n2);
#pragma unroll
        for (int j = 0; j < W; ++j) {
            int my = my0 + j;
            if (my >= g.n2) my -= g.n2;
            atomicAdd(row + 2 * my, bxr * wy[j]);
            atomicAdd(row + 2 * my + 1, bxi * wy[j]);
        }
    }
}

// Row accumulation for one staged point whose stencil starts D rows below the
// warp tile's first row: rows r in [max(0,D), min(kTileR, D+W)) get
// acc[r] += (b wx)[r-D] * wy[lane]. D is a template parameter so the row range
// is straight-line code; rows_dispatch picks it with a binary search on d.
template <int W, int TR, int D>
__device__ __forceinline__ void rows_acc(const double2* __restrict__ bwx, double wyl,
                                         double (&ar)[TR], double (&ai)[TR]) {
    constexpr int r0 = D > 0 ? D : 0;
    constexpr int r1 = D + W < TR ? D + W : TR;
#pragma unroll
    for (int r = r0; r < r1; ++r) {
        const double2 v = bwx[r - D];
        ar[r] = fma(v.x, wyl, ar[r]);
        ai[r] = fma(v.y, wyl, ai[r]);
    }
}

template <int W, int TR, int Lo, int Hi>
__device__ __forceinline__ void rows_dispatch(int d, const double2* __restrict__ bwx, double wyl,
                                              double (&ar)[TR], double (&ai)[TR]) {
    if constexpr (Hi - Lo == 1) {
        rows_acc<W, TR, Lo>(bwx, wyl, ar, ai);
    } else {
        constexpr int Mid = (Lo + Hi) / 2;
        if (d < Mid)
            rows_dispatch<W, TR, Lo, Mid>(d, bwx, wyl, ar, ai);
        else
            rows_dispatch<W, TR, Mid, Hi>(d, bwx, wyl, ar, ai);
    }
}

// Tile-owned spread (nufft.cpp:229-250 restated output-stationary). One warp
// owns a kTileR x kTileC block of grid cells: lane = column, the kTileR rows of
// that column live in registers. The warp scans the points binned in its own
// tile and the three tiles above/left of it (a stencil starting there can
// reach into this tile), queues the intersecting ones, evaluates their
// windows 32 at a time (lane = point; b*wx and wy go to the warp's
// shared-memory slice), then accumulates acc[r] += (b wx)[row] * wy[lane]
// point by point. Every cell of the tile is written exactly once: no atomics
// and no zero-fill of the grid.
template <int W, int TR>
__global__ void __launch_bounds__(128, TR == 16 ? 4 : 5) k_spread_tiles(WindowPoly P, GridGeom g, TileGeom tg,
                                                      const uint32_t* __restrict__ bin_start,
                                                      const double2* __restrict__ bsorted,
                                                      const double2* __restrict__ pos,
                                                      double2* __restrict__ grid,
                                                      const uint32_t* __restrict__ bin_start2,
                                                      const int* __restrict__ herm) {
    extern __shared__ double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per warp: bwx[32*W] (double2), wy[32*W] (double), queue k[64], ix[32], iy[32]
    double2* s_bwx = reinterpret_cast<double2*>(smem) + warp * 32 * W;
    double* s_wy = smem + 4 * 64 * W + warp * 32 * W;
    uint32_t* s_q = reinterpret_cast<uint32_t*>(smem + 4 * 96 * W) + warp * 128;
    int* s_ix = reinterpret_cast<int*>(s_q + 64);
    int* s_iy = s_ix + 32;
    const int tile = blockIdx.x * 4 + warp;
    if (tile >= tg.nbx * tg.nby) return;
    const int bx = tile / tg.nby, by = tile - (tile / tg.nby) * tg.nby;
    const int X0 = tg.rlo + bx * TR, Y0 = tg.clo + by * kTileC;
    double ar[TR], ai[TR];
#pragma unroll
    for (int r = 0; r < TR; ++r) ar[r] = ai[r] = 0.0;

    int queued = 0; // warp-uniform
    // Evaluate windows for the first n (<= 32) queued points and accumulate them.
    auto flush = [&](int n) {
        if (lane < n) {
            const uint32_t k = s_q[lane];
            const double2 t = pos[k];
            const int ix0 = (int)ceil(t.x - g.half), iy0 = (int)ceil(t.y - g.half);
            const double2 b2 = bsorted[k];
            s_ix[lane] = ix0 - X0;
            s_iy[lane] = iy0;
            double2* bw = s_bwx + lane * W;
            double* wyp = s_wy + lane * W;
            kb_taps_each<W>((ix0 - t.x) + g.half, P,
                            [&](int i, double v) { bw[i] = make_double2(b2.x * v, b2.y * v); });
            kb_taps_each<W>((iy0 - t.y) + g.half, P, [&](int i, double v) { wyp[i] = v; });
        }
        __syncwarp();
        for (int p = 0; p < n; ++p) {
            const int d = s_ix[p];
            const int jl = Y0 + lane - s_iy[p];
            const double wyl = (unsigned)jl < (unsigned)W ? s_wy[p * W + jl] : 0.0;
            rows_dispatch<W, TR, 1 - W, TR>(d, s_bwx + p * W, wyl, ar, ai);
        }
        __syncwarp();
    };

    const int nq = (bin_start2 && !(herm && *herm)) ? 8 : 4;
    for (int q = 0; q < nq; ++q) {
        const int cbx = bx - ((q >> 1) & 1), cby = by - (q & 1);
        if (cbx < 0 || cby < 0) continue;
        const int b = cbx * tg.nby + cby;
        const uint32_t* bs = q < 4 ? bin_start : bin_start2;
        const uint32_t s0 = bs[b], s1 = bs[b + 1];
        for (uint32_t s = s0; s < s1; s += 32) {
            const uint32_t k = s + lane;
            bool take = false;
            if (k < s1) {
                const double2 t = pos[k];
                const int ix0 = (int)ceil(t.x - g.half), iy0 = (int)ceil(t.y - g.half);
                take = ix0 < X0 + TR && ix0 + W > X0 && iy0 < Y0 + kTileC && iy0 + W > Y0;
            }
            const unsigned m = __ballot_sync(0xffffffffu, take);
            if (take) s_q[queued + __popc(m & ((1u << lane) - 1u))] = k;
            queued += __popc(m);
            __syncwarp();
            if (queued >= 32) {
                flush(32);
                if (lane < queued - 32) s_q[lane] = s_q[32 + lane];
                queued -= 32;
                __syncwarp();
            }
        }
    }
    if (queued) flush(queued);
    const int col = Y0 + lane;
    const int rend = tg.pitch ? tg.rhi : g.n1, cend = tg.pitch ? tg.chi : g.n2;
    const size_t pitch = tg.pitch ? (size_t)tg.pitch : (size_t)g.n2;
    const int r0 = tg.pitch ? tg.rlo : 0, c0 = tg.pitch ? tg.clo : 0;
    if (lane < kTileC && col < cend) {
#pragma unroll
        for (int r = 0; r < TR; ++r) {
            const int row = X0 + r;
            if (row < rend) grid[(size_t)(row - r0) * pitch + (col - c0)] = make_double2(ar[r], ai[r]);
        }
    }
}

// reflection m -> -m (mod n). The image's stencil must be exactly the mirror
// of the point's (start n - s - w + 1 for start s = ceil(t - w/2)); when
// rounding puts ceil(t' - w/2) one cell off (t - w/2 within an ulp of an
// integer), t' is nudged by ulps, which moves the taps by rounding only.
__device__ __forceinline__ double mirror_coord(double t, int n, int w) {
    const double h = 0.5 * w;
    const int want = n - (int)ceil(t - h) - w + 1;
    double m = (double)n - t;
    for (int it = 0; it < 8 && (int)ceil(m - h) > want; ++it) m = nextafter(m, -1e300);
    for (int it = 0; it < 8 && (int)ceil(m - h) < want; ++it) m = nextafter(m, 1e300);
    return m;
}

// coefficient of mirror image k (second point set): conj of its tag-0
// partner's coefficient when the partner map is given, else stored
__device__ __forceinline__ double2 mirror_coef(const SpreadOut& so, const double2* __restrict__ b,
                                               uint32_t k) {
    if (so.src2) {
        const double2 v = b[so.src2[k]];
        return make_double2(v.x, -v.y);
    }
    return so.b2[k];
}

// storage position of mode j of a column transformed by a radix-r first pass
// (k_untangle_dif): (j mod r) M + j / r, the quotient by multiply-high
__device__ __forceinline__ int rad_pos(const GridGeom& g, int j) {
    if (g.rad <= 1) return j;
    const int q = (int)__umulhi((unsigned)j, g.rad_magic);
    return (j - q * g.rad) * g.rad_m + q;
}

// fp64 tensor-core MMA: D(8x8) = A(8x4) B(4x8) + C (mma.sync m8n8k4 f64; SASS
// DMMA.8x8x4). Fragments: a = A[lane/4][lane%4], b = B[lane%4][lane/4],
// c = {C[lane/4][2(lane%4)], C[lane/4][2(lane%4)+1]}.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Spread on the fp64 tensor cores. Same tile ownership as k_spread_tiles (one
// warp owns 16 x 32 cells, every cell written once), but the accumulation is
// a sequence of 8x8x4 MMAs: for a group of 4 staged points,
//   G[8 rows x 8 cols] += A[8 rows x 4 pts] B[4 pts x 8 cols],
//   A[r][k] = (b_k wx_k)(row r) (real and imaginary parts: two MMAs),
//   B[k][c] = wy_k(col c),
// issued only for the 8x8 sub-tiles the group's stencils touch. One DMMA does
// 256 multiply-adds, which removes the instruction-issue bound of the scalar
// version; points are sorted by 4x4 sub-tile so a group's footprint is small.
template <int W>
__global__ void __launch_bounds__(128, 4) k_spread_mma(WindowPoly P, GridGeom g, TileGeom tg,
                                                    const uint32_t* __restrict__ bin_start,
                                                    const double2* __restrict__ bsorted,
                                                    const double2* __restrict__ pos,
                                                    double2* __restrict__ grid,
                                                      const uint32_t* __restrict__ bin_start2,
                                                      const int* __restrict__ herm, SpreadOut so) {
    constexpr int TR = 16;
    extern __shared__ double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* s_bwx = reinterpret_cast<double2*>(smem) + warp * 32 * W;
    double* s_wy = smem + 4 * 64 * W + warp * 32 * W;
    uint32_t* s_q = reinterpret_cast<uint32_t*>(smem + 4 * 96 * W) + warp * 128;
    int* s_ix = reinterpret_cast<int*>(s_q + 64);
    int* s_iy = s_ix + 32;
    const int tile = blockIdx.x * 4 + warp;
    const int nrun = so.nby_run;  // tile columns run (a prefix of the tg.nby columns)
    if (tile >= tg.nbx * nrun) return;
    const int bx = tile / nrun, by = tile - (tile / nrun) * nrun;
    const int X0 = tg.rlo + bx * TR, Y0 = tg.clo + by * kTileC;
    const int gid = lane >> 2, kq = lane & 3;
    constexpr int NJ = kTileC / 8;
    double cr[2][NJ][2], ci[2][NJ][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

    // 8 tiles x 32 list entries per warp, after all four warps' queues
    uint32_t* s_list = reinterpret_cast<uint32_t*>(smem + 4 * 96 * W) + 4 * 128 + warp * 256;
    int queued = 0;
    // Evaluate the windows of the first n queued points (lane = point), build
    // per-8x8-tile lists of the points whose stencil reaches that tile, and
    // feed each tile's list to the tensor cores 4 points at a time.
    auto flush = [&](int n) {
        int dx = -4 * W, dy = -4 * W;
        if (lane < n) {
            const uint32_t e = s_q[lane];
            const uint32_t k = e & 0x7fffffffu;  // bit 31: second point set
            const double2 t = (e >> 31) ? so.pos2[k] : pos[k];
            const int ix0 = (int)ceil(t.x - g.half), iy0 = (int)ceil(t.y - g.half);
            const double2 b2 = (e >> 31) ? mirror_coef(so, bsorted, k) : bsorted[k];
            dx = ix0 - X0;
            dy = iy0 - Y0;
            double2* bw = s_bwx + lane * W;
            double* wyp = s_wy + lane * W;
            kb_taps_each<W>((ix0 - t.x) + g.half, P,
                            [&](int i, double v) { bw[i] = make_double2(b2.x * v, b2.y * v); });
            kb_taps_each<W>((iy0 - t.y) + g.half, P, [&](int i, double v) { wyp[i] = v; });
        }
        const uint32_t packed = (uint32_t)lane | ((uint32_t)(dx + 64) << 8) | ((uint32_t)(dy + 64) << 16);
        int cnt[2 * NJ];
#pragma unroll
        for (int t = 0; t < 2 * NJ; ++t) {
            const int i = t / NJ, j = t % NJ;
            const bool hit = dx < 8 * i + 8 && dx + W > 8 * i && dy < 8 * j + 8 && dy + W > 8 * j;
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (hit) s_list[t * 32 + __popc(m & ((1u << lane) - 1u))] = packed;
            cnt[t] = __popc(m);
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 2 * NJ; ++t) {
            const int i = t / NJ, j = t % NJ;
            for (int grp = 0; grp < cnt[t]; grp += 4) {
                const int idx = grp + kq;
                double a_r = 0.0, a_i = 0.0, bv = 0.0;
                if (idx < cnt[t]) {
                    const uint32_t e = s_list[t * 32 + idx];
                    const int node = e & 255;
                    const int rr = 8 * i + gid - ((int)((e >> 8) & 255) - 64);
                    const int cc = 8 * j + gid - ((int)(e >> 16) - 64);
                    if ((unsigned)rr < (unsigned)W) {
                        const double2 v = s_bwx[node * W + rr];
                        a_r = v.x;
                        a_i = v.y;
                    }
                    if ((unsigned)cc < (unsigned)W) bv = s_wy[node * W + cc];
                }
                dmma(cr[i][j][0], cr[i][j][1], a_r, bv);
                if (so.mode < 3) dmma(ci[i][j][0], ci[i][j][1], a_i, bv);  // mode 3: real grid
            }
        }
        __syncwarp();
    };

    const int nq = (bin_start2 && !(herm && *herm)) ? 8 : 4;
    for (int q = 0; q < nq; ++q) {
        const int cbx = bx - ((q >> 1) & 1), cby = by - (q & 1);
        if (cbx < 0 || cby < 0) continue;
        const int b = cbx * tg.nby + cby;
        const uint32_t* bs = q < 4 ? bin_start : bin_start2;
        const uint32_t s0 = bs[b], s1 = bs[b + 1];
        const bool second = q >= 4 && so.pos2;
        const double2* P2 = second ? so.pos2 : pos;
        const uint32_t tagbit = second ? 0x80000000u : 0u;
        for (uint32_t s = s0; s < s1; s += 128) {
            // four independent position loads in flight per lane
            double2 tt[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t k = s + 32 * u + lane;
                tt[u] = k < s1 ? P2[k] : make_double2(-1e30, -1e30);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t k = s + 32 * u + lane;
                const int ix0 = (int)ceil(tt[u].x - g.half), iy0 = (int)ceil(tt[u].y - g.half);
                const bool take = k < s1 && ix0 < X0 + TR && ix0 + W > X0 && iy0 < Y0 + kTileC &&
                                  iy0 + W > Y0;
                const unsigned m = __ballot_sync(0xffffffffu, take);
                if (take) s_q[queued + __popc(m & ((1u << lane) - 1u))] = k | tagbit;
                queued += __popc(m);
                __syncwarp();
                if (queued >= 32) {
                    flush(32);
                    if (lane < queued - 32) s_q[lane] = s_q[32 + lane];
                    queued -= 32;
                    __syncwarp();
                }
            }
        }
    }
    if (queued) flush(queued);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int row = X0 + 8 * i + gid;
        if (row >= so.rend) continue;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int col = Y0 + 8 * j + 2 * kq;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (col + h >= so.cend) continue;
                const double re = cr[i][j][h], im = ci[i][j][h];
                if (so.mode == 0)
                    grid[(size_t)(row - so.r0) * so.pitch + (col + h - so.c0)] = make_double2(re, im);
                else if (so.mode == 1)  // real grid rows (the imaginary part is zero)
                    so.rgrid[(size_t)(row - so.r0) * so.pitch + (col + h - so.c0)] = re;
                else if (so.mode == 3)  // real rows packed in pairs: row 2k -> .x, 2k+1 -> .y of row k
                    so.rgrid[2 * ((size_t)((row - so.r0) >> 1) * so.pitch + (col + h - so.c0)) +
                             ((row - so.r0) & 1)] = re;
                else  // transposed: column-major, full-length columns
                    grid[(size_t)(col + h - so.c0) * so.pitch + (row - so.r0)] = make_double2(re, im);
            }
        }
    }
}

// Window taps i in [I0, I1) of the pairs (i, W-1-i), plus the middle tap when
// MID (odd W): a slice of kb_taps_each, for splitting one point over threads.
template <int W, int I0, int I1, bool MID, typename F>
__device__ __forceinline__ void kb_taps_slice(double u, const WindowPoly& P, F&& f) {
    const double v = 2.0 * u - 1.0;
    const double v2 = v * v;
#pragma unroll
    for (int i = I0; i < I1; ++i) {
        double e = P.e[i][kHorner - 1], o = P.o[i][kHorner - 1];
#pragma unroll
        for (int h = kHorner - 2; h >= 0; --h) {
            e = fma(e, v2, P.e[i][h]);
            o = fma(o, v2, P.o[i][h]);
        }
        f(i, fma(v, o, e));
        f(W - 1 - i, fma(-v, o, e));
    }
    if (MID && (W & 1)) {
        constexpr int m = W / 2;
        double e = P.e[m][kHorner - 1];
#pragma unroll
        for (int h = kHorner - 2; h >= 0; --h) e = fma(e, v2, P.e[m][h]);
        f(m, e);
    }
}

// CTA-cooperative DMMA spread (default). One CTA owns a 32 x 32 cell region:
// four 16 x 16 warp tiles with the accumulators of k_spread_mma in registers.
// Against the per-warp kernel it
//  * scans the 3 x 3 bins that can reach the region once per CTA, as one
//    flattened candidate stream (the two point sets and all nine bins in
//    128-candidate chunks), compacting the hits into a shared ring in block
//    prefix order (deterministic: applies stay bitwise reproducible);
//  * evaluates each queued point's taps once for all four warps (a point is
//    staged (1 + (W-1)/32)^2 ~ 1.7 times instead of (1 + (W-1)/16)^2 ~ 2.6),
//    two threads per point (x taps times the coefficient, y taps);
//  * stores the taps in zero-padded rows (7 zeros, W taps, 7 zeros) and
//    gives every (point, 8 x 8 sub-tile) list entry the row offsets of its
//    fragments, so the MMA loop is a list load, two fragment loads and the
//    DMMAs -- no bounds checks (lists are padded to a multiple of 4 with an
//    all-zero point).
constexpr int kSCB = 32;   // points per staged batch (one per lane; keeps 7 CTAs per SM resident)
constexpr int kSCQ = 256;  // candidate ring (>= kSCB - 1 + 128)
constexpr int kSCS = 18;   // scan segments: 2 point sets x 3 x 3 bins

template <int W>
struct SCta {
    static constexpr int L = W + 14;     // padded tap row (y taps)
    static constexpr int LA = W + 15;    // x-tap row: one more cell for the even-start shift
    static constexpr int NP = kSCB + 1;  // staged points + the zero point
    static constexpr int LS = kSCB + 4;  // list stride (room for the padding)
    static constexpr size_t smem = (size_t)NP * (LA * sizeof(double2) + L * sizeof(double)) +
                                   (size_t)kSCQ * 2 * sizeof(double2) + (size_t)16 * LS * 4 +
                                   (size_t)2 * kSCB * 4;
    static constexpr size_t smem_list = smem - (size_t)kSCQ * 2 * sizeof(double2);  // LIST: no ring
};

// PROC (LIST only): the points are procedural ring nodes -- their grid
// coordinates are regenerated from so.gen.id (a mirror image's from its tag-0
// partner) instead of read from pos / so.pos2.
template <int W, bool CPLX, bool LIST, bool PROC = false>
__global__ void __launch_bounds__(128, LIST ? (CPLX ? 8 : 9) : 7) k_spread_cta(WindowPoly P, GridGeom g, TileGeom tg,
                                                     const uint32_t* __restrict__ bin_start,
                                                     const double2* __restrict__ bsorted,
                                                     const double2* __restrict__ pos,
                                                     double2* __restrict__ grid,
                                                     const uint32_t* __restrict__ bin_start2,
                                                     const int* __restrict__ herm, SpreadOut so) {
    using S = SCta<W>;
    constexpr int L = S::L;
    // b * x taps: complex for a complex grid, one double for a real one (half
    // the A-fragment shared-memory traffic of the real spread)
    using AT = typename std::conditional<CPLX, double2, double>::type;
    extern __shared__ __align__(16) double smem_sc[];
    AT* sA = reinterpret_cast<AT*>(smem_sc);            // [NP][LA]: b * x taps
    constexpr size_t kABytes = ((size_t)S::NP * S::LA * sizeof(AT) + 15) & ~(size_t)15;
    double2* sQt = reinterpret_cast<double2*>(reinterpret_cast<char*>(smem_sc) + kABytes);  // queued positions
    double2* sQb = sQt + (LIST ? 0 : kSCQ);              // queued coefficients (scan mode only)
    double* sB = reinterpret_cast<double*>(sQb + (LIST ? 0 : kSCQ));  // [NP][L]: y taps
    uint32_t* sL = reinterpret_cast<uint32_t*>(sB + S::NP * L);  // [4 warps][4 sub-tiles][LS]
    // per staged point: fragment row base << 4 | mask of the region's 4
    // sub-tile rows (x) / columns (y) its stencil covers
    int* sDX = reinterpret_cast<int*>(sL + 16 * S::LS);
    int* sDY = sDX + kSCB;
    __shared__ int sCnt[4];
    __shared__ uint32_t sSeg[kSCS], sPre[kSCS + 1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gid = lane >> 2, kq = lane & 3;
    const int nrun = so.nby_run;
    const int ncy = (nrun + 1) >> 1;
    const int cx = blockIdx.x / ncy + so.cx0, cy = blockIdx.x - (blockIdx.x / ncy) * ncy;
    const int X0 = tg.rlo + cx * 32, Y0 = tg.clo + cy * kTileC * 2;
    // warp w owns the 8 x 8 sub-tiles (wr + 2p, wc + 2q), p, q in {0, 1}, of the
    // region's 4 x 4: every stencil (>= 2 sub-tiles wide) feeds all four warps,
    // so a batch of neighbouring points loads them evenly
    const int wr = warp >> 1, wc = warp & 1;
    const unsigned lt = (1u << lane) - 1u;

    for (int i = tid; i < S::NP * S::LA; i += 128) {
        sA[i] = AT{};
        if (i < S::NP * L) sB[i] = 0.0;
    }
    // scan segments: (set, bin) -> [first sorted position, size), prefix sums
    if (!LIST && warp == 0) {
        uint32_t k0 = 0, sz = 0;
        const bool use2 = bin_start2 && !(herm && *herm);
        if (lane < kSCS) {
            const int set = lane / 9, qb = lane % 9;
            const int cbx = 2 * cx - 1 + qb / 3, cby = 2 * cy - 1 + qb % 3;
            if ((set == 0 || use2) && cbx >= 0 && cby >= 0 && cbx < tg.nbx && cby < tg.nby) {
                const uint32_t* bs = set ? bin_start2 : bin_start;
                const uint32_t b = (uint32_t)cbx * (uint32_t)tg.nby + (uint32_t)cby;
                k0 = bs[b];
                sz = bs[b + 1] - k0;
            }
            const bool second = set && so.pos2;
            sSeg[lane] = k0 | (second ? 0x80000000u : 0u);
        }
        uint32_t inc = sz;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        if (lane < kSCS) sPre[lane + 1] = inc;
        if (lane == 0) sPre[0] = 0;
    }
    double cr[2][2][2], ci[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
    __syncthreads();

    uint32_t head = 0, tail = 0;  // ring positions (uniform across the CTA)
    // t, b2: position and coefficient of point (tid & 63) of the batch
    auto flush = [&](int n, double2 t, double2 b2) {
        // 1. taps: warp -> (axis, half of the tap pairs), lane -> point
        {
            const int p = lane;
            constexpr int H = (W / 2 + 1) / 2;  // pairs [0, H) | [H, W/2) + middle
            if (p < n) {
                if (warp < 2) {
                    const int ix0 = (int)ceil(t.x - g.half);
                    const double u = (ix0 - t.x) + g.half;
                    // every A-fragment read of this point starts on an even
                    // 16-byte bank group (the row shifted by one cell when
                    // needed): a quarter-warp's 4 points x 2 rows then fall in
                    // aligned bank-group pairs (fewer conflicts)
                    const int dx = ix0 - X0;  // in [1 - W, 32)
                    const int sh = (p * S::LA - dx + 7) & 1;
                    AT* a = sA + p * S::LA + sh + 7;
                    auto put = [&](int i, double v) {
                        if constexpr (CPLX)
                            a[i] = make_double2(b2.x * v, b2.y * v);
                        else
                            a[i] = b2.x * v;
                    };
                    if (warp == 0) {
                        const int r0 = max(0, ((dx + 64) >> 3) - 8), r1 = min(3, ((dx + W - 1 + 64) >> 3) - 8);
                        sDX[p] = ((p * S::LA + sh - dx + 7) << 4) | (((2 << r1) - 1) & ~((1 << r0) - 1));
                        a[-1] = AT{};  // a previous batch's tap one cell before ...
                        kb_taps_slice<W, 0, H, false>(u, P, put);
                    } else {
                        a[W] = AT{};   // ... or one cell after
                        kb_taps_slice<W, H, W / 2, true>(u, P, put);
                    }
                } else {
                    const int iy0 = (int)ceil(t.y - g.half);
                    const double u = (iy0 - t.y) + g.half;
                    double* bb = sB + p * L + 7;
                    auto put = [&](int i, double v) { bb[i] = v; };
                    if (warp == 2) {
                        const int dy = iy0 - Y0;
                        const int c0 = max(0, ((dy + 64) >> 3) - 8), c1 = min(3, ((dy + W - 1 + 64) >> 3) - 8);
                        sDY[p] = ((p * L - dy + 7) << 4) | (((2 << c1) - 1) & ~((1 << c0) - 1));
                        kb_taps_slice<W, 0, H, false>(u, P, put);
                    } else {
                        kb_taps_slice<W, H, W / 2, true>(u, P, put);
                    }
                }
            }
        }
        __syncthreads();
        // 2. this warp's four sub-tile lists: fragment row offsets per entry
        uint32_t* lst = sL + warp * 4 * S::LS;
        int cnt[4] = {0, 0, 0, 0};
#pragma unroll
        for (int h = 0; h < (kSCB + 31) / 32; ++h) {
            const int p = h * 32 + lane;
            int ex = 0, ey = 0;
            if (p < n) {
                ex = sDX[p] >> wr;  // row mask bit 0 = sub-tile row wr
                ey = sDY[p] >> wc;
                ex = (ex & 0xf) | ((sDX[p] >> 4) + 8 * wr) << 4;
                ey = (ey & 0xf) | ((sDY[p] >> 4) + 8 * wc) << 4;
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int i = 2 * (t >> 1), j = 2 * (t & 1);  // sub-tile (wr + i, wc + j)
                const bool hit = (ex >> i) & (ey >> j) & 1;
                const unsigned m = __ballot_sync(0xffffffffu, hit);
                if (hit)
                    lst[t * S::LS + cnt[t] + __popc(m & lt)] =
                        (uint32_t)((ex >> 4) + 8 * i) | ((uint32_t)((ey >> 4) + 8 * j) << 16);
                cnt[t] += __popc(m);
            }
        }
        constexpr uint32_t zero = (uint32_t)(kSCB * S::LA) | ((uint32_t)(kSCB * L) << 16);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (lane < ((-cnt[t]) & 3)) lst[t * S::LS + cnt[t] + lane] = zero;
            cnt[t] = (cnt[t] + 3) & ~3;
        }
        __syncwarp();
        // 3. G[8 x 8] += A[8 x 4] B[4 x 8] per sub-tile, 4 listed points at a time
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int i = t >> 1, j = t & 1;
            const uint32_t* lt4 = lst + t * S::LS + kq;
            for (int grp = 0; grp < cnt[t]; grp += 4) {
                const uint32_t e = lt4[grp];
                const AT a = sA[(e & 0xffffu) + gid];
                const double bv = sB[(e >> 16) + gid];
                if constexpr (CPLX) {
                    dmma(cr[i][j][0], cr[i][j][1], a.x, bv);
                    dmma(ci[i][j][0], ci[i][j][1], a.y, bv);
                } else {
                    dmma(cr[i][j][0], cr[i][j][1], a, bv);
                }
            }
        }
        __syncthreads();  // staged rows, starts and lists are rewritten next batch
    };

    if (LIST) {
        // plan-time region lists (SpreadLists): the batches are the region's
        // entries in order, positions and coefficients loaded one batch ahead
        const uint32_t region = (uint32_t)cx * (uint32_t)so.lists.ncy + (uint32_t)cy;
        const uint32_t s1 = so.lists.s1[region], e1 = so.lists.s1[region + 1];
        uint32_t s2 = 0, e2 = 0;
        if (so.lists.s2 && !(herm && *herm)) {
            s2 = so.lists.s2[region];
            e2 = so.lists.s2[region + 1];
        }
        const uint32_t n1 = e1 - s1, nall = n1 + (e2 - s2);
        const int p = lane;
        // two-stage prefetch: list entries two batches ahead, positions and
        // coefficients one batch ahead
        auto entry = [&](uint32_t q0) -> uint32_t {
            const uint32_t q = q0 + p;
            if (q >= nall) return 0xffffffffu;
            return q < n1 ? so.lists.e1[s1 + q] : so.lists.e2[s2 + (q - n1)];
        };
        auto fetch = [&](uint32_t e, double2& t, double2& b2) {
            if (e != 0xffffffffu) {
                const uint32_t k = e & 0x7fffffffu;
                if constexpr (PROC) {
                    const uint32_t kp = (e >> 31) ? so.src2[k] : k;
                    t = plan_point_pos(ring_node(so.gen.id[kp], so.gen.rings), so.gen.px, so.gen.py);
                    if (e >> 31) t = make_double2(mirror_coord(t.x, g.n1, W), mirror_coord(t.y, g.n2, W));
                } else {
                    t = (e >> 31) ? so.pos2[k] : pos[k];
                }
                if (warp < 2) b2 = (e >> 31) ? mirror_coef(so, bsorted, k) : bsorted[k];
            }
        };
        double2 tn = make_double2(0.0, 0.0), bn = tn;
        uint32_t en = entry(kSCB);
        fetch(entry(0), tn, bn);
        for (uint32_t q0 = 0; q0 < nall; q0 += kSCB) {
            const double2 t = tn, b2 = bn;
            fetch(en, tn, bn);
            en = entry(q0 + 2 * kSCB);
            flush((int)min((uint32_t)kSCB, nall - q0), t, b2);
        }
    } else {
        const uint32_t total = sPre[kSCS];
        constexpr int kU = 2;  // candidate loads in flight per thread
        int seg = 0;           // segment of the current sub-chunk's first candidate (uniform)
        for (uint32_t s = 0; s < total; s += 128 * kU) {
            double2 tt[kU], tb[kU];
            uint32_t ent[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t i = s + u * 128 + tid;
                ent[u] = 0xffffffffu;
                tt[u] = make_double2(-1e30, -1e30);
                while (seg < kSCS - 1 && s + u * 128 >= sPre[seg + 1]) ++seg;
                if (i < total) {
                    int sg = seg;
                    while (i >= sPre[sg + 1]) ++sg;
                    const uint32_t e0 = sSeg[sg];
                    const uint32_t k = (e0 & 0x7fffffffu) + (i - sPre[sg]);
                    tt[u] = (e0 >> 31) ? so.pos2[k] : pos[k];
                    tb[u] = (e0 >> 31) ? mirror_coef(so, bsorted, k) : bsorted[k];
                    ent[u] = k | (e0 & 0x80000000u);
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                if (s + u * 128 >= total) break;  // uniform
                const int ix0 = (int)ceil(tt[u].x - g.half), iy0 = (int)ceil(tt[u].y - g.half);
                const bool take = ent[u] != 0xffffffffu && ix0 < X0 + 32 && ix0 + W > X0 && iy0 < Y0 + 32 &&
                                  iy0 + W > Y0;
                const unsigned m = __ballot_sync(0xffffffffu, take);
                if (lane == 0) sCnt[warp] = __popc(m);
                __syncthreads();
                int off = 0, tot = 0;
#pragma unroll
                for (int w2 = 0; w2 < 4; ++w2) {
                    const int c = sCnt[w2];
                    off += w2 < warp ? c : 0;
                    tot += c;
                }
                if (take) {
                    const uint32_t slot = (tail + off + __popc(m & lt)) & (kSCQ - 1);
                    sQt[slot] = tt[u];
                    sQb[slot] = tb[u];
                }
                tail += tot;
                __syncthreads();
                while (tail - head >= (uint32_t)kSCB) {
                    flush(kSCB, sQt[(head + lane) & (kSCQ - 1)], sQb[(head + lane) & (kSCQ - 1)]);
                    head += kSCB;
                }
            }
        }
        if (tail != head) {
            flush((int)(tail - head), sQt[(head + lane) & (kSCQ - 1)], sQb[(head + lane) & (kSCQ - 1)]);
        }
    }


#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int row = X0 + 8 * (wr + 2 * i) + gid;
        if (row >= so.rend || 2 * cx + i >= tg.nbx) continue;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            if (2 * cy + j >= nrun) continue;
            const int col = Y0 + 8 * (wc + 2 * j) + 2 * kq;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (col + h >= so.cend) continue;
                const double re = cr[i][j][h], im = CPLX ? ci[i][j][h] : 0.0;
                if (so.mode == 0)
                    grid[(size_t)(row - so.r0) * so.pitch + (col + h - so.c0)] = make_double2(re, im);
                else if (so.mode == 1)
                    so.rgrid[(size_t)(row - so.r0) * so.pitch + (col + h - so.c0)] = re;
                else if (so.mode == 3)
                    so.rgrid[2 * ((size_t)((row - so.r0) >> 1) * so.pitch + (col + h - so.c0)) +
                             ((row - so.r0) & 1)] = re;
                else
                    grid[(size_t)(col + h - so.c0) * so.pitch + (row - so.r0)] = make_double2(re, im);
            }
        }
    }
}

// Interp (nufft.cpp:254-283): one thread per output; deconvolution folded
// into the taps (exact: stencils never leave the band).
template <int W, bool TRANS>
__global__ void __launch_bounds__(256) k_interp(WindowPoly P, GridGeom g, uint64_t n,
                                                const double2* __restrict__ pos,
                                                const double2* __restrict__ phase,
                                                const double2* __restrict__ mult,
                                                const double* __restrict__ dxt,
                                                const double* __restrict__ dyt,
                                                const double2* __restrict__ grid,
                                                const uint32_t* __restrict__ perm,
                                                const double2* __restrict__ addend,
                                                double2* __restrict__ out, int accumulate,
                                                int conj_out, HermArgs h) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const bool hon = h.flag && *h.flag;
    if (v >= (hon && h.n < n ? h.n : n)) return;
    if (hon && h.mult) mult = h.mult;
    const double2 s = pos[v];
    const int jx0 = (int)ceil(s.x - g.half), jy0 = (int)ceil(s.y - g.half);
    double wx[W], wy[W];
    kb_taps<W>((jx0 - s.x) + g.half, P, wx);
    kb_taps<W>((jy0 - s.y) + g.half, P, wy);
    const int mx0 = wrap_base(jx0, g.n1), my0 = wrap_base(jy0, g.n2);
    int myj[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
        int my = my0 + j;
        if (my >= g.n2) my -= g.n2;
        myj[j] = my;
        if (dyt) wy[j] *= dyt[my];
    }
    double ar = 0.0, ai = 0.0;
    if constexpr (TRANS) {
        // grid stored [my][mx] (pitch n1): columns of the stencil are contiguous
        int mxi[W];
#pragma unroll
        for (int i = 0; i < W; ++i) {
            int mx = mx0 + i;
            if (mx >= g.n1) mx -= g.n1;
            mxi[i] = rad_pos(g, mx);  // (rows stored in a radix first pass's order)
            if (dxt) wx[i] *= dxt[mx];
        }
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const double2* col = grid + (size_t)myj[j] * g.n1;
            double rr = 0.0, ri = 0.0;
#pragma unroll
            for (int i = 0; i < W; ++i) {
                const double2 gv = __ldg(col + mxi[i]);
                rr = fma(gv.x, wx[i], rr);
                ri = fma(gv.y, wx[i], ri);
            }
            ar = fma(rr, wy[j], ar);
            ai = fma(ri, wy[j], ai);
        }
    } else {
#pragma unroll
    for (int i = 0; i < W; ++i) {
        int mx = mx0 + i;
        if (mx >= g.n1) mx -= g.n1;
        const double2* row = grid + (size_t)mx * g.n2;
        double rr = 0.0, ri = 0.0;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const double2 gv = __ldg(row + myj[j]);
            rr = fma(gv.x, wy[j], rr);
            ri = fma(gv.y, wy[j], ri);
        }
        const double wxi = dxt ? wx[i] * dxt[mx] : wx[i];
        ar = fma(rr, wxi, ar);
        ai = fma(ri, wxi, ai);
    }
    }
    double2 o = cmul(make_double2(ar, ai), phase[v]);
    if (mult) o = cmul(o, mult[v]);
    if (hon && h.two_re) o = make_double2(2.0 * o.x, 0.0);
    if (conj_out) o.y = -o.y;
    if (addend) {
        const double2 a = addend[v];
        o.x += a.x;
        o.y += a.y;
    }
    const uint64_t dst = perm ? perm[v] : v;
    if (accumulate) {
        double2 q = out[dst];
        q.x += o.x;
        q.y += o.y;
        out[dst] = q;
    } else {
        out[dst] = o;
    }
}

// Interp on the fp64 tensor cores (nufft.cpp:254-283 restated). A warp
// takes 32 consecutive sorted outputs (Z-ordered, so groups of 8 share a small
// footprint), evaluates their windows (lane = output), then handles them 8 at
// a time:
//   H[8 rows x 8 outputs] = G[8 rows x 4 cols] WY[4 cols x 8 outputs]
// over the group's column footprint (two MMAs: Re G, Im G) for each 8-row
// slice; each thread then applies its row's x taps (and the row's
// deconvolution factor) to its two outputs, and the 8 row-lanes are reduced
// with shuffles. The column deconvolution factor rides in the WY fragment.
// Footprints up to 24 x 24 cells use exact-shape straight-line code; larger
// ones (rare) take a per-output scalar loop.
template <int W, bool TRANS, int NRT, int NCT>
__device__ __forceinline__ void mma_group(const double2* __restrict__ grid, GridGeom g, int rmin,
                                          int cmin, int gid, int kq, const double* wys, int nb,
                                          int jyb, const double* __restrict__ dxt,
                                          const double* __restrict__ dyt, const double* wxs,
                                          int na, int jxa0, int jxa1, double& p0r, double& p0i,
                                          double& p1r, double& p1i) {
    double2 a[NRT][NCT];
    int rows[NRT];
#pragma unroll
    for (int t = 0; t < NRT; ++t) {
        rows[t] = wrap_near(rmin + 8 * t + gid, g.n1);
#pragma unroll
        for (int c = 0; c < NCT; ++c) {
            const int col = wrap_near(cmin + 4 * c + kq, g.n2);
            a[t][c] = __ldg(TRANS ? grid + (size_t)col * g.n1 + rad_pos(g, rows[t])
                                  : grid + (size_t)rows[t] * g.n2 + col);
        }
    }
    double hr[NRT][2], hi[NRT][2];
#pragma unroll
    for (int t = 0; t < NRT; ++t) hr[t][0] = hr[t][1] = hi[t][0] = hi[t][1] = 0.0;
#pragma unroll
    for (int c = 0; c < NCT; ++c) {
        const int cc = cmin + 4 * c + kq;
        const int jb = cc - jyb;
        double b = (unsigned)jb < (unsigned)W ? wys[nb * W + jb] : 0.0;
        if (dyt) b *= __ldg(dyt + wrap_near(cc, g.n2));
#pragma unroll
        for (int t = 0; t < NRT; ++t) {
            dmma(hr[t][0], hr[t][1], a[t][c].x, b);
            dmma(hi[t][0], hi[t][1], a[t][c].y, b);
        }
    }
#pragma unroll
    for (int t = 0; t < NRT; ++t) {
        const int row = rmin + 8 * t + gid;
        const double dxr = dxt ? __ldg(dxt + rows[t]) : 1.0;
        const int i0 = row - jxa0, i1 = row - jxa1;
        const double w0 = (unsigned)i0 < (unsigned)W ? wxs[na * W + i0] * dxr : 0.0;
        const double w1 = (unsigned)i1 < (unsigned)W ? wxs[(na + 1) * W + i1] * dxr : 0.0;
        p0r = fma(hr[t][0], w0, p0r);
        p0i = fma(hi[t][0], w0, p0i);
        p1r = fma(hr[t][1], w1, p1r);
        p1i = fma(hi[t][1], w1, p1i);
    }
}

template <int W, bool TRANS>
__global__ void __launch_bounds__(128) k_interp_mma(WindowPoly P, GridGeom g, uint64_t n,
                                                    const double2* __restrict__ pos,
                                                    const double2* __restrict__ phase,
                                                    const double2* __restrict__ mult,
                                                    const double* __restrict__ dxt,
                                                    const double* __restrict__ dyt,
                                                    const double2* __restrict__ grid,
                                                    const uint32_t* __restrict__ perm,
                                                    const double2* __restrict__ addend,
                                                    double2* __restrict__ out, HermArgs hh) {
    const bool hon = hh.flag && *hh.flag;
    if (hon) {
        if (hh.n < n) n = hh.n;
        if (hh.mult) mult = hh.mult;
    }
    __shared__ double s_wx[4][32 * W];
    __shared__ double s_wy[4][32 * W];
    __shared__ int s_jx[4][32], s_jy[4][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, kq = lane & 3;
    double* wxs = s_wx[warp];
    double* wys = s_wy[warp];
    int* jxs = s_jx[warp];
    int* jys = s_jy[warp];
    const uint64_t nwarps = (uint64_t)gridDim.x * 4;
    for (uint64_t base = ((uint64_t)blockIdx.x * 4 + warp) * 32; base < n; base += nwarps * 32) {
        {
            const uint64_t v = base + lane;
            int jx0 = 1 << 28, jy0 = 1 << 28;
            if (v < n) {
                const double2 s = pos[v];
                jx0 = (int)ceil(s.x - g.half);
                jy0 = (int)ceil(s.y - g.half);
                double* wxp = wxs + lane * W;
                double* wyp = wys + lane * W;
                kb_taps_each<W>((jx0 - s.x) + g.half, P, [&](int i, double w) { wxp[i] = w; });
                kb_taps_each<W>((jy0 - s.y) + g.half, P, [&](int j, double w) { wyp[j] = w; });
            }
            jxs[lane] = jx0;
            jys[lane] = jy0;
        }
        __syncwarp();
#pragma unroll 1
        for (int grp = 0; grp < 4; ++grp) {
            const int o8 = grp * 8;
            const int e = lane & 7;
            const int jxe = jxs[o8 + e], jye = jys[o8 + e];
            const bool real = jxe != (1 << 28);
            int rmin = real ? jxe : 1 << 29, rmax = real ? jxe + W : -(1 << 29);
            int cmin = real ? jye : 1 << 29, cmax = real ? jye + W : -(1 << 29);
#pragma unroll
            for (int o = 1; o <= 4; o <<= 1) {
                rmin = min(rmin, __shfl_xor_sync(0xffffffffu, rmin, o));
                rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
                cmin = min(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
                cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
            }
            if (rmax < rmin) break;
            const int nb = o8 + gid;
            const int jyb = jys[nb];
            const int na = o8 + 2 * kq;
            const int jxa0 = jxs[na], jxa1 = jxs[na + 1];
            double p0r = 0.0, p0i = 0.0, p1r = 0.0, p1i = 0.0;
            const int nrt = (rmax - rmin + 7) >> 3, nct = (cmax - cmin + 3) >> 2;
            const int shape = (nrt <= 3 && nct <= 6 && nct >= 3) ? (nrt - 1) * 4 + (nct - 3) : -1;
#define SBD_MMA_CASE(R, C)                                                                         \
    case (R - 1) * 4 + (C - 3):                                                                    \
        mma_group<W, TRANS, R, C>(grid, g, rmin, cmin, gid, kq, wys, nb, jyb, dxt, dyt, wxs, na,   \
                                  jxa0, jxa1, p0r, p0i, p1r, p1i);                                 \
        break;
            switch (shape) {
                SBD_MMA_CASE(1, 3) SBD_MMA_CASE(1, 4) SBD_MMA_CASE(1, 5) SBD_MMA_CASE(1, 6)
                SBD_MMA_CASE(2, 3) SBD_MMA_CASE(2, 4) SBD_MMA_CASE(2, 5) SBD_MMA_CASE(2, 6)
                SBD_MMA_CASE(3, 3) SBD_MMA_CASE(3, 4) SBD_MMA_CASE(3, 5) SBD_MMA_CASE(3, 6)
                default: {
                    // large footprint: each of lanes 0..7 interpolates one output directly
                    if (lane < 8 && jxs[o8 + lane] != (1 << 28)) {
                        const int node = o8 + lane;
                        const int jx0 = jxs[node], jy0 = jys[node];
                        double ar = 0.0, ai = 0.0;
                        for (int i = 0; i < W; ++i) {
                            const int mx = wrap_near(jx0 + i, g.n1);
                            const double wxi = wxs[node * W + i] * (dxt ? dxt[mx] : 1.0);
                            double rr = 0.0, ri = 0.0;
                            for (int j = 0; j < W; ++j) {
                                const int my = wrap_near(jy0 + j, g.n2);
                                const double wyj = wys[node * W + j] * (dyt ? dyt[my] : 1.0);
                                const double2 gv = __ldg(TRANS ? grid + (size_t)my * g.n1 + rad_pos(g, mx)
                                                               : grid + (size_t)mx * g.n2 + my);
                                rr = fma(gv.x, wyj, rr);
                                ri = fma(gv.y, wyj, ri);
                            }
                            ar = fma(rr, wxi, ar);
                            ai = fma(ri, wxi, ai);
                        }
                        // park the result where the reduction below picks it up
                        jxs[node] = jxs[node];
                        wxs[node * W] = ar;
                        wys[node * W] = ai;
                    }
                    __syncwarp();
                    break;
                }
            }
#undef SBD_MMA_CASE
            if (shape < 0) {
                if (gid == 0) {
                    p0r = wxs[na * W];
                    p0i = wys[na * W];
                    p1r = wxs[(na + 1) * W];
                    p1i = wys[(na + 1) * W];
                } else {
                    p0r = p0i = p1r = p1i = 0.0;
                }
            }
#pragma unroll
            for (int o = 4; o <= 16; o <<= 1) {
                p0r += __shfl_xor_sync(0xffffffffu, p0r, o);
                p0i += __shfl_xor_sync(0xffffffffu, p0i, o);
                p1r += __shfl_xor_sync(0xffffffffu, p1r, o);
                p1i += __shfl_xor_sync(0xffffffffu, p1i, o);
            }
            if (gid == 0) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint64_t v = base + na + h;
                    if (v >= n) continue;
                    double2 o2 = cmul(h ? make_double2(p1r, p1i) : make_double2(p0r, p0i), phase[v]);
                    if (mult) o2 = cmul(o2, mult[v]);
                    if (hon && hh.two_re) o2 = make_double2(2.0 * o2.x, 0.0);
                    if (addend) {
                        const double2 ad = addend[v];
                        o2.x += ad.x;
                        o2.y += ad.y;
                    }
                    out[perm ? perm[v] : v] = o2;
                }
            }
            __syncwarp();
        }
        __syncwarp();
    }
}

// Interpolation from a real band grid (the Hermitian-FFT mode's output,
// row-major [r][c] with pitch g.n2): one thread per output, the real part of
// sum * phase, plus the addend. Same taps and order as k_interp.
template <int W>
__global__ void __launch_bounds__(256) k_interp_real(WindowPoly P, GridGeom g, uint64_t n,
                                                     const double2* __restrict__ pos,
                                                     const double2* __restrict__ phase,
                                                     const double* __restrict__ dxt,
                                                     const double* __restrict__ dyt,
                                                     const double* __restrict__ grid,
                                                     const uint32_t* __restrict__ perm,
                                                     const double2* __restrict__ addend,
                                                     double2* __restrict__ out) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    const double2 s = pos[v];
    const int jx0 = (int)ceil(s.x - g.half), jy0 = (int)ceil(s.y - g.half);
    double wx[W], wy[W];
    kb_taps<W>((jx0 - s.x) + g.half, P, wx);
    kb_taps<W>((jy0 - s.y) + g.half, P, wy);
    const int mx0 = wrap_base(jx0, g.n1), my0 = wrap_base(jy0, g.n2);
    int myj[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
        int my = my0 + j;
        if (my >= g.n2) my -= g.n2;
        myj[j] = my;
        if (dyt) wy[j] *= dyt[my];
    }
    double ar = 0.0;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        int mx = mx0 + i;
        if (mx >= g.n1) mx -= g.n1;
        // rows packed in pairs: row mx is component (mx & 1) of complex row mx >> 1
        const double* row = grid + 2 * (size_t)(mx >> 1) * g.n2 + (mx & 1);
        double rr = 0.0;
#pragma unroll
        for (int j = 0; j < W; ++j) rr = fma(__ldg(row + 2 * myj[j]), wy[j], rr);
        ar = fma(rr, dxt ? wx[i] * dxt[mx] : wx[i], ar);
    }
    const double2 ph = phase[v];
    double2 o = make_double2(ar * ph.x, 0.0);
    if (addend) {
        const double2 a = addend[v];
        o.x += a.x;
        o.y += a.y;
    }
    out[perm ? perm[v] : v] = o;
}

// Staged variant of k_interp_real for Z-ordered outputs: one CTA per 32x32
// block of stencil cells stages the block's (32 + W - 1)^2 footprint of the
// real band (deconvolution folded in) in shared memory; each thread then
// interpolates one output of the block from shared memory. The band is read
// from L2 once per block instead of W^2 times per output.
// sum_i wx_i sum_j wy_j base[i PE + j] from a staged real tile, the row taps
// produced a symmetric pair at a time (rows i and W-1-i share one even/odd
// split) so that only the column taps stay live: ~half the registers of
// holding both tap vectors, which keeps the shared-memory loads pipelined.
template <int W, int PE>
__device__ __forceinline__ double interp_rows_real(const double* __restrict__ base, double ux, double uy,
                                                   const WindowPoly& P) {
    double wy[W];
    kb_taps<W>(uy, P, wy);
    const double v = 2.0 * ux - 1.0;
    const double v2 = v * v;
    double ar = 0.0;
#pragma unroll
    for (int i = 0; i < W / 2; ++i) {
        double e = P.e[i][kHorner - 1], o = P.o[i][kHorner - 1];
#pragma unroll
        for (int h = kHorner - 2; h >= 0; --h) {
            e = fma(e, v2, P.e[i][h]);
            o = fma(o, v2, P.o[i][h]);
        }
        double r0 = 0.0, r1 = 0.0;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            r0 = fma(base[i * PE + j], wy[j], r0);
            r1 = fma(base[(W - 1 - i) * PE + j], wy[j], r1);
        }
        ar = fma(r0, fma(v, o, e), ar);
        ar = fma(r1, fma(-v, o, e), ar);
    }
    if (W & 1) {
        constexpr int m = W / 2;
        double e = P.e[m][kHorner - 1];
#pragma unroll
        for (int h = kHorner - 2; h >= 0; --h) e = fma(e, v2, P.e[m][h]);
        double r0 = 0.0;
#pragma unroll
        for (int j = 0; j < W; ++j) r0 = fma(base[m * PE + j], wy[j], r0);
        ar = fma(r0, e, ar);
    }
    return ar;
}

// The rows i = part, part + K, ... of the same sum (K lanes share an output);
// each row's tap evaluated on its own (pair index from the row), so every
// index stays static except the tap-polynomial row (a constant-bank load).
template <int W, int PE, int K>
__device__ __forceinline__ double interp_rows_part(const double* __restrict__ base, double ux, double uy,
                                                   const WindowPoly& P, int part) {
    double wy[W];
    kb_taps<W>(uy, P, wy);
    const double v = 2.0 * ux - 1.0;
    const double v2 = v * v;
    const double* b = base + part * PE;
    double ar = 0.0;
#pragma unroll
    for (int m = 0; m < (W + K - 1) / K; ++m) {
        const int i = part + K * m;
        if (i < W) {
            const int p = i < W - 1 - i ? i : W - 1 - i;
            double e = P.e[p][kHorner - 1], o = P.o[p][kHorner - 1];
#pragma unroll
            for (int h = kHorner - 2; h >= 0; --h) {
                e = fma(e, v2, P.e[p][h]);
                o = fma(o, v2, P.o[p][h]);
            }
            const double tap = 2 * i == W - 1 ? e : (i < W - 1 - i ? fma(v, o, e) : fma(-v, o, e));
            double rr = 0.0;
#pragma unroll
            for (int j = 0; j < W; ++j) rr = fma(b[K * m * PE + j], wy[j], rr);
            ar = fma(rr, tap, ar);
        }
    }
    return ar;
}

template <int W>
__global__ void __launch_bounds__(128, 8) k_interp_real_tile(
    WindowPoly P, GridGeom g, const uint32_t* __restrict__ tstart, uint32_t ntiles, int shift,
    uint64_t out_lo, uint64_t n, const double2* __restrict__ pos, const double2* __restrict__ phase,
    const double* __restrict__ dxt, const double* __restrict__ dyt, const double* __restrict__ grid,
    const uint32_t* __restrict__ perm, const double2* __restrict__ addend, double2* __restrict__ out) {
    constexpr int E = 32 + W - 1;
    constexpr int PE = E | 1;  // odd pitch (in doubles): rows start on different banks
    __shared__ double S[E * PE];
    __shared__ double s_fx[E], s_fy[E];
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t t0 = tstart[tile], t1 = tstart[tile + 1];
        const uint64_t a0 = t0 > out_lo ? t0 : out_lo, a1 = t1 < out_lo + n ? t1 : out_lo + n;
        if (a0 >= a1) continue;
        const double2 s0 = pos[a0 - out_lo];
        const int X0 = (((int)ceil(s0.x - g.half) + shift) & ~31) - shift;
        const int Y0 = (((int)ceil(s0.y - g.half) + shift) & ~31) - shift;
        __syncthreads();  // previous block's readers are done
        for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) {
            if (i < E)
                s_fx[i] = dxt ? __ldg(dxt + wrap_near(X0 + i, g.n1)) : 1.0;
            else
                s_fy[i - E] = dyt ? __ldg(dyt + wrap_near(Y0 + i - E, g.n2)) : 1.0;
        }
        __syncthreads();
        constexpr int kB = 8;
        for (int ib = 0; ib < E * E; ib += kB * 128) {
            double v[kB];
#pragma unroll
            for (int u = 0; u < kB; ++u) {
                const int i = ib + u * 128 + threadIdx.x;
                v[u] = 0.0;
                if (i < E * E) {
                    const int r = i / E, c = i - (i / E) * E;
                    const int gr = wrap_near(X0 + r, g.n1), gc = wrap_near(Y0 + c, g.n2);
                    // rows packed in pairs (component gr & 1 of complex row gr >> 1)
                    v[u] = __ldg(grid + 2 * ((size_t)(gr >> 1) * g.n2 + rad_pos(g, gc)) + (gr & 1));
                }
            }
#pragma unroll
            for (int u = 0; u < kB; ++u) {
                const int i = ib + u * 128 + threadIdx.x;
                if (i < E * E) {
                    const int r = i / E, c = i - (i / E) * E;
                    S[r * PE + c] = v[u] * s_fx[r] * s_fy[c];
                }
            }
        }
        __syncthreads();
        // one thread per output for whole rounds of 128; the last partial round
        // splits each remaining output's rows over K = 4 / 2 / 1 lanes, so a
        // block with a few more outputs than threads (~30% of the blocks at
        // 0.12 outputs per cell) does not pay a second full output latency
        const uint32_t cnt = (uint32_t)(a1 - a0);
        const uint32_t full = cnt & ~127u;
        auto emit = [&](uint64_t va, double ar) {
            const uint64_t v = va - out_lo;
            const double2 ph = phase[v];
            const double2 ad = addend ? addend[v] : make_double2(0.0, 0.0);
            out[perm ? perm[v] : (uint32_t)v] = make_double2(ar * ph.x + ad.x, ad.y);
        };
        for (uint32_t k = threadIdx.x; k < full; k += 128) {
            const double2 sv = pos[a0 + k - out_lo];
            const int ix = (int)ceil(sv.x - g.half), iy = (int)ceil(sv.y - g.half);
            emit(a0 + k, interp_rows_real<W, PE>(S + (ix - X0) * PE + (iy - Y0), (ix - sv.x) + g.half,
                                                 (iy - sv.y) + g.half, P));
        }
        const uint32_t rem = cnt - full;
        if (rem) {
            const int K = rem <= 32 ? 4 : rem <= 64 ? 2 : 1;
            const uint32_t k = threadIdx.x / K;
            const int part = threadIdx.x % K;
            double ar = 0.0;
            if (k < rem) {
                const double2 sv = pos[a0 + full + k - out_lo];
                const int ix = (int)ceil(sv.x - g.half), iy = (int)ceil(sv.y - g.half);
                const double* base = S + (ix - X0) * PE + (iy - Y0);
                const double ux = (ix - sv.x) + g.half, uy = (iy - sv.y) + g.half;
                if (K == 1)
                    ar = interp_rows_real<W, PE>(base, ux, uy, P);
                else if (K == 2)
                    ar = interp_rows_part<W, PE, 2>(base, ux, uy, P, part);
                else
                    ar = interp_rows_part<W, PE, 4>(base, ux, uy, P, part);
            }
            if (K > 1) ar += __shfl_xor_sync(0xffffffffu, ar, 1);
            if (K > 2) ar += __shfl_xor_sync(0xffffffffu, ar, 2);
            if (k < rem && part == 0) emit(a0 + full + k, ar);
        }
    }
}


// ---- tile-staged tensor-core interpolation -------------------------------
// Outputs are Z-ordered by stencil cell, so the outputs whose stencil starts
// in one 32 x 32 cell block are contiguous ("tiles", starts built at plan
// time). One CTA stages the block's (32 + W - 1)^2 footprint of the grid,
// pre-multiplied by the row and column deconvolution factors, into shared
// memory once; its warps then run the 8-output MMA groups of k_interp_mma
// from shared memory. The grid is read from L2 once per tile instead of once
// per 8-output group.
__device__ __forceinline__ void cp_async16(double2* smem_dst, const double2* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem_dst)),
                 "l"(gsrc));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

constexpr int kIT = 32;  // tile edge (Morton level 5)
constexpr int kITW = 6;  // warps per CTA sharing one staged block

template <int W, bool TRANS>
struct ITile {
    static constexpr int E = kIT + W - 1;  // footprint edge
    static constexpr int RE = E + 3;       // rows incl. the zero rows a 4-row MMA slice may touch
    static constexpr int CE = E + 7;       // cols incl. the zero cols an 8-col MMA slice may touch
    // [col][row] (TRANS) or [row][col] layout, pitch chosen so the 4-row x
    // 8-col B-fragment reads of one quarter-warp hit distinct 16-byte bank groups
    static constexpr int ext = TRANS ? RE : CE;
    static constexpr int mod = TRANS ? 4 : 2;
    static constexpr int P = ext + ((mod - ext % 8) + 8) % 8;
    static constexpr int cells = (TRANS ? CE : RE) * P;
    static constexpr size_t smem = (size_t)cells * sizeof(double2) + 2 * kITW * 32 * W * sizeof(double);
    __device__ static int at(int r, int c) { return TRANS ? c * P + r : r * P + c; }
};

// One 8-output group on the tensor cores, rows contracted first:
//   C[node][col] = sum_row Wx[node][row] S[row][col]  (m8n8k4: m = node,
//   k = 4 rows, n = 8 cols; NRC row chunks x NC8 column tiles), then each lane
//   weights its two columns by Wy and the four lanes of a node reduce.
// Lane (gid, kq) ends with a partial of output `node` = o8 + gid.
template <int W, bool TRANS, int NRC, int NC8>
__device__ __forceinline__ void mma_group_t(const double2* __restrict__ S, int rl, int cl, int gid, int kq,
                                            const double* wxs, const double* wys, int node, int jx0, int jy0,
                                            double& pr, double& pi) {
    using TT = ITile<W, TRANS>;
    double hr[NC8][2], hi[NC8][2];
#pragma unroll
    for (int t = 0; t < NC8; ++t) hr[t][0] = hr[t][1] = hi[t][0] = hi[t][1] = 0.0;
#pragma unroll
    for (int c = 0; c < NRC; ++c) {
        const int row = rl + 4 * c + kq;
        const int ix = row - jx0;
        const double a = (unsigned)ix < (unsigned)W ? wxs[node * W + ix] : 0.0;
#pragma unroll
        for (int t = 0; t < NC8; ++t) {
            const double2 b = S[TT::at(row, cl + 8 * t + gid)];
            dmma(hr[t][0], hr[t][1], a, b.x);
            dmma(hi[t][0], hi[t][1], a, b.y);
        }
    }
#pragma unroll
    for (int t = 0; t < NC8; ++t) {
        const int j0 = cl + 8 * t + 2 * kq - jy0;
        const double w0 = (unsigned)j0 < (unsigned)W ? wys[node * W + j0] : 0.0;
        const double w1 = (unsigned)(j0 + 1) < (unsigned)W ? wys[node * W + j0 + 1] : 0.0;
        pr = fma(hr[t][0], w0, pr);
        pr = fma(hr[t][1], w1, pr);
        pi = fma(hi[t][0], w0, pi);
        pi = fma(hi[t][1], w1, pi);
    }
}

// PROC: the outputs are procedural ring nodes -- positions, postphase and
// kappa (omega-hat times the next plan's prephase, `mult` of the fused path)
// are regenerated from gen.id instead of read from pos / phase / mult.
// ASYNC: the footprint is staged by cp.async, see below.
template <int W, bool TRANS, bool PROC = false, bool ASYNC = false>
__global__ void __launch_bounds__(kITW * 32, 3) k_interp_tile(
    WindowPoly P, GridGeom g, const uint32_t* __restrict__ tstart, uint32_t ntiles, int shift,
    uint64_t out_lo, uint64_t n, const double2* __restrict__ pos, const double2* __restrict__ phase,
    const double2* __restrict__ mult, const double* __restrict__ dxt, const double* __restrict__ dyt,
    const double2* __restrict__ grid, const uint32_t* __restrict__ perm,
    const double2* __restrict__ addend, double2* __restrict__ out, HermArgs hh, NodeGen gen) {
    using TT = ITile<W, TRANS>;
    const bool hon = hh.flag && *hh.flag;
    if (hon) {
        if (hh.n < n) n = hh.n;
        if (hh.mult) mult = hh.mult;
    }
    const int hcols = hon ? hh.hcols : 0;
    extern __shared__ __align__(16) double sm_it[];
    double2* S = reinterpret_cast<double2*>(sm_it);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, kq = lane & 3;
    double* wxs = sm_it + 2 * TT::cells + warp * 2 * 32 * W;
    double* wys = wxs + 32 * W;
    __shared__ int s_jx[kITW][32], s_jy[kITW][32];
    __shared__ double s_dx[TT::E], s_dy[TT::E];  // row / column factors of the staged footprint (cp.async staging)
    int* jxs = s_jx[warp];
    int* jys = s_jy[warp];
    // (the cells of S outside the footprint are never written: zero them once)
    for (int i = threadIdx.x; i < TT::cells; i += kITW * 32) S[i] = make_double2(0.0, 0.0);
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // tile range in sorted order, clipped to this call's output range
        const uint64_t t0 = tstart[tile], t1 = tstart[tile + 1];
        const uint64_t a0 = t0 > out_lo ? t0 : out_lo, a1 = t1 < out_lo + n ? t1 : out_lo + n;
        if (a0 >= a1) continue;
        const double2 s0 = PROC ? plan_output_pos(ring_node(gen.id[a0 - out_lo], gen.rings), gen.ox, gen.oy, gen.osgn)
                                : pos[a0 - out_lo];
        const int X0 = (((int)ceil(s0.x - g.half) + shift) & ~(kIT - 1)) - shift;
        const int Y0 = (((int)ceil(s0.y - g.half) + shift) & ~(kIT - 1)) - shift;
        __syncthreads();  // previous tile's readers are done
        // The footprint is a plain copy, sent straight to shared memory by
        // 16-byte cp.async (LDGSTS: no staging registers, every load of a
        // thread in flight at once); the deconvolution factors of its rows and
        // columns go into each output's x and y taps instead. Cells read by
        // conjugate symmetry take the register path.
        constexpr bool async_copy = ASYNC;
        if constexpr (ASYNC) {
            if (threadIdx.x < TT::E)
                s_dx[threadIdx.x] = dxt ? __ldg(dxt + wrap_near(X0 + (int)threadIdx.x, g.n1)) : 1.0;
            else if (threadIdx.x >= 64 && threadIdx.x < 64 + TT::E)
                s_dy[threadIdx.x - 64] = dyt ? __ldg(dyt + wrap_near(Y0 + (int)threadIdx.x - 64, g.n2)) : 1.0;
            for (int i = threadIdx.x; i < TT::cells; i += kITW * 32) {
                const int q = i / TT::P, rr = i - q * TT::P;
                const int r = TRANS ? rr : q, c = TRANS ? q : rr;
                if (r < TT::E && c < TT::E) {
                    const int gr = wrap_near(X0 + r, g.n1), gc = wrap_near(Y0 + c, g.n2);
                    if (TRANS && hcols && gc >= hcols) {
                        const double2 m = __ldg(grid + (size_t)(g.n2 - gc) * g.n1 + rad_pos(g, gr ? g.n1 - gr : 0));
                        S[i] = make_double2(m.x, -m.y);
                    } else {
                        cp_async16(S + i, TRANS ? grid + (size_t)gc * g.n1 + rad_pos(g, gr)
                                                : grid + (size_t)gr * g.n2 + gc);
                    }
                }
            }
        }
        // this lane's position (or node id) of the warp's first 32 outputs: in
        // flight while the footprint lands; later rounds are fetched a round ahead
        double2 svn = make_double2(0.0, 0.0);
        uint32_t nidn = 0;
        {
            const uint64_t v0 = a0 + 32 * warp + lane;
            if (v0 < a1) {
                if constexpr (PROC)
                    nidn = gen.id[v0 - out_lo];
                else
                    svn = pos[v0 - out_lo];
            }
        }
        if constexpr (ASYNC) cp_async_wait_all();
        // footprint -> shared memory times the deconvolution factors of its
        // row and column (L1-resident tables), eight loads in flight per thread
        constexpr int kB = 8;
        for (int ib = 0; !ASYNC && ib < TT::cells; ib += kB * kITW * 32) {
            double2 v[kB];
            double f[kB];
#pragma unroll
            for (int u = 0; u < kB; ++u) {
                const int i = ib + u * kITW * 32 + threadIdx.x;
                const int q = i / TT::P, rr = i - q * TT::P;
                const int r = TRANS ? rr : q, c = TRANS ? q : rr;
                v[u] = make_double2(0.0, 0.0);
                f[u] = 0.0;
                if (i < TT::cells && r < TT::E && c < TT::E) {
                    const int gr = wrap_near(X0 + r, g.n1), gc = wrap_near(Y0 + c, g.n2);
                    if (TRANS && hcols && gc >= hcols) {
                        // negative column: conjugate of the mirrored stored cell
                        const double2 m =
                            __ldg(grid + (size_t)(g.n2 - gc) * g.n1 + rad_pos(g, gr ? g.n1 - gr : 0));
                        v[u] = make_double2(m.x, -m.y);
                    } else {
                        v[u] = __ldg(TRANS ? grid + (size_t)gc * g.n1 + rad_pos(g, gr) : grid + (size_t)gr * g.n2 + gc);
                    }
                    f[u] = (dxt ? __ldg(dxt + gr) : 1.0) * (dyt ? __ldg(dyt + gc) : 1.0);
                }
            }
#pragma unroll
            for (int u = 0; u < kB; ++u) {
                const int i = ib + u * kITW * 32 + threadIdx.x;
                if (i < TT::cells) S[i] = make_double2(v[u].x * f[u], v[u].y * f[u]);
            }
        }
        __syncthreads();
        for (uint64_t base = a0 + 32 * warp; base < a1; base += 32 * kITW) {
            // this lane's output: position now, epilogue operands prefetched
            const uint64_t vmy = base + lane;
            const bool mine = vmy < a1;
            const uint64_t vr = mine ? vmy - out_lo : 0;
            double2 sv = svn, ph = make_double2(0.0, 0.0), mu = make_double2(1.0, 0.0), ad = ph;
            uint32_t dst = 0;
            const uint32_t nid = nidn;
            double2 xi = ph;
            {
                const uint64_t vnx = vmy + 32 * kITW;
                if (vnx < a1) {
                    if constexpr (PROC)
                        nidn = gen.id[vnx - out_lo];
                    else
                        svn = pos[vnx - out_lo];
                }
            }
            if (mine) {
                if constexpr (PROC) {
                    xi = ring_node(nid, gen.rings, &mu);
                    sv = plan_output_pos(xi, gen.ox, gen.oy, gen.osgn);
                } else {
                    ph = phase[vr];
                    if (mult) mu = mult[vr];
                }
                if (addend) ad = addend[vr];
                dst = perm ? perm[vr] : (uint32_t)vr;
            }
            {
                int jx0 = 1 << 28, jy0 = 1 << 28;
                if (mine) {
                    const int ix = (int)ceil(sv.x - g.half), iy = (int)ceil(sv.y - g.half);
                    double* wxp = wxs + lane * W;
                    double* wyp = wys + lane * W;
                    jx0 = ix - X0;  // tile-local stencil start, in [0, 32)
                    jy0 = iy - Y0;
                    if constexpr (async_copy) {
                        const double* fx = s_dx + jx0;
                        const double* fy = s_dy + jy0;
                        kb_taps_each<W>((ix - sv.x) + g.half, P, [&](int i, double w) { wxp[i] = w * fx[i]; });
                        kb_taps_each<W>((iy - sv.y) + g.half, P, [&](int j, double w) { wyp[j] = w * fy[j]; });
                    } else {
                        kb_taps_each<W>((ix - sv.x) + g.half, P, [&](int i, double w) { wxp[i] = w; });
                        kb_taps_each<W>((iy - sv.y) + g.half, P, [&](int j, double w) { wyp[j] = w; });
                    }
                }
                jxs[lane] = jx0;
                jys[lane] = jy0;
            }
            __syncwarp();
            double accr = 0.0, acci = 0.0;  // this lane's output after the group loop
#pragma unroll 1
            for (int grp = 0; grp < 4; ++grp) {
                const int o8 = grp * 8;
                const int e = lane & 7;
                const int jxe = jxs[o8 + e], jye = jys[o8 + e];
                const bool real = jxe != (1 << 28);
                // group bounding box: (row, col) starts packed in 16-bit halves
                // (tile-local, < 2^15), min/max by SIMD-in-word over 8 lanes
                unsigned lo = real ? ((unsigned)jxe << 16) | (unsigned)jye : 0xffffffffu;
                unsigned hi = real ? ((unsigned)(jxe + W) << 16) | (unsigned)(jye + W) : 0u;
#pragma unroll
                for (int o = 1; o <= 4; o <<= 1) {
                    lo = __vminu2(lo, __shfl_xor_sync(0xffffffffu, lo, o));
                    hi = __vmaxu2(hi, __shfl_xor_sync(0xffffffffu, hi, o));
                }
                if (hi == 0u) break;
                const int rmin = (int)(lo >> 16), cmin = (int)(lo & 0xffffu);
                const int rmax = (int)(hi >> 16), cmax = (int)(hi & 0xffffu);
                const int node = o8 + gid;
                const int jxn = jxs[node], jyn = jys[node];
                double pr = 0.0, pi = 0.0;
                const int nrc = (rmax - rmin + 3) >> 2, nc8 = (cmax - cmin + 7) >> 3;
                const int shape = (nrc >= 3 && nrc <= 6 && nc8 >= 2 && nc8 <= 3) ? (nrc - 3) * 2 + (nc8 - 2) : -1;
#define SBD_MMA_CASE(R, C)                                                                              \
    case (R - 3) * 2 + (C - 2):                                                                         \
        mma_group_t<W, TRANS, R, C>(S, rmin, cmin, gid, kq, wxs, wys, node, jxn, jyn, pr, pi);          \
        break;
                switch (shape) {
                    SBD_MMA_CASE(3, 2) SBD_MMA_CASE(3, 3) SBD_MMA_CASE(4, 2) SBD_MMA_CASE(4, 3)
                    SBD_MMA_CASE(5, 2) SBD_MMA_CASE(5, 3) SBD_MMA_CASE(6, 2) SBD_MMA_CASE(6, 3)
                    default: {
                        // wide group: four lanes per output (rows part, part + 4, ...),
                        // reduced over the four, from the staged tile
                        double ar = 0.0, ai = 0.0;
                        const int node = o8 + (lane >> 2), part = lane & 3;
                        if (jxs[node] != (1 << 28)) {
                            const int jx0 = jxs[node], jy0 = jys[node];
                            for (int i = part; i < W; i += 4) {
                                double rr = 0.0, ri = 0.0;
#pragma unroll
                                for (int j = 0; j < W; ++j) {
                                    const double2 gv = S[TT::at(jx0 + i, jy0 + j)];
                                    const double wyj = wys[node * W + j];
                                    rr = fma(gv.x, wyj, rr);
                                    ri = fma(gv.y, wyj, ri);
                                }
                                ar = fma(rr, wxs[node * W + i], ar);
                                ai = fma(ri, wxs[node * W + i], ai);
                            }
                        }
                        ar += __shfl_xor_sync(0xffffffffu, ar, 1);
                        ai += __shfl_xor_sync(0xffffffffu, ai, 1);
                        ar += __shfl_xor_sync(0xffffffffu, ar, 2);
                        ai += __shfl_xor_sync(0xffffffffu, ai, 2);
                        // lanes 4k hold output o8 + k: hand them to the owners
                        ar = __shfl_sync(0xffffffffu, ar, (lane & 7) << 2);
                        ai = __shfl_sync(0xffffffffu, ai, (lane & 7) << 2);
                        if ((lane >> 3) == grp) {
                            accr = ar;
                            acci = ai;
                        }
                        break;
                    }
                }
#undef SBD_MMA_CASE
                if (shape >= 0) {
                    // the four lanes of each node, then lanes 4k hold output o8 + k
                    pr += __shfl_xor_sync(0xffffffffu, pr, 1);
                    pi += __shfl_xor_sync(0xffffffffu, pi, 1);
                    pr += __shfl_xor_sync(0xffffffffu, pr, 2);
                    pi += __shfl_xor_sync(0xffffffffu, pi, 2);
                    pr = __shfl_sync(0xffffffffu, pr, (lane & 7) << 2);
                    pi = __shfl_sync(0xffffffffu, pi, (lane & 7) << 2);
                    if ((lane >> 3) == grp) {
                        accr = pr;
                        acci = pi;
                    }
                }
            }
            if (mine) {
                if constexpr (PROC) {
                    // after the group loop: the phases' registers are not live across it
                    ph = plan_output_post(xi, gen.ox, gen.oy, gen.osgn, gen.ocxy);
                    mu = cmul(mu, plan_point_pre(xi, gen.px, gen.py, gen.pbeta));
                    if (hon && (nid & kRingHalve)) mu = make_double2(0.5 * mu.x, 0.5 * mu.y);
                }
                double2 o2 = cmul(make_double2(accr, acci), ph);
                if (PROC || mult) o2 = cmul(o2, mu);
                if (hon && hh.two_re) o2 = make_double2(2.0 * o2.x, 0.0);
                if (hon && hh.out2) hh.out2[hh.perm2[vr]] = make_double2(o2.x, -o2.y);
                o2.x += ad.x;
                o2.y += ad.y;
                out[dst] = o2;
            }
            __syncwarp();
        }
    }
}

// tile t of the Z-ordered outputs = sorted positions [start[t], start[t+1])
__global__ void k_tile_flags(const uint32_t* __restrict__ key, uint64_t n, int bits,
                             uint32_t* __restrict__ flag) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    flag[i] = (i == 0 || (key[i] >> bits) != (key[i - 1] >> bits)) ? 1u : 0u;
}
__global__ void k_tile_scatter(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ idx,
                               uint64_t n, uint32_t* __restrict__ start) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (flag[i]) start[idx[i]] = (uint32_t)i;
    if (i == n - 1) start[idx[i] + flag[i]] = (uint32_t)n;
}

// Direct sum (nufft.cpp:76-93): thread per output, sequential over points in
// the caller's order (same summation order as the reference).
__global__ void k_ndft(const double2* __restrict__ pts, uint64_t np,
                       const double2* __restrict__ frq, uint64_t nf,
                       const double2* __restrict__ c, double sgn, double2* __restrict__ out) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (v >= nf) return;
    const double fx = __dmul_rn(sgn, frq[v].x), fy = __dmul_rn(sgn, frq[v].y);
    double ar = 0.0, ai = 0.0;
    for (uint64_t k = 0; k < np; ++k) {
        const double2 z = pts[k];
        const double phase = __dadd_rn(__dmul_rn(z.x, fx), __dmul_rn(z.y, fy));
        double sn, cs;
        sincos(phase, &sn, &cs);
        const double2 ck = c[k];
        ar = __dadd_rn(ar, __dsub_rn(__dmul_rn(ck.x, cs), __dmul_rn(ck.y, sn)));
        ai = __dadd_rn(ai, __dadd_rn(__dmul_rn(ck.x, sn), __dmul_rn(ck.y, cs)));
    }
    out[v] = make_double2(ar, ai);
}

// b[k] = in[perm[k]] * phase[k]; raw[k] = in[perm[k]] (optional): the spread
// coefficients (nufft.cpp:233) and the sorted copy of f for the CSR pass.
__global__ void k_gather_mul(const double2* __restrict__ in, const uint32_t* __restrict__ perm,
                             const double2* __restrict__ phase, double2* __restrict__ b,
                             double2* __restrict__ raw, uint64_t n, uint64_t lo, uint64_t hi,
                             int* __restrict__ clear, double* __restrict__ raw_re) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double2 c = in[perm ? perm[k] : k];
    if (clear && c.y != 0.0) *clear = 0;
    b[k] = (k >= lo && k < hi) ? cmul(c, phase[k]) : make_double2(0.0, 0.0);
    if (raw) raw[k] = c;
    if (raw_re) raw_re[k] = c.x;
}

// qs[r] = sum_{i in row r} D'_i f'_{col'_i} (point_cloud.cpp:116-123 on the
// renumbered matrix); 8 lanes per row, coalesced over the row's entries.
// Same product when every value of D is real (Laplace: log r and a real
// omega-hat): the values are stored as 8-byte reals, 12 instead of 20 bytes
// per nonzero streamed from HBM; the result is bitwise the complex kernel's
// (the imaginary parts it would multiply are exact zeros).
// Real D' times a real f (the caller said so): the gathers read 8-byte
// entries of Re(f) (four per 32-byte sector instead of two), q is exactly real.
__global__ void __launch_bounds__(256) k_spmv_vec_rr(uint64_t rows, const uint64_t* __restrict__ ro,
                                                     const uint32_t* __restrict__ cols,
                                                     const double* __restrict__ vals,
                                                     const double* __restrict__ fr, double2* __restrict__ qs) {
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t r = g >> 3;
    const int sub = (int)(g & 7);
    double ar = 0.0;
    if (r < rows) {
        const uint64_t e = ro[r + 1];
        for (uint64_t i = ro[r] + sub; i < e; i += 8) ar = fma(vals[i], fr[cols[i]], ar);
    }
#pragma unroll
    for (int o = 4; o; o >>= 1) ar += __shfl_xor_sync(0xffffffffu, ar, o);
    if (r < rows && sub == 0) qs[r] = make_double2(ar, 0.0);
}

__global__ void __launch_bounds__(256) k_spmv_vec_real(uint64_t rows, const uint64_t* __restrict__ ro,
                                                       const uint32_t* __restrict__ cols,
                                                       const double* __restrict__ vals,
                                                       const double2* __restrict__ f,
                                                       double2* __restrict__ qs) {
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t r = g >> 3;
    const int sub = (int)(g & 7);
    double ar = 0.0, ai = 0.0;
    if (r < rows) {
        const uint64_t e = ro[r + 1];
        for (uint64_t i = ro[r] + sub; i < e; i += 8) {
            const double v = vals[i];
            const double2 x = f[cols[i]];
            ar = fma(v, x.x, ar);
            ai = fma(v, x.y, ai);
        }
    }
#pragma unroll
    for (int o = 4; o; o >>= 1) {
        ar += __shfl_xor_sync(0xffffffffu, ar, o);
        ai += __shfl_xor_sync(0xffffffffu, ai, o);
    }
    if (r < rows && sub == 0) qs[r] = make_double2(ar, ai);
}

__global__ void __launch_bounds__(256) k_spmv_vec(uint64_t rows, const uint64_t* __restrict__ ro,
                                                  const uint32_t* __restrict__ cols,
                                                  const double2* __restrict__ vals,
                                                  const double2* __restrict__ f,
                                                  double2* __restrict__ qs, int acc) {
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t r = g >> 3;
    const int sub = (int)(g & 7);
    double ar = 0.0, ai = 0.0;
    if (r < rows) {
        const uint64_t e = ro[r + 1];
        for (uint64_t i = ro[r] + sub; i < e; i += 8) {
            const double2 v = vals[i];
            const double2 x = f[cols[i]];
            ar = fma(v.x, x.x, ar);
            ar = fma(-v.y, x.y, ar);
            ai = fma(v.x, x.y, ai);
            ai = fma(v.y, x.x, ai);
        }
    }
#pragma unroll
    for (int o = 4; o; o >>= 1) {
        ar += __shfl_xor_sync(0xffffffffu, ar, o);
        ai += __shfl_xor_sync(0xffffffffu, ai, o);
    }
    if (r < rows && sub == 0) {
        if (acc) {
            const double2 o = qs[r];
            ar += o.x;
            ai += o.y;
        }
        qs[r] = make_double2(ar, ai);
    }
}

// b[k] = conj?(in[perm[k]]) phase[k]: the transposed NUFFT's input times its
// postphase (nufft.cpp:313-314)
__global__ void k_gather_conj_mul(const double2* __restrict__ in, const uint32_t* __restrict__ perm,
                                  const double2* __restrict__ phase, int conj_in, double2* __restrict__ b,
                                  uint64_t n) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    double2 c = in[perm ? perm[k] : k];
    if (conj_in) c.y = -c.y;
    b[k] = cmul(c, phase[k]);
}

// Deconvolution of the transposed spread (nufft.cpp:325-335) restricted to the
// band (the factors are zero outside it), folded from the compact spread region
// into the transposed band layout of the column transforms.
__global__ void k_band_fold(const double2* __restrict__ Z, int pz, int rlo, int rhi, int clo, int chi, int b1,
                            int n1, int b2, int B, int n2, const double* __restrict__ dx,
                            const double* __restrict__ dy, double2* __restrict__ V) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const int R = 2 * b1 + 1;
    if (k >= (uint64_t)R * B) return;
    const int c = (int)(k / R), jx = (int)(k - (uint64_t)c * R) - b1;
    const int jy = c <= b2 ? c : c - B;
    const int mx = jx < 0 ? jx + n1 : jx, my = jy < 0 ? jy + n2 : jy;
    double2 v = make_double2(0.0, 0.0);
    if (jx >= rlo && jx < rhi && jy >= clo && jy < chi) {
        const double2 z = Z[(size_t)(jx - rlo) * pz + (jy - clo)];
        const double f = dx[mx] * dy[my];
        v = make_double2(z.x * f, z.y * f);
    }
    V[(size_t)c * n1 + mx] = v;
}

// Tz[(r - r0) n2 + m(c)] = Wt[c n1 + r]: the transposed band back into rows
// (32 x 32 tiles through shared memory, both sides coalesced)
__global__ void __launch_bounds__(256) k_band_untranspose(const double2* __restrict__ Wt, int n1, int r0, int r1,
                                                          int b, int B, double2* __restrict__ Tz, int n2, int rin) {
    // rin > 1: the columns of Wt come from a radix-rin first pass + length
    // n1 / rin transforms: row r sits at (r mod rin) M + r / rin, and a CTA takes
    // 32 consecutive positions of one residue class
    __shared__ double2 tile[32][33];
    const int cb = blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    auto row_of = [&](int i, int& at) -> int {
        if (rin > 1) {
            const int M = n1 / rin, pos = blockIdx.y * 32 + i;
            at = pos;
            if (pos >= n1) return -1;
            const int cls = pos / M, r = rin * (pos - cls * M) + cls;
            return (r >= r0 && r < r1) ? r : -1;
        }
        const int r = r0 + blockIdx.y * 32 + i;
        at = r;
        return r < r1 ? r : -1;
    };
#pragma unroll
    for (int q = 0; q < 32; q += 8) {
        const int c = cb + ty + q;
        int at;
        const int r = row_of(tx, at);
        if (r >= 0 && c < B) tile[ty + q][tx] = Wt[(size_t)c * n1 + at];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 32; q += 8) {
        const int c = cb + tx;
        int at;
        const int r = row_of(ty + q, at);
        if (r >= 0 && c < B) {
            const int m = c <= b ? c : n2 - B + c;
            Tz[(size_t)(r - r0) * n2 + m] = tile[tx][ty + q];
        }
    }
}

// Tt[c'][r] = T[r][m(c')] for r in [r0, r1) and the band columns c' in [0, B)
// (m = c' for c' <= b, n2 - B + c' otherwise): 32 x 32 tiles through shared
// memory so both the reads (along rows of T) and writes (along rows of Tt)
// are coalesced.
// rin > 1: the rows of T come from a radix-rin first pass + length n2 / rin
// transforms (k_dif_rows): mode j sits at (j mod rin) MR + j / rin, and a CTA
// takes 32 consecutive positions of one residue class (the modes rin l + cls),
// keeping those that are band modes.
__device__ __forceinline__ int band_col_of_pos(int pos, int n2, int b, int B, int rin, int& at) {
    at = pos;
    if (pos >= n2) return -1;
    int j = pos;
    if (rin > 1) {
        const int MR = n2 / rin, cls = pos / MR;
        j = rin * (pos - cls * MR) + cls;
    }
    if (j >= n2) return -1;
    if (j <= b) return j;
    return j >= n2 - b ? j - (n2 - B) : -1;
}

__global__ void __launch_bounds__(256) k_band_transpose(const double2* __restrict__ T, int n2,
                                                        int r0, int r1, int b, int B,
                                                        double2* __restrict__ Tt, int n1, int rin0,
                                                        int conj_out, int rin) {
    __shared__ double2 tile[32][33];
    const int cb = blockIdx.x * 32, rb = r0 + blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    // column handled by lane i of this CTA: band column c_of(i) read at position at_of(i)
    auto col_of = [&](int i, int& at) -> int {
        if (rin > 1) return band_col_of_pos(cb + i, n2, b, B, rin, at);
        const int c = cb + i;
        at = c <= b ? c : n2 - B + c;
        return c < B ? c : -1;
    };
#pragma unroll
    for (int q = 0; q < 32; q += 8) {
        const int r = rb + ty + q;
        int at;
        const int c = col_of(tx, at);
        if (r < r1 && c >= 0) tile[ty + q][tx] = T[(size_t)(r - rin0) * n2 + at];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 32; q += 8) {
        const int r = rb + tx;
        int at;
        const int c = col_of(ty + q, at);
        if (r < r1 && c >= 0) {
            double2 v = tile[tx][ty + q];
            if (conj_out) v.y = -v.y;
            Tt[(size_t)c * n1 + r] = v;
        }
    }
}


// Mirrored grid coordinates t' = n - t: the image of a point under the grid
__global__ void k_mirror_points(const double2* __restrict__ t, uint64_t n, int n1, int n2, int w,
                                double2* __restrict__ out) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double2 p = t[k];
    out[k] = make_double2(mirror_coord(p.x, n1, w), mirror_coord(p.y, n2, w));
}

// out[idx[k]] = conj(in[k])
__global__ void k_conj_scatter(const double2* __restrict__ in, uint64_t n, const uint32_t* __restrict__ idx,
                               double2* __restrict__ out) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double2 v = in[k];
    out[idx[k]] = make_double2(v.x, -v.y);
}

// *flag |= (some im(x[k]) != 0)
__global__ void k_any_imag(const double2* __restrict__ x, uint64_t n, int* __restrict__ flag) {
    int any = 0;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x)
        any |= x[k].y != 0.0;
    if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(flag, 1);
}

// Packed real rows (row 2k in Re, 2k+1 in Im of row k of T, transformed with
// e^{+}): untangle Z_a(j) = (Z(j) + conj Z(-j))/2, Z_b(j) = (Z(j) - conj Z(-j))/(2i)
// for columns j in [0, B) and write them transposed: Tt[j * n1 + r0 + r].
__global__ void __launch_bounds__(256) k_untangle_transpose(const double2* __restrict__ T, int n2, int nr,
                                                            int B, double2* __restrict__ Tt, int n1,
                                                            int r0) {
    __shared__ double2 sa[16][33], sb[16][33];
    const int cb = blockIdx.x * 32, kb = blockIdx.y * 16;  // 32 columns x 16 packed rows
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
    for (int q = 0; q < 16; q += 8) {
        const int k = kb + ty + q, c = cb + tx;
        if (k < nr && c < B) {
            sa[ty + q][tx] = T[(size_t)k * n2 + c];
            sb[ty + q][tx] = T[(size_t)k * n2 + (c ? n2 - c : 0)];
        }
    }
    __syncthreads();
    // output: 32 columns x 32 real rows (two per packed row)
#pragma unroll
    for (int q = 0; q < 32; q += 8) {
        const int c = cb + ty + q, rr = tx;  // rr: real row within the block
        const int k = kb + (rr >> 1);
        if (k < nr && c < B) {
            const double2 a = sa[rr >> 1][ty + q], b = sb[rr >> 1][ty + q];
            double2 v;
            if (rr & 1)
                v = make_double2(0.5 * (a.y + b.y), -0.5 * (a.x - b.x));
            else
                v = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
            Tt[(size_t)c * n1 + r0 + 2 * k + (rr & 1)] = v;
        }
    }
}

// Pack pairs of Hermitian band rows for one complex transform each: band row
// c (mode j1(c)) has half-spectrum X_c[m] = Y[(m - m0) * n1 + j1(c)] for m in
// [m0, n2/2] (zero below m0); row k of Z (full length n2, m in [m0, n2 - m0])
// = X_{2k}(m) + i X_{2k+1}(m) with X(m) = conj X(n2 - m) for m > n2/2.
// ---- radix-r first pass of a length n = r M transform (FFTW_BACKWARD sign) --
// Decimation in frequency: X[r j' + s] = DFT_M(y_s)[j'] with
//   y_s[k] = w_n^{s k} sum_rho x[k + M rho] w_r^{s rho},  w_m = e^{+2 pi i/m},
// so the producer of x writes y (position s M + k), one batched length-M
// cuFFT pass follows, and mode j is read at position (j mod r) M + j / r.
// tw[m] = w_n^m for m < n.
template <int R>
__device__ __forceinline__ void dft_small(const double2 (&x)[R], double2 (&y)[R], const double2* __restrict__ tw,
                                          int M) {
    if (R == 9) {
        // 9 = 3 x 3: rho = 3 a + b, s = s1 + 3 s2
        const double h = 0.8660254037844386467637231707529362;  // sqrt(3) / 2
        double2 t[3][3];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const double2 p = x[b], q = x[3 + b], u = x[6 + b];
            const double2 sum = make_double2(q.x + u.x, q.y + u.y), dif = make_double2(q.x - u.x, q.y - u.y);
            const double2 m = make_double2(p.x - 0.5 * sum.x, p.y - 0.5 * sum.y);
            t[b][0] = make_double2(p.x + sum.x, p.y + sum.y);
            t[b][1] = make_double2(m.x - h * dif.y, m.y + h * dif.x);
            t[b][2] = make_double2(m.x + h * dif.y, m.y - h * dif.x);
            if (b) {
                t[b][1] = cmul(t[b][1], __ldg(tw + b * M));      // w_9^{b s1}, s1 = 1
                t[b][2] = cmul(t[b][2], __ldg(tw + 2 * b * M));  // s1 = 2
            }
        }
#pragma unroll
        for (int s1 = 0; s1 < 3; ++s1) {
            const double2 p = t[0][s1], q = t[1][s1], u = t[2][s1];
            const double2 sum = make_double2(q.x + u.x, q.y + u.y), dif = make_double2(q.x - u.x, q.y - u.y);
            const double2 m = make_double2(p.x - 0.5 * sum.x, p.y - 0.5 * sum.y);
            y[s1] = make_double2(p.x + sum.x, p.y + sum.y);
            y[s1 + 3] = make_double2(m.x - h * dif.y, m.y + h * dif.x);
            y[s1 + 6] = make_double2(m.x + h * dif.y, m.y - h * dif.x);
        }
    } else {
#pragma unroll
        for (int k = 0; k < R; ++k) {
            double2 a = x[0];
#pragma unroll
            for (int rho = 1; rho < R; ++rho) {
                const double2 w = __ldg(tw + ((k * rho) % R) * M);
                a.x += x[rho].x * w.x - x[rho].y * w.y;
                a.y += x[rho].x * w.y + x[rho].y * w.x;
            }
            y[k] = a;
        }
    }
}

// The band transpose with the radix-R first pass of the length n1 = R M column
// transform folded in (the complex pipeline's k_untangle_dif): band column c
// of the rows [r0, r1) of T (zero elsewhere) leaves as y_s[k] at c n1 + s M + k
// for a batched length-M column transform. Columns by position as above.
template <int R>
__global__ void __launch_bounds__(256, 5) k_band_transpose_dif(const double2* __restrict__ T, int n2, int r0, int r1,
                                                            int b, int B, double2* __restrict__ Tt, int n1, int M,
                                                            const double2* __restrict__ tw, int rin) {
    __shared__ double2 so[R][8][33];
    __shared__ int s_col[32];
    const int cb = blockIdx.x * 32, k0 = blockIdx.y * 8;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int at = 0;
    int c;
    if (rin > 1) {
        c = band_col_of_pos(cb + lane, n2, b, B, rin, at);
    } else {
        c = cb + lane < B ? cb + lane : -1;
        at = c <= b ? c : n2 - B + c;
    }
    if (w == 0) s_col[lane] = c;
    if (__syncthreads_and(c < 0)) return;  // no band column among these positions
    const int k = k0 + w;
    double2 x[R], y[R];
#pragma unroll
    for (int rho = 0; rho < R; ++rho) {
        const int m1 = k + M * rho;
        x[rho] = (c >= 0 && m1 >= r0 && m1 < r1) ? T[(size_t)(m1 - r0) * n2 + at] : make_double2(0.0, 0.0);
    }
    dft_small<R>(x, y, tw, M);
#pragma unroll
    for (int sI = 0; sI < R; ++sI) so[sI][w][lane] = sI ? cmul(y[sI], __ldg(tw + sI * k)) : y[sI];
    __syncthreads();
    const int kl = threadIdx.x & 7;
    for (int p = threadIdx.x >> 3; p < 32 * R; p += 32) {
        const int sI = p >> 5, cl = p & 31;
        const int co = s_col[cl];
        if (co >= 0) Tt[(size_t)co * n1 + (size_t)sI * M + k0 + kl] = so[sI][kl][cl];
    }
}

// Radix-R first pass of contiguous length n = R M transforms (rows of X, row
// pitch n), as its own streaming kernel: Y[row][s M + k] = w_n^{s k} sum_rho
// X[row][k + M rho] w_R^{s rho}. A batched contiguous length-M cuFFT pass then
// leaves mode j at (j mod R) M + j / R, where the consumer reads it -- cuFFT's
// own second pass of a length-n transform writes with stride R at ~58% of the
// contiguous pass's bandwidth. Columns outside [c_lo, c_hi) are known zeros
// (the spread's populated range) and are not read.
template <int R>
__global__ void __launch_bounds__(256) k_dif_rows(const double2* __restrict__ X, int n, int M, int c_lo, int c_hi,
                                                  const double2* __restrict__ tw, double2* __restrict__ Y) {
    const int k = blockIdx.x * 256 + threadIdx.x;
    if (k >= M) return;
    const size_t row = (size_t)blockIdx.y * (size_t)n;
    double2 x[R], y[R];
#pragma unroll
    for (int rho = 0; rho < R; ++rho) {
        const int c = k + M * rho;
        x[rho] = (c >= c_lo && c < c_hi) ? X[row + c] : make_double2(0.0, 0.0);
    }
    dft_small<R>(x, y, tw, M);
#pragma unroll
    for (int sI = 0; sI < R; ++sI) Y[row + (size_t)sI * M + k] = sI ? cmul(y[sI], __ldg(tw + sI * k)) : y[sI];
}

// k_untangle_transpose with the radix-R first pass of the column transform
// folded in: the band columns c < B of the untangled real rows x[m1] (rows
// [r0, r0 + 2 nr), zero elsewhere) leave as y_s[k] (column c at c * n1 +
// s M + k, n1 = R M) for a batched length-M column transform.
// RIN > 1: the rows of T come from a radix-RIN first pass + length n2 / RIN
// transforms (k_dif_rows), mode j at (j mod RIN) MR + j / RIN; a CTA then takes
// the 32 columns RIN (l0 + lane) + cls of one residue class, which are
// contiguous there (and so are their mirrors n2 - c).
template <int R, int RIN = 1>
__global__ void __launch_bounds__(256, 5) k_untangle_dif(const double2* __restrict__ T, int n2, int nr, int B,
                                                      double2* __restrict__ Tt, int n1, int r0, int M,
                                                      const double2* __restrict__ tw,
                                                      const double* __restrict__ colf) {
    __shared__ double2 so[R][8][33];
    const int k0 = blockIdx.y * 8;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int MR = n2 / RIN;
    // columns of this CTA: c(i) = cbase + cstep i, i < 32
    int cbase, cstep, pa, pb, pbstep;  // positions of column c and of its mirror in a row of T
    if (RIN > 1) {
        const int per = ((B + RIN - 1) / RIN + 31) / 32;  // CTAs per residue class
        const int cls = blockIdx.x / per, l0 = (blockIdx.x - cls * per) * 32;
        cbase = RIN * l0 + cls;
        cstep = RIN;
        pa = cls * MR + l0 + lane;
        // n2 - c = RIN (MR - l) (cls 0) or RIN (MR - 1 - l) + (RIN - cls)
        pb = cls ? (RIN - cls) * MR + MR - 1 - (l0 + lane) : (l0 + lane ? MR - (l0 + lane) : 0);
        pbstep = 0;
    } else {
        cbase = blockIdx.x * 32;
        cstep = 1;
        pa = cbase + lane;
        pb = pa ? n2 - pa : 0;
        pbstep = 0;
    }
    (void)pbstep;
    const int c = cbase + cstep * lane, k = k0 + w;
    double2 x[R], y[R];
#pragma unroll
    for (int rho = 0; rho < R; ++rho) {
        const int m1 = k + M * rho;
        x[rho] = make_double2(0.0, 0.0);
        if (c < B && m1 >= r0 && m1 < r0 + 2 * nr) {
            const int kk = (m1 - r0) >> 1;
            const double2 a = T[(size_t)kk * n2 + pa], b = T[(size_t)kk * n2 + pb];
            x[rho] = ((m1 - r0) & 1) ? make_double2(0.5 * (a.y + b.y), -0.5 * (a.x - b.x))
                                     : make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
        }
    }
    dft_small<R>(x, y, tw, M);
    // the column's deconvolution factor (exact here: the column transform does
    // not mix columns, and the factor is even in the mode, so the mirrored
    // negative columns the interpolation reads carry theirs too)
    const double fc = (colf && c < B) ? __ldg(colf + c) : 1.0;
#pragma unroll
    for (int sI = 0; sI < R; ++sI) {
        const double2 v = sI ? cmul(y[sI], __ldg(tw + sI * k)) : y[sI];
        so[sI][w][lane] = make_double2(v.x * fc, v.y * fc);
    }
    __syncthreads();
    const int kl = threadIdx.x & 7;
    for (int p = threadIdx.x >> 3; p < 32 * R; p += 32) {
        const int sI = p >> 5, cl = p & 31;
        const int co = cbase + cstep * cl;
        if (co < B) Tt[(size_t)co * n1 + (size_t)sI * M + k0 + kl] = so[sI][kl][cl];
    }
}

// k_pack_rows with the radix-R first pass of the length n2 = R M row
// transform folded in: packed row k (band rows 2k, 2k+1 as z = a + i b, the
// columns above n2/2 their conjugate mirror) leaves as y_s[k1] at
// k n2 + s M + k1 for a batched length-M row transform.
// RIN > 1: the columns of Y (length n1) come from a radix-RIN first pass +
// length n1 / RIN transforms (k_dif_rows), mode j at (j mod RIN) M1 + j / RIN;
// a CTA then takes the 32 packed rows RIN (l0 + lane) + cls, whose band rows
// sit two cells apart there.
template <int R, int RIN = 1>
__global__ void __launch_bounds__(256, 5) k_pack_dif(const double2* __restrict__ Y, int n1, int m0, int n2,
                                                  int b1, int B1, double2* __restrict__ Z, int M,
                                                  const double2* __restrict__ tw) {
    __shared__ double2 so[R][8][33];  // [s][k1][packed row]
    const int k10 = blockIdx.y * 8;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int mhi = n2 / 2, K = (B1 + 1) / 2;
    int kb, kstep;
    if (RIN > 1) {
        const int per = ((K + RIN - 1) / RIN + 31) / 32;  // CTAs per residue class
        const int cls = blockIdx.x / per;
        kb = RIN * ((blockIdx.x - cls * per) * 32) + cls;
        kstep = RIN;
    } else {
        kb = blockIdx.x * 32;
        kstep = 1;
    }
    const int k = kb + kstep * lane, k1 = k10 + w;
    const int ra = 2 * k, rb = 2 * k + 1;
    int ia = ra <= b1 ? ra : n1 - B1 + ra, ib = rb <= b1 ? rb : n1 - B1 + rb;
    if (RIN > 1 && k < K) {
        const int M1 = n1 / RIN;
        ia = (ia % RIN) * M1 + ia / RIN;
        if (rb < B1) ib = (ib % RIN) * M1 + ib / RIN;
    }
    double2 z[R], y[R];
#pragma unroll
    for (int rho = 0; rho < R; ++rho) {
        const int m = k1 + M * rho;
        z[rho] = make_double2(0.0, 0.0);
        if (k < K) {
            const bool dir = m >= m0 && m <= mhi;
            const int mm = dir ? m : n2 - m;  // mirrored source column
            if (dir || (m > mhi && mm >= m0)) {
                const double2 a = Y[(size_t)(mm - m0) * n1 + ia];
                const double2 b = rb < B1 ? Y[(size_t)(mm - m0) * n1 + ib] : make_double2(0.0, 0.0);
                z[rho] = dir ? make_double2(a.x - b.y, a.y + b.x) : make_double2(a.x + b.y, -a.y + b.x);
            }
        }
    }
    dft_small<R>(z, y, tw, M);
#pragma unroll
    for (int sI = 0; sI < R; ++sI) so[sI][w][lane] = sI ? cmul(y[sI], __ldg(tw + sI * k1)) : y[sI];
    __syncthreads();
    const int kl = threadIdx.x & 7;
    for (int p = threadIdx.x >> 3; p < 32 * R; p += 32) {
        const int sI = p >> 5, rl = p & 31;
        const int ko = kb + kstep * rl;
        if (ko < K) Z[(size_t)ko * n2 + (size_t)sI * M + k10 + kl] = so[sI][kl][rl];
    }
}

__global__ void __launch_bounds__(256) k_pack_rows(const double2* __restrict__ Y, int n1, int m0,
                                                   int n2, int b1, int B1, double2* __restrict__ Z) {
    __shared__ double2 sy[32][33];  // [m][band row]
    const int mb = m0 + blockIdx.x * 32, cb = blockIdx.y * 32;  // 32 source columns m x 32 band rows
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int mhi = n2 / 2;
#pragma unroll
    for (int q = 0; q < 32; q += 8) {
        const int m = mb + ty + q, c = cb + tx;
        double2 v = make_double2(0.0, 0.0);
        if (m <= mhi && c < B1) v = Y[(size_t)(m - m0) * n1 + (c <= b1 ? c : n1 - B1 + c)];
        sy[ty + q][tx] = v;
    }
    __syncthreads();
    // each source column m feeds output columns m and (if m < n2/2, m > 0) n2 - m (conjugated)
#pragma unroll
    for (int q = 0; q < 16; q += 8) {
        const int kk = ty + q;  // packed row within the block (16 per block)
        const int k = (cb >> 1) + kk;
        const int m = mb + tx;
        if (m > mhi || 2 * k >= B1) continue;
        const double2 a = sy[tx][2 * kk];
        const double2 b = (2 * k + 1 < B1) ? sy[tx][2 * kk + 1] : make_double2(0.0, 0.0);
        // a + i b, and for the mirrored column conj(a) + i conj(b)
        Z[(size_t)k * n2 + m] = make_double2(a.x - b.y, a.y + b.x);
        if (m > 0 && m < mhi) Z[(size_t)k * n2 + (n2 - m)] = make_double2(a.x + b.y, -a.y + b.x);
    }
}

__global__ void k_mul(double2* x, const double2* __restrict__ m, uint64_t n) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k < n) x[k] = cmul(x[k], m[k]);
}

__global__ void k_conj(const double2* __restrict__ in, double2* out, uint64_t n) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = make_double2(in[k].x, -in[k].y);
}

// q_k += sum_{i in row k} D_i f_{col i}, sequential in CSR order like
// point_cloud.cpp:116-123.
__global__ void k_spmv(uint64_t rows, const uint64_t* __restrict__ ro,
                       const uint32_t* __restrict__ cols, const double2* __restrict__ vals,
                       const double2* __restrict__ f, double2* __restrict__ q) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= rows) return;
    double ar = 0.0, ai = 0.0;
    for (uint64_t i = ro[k]; i < ro[k + 1]; ++i) {
        const double2 v = vals[i];
        const double2 x = f[cols[i]];
        ar += v.x * x.x - v.y * x.y;
        ai += v.x * x.y + v.y * x.x;
    }
    double2 o = q[k];
    o.x += ar;
    o.y += ai;
    q[k] = o;
}

// q_{col} += conj(D_i) u_k (point_cloud.cpp:125-132), fp64 reductions.
__global__ void k_spmv_adjoint(uint64_t rows, const uint64_t* __restrict__ ro,
                               const uint32_t* __restrict__ cols,
                               const double2* __restrict__ vals,
                               const double2* __restrict__ u, double2* q) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= rows) return;
    const double2 uk = u[k];
    for (uint64_t i = ro[k]; i < ro[k + 1]; ++i) {
        const double2 v = vals[i];
        double* dst = reinterpret_cast<double*>(q + cols[i]);
        atomicAdd(dst, v.x * uk.x + v.y * uk.y);
        atomicAdd(dst + 1, v.x * uk.y - v.y * uk.x);
    }
}

inline unsigned blocks(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

template <template <int> class F, typename... Args>
void dispatch_w(int w, Args&&... args) {
    switch (w) {
#define SBD_W(N) \
    case N: F<N>::run(args...); break;
        SBD_W(4) SBD_W(5) SBD_W(6) SBD_W(7) SBD_W(8) SBD_W(9) SBD_W(10) SBD_W(11) SBD_W(12)
        SBD_W(13) SBD_W(14) SBD_W(15) SBD_W(16) SBD_W(17)
#undef SBD_W
        default: throw Error(3, "unsupported kernel width");
    }
}

template <int W>
struct SpreadRun {
    static void run(const WindowPoly& P, GridGeom g, uint64_t n, const uint32_t* perm,
                    const double2* in, const double2* pos, const double2* phase,
                    const double2* mult, const double* dx, const double* dy, double2* grid,
                    int conj_in, cudaStream_t st) {
        k_spread<W><<<blocks(n, 256), 256, 0, st>>>(P, g, n, perm, in, pos, phase, mult, dx, dy,
                                                    grid, conj_in);
    }
};

template <int W>
struct SpreadTilesRun {
    static size_t smem() { return (size_t)4 * 32 * W * 24 + 4 * 128 * sizeof(uint32_t) + 4 * 256 * sizeof(uint32_t); }
    static void run(const WindowPoly& P, GridGeom g, TileGeom tg, const uint32_t* bs,
                    const double2* b, const double2* pos, double2* grid, cudaStream_t st,
                    const uint32_t* bs2, const int* herm, const SpreadOut* out, const SpreadLists* lists,
                    int variant) {
        static bool attr = false;
        if (!attr) {
            ck(cudaFuncSetAttribute(k_spread_tiles<W, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem()),
               "smem attr");
            ck(cudaFuncSetAttribute(k_spread_tiles<W, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem()),
               "smem attr");
            attr = true;
        }
        const int tiles = tg.nbx * tg.nby;
        // variant 0: CTA spread over the plan's region lists; 1: CTA spread
        // scanning the bins; 2: per-warp DMMA spread; 3: scalar
        const int use_mma = variant != 3;
        const int use_cta = variant == 0 ? 1 : variant == 1 ? 2 : 0;
        static bool attr2 = false;
        if (!attr2) {
            attr2 = true;
            ck(cudaFuncSetAttribute(k_spread_mma<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem()),
               "smem attr");
            ck(cudaFuncSetAttribute(k_spread_cta<W, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)SCta<W>::smem),
               "smem attr");
            ck(cudaFuncSetAttribute(k_spread_cta<W, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)SCta<W>::smem_list),
               "smem attr");
            ck(cudaFuncSetAttribute(k_spread_cta<W, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)SCta<W>::smem),
               "smem attr");
            ck(cudaFuncSetAttribute(k_spread_cta<W, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)SCta<W>::smem_list),
               "smem attr");
            ck(cudaFuncSetAttribute(k_spread_cta<W, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)SCta<W>::smem_list),
               "smem attr");
        }
        SpreadOut so;
        if (out) {
            so = *out;
        } else {
            so.mode = 0;
            so.rend = tg.pitch ? tg.rhi : g.n1;
            so.cend = tg.pitch ? tg.chi : g.n2;
            so.pitch = tg.pitch ? (size_t)tg.pitch : (size_t)g.n2;
            so.r0 = tg.pitch ? tg.rlo : 0;
            so.c0 = tg.pitch ? tg.clo : 0;
            so.nby_run = tg.nby;
        }
        if (out && !(use_mma && tg.tr == 16)) throw Error(3, "spread output modes need the DMMA spread");
        if (lists) so.lists = *lists;
        if (use_cta && tg.tr == 16) {
            const int nblk = (so.ncx_run > 0 ? so.ncx_run : (tg.nbx + 1) / 2) * ((so.nby_run + 1) / 2);
            if (nblk <= 0) return;
            const bool cplx = so.mode == 0 || so.mode == 2, list = so.lists.s1 && use_cta == 1;
#define SBD_SPREAD_CTA(C, LI) \
    k_spread_cta<W, C, LI><<<nblk, 128, LI ? SCta<W>::smem_list : SCta<W>::smem, st>>>(P, g, tg, bs, b, pos, \
                                                                                       grid, bs2, herm, so)
            if (so.gen.id && !(cplx && list)) throw Error(3, "procedural nodes need the complex list spread");
            if (so.gen.id)
                k_spread_cta<W, true, true, true><<<nblk, 128, SCta<W>::smem_list, st>>>(P, g, tg, bs, b, pos, grid, bs2,
                                                                                       herm, so);
            else if (cplx && list) SBD_SPREAD_CTA(true, true);
            else if (cplx) SBD_SPREAD_CTA(true, false);
            else if (list) SBD_SPREAD_CTA(false, true);
            else SBD_SPREAD_CTA(false, false);
#undef SBD_SPREAD_CTA
        } else if (so.gen.id)
            throw Error(3, "procedural nodes need the CTA list spread");
        else if (use_mma && tg.tr == 16)
            k_spread_mma<W><<<(tg.nbx * so.nby_run + 3) / 4, 128, smem(), st>>>(P, g, tg, bs, b, pos, grid, bs2,
                                                                               herm, so);
        else if (tg.tr == 8)
            k_spread_tiles<W, 8><<<(tiles + 3) / 4, 128, smem(), st>>>(P, g, tg, bs, b, pos, grid, bs2, herm);
        else
            k_spread_tiles<W, 16><<<(tiles + 3) / 4, 128, smem(), st>>>(P, g, tg, bs, b, pos, grid, bs2, herm);
    }
};

template <int W>
struct InterpRun {
    static void run(const WindowPoly& P, GridGeom g, uint64_t n, const double2* pos,
                    const double2* phase, const double2* mult, const double* dx, const double* dy,
                    const double2* grid, const uint32_t* perm, const double2* addend, double2* out,
                    int acc, int cj, cudaStream_t st, bool trans, const InterpTiles* tiles,
                    const HermArgs* herm, int variant, const NodeGen* gen) {
        const HermArgs hh = herm ? *herm : HermArgs{};
        const NodeGen ng = gen ? *gen : NodeGen{};
        // tensor-core interpolation pays off when outputs are dense on the band
        // (>= 0.25 per cell: the xi side); variant 1 (staged tiles, needs the
        // tile list), 2 (DMMA per warp) or 3 (scalar) forces a choice
        const double density = (double)n / ((double)g.n1 * (double)g.n2 / (trans ? 2.0 : 4.0));
        const bool use_mma = variant ? (variant == 1 || variant == 2) : density >= 0.25;
        // sparser outputs on a band layout (the complex pipeline's targets) still
        // gain from the staged block: the wide-group path reads the footprint from
        // shared memory instead of L2 (config 4 with a complex f: 3.0 -> 1.95 ms)
        const bool sparse_tile = !variant && trans && density >= 0.05;
        const bool use_tile = ((use_mma || sparse_tile) && tiles && tiles->n && variant != 2) || hh.hcols;
        if (hh.hcols && !(tiles && tiles->n)) throw Error(3, "Hermitian band needs the staged interpolation");
        if (use_tile && !acc && !cj) {
            auto go = [&](auto kern, size_t smem, size_t& attr) {
                if (smem > attr) {
                    ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                       "interp tile smem");
                    attr = smem;
                }
                int dev = 0, sms = 148, per = 1;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kITW * 32, smem);
                const unsigned nb = (unsigned)std::min<uint64_t>(tiles->n, (uint64_t)sms * std::max(per, 1) * 8);
                kern<<<nb, kITW * 32, smem, st>>>(P, g, tiles->start, tiles->n, tiles->shift, tiles->out_lo, n, pos,
                                            phase, mult, dx, dy, grid, perm, addend, out, hh, ng);
            };
            static size_t attr_t = 0, attr_n = 0, attr_p = 0;  // per W (this template)
            if (ng.id && !trans) throw Error(3, "procedural nodes need the transposed staged interpolation");
            // every staged layout is copied by cp.async
            if (ng.id)
                go(k_interp_tile<W, true, true, true>, ITile<W, true>::smem, attr_p);
            else if (trans)
                go(k_interp_tile<W, true, false, true>, ITile<W, true>::smem, attr_t);
            else
                go(k_interp_tile<W, false, false, true>, ITile<W, false>::smem, attr_n);
            return;
        }
        if (ng.id) throw Error(3, "procedural nodes need the staged interpolation");
        if (use_mma && !acc && !cj) {
            const uint64_t warps = (n + 31) / 32;
            const unsigned grid_blocks = (unsigned)std::min<uint64_t>((warps + 3) / 4, 148ull * 16);
            if (trans)
                k_interp_mma<W, true><<<grid_blocks, 128, 0, st>>>(P, g, n, pos, phase, mult, dx, dy,
                                                                    grid, perm, addend, out, hh);
            else
                k_interp_mma<W, false><<<grid_blocks, 128, 0, st>>>(P, g, n, pos, phase, mult, dx, dy,
                                                                     grid, perm, addend, out, hh);
            return;
        }
        if (trans) {
            k_interp<W, true><<<blocks(n, 256), 256, 0, st>>>(P, g, n, pos, phase, mult, dx, dy, grid,
                                                              perm, addend, out, acc, cj, hh);
            return;
        }
        k_interp<W, false><<<blocks(n, 256), 256, 0, st>>>(P, g, n, pos, phase, mult, dx, dy, grid,
                                                           perm, addend, out, acc, cj, hh);
    }
};

} // namespace

void launch_ring_nodes(const uint32_t* id, uint64_t n, const RingRow* rings, double2* xi, double2* w,
                       cudaStream_t st) {
    if (!n) return;
    k_ring_nodes<<<blocks(n, 256), 256, 0, st>>>(id, n, rings, xi, w);
    count_launch();
    ck(cudaGetLastError(), "k_ring_nodes");
}

double node_deviation(const double2* a, const double2* b, uint64_t n, cudaStream_t st) {
    if (!n) return 0.0;
    DevBuf<unsigned long long> worst(1);
    ck(cudaMemsetAsync(worst.p, 0, sizeof(unsigned long long), st), "node deviation");
    k_node_deviation<<<blocks(n, 256), 256, 0, st>>>(a, b, n, worst.p);
    count_launch();
    unsigned long long bits = 0;
    ck(cudaMemcpyAsync(&bits, worst.p, sizeof(bits), cudaMemcpyDeviceToHost, st), "node deviation");
    ck(cudaStreamSynchronize(st), "node deviation");
    double d;
    static_assert(sizeof(d) == sizeof(bits), "double bits");
    std::memcpy(&d, &bits, sizeof(d));
    return d;
}

void launch_ring_point_arrays(const NodeGen& gen, uint64_t n, double2* t, double2* pre, cudaStream_t st) {
    if (!n) return;
    k_ring_point_arrays<<<blocks(n, 256), 256, 0, st>>>(gen, n, t, pre);
    count_launch();
    ck(cudaGetLastError(), "k_ring_point_arrays");
}

void launch_ring_output_arrays(const NodeGen& gen, uint64_t n, double2* s, double2* post, double2* kappa,
                               double2* kappa_h, cudaStream_t st) {
    if (!n) return;
    k_ring_output_arrays<<<blocks(n, 256), 256, 0, st>>>(gen, n, s, post, kappa, kappa_h);
    count_launch();
    ck(cudaGetLastError(), "k_ring_output_arrays");
}

void launch_plan_points(const double2* pts, uint64_t n, Axis ax, Axis ay, double beta,
                        double2* t, double2* pre, cudaStream_t st) {
    if (!n) return;
    k_plan_points<<<blocks(n, 256), 256, 0, st>>>(pts, n, ax, ay, beta, t, pre);
    count_launch();
    ck(cudaGetLastError(), "k_plan_points");
}

void launch_plan_outputs(const double2* frq, uint64_t n, Axis ax, Axis ay, double sgn,
                         double2* s, double2* post, cudaStream_t st) {
    if (!n) return;
    const double cx = 2.0 * kPi / (ax.n * ax.gamma);
    const double cy = 2.0 * kPi / (ay.n * ay.gamma);
    k_plan_outputs<<<blocks(n, 256), 256, 0, st>>>(frq, n, ax, ay, sgn, cx * cy, s, post);
    count_launch();
    ck(cudaGetLastError(), "k_plan_outputs");
}

void launch_bin_keys(const double2* pos, uint64_t n, GridGeom g, int tile, uint32_t* keys,
                     cudaStream_t st) {
    if (!n) return;
    k_bin_keys<<<blocks(n, 256), 256, 0, st>>>(pos, n, g, tile, keys);
    count_launch();
    ck(cudaGetLastError(), "k_bin_keys");
}

void launch_stencil_extent(const double2* pos, uint64_t n, double half, int* ext, cudaStream_t st) {
    const int init[4] = {INT_MAX, INT_MIN, INT_MAX, INT_MIN};
    ck(cudaMemcpyAsync(ext, init, sizeof(init), cudaMemcpyHostToDevice, st), "ext init");
    if (n) {
        k_stencil_extent<<<(unsigned)std::min<uint64_t>(blocks(n, 256), 148 * 16), 256, 0, st>>>(
            pos, n, half, ext);
        count_launch();
    }
    ck(cudaGetLastError(), "k_stencil_extent");
}

void launch_tile_keys(const double2* pos, uint64_t n, double half, TileGeom tg, uint32_t* keys,
                      cudaStream_t st, const uint8_t* tag) {
    if (!n) return;
    k_tile_keys<<<blocks(n, 256), 256, 0, st>>>(pos, n, half, tg, keys, tag);
    count_launch();
    ck(cudaGetLastError(), "k_tile_keys");
}

void build_region_lists(const double2* pos, uint64_t n, int w, TileGeom tg, uint32_t base, uint32_t tagbit,
                        DevBuf<uint32_t>& start, DevBuf<uint32_t>& ent, cudaStream_t st) {
    const int ncx = (tg.nbx + 1) / 2, ncy = (tg.nby + 1) / 2;
    const uint32_t nreg = (uint32_t)ncx * (uint32_t)ncy;
    start.alloc((uint64_t)nreg + 1);
    if (!n) {
        ck(cudaMemsetAsync(start.p, 0, ((uint64_t)nreg + 1) * 4, st), "region lists");
        ent.alloc(1);
        return;
    }
    DevBuf<uint32_t> keys(4 * n), vals(4 * n);
    k_region_pairs<<<blocks(n, 256), 256, 0, st>>>(pos, n, 0.5 * w, w, tg, ncx, ncy, base, tagbit, keys.p,
                                                   vals.p);
    count_launch();
    ck(cudaGetLastError(), "k_region_pairs");
    sort_by_key(keys.p, vals.p, 4 * n, st);
    // k_bin_bounds reads key >> 5; the unused slots (key nreg) sort last
    k_shift_keys<<<blocks(4 * n, 256), 256, 0, st>>>(keys.p, 4 * n);
    launch_bin_bounds(keys.p, 4 * n, nreg, start.p, st);
    uint32_t used = 0;
    ck(cudaMemcpyAsync(&used, start.p + nreg, 4, cudaMemcpyDeviceToHost, st), "region lists");
    ck(cudaStreamSynchronize(st), "region lists");
    ent.alloc(std::max<uint32_t>(used, 1));
    ck(cudaMemcpyAsync(ent.p, vals.p, (size_t)used * 4, cudaMemcpyDeviceToDevice, st), "region lists");
    ck(cudaStreamSynchronize(st), "region lists");
}

void launch_bin_bounds(const uint32_t* sorted_keys, uint64_t n, uint32_t nbins, uint32_t* start,
                       cudaStream_t st, uint32_t base, uint32_t mask) {
    k_bin_bounds<<<blocks(n + 1, 256), 256, 0, st>>>(sorted_keys, n, nbins, start, base, mask);
    count_launch();
    ck(cudaGetLastError(), "k_bin_bounds");
}

void launch_spread_tiles(int w, const WindowPoly& win, GridGeom g, TileGeom tg,
                         const uint32_t* bin_start, const double2* b, const double2* pos,
                         double2* grid, cudaStream_t st, const uint32_t* bin_start2,
                         const int* herm, const SpreadOut* out, const SpreadLists* lists, int variant) {
    if (tg.nbx * tg.nby == 0) return;
    dispatch_w<SpreadTilesRun>(w, win, g, tg, bin_start, b, pos, grid, st, bin_start2, herm, out, lists, variant);
    count_launch();
    ck(cudaGetLastError(), "k_spread_tiles");
}

void launch_morton_keys(const double2* pos, uint64_t n, double half, int shift, uint32_t* keys,
                        cudaStream_t st, const uint8_t* tag) {
    if (!n) return;
    k_morton_keys<<<blocks(n, 256), 256, 0, st>>>(pos, n, half, shift, keys, tag);
    count_launch();
    ck(cudaGetLastError(), "k_morton_keys");
}

void launch_iota(uint32_t* v, uint64_t n, cudaStream_t st) {
    if (!n) return;
    k_iota<<<blocks(n, 256), 256, 0, st>>>(v, n);
    count_launch();
}

void sort_by_key(uint32_t* keys, uint32_t* vals, uint64_t n, cudaStream_t st) {
    if (n < 2) return;
    DevBuf<uint32_t> k2(n), v2(n);
    size_t tmp = 0;
    ck(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, k2.p, vals, v2.p, (int)n, 0, 32, st),
       "cub sort (size)");
    DevBuf<unsigned char> t(tmp);
    ck(cub::DeviceRadixSort::SortPairs(t.p, tmp, keys, k2.p, vals, v2.p, (int)n, 0, 32, st),
       "cub sort");
    count_launch(4);
    ck(cudaMemcpyAsync(keys, k2.p, n * 4, cudaMemcpyDeviceToDevice, st), "sort copy");
    ck(cudaMemcpyAsync(vals, v2.p, n * 4, cudaMemcpyDeviceToDevice, st), "sort copy");
    ck(cudaStreamSynchronize(st), "sort sync");
}

template <typename T>
void launch_gather(const T* src, const uint32_t* perm, T* dst, uint64_t n, cudaStream_t st) {
    if (!n) return;
    k_gather<T><<<blocks(n, 256), 256, 0, st>>>(src, perm, dst, n);
    count_launch();
}
template void launch_gather<double2>(const double2*, const uint32_t*, double2*, uint64_t,
                                     cudaStream_t);
template void launch_gather<uint32_t>(const uint32_t*, const uint32_t*, uint32_t*, uint64_t,
                                      cudaStream_t);

void launch_spread(int w, const WindowPoly& win, GridGeom g, uint64_t n, const uint32_t* perm,
                   const double2* in, const double2* pos, const double2* phase,
                   const double2* mult, const double* dx, const double* dy, double2* grid,
                   int conj_in, cudaStream_t st) {
    if (!n) return;
    dispatch_w<SpreadRun>(w, win, g, n, perm, in, pos, phase, mult, dx, dy, grid, conj_in, st);
    count_launch();
    ck(cudaGetLastError(), "k_spread");
}

void launch_interp(int w, const WindowPoly& win, GridGeom g, uint64_t n, const double2* pos,
                   const double2* phase, const double2* mult, const double* dx, const double* dy,
                   const double2* grid, const uint32_t* perm, double2* out, int accumulate,
                   int conj_out, cudaStream_t st, const double2* addend, bool transposed,
                   const InterpTiles* tiles, const HermArgs* herm, int variant, const NodeGen* gen) {
    if (!n) return;
    dispatch_w<InterpRun>(w, win, g, n, pos, phase, mult, dx, dy, grid, perm, addend, out,
                          accumulate, conj_out, st, transposed, tiles, herm, variant, gen);
    count_launch();
    ck(cudaGetLastError(), "k_interp");
}

template <int W>
struct InterpRealRun {
    static void run(const WindowPoly& P, GridGeom g, uint64_t n, const double2* pos, const double2* phase,
                    const double* dx, const double* dy, const double* grid, const uint32_t* perm,
                    const double2* addend, double2* out, cudaStream_t st, const InterpTiles* tiles,
                    int variant) {
        const bool staged = variant != 3;
        if (staged && tiles && tiles->n) {
            int dev = 0, sms = 148, per = 1;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_interp_real_tile<W>, 128, 0);
            const unsigned nb = (unsigned)std::min<uint64_t>(tiles->n, (uint64_t)sms * std::max(per, 1) * 8);
            k_interp_real_tile<W><<<nb, 128, 0, st>>>(P, g, tiles->start, tiles->n, tiles->shift, tiles->out_lo,
                                                       n, pos, phase, dx, dy, grid, perm, addend, out);
            return;
        }
        k_interp_real<W><<<blocks(n, 256), 256, 0, st>>>(P, g, n, pos, phase, dx, dy, grid, perm, addend, out);
    }
};

void launch_interp_real(int w, const WindowPoly& win, GridGeom g, uint64_t n, const double2* pos,
                        const double2* phase, const double* dx, const double* dy, const double* grid,
                        const uint32_t* perm, const double2* addend, double2* out, cudaStream_t st,
                        const InterpTiles* tiles, int variant) {
    if (!n) return;
    dispatch_w<InterpRealRun>(w, win, g, n, pos, phase, dx, dy, grid, perm, addend, out, st, tiles, variant);
    count_launch();
    ck(cudaGetLastError(), "k_interp_real");
}

// Within each 32 x 32 block of Z-ordered outputs, deal the outputs round-robin
// over the 16 shared-memory double-banks their staged-tile reads start on
// (k_interp_real_tile: lane = output, address (ix - X0) PE + (iy - Y0) + i PE
// + j), so each warp's 32 outputs spread ~2 per double-bank: the tap loads of
// the staged target interpolation need ~2 wavefronts instead of ~4.6 for
// random positions. The order inside a block is otherwise free.
// map[new sorted position] = old sorted position.
__global__ void __launch_bounds__(128) k_bank_interleave(const uint32_t* __restrict__ tstart, uint32_t ntiles,
                                                         const double2* __restrict__ pos, double half, int shift,
                                                         int pe, uint32_t* __restrict__ map) {
    constexpr int kMax = 1024;
    __shared__ uint8_t sb[kMax];
    __shared__ uint16_t srank[kMax];
    __shared__ int cntb[16];
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint32_t t0 = tstart[t], t1 = tstart[t + 1];
        const uint32_t c = t1 - t0;
        if (c > kMax) {  // (dense block: keep the Z order)
            for (uint32_t k = threadIdx.x; k < c; k += blockDim.x) map[t0 + k] = t0 + k;
            continue;
        }
        const double2 s0 = pos[t0];
        const int X0 = (((int)ceil(s0.x - half) + shift) & ~31) - shift;
        const int Y0 = (((int)ceil(s0.y - half) + shift) & ~31) - shift;
        __syncthreads();
        if (threadIdx.x < 16) cntb[threadIdx.x] = 0;
        for (uint32_t k = threadIdx.x; k < c; k += blockDim.x) {
            const double2 sv = pos[t0 + k];
            const int ix = (int)ceil(sv.x - half), iy = (int)ceil(sv.y - half);
            sb[k] = (uint8_t)((((ix - X0) * pe + (iy - Y0)) % 16 + 16) % 16);
        }
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < c; k += blockDim.x) {
            int r = 0;
            for (uint32_t q = 0; q < k; ++q) r += sb[q] == sb[k];
            srank[k] = (uint16_t)r;
            atomicAdd(&cntb[sb[k]], 1);
        }
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < c; k += blockDim.x) {
            const int r = srank[k], b = sb[k];
            int p = 0;
            for (int q = 0; q < 16; ++q) p += min(cntb[q], r) + (q < b && cntb[q] > r ? 1 : 0);
            map[t0 + p] = t0 + k;
        }
    }
}

void bank_interleave_outputs(const uint32_t* tile_start, uint32_t ntiles, const double2* pos, uint64_t n, int w,
                             int shift, DevBuf<uint32_t>& map, cudaStream_t st) {
    map.alloc(std::max<uint64_t>(n, 1));
    if (!ntiles) return;
    const int pe = (32 + w - 1) | 1;  // k_interp_real_tile's staged-tile pitch
    k_bank_interleave<<<std::min<uint32_t>(ntiles, 148 * 16), 128, 0, st>>>(tile_start, ntiles, pos, 0.5 * w, shift,
                                                                          pe, map.p);
    count_launch();
    ck(cudaGetLastError(), "k_bank_interleave");
}

void build_tile_starts(const uint32_t* sorted_keys, uint64_t n, int bits, DevBuf<uint32_t>& start,
                       uint32_t& ntiles, cudaStream_t st) {
    ntiles = 0;
    if (!n) return;
    DevBuf<uint32_t> flag(n), idx(n);
    k_tile_flags<<<blocks(n, 256), 256, 0, st>>>(sorted_keys, n, bits, flag.p);
    size_t tmp = 0;
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag.p, idx.p, (int)n, st), "tile scan (size)");
    DevBuf<unsigned char> t(tmp);
    ck(cub::DeviceScan::ExclusiveSum(t.p, tmp, flag.p, idx.p, (int)n, st), "tile scan");
    uint32_t last[2];
    ck(cudaMemcpyAsync(&last[0], idx.p + n - 1, 4, cudaMemcpyDeviceToHost, st), "tile count");
    ck(cudaMemcpyAsync(&last[1], flag.p + n - 1, 4, cudaMemcpyDeviceToHost, st), "tile count");
    ck(cudaStreamSynchronize(st), "tile count");
    ntiles = last[0] + last[1];
    start.alloc((size_t)ntiles + 1);
    k_tile_scatter<<<blocks(n, 256), 256, 0, st>>>(flag.p, idx.p, n, start.p);
    count_launch(4);
    ck(cudaStreamSynchronize(st), "tile starts");
}

void launch_ndft(const double2* pts, uint64_t np, const double2* frq, uint64_t nf,
                 const double2* c, int sign, double2* out, cudaStream_t st) {
    if (!nf) return;
    k_ndft<<<blocks(nf, 128), 128, 0, st>>>(pts, np, frq, nf, c, sign > 0 ? 1.0 : -1.0, out);
    count_launch();
    ck(cudaGetLastError(), "k_ndft");
}

void launch_gather_mul(const double2* in, const uint32_t* perm, const double2* phase, double2* b,
                       double2* raw, uint64_t n, cudaStream_t st, uint64_t lo, uint64_t hi,
                       int* clear, double* raw_re) {
    if (!n) return;
    k_gather_mul<<<blocks(n, 256), 256, 0, st>>>(in, perm, phase, b, raw, n, lo, hi, clear, raw_re);
    count_launch();
    ck(cudaGetLastError(), "k_gather_mul");
}

void launch_spmv_vec(uint64_t rows, const uint64_t* ro, const uint32_t* cols, const double2* vals,
                     const double2* f, double2* qs, cudaStream_t st, bool accumulate) {
    if (!rows) return;
    k_spmv_vec<<<blocks(rows * 8, 256), 256, 0, st>>>(rows, ro, cols, vals, f, qs, accumulate ? 1 : 0);
    count_launch();
    ck(cudaGetLastError(), "k_spmv_vec");
}

// k_spmv_vec / k_spmv_vec_real for NR right-hand sides at once: each
// nonzero's value and column are loaded once; per column the summation
// order is the single-RHS kernels' (bitwise equal results).
template <int NR, bool RD>
__global__ void __launch_bounds__(256) k_spmm(uint64_t rows, const uint64_t* __restrict__ ro,
                                              const uint32_t* __restrict__ cols,
                                              const double2* __restrict__ vals,
                                              const double* __restrict__ vals_r,
                                              const double2* __restrict__ f, uint64_t ldf,
                                              double2* __restrict__ qs, uint64_t ldq, SpmmCols cs) {
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t r = g >> 3;
    const int sub = (int)(g & 7);
    double ar[NR], ai[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) ar[j] = ai[j] = 0.0;
    if (r < rows) {
        const uint64_t e = ro[r + 1];
        for (uint64_t i = ro[r] + sub; i < e; i += 8) {
            const uint32_t c = cols[i];
            if (RD) {
                const double v = vals_r[i];
#pragma unroll
                for (int j = 0; j < NR; ++j) {
                    const double2 x = f[(size_t)cs.idx[j] * ldf + c];
                    ar[j] = fma(v, x.x, ar[j]);
                    ai[j] = fma(v, x.y, ai[j]);
                }
            } else {
                const double2 v = vals[i];
#pragma unroll
                for (int j = 0; j < NR; ++j) {
                    const double2 x = f[(size_t)cs.idx[j] * ldf + c];
                    ar[j] = fma(v.x, x.x, ar[j]);
                    ar[j] = fma(-v.y, x.y, ar[j]);
                    ai[j] = fma(v.x, x.y, ai[j]);
                    ai[j] = fma(v.y, x.x, ai[j]);
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < NR; ++j)
#pragma unroll
        for (int o = 4; o; o >>= 1) {
            ar[j] += __shfl_xor_sync(0xffffffffu, ar[j], o);
            ai[j] += __shfl_xor_sync(0xffffffffu, ai[j], o);
        }
    if (r < rows && sub == 0)
#pragma unroll
        for (int j = 0; j < NR; ++j) qs[(size_t)cs.idx[j] * ldq + r] = make_double2(ar[j], ai[j]);
}

template <int NR>
static void spmm_nr(uint64_t rows, const uint64_t* ro, const uint32_t* cols, const double2* vals,
                    const double* vals_r, const double2* f, uint64_t ldf, double2* qs, uint64_t ldq,
                    const SpmmCols& cs, cudaStream_t st) {
    if (vals_r)
        k_spmm<NR, true><<<blocks(rows * 8, 256), 256, 0, st>>>(rows, ro, cols, vals, vals_r, f, ldf, qs, ldq, cs);
    else
        k_spmm<NR, false><<<blocks(rows * 8, 256), 256, 0, st>>>(rows, ro, cols, vals, vals_r, f, ldf, qs, ldq, cs);
}

void launch_spmm(uint64_t rows, const uint64_t* ro, const uint32_t* cols, const double2* vals,
                 const double* vals_r, const double2* f, uint64_t ldf, double2* qs, uint64_t ldq,
                 const SpmmCols& cs, cudaStream_t st) {
    if (!rows || !cs.n) return;
    switch (cs.n) {
        case 1: spmm_nr<1>(rows, ro, cols, vals, vals_r, f, ldf, qs, ldq, cs, st); break;
        case 2: spmm_nr<2>(rows, ro, cols, vals, vals_r, f, ldf, qs, ldq, cs, st); break;
        case 3: spmm_nr<3>(rows, ro, cols, vals, vals_r, f, ldf, qs, ldq, cs, st); break;
        case 4: spmm_nr<4>(rows, ro, cols, vals, vals_r, f, ldf, qs, ldq, cs, st); break;
        case 5: spmm_nr<5>(rows, ro, cols, vals, vals_r, f, ldf, qs, ldq, cs, st); break;
        case 6: spmm_nr<6>(rows, ro, cols, vals, vals_r, f, ldf, qs, ldq, cs, st); break;
        case 7: spmm_nr<7>(rows, ro, cols, vals, vals_r, f, ldf, qs, ldq, cs, st); break;
        default: spmm_nr<8>(rows, ro, cols, vals, vals_r, f, ldf, qs, ldq, cs, st); break;
    }
    count_launch();
    ck(cudaGetLastError(), "k_spmm");
}

void launch_spmv_vec_real(uint64_t rows, const uint64_t* ro, const uint32_t* cols, const double* vals,
                          const double2* f, double2* qs, cudaStream_t st, const double* f_re) {
    if (!rows) return;
    if (f_re)
        k_spmv_vec_rr<<<blocks(rows * 8, 256), 256, 0, st>>>(rows, ro, cols, vals, f_re, qs);
    else
        k_spmv_vec_real<<<blocks(rows * 8, 256), 256, 0, st>>>(rows, ro, cols, vals, f, qs);
    count_launch();
    ck(cudaGetLastError(), "k_spmv_vec_real");
}

void launch_gather_conj_mul(const double2* in, const uint32_t* perm, const double2* phase, int conj_in,
                            double2* b, uint64_t n, cudaStream_t st) {
    if (!n) return;
    k_gather_conj_mul<<<blocks(n, 256), 256, 0, st>>>(in, perm, phase, conj_in, b, n);
    count_launch();
    ck(cudaGetLastError(), "k_gather_conj_mul");
}

void launch_band_fold(const double2* Z, int pz, int rlo, int rhi, int clo, int chi, int b1, int n1, int b2,
                      int B, int n2, const double* dx, const double* dy, double2* V, cudaStream_t st) {
    const uint64_t n = (uint64_t)(2 * b1 + 1) * (uint64_t)B;
    k_band_fold<<<blocks(n, 256), 256, 0, st>>>(Z, pz, rlo, rhi, clo, chi, b1, n1, b2, B, n2, dx, dy, V);
    count_launch();
    ck(cudaGetLastError(), "k_band_fold");
}

void launch_band_untranspose(const double2* Wt, int n1, int r0, int r1, int b, int B, double2* Tz, int n2,
                             cudaStream_t st, int rin) {
    if (r1 <= r0) return;
    dim3 grid((unsigned)((B + 31) / 32), (unsigned)(((rin > 1 ? n1 : r1 - r0) + 31) / 32));
    k_band_untranspose<<<grid, 256, 0, st>>>(Wt, n1, r0, r1, b, B, Tz, n2, rin);
    count_launch();
    ck(cudaGetLastError(), "k_band_untranspose");
}

__global__ void __launch_bounds__(256) k_wrap_transpose(const double2* __restrict__ in, size_t ipitch, int nin,
                                                        int j0, int L, int Q, double2* __restrict__ out,
                                                        size_t opitch) {
    __shared__ double2 tile[32][33];
    const int lb = blockIdx.x * 32, qb = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const int q = qb + ty + k, l = lb + tx;
        if (q < Q && l < L) {
            int c = (j0 + l) % nin;
            if (c < 0) c += nin;
            tile[ty + k][tx] = in[(size_t)q * ipitch + c];
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const int l = lb + ty + k, q = qb + tx;
        if (q < Q && l < L) out[(size_t)l * opitch + q] = tile[tx][ty + k];
    }
}

void launch_wrap_transpose(const double2* in, size_t ipitch, int nin, int j0, int L, int Q, double2* out,
                           size_t opitch, cudaStream_t st) {
    if (L <= 0 || Q <= 0) return;
    dim3 grid((unsigned)((L + 31) / 32), (unsigned)((Q + 31) / 32));
    k_wrap_transpose<<<grid, 256, 0, st>>>(in, ipitch, nin, j0, L, Q, out, opitch);
    count_launch();
    ck(cudaGetLastError(), "k_wrap_transpose");
}

void launch_band_transpose(const double2* T, int n2, int r0, int r1, int b, int B, double2* Tt,
                           int n1, cudaStream_t st, int rin0, int conj_out, int rin) {
    if (r1 <= r0) return;
    // permuted rows: CTAs walk the row positions (about half hold band modes)
    dim3 grid((unsigned)(((rin > 1 ? n2 : B) + 31) / 32), (unsigned)((r1 - r0 + 31) / 32));
    k_band_transpose<<<grid, 256, 0, st>>>(T, n2, r0, r1, b, B, Tt, n1, rin0, conj_out, rin);
    count_launch();
    ck(cudaGetLastError(), "k_band_transpose");
}

void launch_band_transpose_dif(const double2* T, int n2, int r0, int r1, int b, int B, double2* Tt, int n1, int R,
                               const double2* tw, cudaStream_t st, int rin) {
    if (r1 <= r0) return;
    const int M = n1 / R;
    dim3 grid((unsigned)(((rin > 1 ? n2 : B) + 31) / 32), (unsigned)(M / 8));
    if (R == 9)
        k_band_transpose_dif<9><<<grid, 256, 0, st>>>(T, n2, r0, r1, b, B, Tt, n1, M, tw, rin);
    else if (R == 5)
        k_band_transpose_dif<5><<<grid, 256, 0, st>>>(T, n2, r0, r1, b, B, Tt, n1, M, tw, rin);
    else if (R == 3)
        k_band_transpose_dif<3><<<grid, 256, 0, st>>>(T, n2, r0, r1, b, B, Tt, n1, M, tw, rin);
    else
        throw Error(3, "band_transpose_dif: unsupported radix");
    count_launch();
    ck(cudaGetLastError(), "k_band_transpose_dif");
}

void launch_dif_rows(const double2* X, int rows, int n, int R, int c_lo, int c_hi, const double2* tw, double2* Y,
                     cudaStream_t st) {
    if (rows <= 0) return;
    const int M = n / R;
    dim3 grid((unsigned)((M + 255) / 256), (unsigned)rows);
    if (R == 9)
        k_dif_rows<9><<<grid, 256, 0, st>>>(X, n, M, c_lo, c_hi, tw, Y);
    else if (R == 5)
        k_dif_rows<5><<<grid, 256, 0, st>>>(X, n, M, c_lo, c_hi, tw, Y);
    else if (R == 3)
        k_dif_rows<3><<<grid, 256, 0, st>>>(X, n, M, c_lo, c_hi, tw, Y);
    else
        throw Error(3, "dif_rows: unsupported radix");
    count_launch();
    ck(cudaGetLastError(), "k_dif_rows");
}

void launch_untangle_dif(const double2* T, int n2, int nr, int B, double2* Tt, int n1, int r0, int R,
                        const double2* tw, cudaStream_t st, const double* colf, int rin) {
    if (nr <= 0 || B <= 0) return;
    const int M = n1 / R;
    dim3 grid((unsigned)((B + 31) / 32), (unsigned)(M / 8));
    if (rin > 1) {
        if (R != 9 || rin != 9) throw Error(3, "untangle_dif: the permuted row input needs radix 9 on both sides");
        grid.x = (unsigned)(9 * (((B + 8) / 9 + 31) / 32));
        k_untangle_dif<9, 9><<<grid, 256, 0, st>>>(T, n2, nr, B, Tt, n1, r0, M, tw, colf);
    } else if (R == 9)
        k_untangle_dif<9><<<grid, 256, 0, st>>>(T, n2, nr, B, Tt, n1, r0, M, tw, colf);
    else if (R == 5)
        k_untangle_dif<5><<<grid, 256, 0, st>>>(T, n2, nr, B, Tt, n1, r0, M, tw, colf);
    else if (R == 3)
        k_untangle_dif<3><<<grid, 256, 0, st>>>(T, n2, nr, B, Tt, n1, r0, M, tw, colf);
    else
        throw Error(3, "untangle_dif: unsupported radix");
    count_launch();
    ck(cudaGetLastError(), "k_untangle_dif");
}

void launch_pack_dif(const double2* Y, int n1, int m0, int n2, int b1, int B1, double2* Z, int R,
                     const double2* tw, cudaStream_t st, int rin) {
    const int K = (B1 + 1) / 2, M = n2 / R;
    if (K <= 0) return;
    dim3 grid((unsigned)((K + 31) / 32), (unsigned)(M / 8));
    if (rin > 1) {
        if (R != 9 || rin != 9) throw Error(3, "pack_dif: the permuted column input needs radix 9 on both sides");
        grid.x = (unsigned)(9 * (((K + 8) / 9 + 31) / 32));
        k_pack_dif<9, 9><<<grid, 256, 0, st>>>(Y, n1, m0, n2, b1, B1, Z, M, tw);
    } else if (R == 9)
        k_pack_dif<9><<<grid, 256, 0, st>>>(Y, n1, m0, n2, b1, B1, Z, M, tw);
    else if (R == 5)
        k_pack_dif<5><<<grid, 256, 0, st>>>(Y, n1, m0, n2, b1, B1, Z, M, tw);
    else if (R == 3)
        k_pack_dif<3><<<grid, 256, 0, st>>>(Y, n1, m0, n2, b1, B1, Z, M, tw);
    else
        throw Error(3, "pack_dif: unsupported radix");
    count_launch();
    ck(cudaGetLastError(), "k_pack_dif");
}

void launch_untangle_transpose(const double2* T, int n2, int nr, int B, double2* Tt, int n1, int r0,
                               cudaStream_t st) {
    if (nr <= 0 || B <= 0) return;
    dim3 grid((unsigned)((B + 31) / 32), (unsigned)((nr + 15) / 16));
    k_untangle_transpose<<<grid, 256, 0, st>>>(T, n2, nr, B, Tt, n1, r0);
    count_launch();
    ck(cudaGetLastError(), "k_untangle_transpose");
}

void launch_pack_rows(const double2* Y, int n1, int m0, int n2, int b1, int B1, double2* Z, cudaStream_t st) {
    const int nm = n2 / 2 - m0 + 1;
    if (nm <= 0) return;
    dim3 grid((unsigned)((nm + 31) / 32), (unsigned)((B1 + 31) / 32));
    k_pack_rows<<<grid, 256, 0, st>>>(Y, n1, m0, n2, b1, B1, Z);
    count_launch();
    ck(cudaGetLastError(), "k_pack_rows");
}

void launch_conj_scatter(const double2* in, uint64_t n, const uint32_t* idx, double2* out, cudaStream_t st) {
    if (!n) return;
    k_conj_scatter<<<blocks(n, 256), 256, 0, st>>>(in, n, idx, out);
    count_launch();
    ck(cudaGetLastError(), "k_conj_scatter");
}

void launch_mirror_points(const double2* t, uint64_t n, int n1, int n2, int w, double2* out,
                          cudaStream_t st) {
    if (!n) return;
    k_mirror_points<<<blocks(n, 256), 256, 0, st>>>(t, n, n1, n2, w, out);
    count_launch();
    ck(cudaGetLastError(), "k_mirror_points");
}

void launch_any_imag(const double2* x, uint64_t n, int* flag, cudaStream_t st) {
    ck(cudaMemsetAsync(flag, 0, sizeof(int), st), "imag flag");
    if (!n) return;
    k_any_imag<<<(unsigned)std::min<uint64_t>(blocks(n, 256), 148 * 8), 256, 0, st>>>(x, n, flag);
    count_launch();
    ck(cudaGetLastError(), "k_any_imag");
}

void launch_mul(double2* x, const double2* m, uint64_t n, cudaStream_t st) {
    if (!n) return;
    k_mul<<<blocks(n, 256), 256, 0, st>>>(x, m, n);
    count_launch();
}

void launch_conj(const double2* in, double2* out, uint64_t n, cudaStream_t st) {
    if (!n) return;
    k_conj<<<blocks(n, 256), 256, 0, st>>>(in, out, n);
    count_launch();
}

void launch_spmv(uint64_t rows, const uint64_t* ro, const uint32_t* cols, const double2* vals,
                 const double2* f, double2* q, cudaStream_t st) {
    if (!rows) return;
    k_spmv<<<blocks(rows, 256), 256, 0, st>>>(rows, ro, cols, vals, f, q);
    count_launch();
    ck(cudaGetLastError(), "k_spmv");
}

void launch_spmv_adjoint(uint64_t rows, const uint64_t* ro, const uint32_t* cols,
                         const double2* vals, const double2* u, double2* q, cudaStream_t st) {
    if (!rows) return;
    k_spmv_adjoint<<<blocks(rows, 256), 256, 0, st>>>(rows, ro, cols, vals, u, q);
    count_launch();
    ck(cudaGetLastError(), "k_spmv_adjoint");
}

} // namespace sbdgpu
