// assemble_kernels.cu -- offline close-correction matrix D on the GPU.
//
// Reference: neighbor_pairs (point_cloud.cpp:74-114, hash grid with cell =
// radius, rows sorted) and assemble_close_matrix (conv_operator.cpp:172-237:
// D = G(|y|) - sum_v w_v e^{i y.xi_v} for every pair closer than delta_min,
// plus the -sum(w) diagonal for a single cloud).
//
// GPU formulation: sources are radix-sorted by cell; a count pass and a fill
// pass scan the 3x3 neighbourhood of each target; each row is sorted in
// registers. The far field at all pair differences comes from ONE type-III
// NUFFT whose grid covers the bounding box of every difference (the reference
// re-spreads all N_xi nodes for every 4 Mi-pair chunk, conv_operator.cpp:186-199,
// which is what makes its offline stage take hours at N = 1e7): the omega-hat
// spectrum is spread once onto a small grid, transformed once, and each pair's
// difference is formed on the fly and interpolated (k_close_values).
#include <cstdlib>
#include <cstdio>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "assemble_gpu.h"
#include "device_common.cuh"

namespace sbdgpu {

namespace {

using namespace dev;

inline unsigned nblk(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

struct CellGrid {
    double ox, oy, cell;
    int ncx, ncy;
};

__device__ __forceinline__ int cell_of(double v, double o, double cell, int nc) {
    int c = (int)floor((v - o) / cell);
    return c < 0 ? 0 : (c >= nc ? nc - 1 : c);
}

__global__ void k_cell_keys(const double2* __restrict__ p, uint64_t n, CellGrid g,
                            uint32_t* __restrict__ keys, uint32_t* __restrict__ idx,
                            uint32_t* __restrict__ counts) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int cx = cell_of(p[i].x, g.ox, g.cell, g.ncx), cy = cell_of(p[i].y, g.oy, g.cell, g.ncy);
    const uint32_t key = (uint32_t)cx * (uint32_t)g.ncy + (uint32_t)cy;
    keys[i] = key;
    idx[i] = (uint32_t)i;
    atomicAdd(counts + key, 1u);
}

// dist^2 <= r^2 exactly as point_cloud.cpp:108 (no FMA contraction)
__device__ __forceinline__ bool close_enough(double2 a, double2 b, double r2) {
    const double dx = __dsub_rn(a.x, b.x), dy = __dsub_rn(a.y, b.y);
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= r2;
}

template <bool kFill>
__global__ void k_pairs(const double2* __restrict__ tgt, uint64_t nt,
                        const double2* __restrict__ src_sorted, const uint32_t* __restrict__ idx,
                        const uint32_t* __restrict__ cell_start, CellGrid g, double r2, int single,
                        uint64_t* __restrict__ counts, const uint64_t* __restrict__ offsets,
                        uint32_t* __restrict__ cols) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= nt) return;
    const double2 z = tgt[k];
    const int cx = (int)floor((z.x - g.ox) / g.cell), cy = (int)floor((z.y - g.oy) / g.cell);
    uint64_t n = 0;
    uint64_t base = kFill ? offsets[k] : 0;
    for (int dx = -1; dx <= 1; ++dx) {
        const int x = cx + dx;
        if (x < 0 || x >= g.ncx) continue;
        for (int dy = -1; dy <= 1; ++dy) {
            const int y = cy + dy;
            if (y < 0 || y >= g.ncy) continue;
            const uint32_t key = (uint32_t)x * (uint32_t)g.ncy + (uint32_t)y;
            for (uint32_t s = cell_start[key]; s < cell_start[key + 1]; ++s) {
                const uint32_t l = idx[s];
                if (single && l == (uint32_t)k) continue;
                if (close_enough(z, src_sorted[s], r2)) {
                    if (kFill) cols[base + n] = l;
                    ++n;
                }
            }
        }
    }
    if (single) { // diagonal slot: -sum(w), conv_operator.cpp:208-236
        if (kFill) cols[base + n] = (uint32_t)k;
        ++n;
    }
    if (!kFill) {
        counts[k] = n;
        return;
    }
    // sort the row ascending (point_cloud.cpp:111-113)
    uint32_t* c = cols + base;
    for (uint64_t i = 1; i < n; ++i) {
        const uint32_t v = c[i];
        uint64_t j = i;
        while (j > 0 && c[j - 1] > v) {
            c[j] = c[j - 1];
            --j;
        }
        c[j] = v;
    }
}

__global__ void k_row_index(const uint64_t* __restrict__ ro, uint64_t nt, uint32_t* __restrict__ row) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= nt) return;
    for (uint64_t i = ro[k]; i < ro[k + 1]; ++i) row[i] = (uint32_t)k;
}

// order-preserving double <-> u64 for atomic min/max
__device__ __forceinline__ unsigned long long ord(double v) {
    const unsigned long long b = __double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_diff_extrema(const double2* __restrict__ tgt, const double2* __restrict__ src,
                               const uint32_t* __restrict__ row, const uint32_t* __restrict__ cols,
                               uint64_t nnz, int single, unsigned long long* __restrict__ ext) {
    double mnx = 1e300, mxx = -1e300, mny = 1e300, mxy = -1e300;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nnz;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = row[i], c = cols[i];
        if (single && r == c) continue;
        const double yx = tgt[r].x - src[c].x, yy = tgt[r].y - src[c].y;
        mnx = fmin(mnx, yx);
        mxx = fmax(mxx, yx);
        mny = fmin(mny, yy);
        mxy = fmax(mxy, yy);
    }
    typedef cub::BlockReduce<double, 256> BR;
    __shared__ typename BR::TempStorage ts;
    const double a = BR(ts).Reduce(mnx, cub::Min());
    __syncthreads();
    const double b = BR(ts).Reduce(mxx, cub::Max());
    __syncthreads();
    const double c = BR(ts).Reduce(mny, cub::Min());
    __syncthreads();
    const double d = BR(ts).Reduce(mxy, cub::Max());
    if (threadIdx.x == 0) {
        atomicMin(ext + 0, ord(a));
        atomicMax(ext + 1, ord(b));
        atomicMin(ext + 2, ord(c));
        atomicMax(ext + 3, ord(d));
    }
}

// far(y) by interpolation on the omega-hat grid (same plan arithmetic as
// k_plan_outputs + k_interp), then D = G(|y|) - far for Laplace (G = log r);
// for Helmholtz only -far is stored and the host adds G.
template <int W>
__global__ void __launch_bounds__(256) k_close_values(
    WindowPoly P, GridGeom g, Axis ax, Axis ay, double cxy, const double* __restrict__ dxt,
    const double* __restrict__ dyt, const double2* __restrict__ grid,
    const double2* __restrict__ tgt, const double2* __restrict__ src,
    const uint32_t* __restrict__ row, const uint32_t* __restrict__ cols, uint64_t nnz, int single,
    double2 diag, int laplace, double2* __restrict__ vals, int* __restrict__ bad) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= nnz) return;
    const uint32_t r = row[i], c = cols[i];
    if (single && r == c) {
        vals[i] = diag;
        return;
    }
    const double yx = __dsub_rn(tgt[r].x, src[c].x), yy = __dsub_rn(tgt[r].y, src[c].y);
    const double sx = __dmul_rn(ax.gamma, __dsub_rn(yx, ax.fcenter));
    const double sy = __dmul_rn(ay.gamma, __dsub_rn(yy, ay.fcenter));
    const double phase = __dadd_rn(__dmul_rn(ax.center, yx), __dmul_rn(ay.center, yy));
    double sn, cs;
    sincos(phase, &sn, &cs);
    const double2 post = make_double2(__dmul_rn(cs, cxy), __dmul_rn(sn, cxy));
    const int jx0 = (int)ceil(sx - g.half), jy0 = (int)ceil(sy - g.half);
    double wx[W], wy[W];
    kb_taps<W>((jx0 - sx) + g.half, P, wx);
    kb_taps<W>((jy0 - sy) + g.half, P, wy);
    const int mx0 = wrap_base(jx0, g.n1), my0 = wrap_base(jy0, g.n2);
    int myj[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
        int my = my0 + j;
        if (my >= g.n2) my -= g.n2;
        myj[j] = my;
        wy[j] *= dyt[my];
    }
    double ar = 0.0, ai = 0.0;
#pragma unroll
    for (int a = 0; a < W; ++a) {
        int mx = mx0 + a;
        if (mx >= g.n1) mx -= g.n1;
        const double2* rowp = grid + (size_t)mx * g.n2;
        double rr = 0.0, ri = 0.0;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const double2 v = rowp[myj[j]];
            rr = fma(v.x, wy[j], rr);
            ri = fma(v.y, wy[j], ri);
        }
        const double wxa = wx[a] * dxt[mx];
        ar = fma(rr, wxa, ar);
        ai = fma(ri, wxa, ai);
    }
    const double2 far = cmul(make_double2(ar, ai), post);
    const double rad = hypot(yx, yy);
    if (!(rad > 0.0)) atomicExch(bad, 1);
    vals[i] = laplace ? make_double2(log(rad) - far.x, -far.y) : make_double2(-far.x, -far.y);
}

template <int W>
struct CloseRun {
    static void run(const WindowPoly& P, GridGeom g, Axis ax, Axis ay, double cxy, const double* dx,
                    const double* dy, const double2* grid, const double2* tgt, const double2* src,
                    const uint32_t* row, const uint32_t* cols, uint64_t nnz, int single,
                    double2 diag, int laplace, double2* vals, int* bad, cudaStream_t st) {
        k_close_values<W><<<nblk(nnz, 256), 256, 0, st>>>(P, g, ax, ay, cxy, dx, dy, grid, tgt, src,
                                                          row, cols, nnz, single, diag, laplace,
                                                          vals, bad);
    }
};

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

template <typename T>
void exclusive_scan(const T* in, T* out, uint64_t n, cudaStream_t st) {
    size_t tmp = 0;
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, st), "scan size");
    DevBuf<unsigned char> t(tmp + 1);
    ck(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, (int)n, st), "scan");
    ck(cudaStreamSynchronize(st), "scan sync");
}

} // namespace

void build_close_matrix_gpu(const CloseMatrixInput& in, CloseMatrixOutput& out) {
    ck(cudaSetDevice(in.device), "cudaSetDevice");
    cudaStream_t st;
    ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    const uint64_t ns = in.n_src, nt = in.n_tgt;
    DevBuf<double2> src, tgt;
    src.upload(reinterpret_cast<const double2*>(in.src_xy), ns, st);
    tgt.upload(reinterpret_cast<const double2*>(in.tgt_xy), nt, st);

    // ---- cell grid over the sources, cell = radius (point_cloud.cpp:80-88)
    double ox = 1e300, oy = 1e300, hx = -1e300, hy = -1e300;
    for (uint64_t i = 0; i < ns; ++i) {
        ox = std::min(ox, in.src_xy[2 * i]);
        hx = std::max(hx, in.src_xy[2 * i]);
        oy = std::min(oy, in.src_xy[2 * i + 1]);
        hy = std::max(hy, in.src_xy[2 * i + 1]);
    }
    CellGrid g;
    g.cell = in.radius;
    g.ox = ox;
    g.oy = oy;
    // cap the cell count (huge radius-less extents) by growing the cell
    double cell = in.radius;
    while ((hx - ox) / cell * (hy - oy) / cell > 4e8) cell *= 2.0;
    g.cell = cell;
    g.ncx = (int)std::floor((hx - ox) / cell) + 1;
    g.ncy = (int)std::floor((hy - oy) / cell) + 1;
    const uint64_t ncells = (uint64_t)g.ncx * g.ncy;

    DevBuf<uint32_t> keys(ns), idx(ns), cnt(ncells + 1), cstart(ncells + 1);
    ck(cudaMemsetAsync(cnt.p, 0, (ncells + 1) * 4, st), "memset");
    k_cell_keys<<<nblk(ns, 256), 256, 0, st>>>(src.p, ns, g, keys.p, idx.p, cnt.p);
    count_launch();
    exclusive_scan(cnt.p, cstart.p, ncells + 1, st);
    {
        DevBuf<uint32_t> k2(ns), i2(ns);
        size_t tmp = 0;
        ck(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys.p, k2.p, idx.p, i2.p, (int)ns, 0, 32, st), "sort");
        DevBuf<unsigned char> t(tmp + 1);
        ck(cub::DeviceRadixSort::SortPairs(t.p, tmp, keys.p, k2.p, idx.p, i2.p, (int)ns, 0, 32, st), "sort");
        count_launch(4);
        ck(cudaStreamSynchronize(st), "sort");
        idx = std::move(i2);
    }
    DevBuf<double2> src_sorted(ns);
    launch_gather(src.p, idx.p, src_sorted.p, ns, st);

    // ---- count, scan, fill (neighbor_pairs, point_cloud.cpp:90-110)
    const double r2 = in.radius * in.radius;
    DevBuf<uint64_t> counts(nt + 1), ro(nt + 1);
    ck(cudaMemsetAsync(counts.p, 0, (nt + 1) * 8, st), "memset");
    k_pairs<false><<<nblk(nt, 128), 128, 0, st>>>(tgt.p, nt, src_sorted.p, idx.p, cstart.p, g, r2,
                                                  in.single, counts.p, nullptr, nullptr);
    count_launch();
    exclusive_scan(counts.p, ro.p, nt + 1, st);
    uint64_t nnz = 0;
    ck(cudaMemcpyAsync(&nnz, ro.p + nt, 8, cudaMemcpyDeviceToHost, st), "nnz");
    ck(cudaStreamSynchronize(st), "nnz sync");
    DevBuf<uint32_t> cols(std::max<uint64_t>(nnz, 1)), row(std::max<uint64_t>(nnz, 1));
    if (nnz) {
        k_pairs<true><<<nblk(nt, 128), 128, 0, st>>>(tgt.p, nt, src_sorted.p, idx.p, cstart.p, g, r2,
                                                     in.single, nullptr, ro.p, cols.p);
        k_row_index<<<nblk(nt, 256), 256, 0, st>>>(ro.p, nt, row.p);
        count_launch(2);
    }
    out.row_offsets.resize(nt + 1);
    out.cols.resize(nnz);
    ck(cudaMemcpyAsync(out.row_offsets.data(), ro.p, (nt + 1) * 8, cudaMemcpyDeviceToHost, st), "D2H");
    if (nnz) ck(cudaMemcpyAsync(out.cols.data(), cols.p, nnz * 4, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "pairs");
    out.values.assign(2 * nnz, 0.0);
    out.laplace_done = in.laplace;
    if (nnz == 0) {
        cudaStreamDestroy(st);
        return;
    }

    // ---- far field at every pair difference (conv_operator.cpp:186-206)
    DevBuf<unsigned long long> ext(4);
    const unsigned long long init[4] = {~0ull, 0ull, ~0ull, 0ull};
    // st is non-blocking: every host transfer goes through st (a legacy-stream
    // cudaMemcpy would not wait for the kernels queued on st)
    ck(cudaMemcpyAsync(ext.p, init, sizeof(init), cudaMemcpyHostToDevice, st), "ext init");
    k_diff_extrema<<<std::min<uint64_t>(nblk(nnz, 256), 148 * 8), 256, 0, st>>>(tgt.p, src.p, row.p, cols.p,
                                                                             nnz, in.single, ext.p);
    count_launch();
    unsigned long long he[4];
    ck(cudaMemcpyAsync(he, ext.p, sizeof(he), cudaMemcpyDeviceToHost, st), "ext D2H");
    ck(cudaStreamSynchronize(st), "ext sync");
    auto unord = [](unsigned long long u) {
        const unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
        double d;
        std::memcpy(&d, &b, 8);
        return d;
    };
    double corners[4] = {unord(he[0]), unord(he[2]), unord(he[1]), unord(he[3])};
    uint64_t n_off = nnz - (in.single ? nt : 0);
    if (n_off == 0) { // only diagonals
        corners[0] = corners[1] = corners[2] = corners[3] = 0.0;
    }
    DevBuf<double2> vals(nnz);
    DevBuf<int> bad(1);
    ck(cudaMemsetAsync(bad.p, 0, 4, st), "memset");
    const double2 diag = make_double2(-in.wsum_re, -in.wsum_im);
    NufftOpts o;
    o.tol = in.nufft_tol;
    o.mode = (double)in.n_xi * (double)n_off > (double)in.direct_threshold ? 2 : 1;
    o.direct_threshold = in.direct_threshold;
    o.max_grid_bytes = in.max_grid_bytes;
    // Plan(xi, {box corners}, +): same geometry as a plan over all differences.
    Plan far(in.xi_xy, in.n_xi, corners, 2, +1, o, in.device, true, false, st);
    if (!(std::isfinite(corners[0]) && std::isfinite(corners[1]) && std::isfinite(corners[2]) &&
          std::isfinite(corners[3])))
        throw Error(3, "assemble: pair-difference extent is not finite");
    if (g_verbose)
        std::fprintf(stderr, "[sbd] far plan: fast %d n %d x %d w %d gamma %.6g %.6g center %.6g %.6g fcenter %.6g %.6g "
                             "corners %.6g %.6g %.6g %.6g nnz %llu n_xi %llu\n",
                     (int)far.fast, far.ax.n, far.ay.n, far.w, far.ax.gamma, far.ay.gamma, far.ax.center, far.ay.center,
                     far.ax.fcenter, far.ay.fcenter, corners[0], corners[1], corners[2], corners[3],
                     (unsigned long long)nnz, (unsigned long long)in.n_xi);
    if (far.fast) {
        DevBuf<double2> grid(far.cells());
        DevBuf<double2> w;
        w.upload(reinterpret_cast<const double2*>(in.w), in.n_xi, st);
        const GridGeom gg{far.ax.n, far.ay.n, 0.5 * far.w};
        ck(cudaMemsetAsync(grid.p, 0, far.cells() * 16, st), "grid zero");
        launch_spread(far.w, far.win, gg, in.n_xi, far.perm_t.n ? far.perm_t.p : nullptr, w.p, far.t.p,
                      far.pre.p, nullptr, nullptr, nullptr, grid.p, 0, st);
        far.full_transform(grid.p, st);
        const double cxy = (2.0 * M_PI / (far.ax.n * far.ax.gamma)) * (2.0 * M_PI / (far.ay.n * far.ay.gamma));
        dispatch_w<CloseRun>(far.w, far.win, gg, far.ax, far.ay, cxy, far.dx.p, far.dy.p, grid.p, tgt.p,
                             src.p, row.p, cols.p, nnz, (int)in.single, diag, (int)in.laplace, vals.p,
                             bad.p, st);
        count_launch(3);
        ck(cudaStreamSynchronize(st), "close values");
    } else {
        // tiny problem: exact sum over the quadrature for every pair, on the host
        ck(cudaStreamSynchronize(st), "sync");
        std::vector<uint32_t> hrow(nnz);
        ck(cudaMemcpy(hrow.data(), row.p, nnz * 4, cudaMemcpyDeviceToHost), "row D2H");
        std::vector<double> hv(2 * nnz);
        for (uint64_t i = 0; i < nnz; ++i) {
            const uint32_t r = hrow[i], c = out.cols[i];
            if (in.single && r == c) {
                hv[2 * i] = -in.wsum_re;
                hv[2 * i + 1] = -in.wsum_im;
                continue;
            }
            const double yx = in.tgt_xy[2 * r] - in.src_xy[2 * c], yy = in.tgt_xy[2 * r + 1] - in.src_xy[2 * c + 1];
            double fr = 0.0, fi = 0.0;
            for (uint64_t v = 0; v < in.n_xi; ++v) {
                const double ph = yx * in.xi_xy[2 * v] + yy * in.xi_xy[2 * v + 1];
                const double cs = std::cos(ph), sn = std::sin(ph);
                fr += in.w[2 * v] * cs - in.w[2 * v + 1] * sn;
                fi += in.w[2 * v] * sn + in.w[2 * v + 1] * cs;
            }
            const double rad = std::hypot(yx, yy);
            if (!(rad > 0.0)) throw Error(3, "assemble: coincident source/target points");
            hv[2 * i] = (in.laplace ? std::log(rad) : 0.0) - fr;
            hv[2 * i + 1] = -fi;
        }
        out.values = std::move(hv);
        cudaStreamDestroy(st);
        return;
    }
    int hbad = 0;
    ck(cudaMemcpy(&hbad, bad.p, 4, cudaMemcpyDeviceToHost), "bad");
    if (hbad) throw Error(3, "assemble: coincident source/target points");
    ck(cudaMemcpy(out.values.data(), vals.p, nnz * 16, cudaMemcpyDeviceToHost), "vals D2H");
    cudaStreamDestroy(st);
}

} // namespace sbdgpu
