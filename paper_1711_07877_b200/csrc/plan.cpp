// plan.cpp -- host side of the device type-III NUFFT plan (reference
// NufftPlan, /root/reference/proj/src/nufft.cpp:97-216, 369-398).
//
// The plan geometry (w, beta, centers, gamma, n, alpha1, alpha2) is restated
// exactly on the host from the coordinate extrema (nufft.cpp:127-160), so the
// device path uses the same grid, stencil starts and window as the reference;
// per-point arrays are computed on the device (k_plan_points/k_plan_outputs)
// with the same operation order. Points and outputs are stored sorted by grid
// tile for locality.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "sbd_internal.h"

namespace sbdgpu {

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kSigma = 2.0; // nufft.cpp:19

void span(const double* v, uint64_t n, int comp, double s, double& lo, double& hi) {
    lo = 1e300;
    hi = -1e300;
    for (uint64_t i = 0; i < n; ++i) {
        const double x = s * v[2 * i + comp];
        lo = std::min(lo, x);
        hi = std::max(hi, x);
    }
    if (n == 0) lo = hi = 0.0;
}

std::vector<double> make_deconv(const Axis& a, double beta) {
    std::vector<double> d(a.n, 0.0);
    const int band = a.n / (int)(2.0 * kSigma);
    for (int m = 0; m < a.n; ++m) {
        const int j = m <= a.n / 2 ? m : m - a.n;
        if (std::abs(j) > band) continue;
        const double psi1 = a.alpha1 * kb_window_hat_host(beta, a.alpha1 * j);
        d[m] = ((j & 1) ? -1.0 : 1.0) / psi1;
    }
    return d;
}

} // namespace

Axis plan_axis(const double* pts_xy, uint64_t np, const double* frq_xy, uint64_t nf, int comp,
               double sg, int w) {
    Axis a;
    double plo, phi, flo, fhi;
    span(pts_xy, np, comp, 1.0, plo, phi);
    span(frq_xy, nf, comp, sg, flo, fhi);
    a.center = 0.5 * (plo + phi);
    a.fcenter = 0.5 * (flo + fhi);
    const double X = std::max(0.5 * (phi - plo), 1e-8 * (1.0 + std::fabs(a.center)));
    const double S = std::max(0.5 * (fhi - flo), 1e-8 * (1.0 + std::fabs(a.fcenter)));
    a.gamma = kSigma * X / kPi;
    a.n = next_fast_even((int)std::ceil(2.0 * kSigma * (a.gamma * S + 0.5 * w + 1.0)));
    a.alpha1 = kPi * w / a.n;
    a.alpha2 = 0.5 * w / a.gamma;
    return a;
}

int stencil_start_point(const Axis& a, double p, int w) {
    // k_plan_points' grid coordinate, then ceil(t - w/2) (same IEEE operations)
    const double u = (p - a.center) / a.gamma;
    const double tt = ((u + kPi) * (double)a.n) / (2.0 * kPi);
    return (int)std::ceil(tt - 0.5 * w);
}

int stencil_start_output(const Axis& a, double f, double sg, int w) {
    // k_plan_outputs' mode coordinate, then ceil(s - w/2)
    const double s = a.gamma * (sg * f - a.fcenter);
    return (int)std::ceil(s - 0.5 * w);
}

static void upload_twiddles(DevBuf<double2>& tw, int n, cudaStream_t st);
static int pick_radix(int n, int mode);

Plan::Plan(const double* pts_xy, uint64_t np_, const double* frq_xy, uint64_t nf_, int sign_,
           const NufftOpts& o, int dev, bool sort_points, bool sort_outputs, cudaStream_t st,
           const uint8_t* pt_tag, const uint8_t* out_tag, const double2* dev_pts, const double2* dev_frq)
    : sign(sign_ > 0 ? 1 : -1), device(dev), np(np_), nf(nf_), opts(o) {
    const uint64_t work = np * nf;
    const bool direct = o.mode == 1 || (o.mode == 0 && work <= o.direct_threshold);
    pts.upload(reinterpret_cast<const double2*>(pts_xy), np, st);
    frq.upload(reinterpret_cast<const double2*>(frq_xy), nf, st);
    if (dev_pts && np) ck(cudaMemcpyAsync(pts.p, dev_pts, np * 16, cudaMemcpyDeviceToDevice, st), "device points");
    if (dev_frq && nf) ck(cudaMemcpyAsync(frq.p, dev_frq, nf * 16, cudaMemcpyDeviceToDevice, st), "device freqs");
    if (direct) {
        fast = false;
        ck(cudaStreamSynchronize(st), "plan upload");
        return;
    }

    // ---- geometry, nufft.cpp:127-160
    w = width_for_tol(o.tol);
    beta = 2.3562 * w;
    const double sg = (double)sign;
    ax = plan_axis(pts_xy, np, frq_xy, nf, 0, sg, w);
    ay = plan_axis(pts_xy, np, frq_xy, nf, 1, sg, w);
    const uint64_t ncell = (uint64_t)ax.n * (uint64_t)ay.n;
    if (ncell * 16u > o.max_grid_bytes)
        throw Error(3, "nufft: oversampled grid exceeds the memory limit");
    win = fit_window(w, beta);
    fast = true;

    // ---- per point / per output arrays (nufft.cpp:163-192), caller order
    t.alloc(np);
    pre.alloc(np);
    this->s.alloc(nf);
    post.alloc(nf);
    launch_plan_points(pts.p, np, ax, ay, beta, t.p, pre.p, st);
    launch_plan_outputs(frq.p, nf, ax, ay, sg, this->s.p, post.p, st);

    // ---- deconvolution tables (nufft.cpp:194-205), host exact
    const std::vector<double> hx = make_deconv(ax, beta), hy = make_deconv(ay, beta);
    dx.upload(hx.data(), hx.size(), st);
    dy.upload(hy.data(), hy.size(), st);

    // ---- populated region of the spread (stencil starts never wrap: points
    // sit in [n/4, 3n/4] of the grid, nufft.cpp:166-169), for the pruned path
    const GridGeom g{ax.n, ay.n, 0.5 * w};
    {
        DevBuf<int> ext(4);
        launch_stencil_extent(t.p, np, g.half, ext.p, st);
        int he[4];
        ck(cudaMemcpyAsync(he, ext.p, sizeof(he), cudaMemcpyDeviceToHost, st), "extent D2H");
        ck(cudaStreamSynchronize(st), "extent");
        pruned = sort_points && np > 0 && he[0] >= 0 && he[1] + w <= ax.n && he[2] >= 0 &&
                 he[3] + w <= ay.n;
        if (pruned) {
            tg.tr = 16;
            tg.rlo = he[0];
            tg.clo = he[2];
            tg.nbx = (he[1] + w - he[0] + tg.tr - 1) / tg.tr;
            tg.nby = (he[3] + w - he[2] + kTileC - 1) / kTileC;
            rlo = tg.rlo;
            clo = tg.clo;
            rhi = std::min(ax.n, tg.rlo + tg.nbx * tg.tr);
            chi = std::min(ay.n, tg.clo + tg.nby * kTileC);
        }
    }

    // ---- sort both sides by grid tile of the stencil start
    // tags: tag-0 entries sort first (key bit 31); needs the tile index below
    // 2^26 (points) or stencil cells below 2^15 after the shift (outputs)
    const int oshift = std::max(ax.n, ay.n) / 2 + w;
    auto count0 = [](const uint8_t* tag, uint64_t n) {
        uint64_t c = 0;
        for (uint64_t i = 0; i < n; ++i) c += tag[i] ? 0 : 1;
        return c;
    };
    if (pt_tag && pruned && (uint64_t)tg.nbx * (uint64_t)tg.nby < (1ull << 26)) {
        tagged_pts = true;
        n0_pts = count0(pt_tag, np);
    }
    if (out_tag && sort_outputs && oshift + std::max(ax.n, ay.n) / 2 + w < 32768) {
        tagged_out = true;
        n0_out = count0(out_tag, nf);
    }
    auto sort_side = [&](DevBuf<double2>& pos, DevBuf<double2>& ph, DevBuf<uint32_t>& perm,
                         uint64_t n, bool tiles) {
        if (n < 1) return;
        DevBuf<uint32_t> keys(n);
        perm.alloc(n);
        const uint8_t* htag = tiles ? (tagged_pts ? pt_tag : nullptr) : (tagged_out ? out_tag : nullptr);
        DevBuf<uint8_t> dtag;
        if (htag) dtag.upload(htag, n, st);
        if (tiles)
            launch_tile_keys(pos.p, n, g.half, tg, keys.p, st, dtag.p);
        else  // outputs: Z-order of the stencil cell (mode units, |j| <= n/2)
            launch_morton_keys(pos.p, n, g.half, oshift, keys.p, st, dtag.p);
        launch_iota(perm.p, n, st);
        sort_by_key(keys.p, perm.p, n, st);
        DevBuf<double2> a(n), b(n);
        launch_gather(pos.p, perm.p, a.p, n, st);
        launch_gather(ph.p, perm.p, b.p, n, st);
        pos = std::move(a);
        ph = std::move(b);
        if (tiles) {
            const uint32_t nbins = (uint32_t)tg.nbx * (uint32_t)tg.nby;
            bin_start.alloc(nbins + 1);
            if (tagged_pts) {
                // tag-0 points [0, n0) and tag-1 points [n0, n) binned separately
                bin_start2.alloc(nbins + 1);
                launch_bin_bounds(keys.p, n0_pts, nbins, bin_start.p, st);
                launch_bin_bounds(keys.p + n0_pts, n - n0_pts, nbins, bin_start2.p, st, (uint32_t)n0_pts,
                                  0x7fffffffu);
            } else {
                launch_bin_bounds(keys.p, n, nbins, bin_start.p, st);
            }
            if (tg.tr == 16) {
                const uint64_t n0 = tagged_pts ? n0_pts : n;
                build_region_lists(pos.p, n0, w, tg, 0u, 0u, rl1_s, rl1_e, st);
                // tag-1 points: entries index the same arrays (from n0)
                if (tagged_pts) build_region_lists(pos.p + n0, n - n0, w, tg, (uint32_t)n0, 0u, rl2_s, rl2_e, st);
            }
        } else {
            // 32 x 32 blocks of the Z order (k_interp_tile)
            out_shift = oshift;
            build_tile_starts(keys.p, n, 10, out_tiles, n_out_tiles, st);
            // sparse outputs (the targets; < 0.25 per band cell) are interpolated
            // one per thread from a staged real tile: order each block for
            // conflict-free shared-memory reads (the dense xi side keeps its
            // Z order for the 8-node tensor-core groups)
            if ((double)n < 0.25 * ((double)ax.n * (double)ay.n / 4.0) && !tagged_out) {
                DevBuf<uint32_t> map;
                bank_interleave_outputs(out_tiles.p, n_out_tiles, pos.p, n, w, oshift, map, st);
                DevBuf<double2> a(n), b(n);
                DevBuf<uint32_t> c(n);
                launch_gather(pos.p, map.p, a.p, n, st);
                launch_gather(ph.p, map.p, b.p, n, st);
                launch_gather(perm.p, map.p, c.p, n, st);
                pos = std::move(a);
                ph = std::move(b);
                perm = std::move(c);
            }
        }
        ck(cudaStreamSynchronize(st), "sort side");
    };
    if (sort_points) sort_side(t, pre, perm_t, np, pruned);
    if (sort_outputs) sort_side(this->s, post, perm_s, nf, false);

    // ---- band-limited FFT plans (pruned path): the interpolation only reads
    // modes |j| <= n/4 (nufft.cpp:194-205), so columns outside the band are
    // never transformed and rows outside the populated region are zero.
    band2 = ay.n / 4;
    bc = 2 * band2 + 1;
    {
        std::vector<double> hb(bc);
        for (int c = 0; c < bc; ++c) hb[c] = hy[c <= band2 ? c : ay.n + c - bc];
        dy_band.upload(hb.data(), bc, st);
    }
    if (pruned) {
        tg.pitch = 0;
        tg.rhi = rhi;
        tg.chi = chi;
    }
    if (pruned) {
        // rows: cuFFT over the populated rows; columns: the band columns
        // transposed (k_band_transpose), then contiguous length-n1 transforms
        int n2[1] = {ay.n}, n1[1] = {ax.n};
        ckfft(cufftPlanMany(&fft_row, 1, n2, n2, 1, ay.n, n2, 1, ay.n, CUFFT_Z2Z, rhi - rlo),
              "cufftPlanMany rows");
        ckfft(cufftPlanMany(&fft_colT, 1, n1, n1, 1, ax.n, n1, 1, ax.n, CUFFT_Z2Z, bc),
              "cufftPlanMany cols T");
        // radix first passes in our own kernels where the lengths split
        crad_row = pick_radix(ay.n, opts.radix);
        crad_col = pick_radix(ax.n, opts.radix);
        if (crad_row > 1) {
            int m2[1] = {ay.n / crad_row};
            ckfft(cufftPlanMany(&fft_row_m, 1, m2, m2, 1, m2[0], m2, 1, m2[0], CUFFT_Z2Z, (rhi - rlo) * crad_row),
                  "cufftPlanMany rows (M)");
            upload_twiddles(ctw_row, ay.n, st);
        }
        if (crad_col > 1) {
            int m1[1] = {ax.n / crad_col};
            ckfft(cufftPlanMany(&fft_colT_m, 1, m1, m1, 1, m1[0], m1, 1, m1[0], CUFFT_Z2Z, bc * crad_col),
                  "cufftPlanMany cols T (M)");
            upload_twiddles(ctw_col, ax.n, st);
        }
    }
    ck(cudaStreamSynchronize(st), "plan build");
}

double Plan::out_cxy() const {
    const double kPi = 3.14159265358979323846;
    return (2.0 * kPi / (ax.n * ax.gamma)) * (2.0 * kPi / (ay.n * ay.gamma));
}

Plan::~Plan() {
    if (fft) cufftDestroy(fft);
    if (fft_row) cufftDestroy(fft_row);
    if (fft_colT) cufftDestroy(fft_colT);
    if (fft_row_m) cufftDestroy(fft_row_m);
    if (fft_colT_m) cufftDestroy(fft_colT_m);
    if (hp1) cufftDestroy(hp1);
    if (hp2) cufftDestroy(hp2);
}

// Radix r of a first pass folded into the producer of a length-n transform
// (n = r M, r in {3, 5, 9}, M <= 4096 a multiple of 8: cuFFT then runs one
// length-M pass instead of two length-n passes). 1: none. Used for n > 4096;
// opts.radix = 0 turns it off, 1 uses it for any such n (tests).
// tw[m] = e^{+2 pi i m / n}, m < n (long double arguments)
static void upload_twiddles(DevBuf<double2>& tw, int n, cudaStream_t st) {
    std::vector<double2> h(n);
    for (int m = 0; m < n; ++m) {
        const long double a = 2.0L * 3.14159265358979323846264338327950288L * m / n;
        h[m] = make_double2((double)cosl(a), (double)sinl(a));
    }
    tw.upload(h.data(), n, st);
    ck(cudaStreamSynchronize(st), "twiddles");
}

static int pick_radix(int n, int mode) {
    if (mode == 0) return 1;
    const bool force = mode == 1;
    if (!force && n <= 4096) return 1;
    for (int r : {3, 5, 9})
        if (n % r == 0 && n / r <= 4096 && (n / r) % 8 == 0) return r;
    return 1;
}

bool Plan::enable_hfft(int role, cudaStream_t st) {
    if (!fast || !pruned) return false;
    const int n1 = ax.n, n2 = ay.n, R = rhi - rlo;
    if (role == 1) {
        // the spread grid is real only when the prephase is (fcenter exactly 0)
        if (!tagged_out || !n_out_tiles || ax.fcenter != 0.0 || ay.fcenter != 0.0) return false;
        // real rows packed in pairs into R/2 complex rows (R is a multiple of 16)
        hcols = band2 + 1;
        hA.alloc((size_t)(R / 2) * n2);
        ck(cudaMemsetAsync(hA.p, 0, hA.bytes(), st), "hfft zero");
        hD.alloc((size_t)(R / 2) * n2);
        hB.alloc((size_t)hcols * n1);
        ck(cudaMemsetAsync(hB.p, 0, hB.bytes(), st), "hfft zero");
        hC.alloc((size_t)hcols * n1);
        int nr[1] = {n2}, nc[1] = {n1};
        hrad = pick_radix(n1, opts.radix);
        // the row transform's own first pass (k_dif_rows) when both sides split by 9
        hrad0 = hrad == 9 && pick_radix(n2, opts.radix) == 9 ? 9 : 1;
        if (hrad0 > 1) {
            int nm0[1] = {n2 / hrad0};
            ckfft(cufftPlanMany(&hp1, 1, nm0, nm0, 1, nm0[0], nm0, 1, nm0[0], CUFFT_Z2Z, (R / 2) * hrad0),
                  "hfft Z2Z rows (M)");
            upload_twiddles(htw0, n2, st);
        } else {
            ckfft(cufftPlanMany(&hp1, 1, nr, nr, 1, n2, nr, 1, n2, CUFFT_Z2Z, R / 2), "hfft Z2Z rows");
        }
        if (hrad > 1) {
            // the untangle does the radix-hrad first pass; cuFFT one length-M pass
            const int M = n1 / hrad;
            int nm[1] = {M};
            ckfft(cufftPlanMany(&hp2, 1, nm, nm, 1, M, nm, 1, M, CUFFT_Z2Z, hcols * hrad), "hfft Z2Z cols (M)");
            upload_twiddles(htw, n1, st);
        } else {
            ckfft(cufftPlanMany(&hp2, 1, nc, nc, 1, n1, nc, 1, n1, CUFFT_Z2Z, hcols), "hfft Z2Z cols");
        }
    } else if (role == 2) {
        if (!tagged_pts || !n0_pts) return false;
        const GridGeom g{n1, n2, 0.5 * w};
        hv_t.alloc(n0_pts);
        launch_mirror_points(t.p, n0_pts, n1, n2, w, hv_t.p, st);
        // the mirror images must fall inside this plan's spread tiles
        DevBuf<int> ext(4);
        const int init[4] = {INT_MAX, INT_MIN, INT_MAX, INT_MIN};
        ck(cudaMemcpyAsync(ext.p, init, sizeof(init), cudaMemcpyHostToDevice, st), "extent init");
        launch_stencil_extent(hv_t.p, n0_pts, g.half, ext.p, st);
        int he[4];
        ck(cudaMemcpyAsync(he, ext.p, sizeof(he), cudaMemcpyDeviceToHost, st), "extent D2H");
        ck(cudaStreamSynchronize(st), "extent");
        if (he[0] < rlo || he[1] + w > rhi || he[2] < clo || he[3] + w > chi || clo > n2 / 2) {
            hv_t = DevBuf<double2>();
            return false;
        }
        // sort the mirror images by spread tile, keep both directions of the map
        DevBuf<uint32_t> keys(n0_pts), src(n0_pts);
        launch_tile_keys(hv_t.p, n0_pts, g.half, tg, keys.p, st);
        launch_iota(src.p, n0_pts, st);
        sort_by_key(keys.p, src.p, n0_pts, st);
        DevBuf<double2> sorted(n0_pts);
        launch_gather(hv_t.p, src.p, sorted.p, n0_pts, st);
        hv_t = std::move(sorted);
        const uint32_t nbins = (uint32_t)tg.nbx * (uint32_t)tg.nby;
        hv_bins.alloc(nbins + 1);
        launch_bin_bounds(keys.p, n0_pts, nbins, hv_bins.p, st);
        std::vector<uint32_t> hs(n0_pts), inv(n0_pts);
        ck(cudaMemcpyAsync(hs.data(), src.p, n0_pts * 4, cudaMemcpyDeviceToHost, st), "mirror map");
        ck(cudaStreamSynchronize(st), "mirror map");
        for (uint64_t i = 0; i < n0_pts; ++i) inv[hs[i]] = (uint32_t)i;
        hv_of.upload(inv.data(), n0_pts, st);
        hv_src = std::move(src);
        if (rl1_s.n) build_region_lists(hv_t.p, n0_pts, w, tg, 0u, 0x80000000u, rlh_s, rlh_e, st);
        // columns m2 in [clo, n2/2] of the Hermitian grid, as full-length columns
        hnm = n2 / 2 - clo + 1;
        hnby = std::min(tg.nby, (n2 / 2 + 1 - clo + kTileC - 1) / kTileC);
        hb1 = n1 / 4;
        hB1 = 2 * hb1 + 1;
        hA.alloc((size_t)hnm * n1);
        ck(cudaMemsetAsync(hA.p, 0, hA.bytes(), st), "hfft zero");
        hB.alloc((size_t)hnm * n1);
        const int K = (hB1 + 1) / 2;  // band rows packed in pairs
        hC.alloc((size_t)K * n2);
        ck(cudaMemsetAsync(hC.p, 0, hC.bytes(), st), "hfft zero");
        hD.alloc((size_t)K * n2);
        std::vector<double> hx(n1), hb(hB1);
        ck(cudaMemcpyAsync(hx.data(), dx.p, n1 * sizeof(double), cudaMemcpyDeviceToHost, st), "deconv");
        ck(cudaStreamSynchronize(st), "deconv");
        for (int r = 0; r < hB1; ++r) hb[r] = hx[r <= hb1 ? r : n1 + r - hB1];
        hdx_band.upload(hb.data(), hB1, st);
        int nc[1] = {n1}, nr[1] = {n2};
        hrad = pick_radix(n2, opts.radix);
        // the column transform's own first pass (k_dif_rows) when both sides split by 9
        hrad0 = hrad == 9 && pick_radix(n1, opts.radix) == 9 ? 9 : 1;
        if (hrad0 > 1) {
            int nm0[1] = {n1 / hrad0};
            ckfft(cufftPlanMany(&hp1, 1, nm0, nm0, 1, nm0[0], nm0, 1, nm0[0], CUFFT_Z2Z, hnm * hrad0),
                  "hfft Z2Z cols (M)");
            upload_twiddles(htw0, n1, st);
        } else {
            ckfft(cufftPlanMany(&hp1, 1, nc, nc, 1, n1, nc, 1, n1, CUFFT_Z2Z, hnm), "hfft Z2Z cols");
        }
        if (hrad > 1) {
            // the packing does the radix-hrad first pass; cuFFT one length-M pass
            const int M = n2 / hrad;
            int nm[1] = {M};
            ckfft(cufftPlanMany(&hp2, 1, nm, nm, 1, M, nm, 1, M, CUFFT_Z2Z, K * hrad), "hfft Z2Z rows (M)");
            upload_twiddles(htw, n2, st);
        } else {
            ckfft(cufftPlanMany(&hp2, 1, nr, nr, 1, n2, nr, 1, n2, CUFFT_Z2Z, K), "hfft Z2Z rows");
        }

    } else {
        return false;
    }
    ck(cudaStreamSynchronize(st), "hfft setup");
    hrole = role;
    return true;
}

void FftWork::ensure(int n1_, int n2_, int bc_, cudaStream_t st) {
    if (n1_ == n1 && n2_ == n2 && bc_ == bc) return;
    n1 = n1_;
    n2 = n2_;
    bc = bc_;
    const size_t cells = (size_t)n1 * n2;
    grid.alloc(std::max<size_t>(cells, 1));
    T.alloc(std::max<size_t>(cells, 1));
    band.alloc(std::max<size_t>((size_t)n1 * bc, 1));
    ck(cudaMemsetAsync(grid.p, 0, grid.bytes(), st), "grid zero");
    ck(cudaMemsetAsync(T.p, 0, T.bytes(), st), "T zero");
    gr0 = gr1 = gc0 = gc1 = tr0 = tr1 = 0;
    g_pitch = t_pitch = 0;
}

void Plan::ensure_work(FftWork& wk, cudaStream_t st) const {
    if (fast) wk.ensure(std::max(wk.n1, ax.n), std::max(wk.n2, ay.n), std::max(wk.bc, bc), st);
    if (fft_colT) {
        const size_t need = (size_t)bc * ax.n;
        if (wk.T1.n < need) {
            wk.T1.alloc(need);
            ck(cudaMemsetAsync(wk.T1.p, 0, wk.T1.bytes(), st), "Tt zero");
            wk.tt_r0 = wk.tt_r1 = 0;
        }
        if (wk.bandT.n < need) wk.bandT.alloc(need);
    }
}

namespace {

// Zero the cells of rectangle D not covered by rectangle O (row-major, pitch n2).
void zero_rect_minus(double2* base, int n2, int r0, int r1, int c0, int c1, int R0, int R1, int C0,
                     int C1, cudaStream_t st) {
    if (r1 <= r0 || c1 <= c0) return;
    const size_t pitch = (size_t)n2 * sizeof(double2);
    auto zero = [&](int a0, int a1, int b0, int b1) {
        if (a1 <= a0 || b1 <= b0) return;
        ck(cudaMemset2DAsync(base + (size_t)a0 * n2 + b0, pitch, 0, (size_t)(b1 - b0) * sizeof(double2),
                             (size_t)(a1 - a0), st),
           "zero strip");
    };
    zero(r0, std::min(r1, R0), c0, c1);           // rows above O
    zero(std::max(r0, R1), r1, c0, c1);           // rows below O
    const int m0 = std::max(r0, R0), m1 = std::min(r1, R1);
    zero(m0, m1, c0, std::min(c1, C0));           // left of O
    zero(m0, m1, std::max(c0, C1), c1);           // right of O
}

void full_fft(const Plan& p, double2* grid, cudaStream_t st) { p.full_transform(grid, st); }

} // namespace

void Plan::full_transform(double2* grid, cudaStream_t st) const {
    if (!fft) ckfft(cufftPlan2d(&fft, ax.n, ay.n, CUFFT_Z2Z), "cufftPlan2d");
    ckfft(cufftSetStream(fft, st), "cufftSetStream");
    ckfft(cufftExecZ2Z(fft, reinterpret_cast<cufftDoubleComplex*>(grid),
                       reinterpret_cast<cufftDoubleComplex*>(grid), CUFFT_INVERSE),
          "cufftExecZ2Z");
    count_launch();
}

size_t Plan::device_bytes() const {
    return pts.bytes() + frq.bytes() + perm_t.bytes() + perm_s.bytes() + t.bytes() + pre.bytes() +
           s.bytes() + post.bytes() + dx.bytes() + dy.bytes() + tpw.b.bytes() + tpw.Z.bytes() + tpw.V.bytes() +
           tpw.Wt.bytes() + tpw.Tz.bytes() + tpw.G.bytes() + tpw.rl_s.bytes() + tpw.rl_e.bytes() +
           tpw.m_tiles.bytes() + tpw.m_src.bytes() + tpw.m_dst.bytes() + tpw.m_t.bytes() + tpw.m_phase.bytes();
}

// nufft.cpp:218-290
void Plan::apply(const double2* in, double2* out, FftWork& wk, cudaStream_t st, StageTimer* tm,
                 const double2* mult, const char* tag_spread, const char* tag_fft,
                 const char* tag_interp) const {
    if (!fast) {
        if (tm) tm->start(tag_interp);
        launch_ndft(pts.p, np, frq.p, nf, in, sign, out, st);
        if (mult) launch_mul(out, mult, nf, st);
        if (tm) tm->stop();
        return;
    }
    ensure_work(wk, st);
    const GridGeom g{ax.n, ay.n, 0.5 * w};
    const int n2 = ay.n;
    if (pruned) {
        apply_pruned(in, false, nullptr, out, mult, nullptr, wk, st, tm, tag_spread, tag_fft, tag_interp);
        return;
    }
    if (tm) tm->start(tag_spread);
    ck(cudaMemsetAsync(wk.grid.p, 0, cells() * sizeof(double2), st), "grid zero");
    launch_spread(w, win, g, np, perm_t.n ? perm_t.p : nullptr, in, t.p, pre.p, nullptr, nullptr,
                  nullptr, wk.grid.p, 0, st);
    if (tm) tm->stop();
    if (tm) tm->start(tag_fft);
    full_fft(*this, wk.grid.p, st);
    if (tm) tm->stop();
    if (tm) tm->start(tag_interp);
    launch_interp(w, win, g, nf, s.p, post.p, mult, dx.p, dy.p, wk.grid.p,
                  perm_s.n ? perm_s.p : nullptr, out, 0, 0, st, nullptr, false, nullptr, nullptr,
                  opts.interp_kernel);
    if (tm) tm->stop();
    wk.gr0 = 0;
    wk.gr1 = ax.n;
    wk.gc0 = 0;
    wk.gc1 = ay.n;
    wk.g_pitch = ay.n;
}

void Plan::apply_pruned(const double2* in, bool in_is_b, double2* raw_sorted, double2* out,
                        const double2* mult, const double2* addend, FftWork& wk, cudaStream_t st,
                        StageTimer* tm, const char* tag_spread, const char* tag_fft,
                        const char* tag_interp, uint64_t in_lo, uint64_t in_hi, uint64_t out_lo,
                        uint64_t out_hi, const HermArgs* herm, cudaEvent_t before_interp) const {
    out_hi = std::min<uint64_t>(out_hi, nf);
    out_lo = std::min(out_lo, out_hi);
    const uint64_t nout = out_hi - out_lo;
    // output-side arrays restricted to the sorted output range [out_lo, out_hi)
    const double2* s_p = s.p + out_lo;
    const double2* post_p = post.p + out_lo;
    const double2* mult_p = mult ? mult + out_lo : nullptr;
    const double2* add_p = addend ? addend + out_lo : nullptr;
    const uint32_t* perm_p = perm_s.n ? perm_s.p + out_lo : nullptr;
    double2* out_p = perm_s.n ? out : out + out_lo;
    if (!pruned) throw Error(3, "apply_pruned on a plan without the pruned path");
    // real-input half split: the output count is relative to this call's range
    HermArgs hz;
    const HermArgs* hp = nullptr;
    if (herm) {
        hz = *herm;
        hz.n = herm->n > out_lo ? std::min<uint64_t>(nout, herm->n - out_lo) : 0;
        hp = &hz;
    }
    int* clear = herm && herm->clear ? herm->flag : nullptr;
    const uint32_t* bs2 = tagged_pts ? bin_start2.p : nullptr;
    const int* hflag = herm ? herm->flag : nullptr;
    InterpTiles otiles;
    otiles.start = out_tiles.p;
    otiles.n = n_out_tiles;
    otiles.shift = out_shift;
    otiles.out_lo = out_lo;
    ensure_work(wk, st);
    const GridGeom g{ax.n, ay.n, 0.5 * w};
    const int n2 = ay.n;
    // procedural sides: ids restricted like the arrays they replace
    NodeGen go = gen_out;
    if (go.id) go.id += out_lo;
    const NodeGen* gop = go.id ? &go : nullptr;
    if (gen_pts.id && !in_is_b) throw Error(3, "procedural points take their coefficients as b");
    if (tm) tm->start(tag_spread);
    const double2* b = in;
    if (!in_is_b) {
        if (wk.bbuf.n < np) wk.bbuf.alloc(np);
        launch_gather_mul(in, perm_t.n ? perm_t.p : nullptr, pre.p, wk.bbuf.p, raw_sorted, np, st, in_lo,
                          in_hi, clear, herm ? herm->raw_re : nullptr);
        b = wk.bbuf.p;
    }
    if (herm && herm->hfft && hrole == 1) {
        // real rows packed in pairs -> Z2Z rows -> untangle + band transpose
        // (columns 0..n2/4) -> Z2Z columns
        SpreadOut so;
        so.mode = 3;
        so.rgrid = reinterpret_cast<double*>(hA.p);
        so.pitch = (size_t)n2;
        so.r0 = rlo;
        so.c0 = 0;
        so.rend = rhi;
        so.cend = chi;
        so.nby_run = tg.nby;
        so.lists = lists(false);
        launch_spread_tiles(w, win, g, tg, bin_start.p, b, t.p, nullptr, st, bs2, hflag, &so, nullptr,
                            opts.spread_kernel);
        if (tm) tm->stop();
        if (tm) tm->start(tag_fft);
        ckfft(cufftSetStream(hp1, st), "cufftSetStream");
        if (hrad0 > 1) {
            // rows: our radix pass, then contiguous length-M transforms in place
            launch_dif_rows(hA.p, (rhi - rlo) / 2, n2, hrad0, clo, chi, htw0.p, hD.p, st);
            ckfft(cufftExecZ2Z(hp1, reinterpret_cast<cufftDoubleComplex*>(hD.p),
                               reinterpret_cast<cufftDoubleComplex*>(hD.p), CUFFT_INVERSE),
                  "hfft Z2Z rows (M)");
        } else {
            ckfft(cufftExecZ2Z(hp1, reinterpret_cast<cufftDoubleComplex*>(hA.p),
                               reinterpret_cast<cufftDoubleComplex*>(hD.p), CUFFT_INVERSE),
                  "hfft Z2Z rows");
        }
        if (hrad > 1)
            launch_untangle_dif(hD.p, n2, (rhi - rlo) / 2, hcols, hB.p, ax.n, rlo, hrad, htw.p, st, dy_band.p,
                                hrad0);
        else
            launch_untangle_transpose(hD.p, n2, (rhi - rlo) / 2, hcols, hB.p, ax.n, rlo, st);
        ckfft(cufftSetStream(hp2, st), "cufftSetStream");
        ckfft(cufftExecZ2Z(hp2, reinterpret_cast<cufftDoubleComplex*>(hB.p),
                           reinterpret_cast<cufftDoubleComplex*>(hC.p), CUFFT_INVERSE),
              "hfft Z2Z");
        count_launch(4);
        if (tm) tm->stop();
        if (before_interp) ck(cudaStreamWaitEvent(st, before_interp, 0), "wait");
        if (tm) tm->start(tag_interp);
        GridGeom gt{ax.n, bc, 0.5 * w};
        if (hrad > 1) {
            gt.rad = hrad;
            gt.rad_m = ax.n / hrad;
            gt.rad_magic = (unsigned)((0x100000000ull + hrad - 1) / hrad);
        }
        // with the radix pass the column factors are already in the band
        launch_interp(w, win, gt, nout, s_p, post_p, mult_p, dx.p, hrad > 1 ? nullptr : dy_band.p, hC.p, perm_p,
                      out_p, 0, 0, st, add_p, /*transposed=*/true, &otiles, hp, opts.interp_kernel, gop);
        if (tm) tm->stop();
        return;
    }
    if (herm && herm->hfft && hrole == 2) {
        // tag-0 points + mirror images -> Hermitian grid columns m2 <= n2/2
        // (transposed) -> Z2Z columns -> band rows -> Z2D rows -> real band
        SpreadOut so;
        so.mode = 2;
        so.pitch = (size_t)ax.n;
        so.r0 = 0;
        so.c0 = clo;
        so.rend = rhi;
        so.cend = clo + hnm;
        so.nby_run = hnby;
        so.pos2 = hv_t.p;
        // the spread reads each mirror image's value as the conjugate of its
        // partner's (only images near the m2 = n2/2 line are ever read)
        so.src2 = hv_src.p;
        so.lists = lists(true);
        so.gen = gen_pts;
        launch_spread_tiles(w, win, g, tg, bin_start.p, b, t.p, hA.p, st, hv_bins.p, nullptr, &so, nullptr,
                            opts.spread_kernel);
        if (tm) tm->stop();
        if (tm) tm->start(tag_fft);
        ckfft(cufftSetStream(hp1, st), "cufftSetStream");
        if (hrad0 > 1) {
            // columns: our radix pass over the populated rows, then contiguous
            // length-M transforms in place
            launch_dif_rows(hA.p, hnm, ax.n, hrad0, rlo, rhi, htw0.p, hB.p, st);
            ckfft(cufftExecZ2Z(hp1, reinterpret_cast<cufftDoubleComplex*>(hB.p),
                               reinterpret_cast<cufftDoubleComplex*>(hB.p), CUFFT_INVERSE),
                  "hfft Z2Z cols (M)");
        } else {
            ckfft(cufftExecZ2Z(hp1, reinterpret_cast<cufftDoubleComplex*>(hA.p),
                               reinterpret_cast<cufftDoubleComplex*>(hB.p), CUFFT_INVERSE),
                  "hfft Z2Z cols");
        }
        // two Hermitian band rows per complex row: their transforms are the
        // real and imaginary parts of one e^{+} transform
        if (hrad > 1)
            launch_pack_dif(hB.p, ax.n, clo, n2, hb1, hB1, hC.p, hrad, htw.p, st, hrad0);
        else
            launch_pack_rows(hB.p, ax.n, clo, n2, hb1, hB1, hC.p, st);
        ckfft(cufftSetStream(hp2, st), "cufftSetStream");
        ckfft(cufftExecZ2Z(hp2, reinterpret_cast<cufftDoubleComplex*>(hC.p),
                           reinterpret_cast<cufftDoubleComplex*>(hD.p), CUFFT_INVERSE),
              "hfft Z2Z rows");
        count_launch(4);
        if (tm) tm->stop();
        if (before_interp) ck(cudaStreamWaitEvent(st, before_interp, 0), "wait");
        if (tm) tm->start(tag_interp);
        GridGeom gr{hB1, n2, 0.5 * w};
        if (hrad > 1) {
            gr.rad = hrad;
            gr.rad_m = n2 / hrad;
            gr.rad_magic = (unsigned)((0x100000000ull + hrad - 1) / hrad);
        }
        launch_interp_real(w, win, gr, nout, s_p, post_p, hdx_band.p, dy.p,
                           reinterpret_cast<const double*>(hD.p), perm_p, add_p, out_p, st, &otiles,
                           opts.interp_kernel);
        if (tm) tm->stop();
        return;
    }
    if (wk.g_pitch == n2)
        zero_rect_minus(wk.grid.p, n2, wk.gr0, wk.gr1, wk.gc0, wk.gc1, rlo, rhi, clo, chi, st);
    else if (wk.g_pitch)  // written by a plan of another grid size: clear all of it
        zero_rect_minus(wk.grid.p, wk.g_pitch, wk.gr0, wk.gr1, wk.gc0, wk.gc1, 0, 0, 0, 0, st);
    const SpreadLists sl = lists(false);
    if (gen_pts.id) {
        SpreadOut so;  // the default full-grid output with the procedural points
        so.mode = 0;
        so.rend = ax.n;
        so.cend = n2;
        so.pitch = (size_t)n2;
        so.nby_run = tg.nby;
        so.gen = gen_pts;
        launch_spread_tiles(w, win, g, tg, bin_start.p, b, t.p, wk.grid.p, st, bs2, hflag, &so, &sl,
                            opts.spread_kernel);
    } else {
        launch_spread_tiles(w, win, g, tg, bin_start.p, b, t.p, wk.grid.p, st, bs2, hflag, nullptr, &sl,
                            opts.spread_kernel);
    }
    wk.gr0 = rlo;
    wk.gr1 = rhi;
    wk.gc0 = clo;
    wk.gc1 = chi;
    wk.g_pitch = n2;
    if (tm) tm->stop();
    if (tm) tm->start(tag_fft);
    // rows [rlo, rhi): grid -> T (out of place; T rows elsewhere stay zero)
    if (wk.t_pitch == n2)
        zero_rect_minus(wk.T.p, n2, wk.tr0, wk.tr1, 0, n2, rlo, rhi, 0, n2, st);
    else if (wk.t_pitch)
        zero_rect_minus(wk.T.p, wk.t_pitch, wk.tr0, wk.tr1, 0, wk.t_pitch, 0, 0, 0, 0, st);
    auto* G = reinterpret_cast<cufftDoubleComplex*>(wk.grid.p);
    auto* T = reinterpret_cast<cufftDoubleComplex*>(wk.T.p);
    if (crad_row > 1) {
        // our radix pass over the written columns, then contiguous length-M
        // transforms in place: mode j of a row at (j mod r) M + j / r
        launch_dif_rows(wk.grid.p + (size_t)rlo * n2, rhi - rlo, n2, crad_row, clo, chi, ctw_row.p,
                        wk.T.p + (size_t)rlo * n2, st);
        ckfft(cufftSetStream(fft_row_m, st), "cufftSetStream");
        ckfft(cufftExecZ2Z(fft_row_m, T + (size_t)rlo * n2, T + (size_t)rlo * n2, CUFFT_INVERSE), "fft rows (M)");
    } else {
        ckfft(cufftSetStream(fft_row, st), "cufftSetStream");
        ckfft(cufftExecZ2Z(fft_row, G + (size_t)rlo * n2, T + (size_t)rlo * n2, CUFFT_INVERSE), "fft rows");
    }
    wk.tr0 = rlo;
    wk.tr1 = rhi;
    wk.t_pitch = n2;
    {
        auto* Tt = reinterpret_cast<cufftDoubleComplex*>(wk.T1.p);
        auto* BT = reinterpret_cast<cufftDoubleComplex*>(wk.bandT.p);
        if (crad_col > 1) {
            // the transpose does the column transform's radix pass and writes
            // every row of the band columns (no zero strips to keep)
            launch_band_transpose_dif(wk.T.p + (size_t)rlo * n2, n2, rlo, rhi, band2, bc, wk.T1.p, ax.n, crad_col,
                                      ctw_col.p, st, crad_row);
            wk.tt_r0 = 0;
            wk.tt_r1 = ax.n;
            wk.tt_pitch = ax.n;
            wk.tt_rows = bc;
            ckfft(cufftSetStream(fft_colT_m, st), "cufftSetStream");
            ckfft(cufftExecZ2Z(fft_colT_m, Tt, BT, CUFFT_INVERSE), "fft cols T (M)");
        } else {
            // Tt[c'][x] (pitch n1) holds band column c' over the populated rows only;
            // every other row x of Tt stays zero (strips a previous plan left are cleared).
            if (wk.tt_r1 > wk.tt_r0) {
                if (wk.tt_pitch == ax.n && wk.tt_rows == bc)
                    zero_rect_minus(wk.T1.p, ax.n, 0, bc, wk.tt_r0, wk.tt_r1, 0, bc, rlo, rhi, st);
                else
                    zero_rect_minus(wk.T1.p, wk.tt_pitch, 0, wk.tt_rows, wk.tt_r0, wk.tt_r1, 0, 0, 0, 0, st);
            }
            launch_band_transpose(wk.T.p, n2, rlo, rhi, band2, bc, wk.T1.p, ax.n, st, 0, 0, crad_row);
            wk.tt_r0 = rlo;
            wk.tt_r1 = rhi;
            wk.tt_pitch = ax.n;
            wk.tt_rows = bc;
            ckfft(cufftSetStream(fft_colT, st), "cufftSetStream");
            ckfft(cufftExecZ2Z(fft_colT, Tt, BT, CUFFT_INVERSE), "fft cols T");
        }
        count_launch(2);
        if (tm) tm->stop();
        if (before_interp) ck(cudaStreamWaitEvent(st, before_interp, 0), "wait");
        if (tm) tm->start(tag_interp);
        GridGeom gt{ax.n, bc, 0.5 * w};
        if (crad_col > 1) {
            gt.rad = crad_col;
            gt.rad_m = ax.n / crad_col;
            gt.rad_magic = (unsigned)((0x100000000ull + crad_col - 1) / crad_col);
        }
        launch_interp(w, win, gt, nout, s_p, post_p, mult_p, dx.p, dy_band.p, wk.bandT.p, perm_p,
                      out_p, 0, 0, st, add_p, /*transposed=*/true, &otiles, hp, opts.interp_kernel, gop);
        if (tm) tm->stop();
        return;
    }
}

// nufft.cpp:295-367 on the pruned plan. Every stage is the exact transpose of
// the corresponding forward stage restricted to the cells that are nonzero or
// read: the deconvolution factors vanish outside the band (|j| <= n/4), so the
// transposed spread only matters there; the DFT is symmetric; the gather at
// the points reads only the populated rows/columns.
void Plan::apply_transpose_pruned(const double2* in, double2* out, cudaStream_t st, StageTimer* tm,
                                  const double2* mult, int conj_in, int conj_out, const double2* addend) const {
    TransposeWork& T = tpw;
    const int n1 = ax.n, n2 = ay.n;
    const int b1 = n1 / 4;
    const GridGeom g{n1, n2, 0.5 * w};
    if (!T.ready) {
        // tile geometry of the output side at its mode coordinates (stencil
        // starts ceil(s - w/2), negative modes included) and its region lists
        DevBuf<int> ext(4);
        const int init[4] = {INT_MAX, INT_MIN, INT_MAX, INT_MIN};
        ck(cudaMemcpyAsync(ext.p, init, sizeof(init), cudaMemcpyHostToDevice, st), "extent init");
        launch_stencil_extent(s.p, nf, g.half, ext.p, st);
        int he[4];
        ck(cudaMemcpyAsync(he, ext.p, sizeof(he), cudaMemcpyDeviceToHost, st), "extent D2H");
        ck(cudaStreamSynchronize(st), "extent");
        TileGeom tg{};
        tg.tr = 16;
        tg.rlo = he[0];
        tg.clo = he[2];
        tg.nbx = (he[1] + w - he[0] + 15) / 16;
        tg.nby = (he[3] + w - he[2] + kTileC - 1) / kTileC;
        tg.rhi = tg.rlo + tg.nbx * 16;
        tg.chi = tg.clo + tg.nby * kTileC;
        tg.pitch = tg.chi - tg.clo;
        T.tg = tg;
        build_region_lists(s.p, nf, w, tg, 0u, 0u, T.rl_s, T.rl_e, st);
        T.b.alloc(std::max<uint64_t>(nf, 1));
        T.Z.alloc((size_t)(tg.rhi - tg.rlo) * tg.pitch);
        T.V.alloc((size_t)bc * n1);
        ck(cudaMemsetAsync(T.V.p, 0, T.V.bytes(), st), "V zero");  // rows outside the band stay zero
        T.Wt.alloc((size_t)bc * n1);
        T.Tz.alloc((size_t)(rhi - rlo) * n2);
        ck(cudaMemsetAsync(T.Tz.p, 0, T.Tz.bytes(), st), "Tz zero");  // columns outside the band stay zero
        T.G.alloc((size_t)n1 * n2);
        ck(cudaMemsetAsync(T.G.p, 0, T.G.bytes(), st), "G zero");
        // a dense point side gets a Z order for the staged gather (32 x 32 blocks)
        T.morton = (double)np >= 0.25 * ((double)n1 * (double)n2 / 4.0) && n1 < 32768 && n2 < 32768;
        if (T.morton) {
            DevBuf<uint32_t> keys(np);
            T.m_shift = 0;
            launch_morton_keys(t.p, np, g.half, T.m_shift, keys.p, st);
            T.m_src.alloc(np);
            launch_iota(T.m_src.p, np, st);
            sort_by_key(keys.p, T.m_src.p, np, st);
            build_tile_starts(keys.p, np, 10, T.m_tiles, T.m_ntiles, st);
            T.m_t.alloc(np);
            launch_gather(t.p, T.m_src.p, T.m_t.p, np, st);
            T.m_dst.alloc(np);
            if (perm_t.n)
                launch_gather(perm_t.p, T.m_src.p, T.m_dst.p, np, st);
            else
                ck(cudaMemcpyAsync(T.m_dst.p, T.m_src.p, np * 4, cudaMemcpyDeviceToDevice, st), "m_dst");
            T.m_phase.alloc(np);
        }
        ck(cudaStreamSynchronize(st), "transpose setup");
        T.ready = true;
    }
    const TileGeom& tg = T.tg;
    if (tm) tm->start("spread_T");
    // postphase multiply, then the tile-owned spread at the mode stencils
    launch_gather_conj_mul(in, perm_s.n ? perm_s.p : nullptr, post.p, conj_in, T.b.p, nf, st);
    SpreadOut so;
    so.mode = 0;
    so.pitch = (size_t)tg.pitch;
    so.r0 = tg.rlo;
    so.c0 = tg.clo;
    so.rend = tg.rhi;
    so.cend = tg.chi;
    so.nby_run = tg.nby;
    so.lists.s1 = T.rl_s.p;
    so.lists.e1 = T.rl_e.p;
    so.lists.ncy = (tg.nby + 1) / 2;
    launch_spread_tiles(w, win, g, tg, nullptr, T.b.p, s.p, T.Z.p, st, nullptr, nullptr, &so, &so.lists, 0);
    // deconvolution (zero outside the band) into the transposed band
    launch_band_fold(T.Z.p, tg.pitch, tg.rlo, tg.rhi, tg.clo, tg.chi, b1, n1, band2, bc, n2, dx.p, dy.p, T.V.p, st);
    if (tm) tm->stop();
    if (tm) tm->start("fft_T");
    auto* V = reinterpret_cast<cufftDoubleComplex*>(T.V.p);
    auto* Wt = reinterpret_cast<cufftDoubleComplex*>(T.Wt.p);
    if (crad_col > 1) {
        // our radix pass along the contiguous band columns, then length-M
        // transforms in place; the untranspose reads the permuted rows
        launch_dif_rows(T.V.p, bc, n1, crad_col, 0, n1, ctw_col.p, T.Wt.p, st);
        ckfft(cufftSetStream(fft_colT_m, st), "cufftSetStream");
        ckfft(cufftExecZ2Z(fft_colT_m, Wt, Wt, CUFFT_INVERSE), "fft cols T (M)");
    } else {
        ckfft(cufftSetStream(fft_colT, st), "cufftSetStream");
        ckfft(cufftExecZ2Z(fft_colT, V, Wt, CUFFT_INVERSE), "fft cols T");
    }
    launch_band_untranspose(T.Wt.p, n1, rlo, rhi, band2, bc, T.Tz.p, n2, st, crad_col);
    ckfft(cufftSetStream(fft_row, st), "cufftSetStream");
    ckfft(cufftExecZ2Z(fft_row, reinterpret_cast<cufftDoubleComplex*>(T.Tz.p),
                       reinterpret_cast<cufftDoubleComplex*>(T.G.p + (size_t)rlo * n2), CUFFT_INVERSE),
          "fft rows T");
    count_launch(2);
    if (tm) tm->stop();
    if (tm) tm->start("interp_T");
    // gather at the point stencils x prephase (x mult)
    if (T.morton && !addend && !conj_out && opts.interp_kernel == 0) {
        if (T.m_mult_of != mult || !mult) {
            launch_gather(pre.p, T.m_src.p, T.m_phase.p, np, st);
            if (mult) {
                DevBuf<double2> mm(np);
                launch_gather(mult, T.m_src.p, mm.p, np, st);
                launch_mul(T.m_phase.p, mm.p, np, st);
                ck(cudaStreamSynchronize(st), "m_phase");
            }
            T.m_mult_of = mult;
        }
        InterpTiles it;
        it.start = T.m_tiles.p;
        it.n = T.m_ntiles;
        it.shift = T.m_shift;
        it.out_lo = 0;
        launch_interp(w, win, g, np, T.m_t.p, T.m_phase.p, nullptr, nullptr, nullptr, T.G.p, T.m_dst.p, out, 0, 0,
                      st, nullptr, false, &it, nullptr, 1);
    } else {
        launch_interp(w, win, g, np, t.p, pre.p, mult, nullptr, nullptr, T.G.p, perm_t.n ? perm_t.p : nullptr, out,
                      0, conj_out, st, addend, false, nullptr, nullptr, opts.interp_kernel);
    }
    if (tm) tm->stop();
}

// nufft.cpp:295-367
void Plan::apply_transpose(const double2* in, double2* out, FftWork& wk, cudaStream_t st,
                           StageTimer* tm, const double2* mult, int conj_in,
                           int conj_out, const double2* addend) const {
    if (fast && pruned) {
        apply_transpose_pruned(in, out, st, tm, mult, conj_in, conj_out, addend);
        return;
    }
    if (addend) throw Error(3, "apply_transpose: addend needs the pruned path");
    if (!fast) {
        if (tm) tm->start("ndft_T");
        const double2* src = in;
        DevBuf<double2> tmp;
        if (conj_in) {
            tmp.alloc(nf);
            launch_conj(in, tmp.p, nf, st);
            src = tmp.p;
        }
        launch_ndft(frq.p, nf, pts.p, np, src, sign, out, st);
        if (mult) launch_mul(out, mult, np, st);
        if (conj_out) launch_conj(out, out, np, st);
        if (tm) tm->stop();
        if (conj_in) ck(cudaStreamSynchronize(st), "ndft_T tmp");
        return;
    }
    ensure_work(wk, st);
    const GridGeom g{ax.n, ay.n, 0.5 * w};
    if (tm) tm->start("spread_T");
    ck(cudaMemsetAsync(wk.grid.p, 0, cells() * sizeof(double2), st), "grid zero");
    // spread at the frequency stencils with postphase, deconv folded in
    launch_spread(w, win, g, nf, perm_s.n ? perm_s.p : nullptr, in, s.p, post.p, nullptr, dx.p,
                  dy.p, wk.grid.p, conj_in, st);
    if (tm) tm->stop();
    if (tm) tm->start("fft_T");
    full_fft(*this, wk.grid.p, st);
    if (tm) tm->stop();
    if (tm) tm->start("interp_T");
    launch_interp(w, win, g, np, t.p, pre.p, mult, nullptr, nullptr, wk.grid.p,
                  perm_t.n ? perm_t.p : nullptr, out, 0, conj_out, st, nullptr, false, nullptr, nullptr,
                  opts.interp_kernel);
    if (tm) tm->stop();
    wk.gr0 = 0;
    wk.gr1 = ax.n;
    wk.gc0 = 0;
    wk.gc1 = ay.n;
    wk.g_pitch = ay.n;
}

std::vector<uint32_t> Plan::adopt_point_order(cudaStream_t st) {
    std::vector<uint32_t> h(np);
    if (perm_t.n) {
        ck(cudaMemcpyAsync(h.data(), perm_t.p, np * 4, cudaMemcpyDeviceToHost, st), "perm D2H");
        ck(cudaStreamSynchronize(st), "perm D2H");
        perm_t.release();
    } else {
        for (uint64_t i = 0; i < np; ++i) h[i] = (uint32_t)i;
    }
    if (!fast) {
        // direct path keeps raw points; reorder them to match
        std::vector<double2> raw(np), sorted(np);
        ck(cudaStreamSynchronize(st), "pts sync");  // st is non-blocking
        ck(cudaMemcpy(raw.data(), pts.p, np * 16, cudaMemcpyDeviceToHost), "pts D2H");
        for (uint64_t i = 0; i < np; ++i) sorted[i] = raw[h[i]];
        pts.upload(sorted.data(), np, st);
        ck(cudaStreamSynchronize(st), "pts H2D");
    }
    return h;
}

// ------------------------------------------------------------ StageTimer
void StageTimer::reset() {
    for (auto e : begin) cudaEventDestroy(e);
    for (auto e : end) cudaEventDestroy(e);
    begin.clear();
    end.clear();
    names.clear();
}
void StageTimer::start(const char* name, cudaStream_t on_stream) {
    if (!on) return;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, on_stream ? on_stream : stream);
    begin.push_back(a);
    end.push_back(b);
    names.emplace_back(name);
}
void StageTimer::stop(cudaStream_t on_stream) {
    if (!on || end.empty()) return;
    cudaEventRecord(end.back(), on_stream ? on_stream : stream);
}
int StageTimer::read(double* ms, const char** nm, int cap) {
    const int n = (int)names.size();
    for (int i = 0; i < n && i < cap; ++i) {
        float f = 0.f;
        cudaEventSynchronize(end[i]);
        cudaEventElapsedTime(&f, begin[i], end[i]);
        if (ms) ms[i] = f;
        if (nm) nm[i] = names[i].c_str();
    }
    return n;
}
StageTimer::~StageTimer() { reset(); }

} // namespace sbdgpu
