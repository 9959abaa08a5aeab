// slab.cpp -- slab decomposition of one CompressedOperator::apply
// (conv_operator.cpp:301-309) over G devices, one rank per device, such that
// no stage is replicated (SURVEY.md section 8e's
// "scaling alternative"). Complex pipeline (every xi node; complex f or not).
//
// Rank h of G holds the whole operator and computes
//   A  spread of all sources, restricted to its row slab [R_h, R_h+1) of the
//      fwd_in grid (a range of region rows of the tile-owned CTA spread), and
//      the row transforms of those rows;               -> exchange 0
//   B  the column transforms of its window of fwd_in band columns (all rows),
//      the xi interpolation at the nodes its fwd_out column slab needs, the
//      tile-owned spread of those nodes into the slab [C_h, C_h+1), and the
//      column transforms of the slab;                   -> exchange 1
//   C  the row transforms of its window of fwd_out band rows, the
//      interpolation at the targets whose x-mode stencils start in its range,
//      plus their rows of D f.
// Exchanges 0 and 1 are all-to-alls (NCCL / gloo through torch.distributed,
// parallel.py): rank h sends every rank h' the columns (rows) of h''s window
// for its own rows (columns). Windows include the stencil halos, so the only
// duplicated work is the interpolation of the xi nodes near a slab boundary.
// Every partition table is computed from the operator alone, identically on
// every rank; slabs are balanced by point counts.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <numeric>

#include "op_internal.h"

using namespace sbdgpu;

struct sbd_slab {
    sbd_op* op = nullptr;
    int rank = 0, world = 1, device = 0, w = 0;
    double half = 0.0;
    // partition tables (world + 1 bounds or world windows)
    std::vector<int> Q, R;        // fwd_in region rows / grid rows of each row slab
    std::vector<int> J0, J1;      // fwd_in y-mode windows (band columns) per rank
    std::vector<int> C;           // fwd_out grid column slabs
    std::vector<int> M0, M1;      // fwd_out x-mode windows (band rows) per rank
    std::vector<uint64_t> cnt[4], off[4];  // send0, recv0, send1, recv1 (complex counts / offsets)
    // stage A
    DevBuf<double2> bsrc, A, A2;
    cufftHandle fftA = 0;
    // stage B
    DevBuf<double2> T, U;
    cufftHandle fftT = 0;
    uint64_t n_need = 0;
    DevBuf<double2> need_s, need_post, need_kappa;
    DevBuf<uint32_t> need_dst, need_tiles;
    uint32_t need_ntiles = 0;
    int need_shift = 0;
    DevBuf<double> dy_loc;
    DevBuf<double2> pts_t, spec;
    TileGeom tgB{};
    DevBuf<uint32_t> rl_s, rl_e;
    DevBuf<double2> Bt, V;
    cufftHandle fftB = 0;
    // stage C
    DevBuf<double2> Wr, X;
    cufftHandle fftW = 0;
    uint64_t n_own = 0;
    DevBuf<double2> tgt_s, tgt_post, f_sorted, qs;
    DevBuf<uint32_t> tgt_dst;
    DevBuf<double> dx_loc;
    DevBuf<uint64_t> ro;
    DevBuf<uint32_t> cols;
    DevBuf<double2> vals;

    ~sbd_slab() {
        for (cufftHandle h : {fftA, fftT, fftB, fftW})
            if (h) cufftDestroy(h);
    }
    int rows(int h) const { return R[h + 1] - R[h]; }
    int ncol(int h) const { return J1[h] - J0[h]; }
    int ncs(int h) const { return C[h + 1] - C[h]; }
    int nrow(int h) const { return M1[h] - M0[h]; }
};

namespace {

template <typename T>
std::vector<T> download(const DevBuf<T>& b, uint64_t n, cudaStream_t st) {
    if (!b.n || !n) return {};
    std::vector<T> h(n);
    ck(cudaMemcpyAsync(h.data(), b.p, n * sizeof(T), cudaMemcpyDeviceToHost, st), "slab D2H");
    return h;
}

// split [0, n) (weights wt) into g contiguous ranges of ~equal weight
std::vector<int> balance(const std::vector<uint64_t>& wt, int g) {
    const int n = (int)wt.size();
    std::vector<uint64_t> pre(n + 1, 0);
    for (int i = 0; i < n; ++i) pre[i + 1] = pre[i] + wt[i];
    std::vector<int> b(g + 1, 0);
    b[g] = n;
    for (int k = 1; k < g; ++k) {
        const uint64_t target = pre[n] * (uint64_t)k / (uint64_t)g;
        int i = (int)(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
        b[k] = std::min(std::max(i, b[k - 1]), n);
    }
    return b;
}

inline int stencil_start(double c, double half) { return (int)std::ceil(c - half); }

void plan_fft(cufftHandle& h, int len, int batch, const char* what) {
    if (batch <= 0) return;
    int n[1] = {len};
    ckfft(cufftPlanMany(&h, 1, n, n, 1, len, n, 1, len, CUFFT_Z2Z, batch), what);
}

void build(sbd_slab& S, cudaStream_t st) {
    sbd_op& op = *S.op;
    const Plan& P1 = *op.fwd_in;
    const Plan& P2 = *op.fwd_out;
    const int G = S.world, h = S.rank;
    const int w = P1.w;
    S.w = w;
    S.half = 0.5 * w;
    const uint64_t ns = op.d.n_src(), nt = op.d.n_tgt(), nx = op.d.n_xi();
    const int n1 = P1.ax.n, n2 = P1.ay.n, m1 = P2.ax.n, m2 = P2.ay.n;

    // ---- fwd_in row slabs: region rows balanced by their list entries
    const int ncx1 = (P1.tg.nbx + 1) / 2, ncy1 = (P1.tg.nby + 1) / 2;
    {
        const std::vector<uint32_t> rs = download(P1.rl1_s, (uint64_t)ncx1 * ncy1 + 1, st);
        ck(cudaStreamSynchronize(st), "slab");
        std::vector<uint64_t> wt(ncx1, 0);
        for (int cx = 0; cx < ncx1; ++cx) wt[cx] = rs[(size_t)(cx + 1) * ncy1] - rs[(size_t)cx * ncy1];
        S.Q = balance(wt, G);
        S.R.resize(G + 1);
        for (int k = 0; k <= G; ++k) S.R[k] = std::min(P1.tg.rlo + 32 * S.Q[k], P1.rhi);
        S.R[G] = P1.rhi;
    }

    // ---- fwd_out column slabs: 32-column region blocks balanced by xi nodes
    const std::vector<double2> t2 = download(P2.t, nx, st);     // canonical xi order
    const std::vector<double2> s1 = download(P1.s, nx, st);     // fwd_in output order
    const std::vector<uint32_t> p1 = download(P1.perm_s, nx, st);
    const std::vector<double2> post1 = download(P1.post, nx, st);
    const std::vector<double2> kap = download(op.kappa, nx, st);
    ck(cudaStreamSynchronize(st), "slab");
    std::vector<uint32_t> pos1(nx);  // canonical -> fwd_in output position
    for (uint64_t k = 0; k < nx; ++k) pos1[p1.empty() ? k : p1[k]] = (uint32_t)k;
    const int ncb = (P2.tg.nby + 1) / 2;
    {
        std::vector<uint64_t> wt(ncb, 0);
        for (uint64_t v = 0; v < nx; ++v) {
            const int b = (stencil_start(t2[v].y, S.half) - P2.tg.clo) >> 5;
            wt[std::min(std::max(b, 0), ncb - 1)] += 1;
        }
        const std::vector<int> bk = balance(wt, G);
        S.C.resize(G + 1);
        for (int k = 0; k <= G; ++k) S.C[k] = std::min(P2.tg.clo + 32 * bk[k], P2.chi);
        S.C[G] = P2.chi;
    }
    // nodes each rank's slab needs, and the fwd_in y-mode windows they read
    // (one column of margin on each side: the shifted coordinates round like
    // the originals up to an ulp)
    S.J0.assign(G, 0);
    S.J1.assign(G, 0);
    std::vector<uint32_t> need;
    for (int k = 0; k < G; ++k) {
        int lo = INT_MAX, hi = INT_MIN;
        for (uint64_t v = 0; v < nx; ++v) {
            const int iy = stencil_start(t2[v].y, S.half);
            if (iy >= S.C[k + 1] || iy + w <= S.C[k]) continue;
            const int jy = stencil_start(s1[pos1[v]].y, S.half);
            lo = std::min(lo, jy);
            hi = std::max(hi, jy + w);
            if (k == h) need.push_back((uint32_t)v);
        }
        if (lo <= hi) {
            // (>= 48 columns: the staged interpolation's 42-column footprints
            // wrap inside the window)
            S.J0[k] = lo - 1;
            S.J1[k] = std::max(hi + 1, S.J0[k] + 48);
        }
    }
    S.n_need = need.size();

    // ---- fwd_out x-mode windows: targets balanced by their stencil rows
    const std::vector<double2> s2 = download(P2.s, nt, st);
    const std::vector<double2> post2 = download(P2.post, nt, st);
    const std::vector<uint32_t> p2 = download(P2.perm_s, nt, st);
    ck(cudaStreamSynchronize(st), "slab");
    int xlo = INT_MAX, xhi = INT_MIN;
    for (uint64_t j = 0; j < nt; ++j) {
        const int ix = stencil_start(s2[j].x, S.half);
        xlo = std::min(xlo, ix);
        xhi = std::max(xhi, ix);
    }
    std::vector<int> Mo(G + 1);
    {
        std::vector<uint64_t> wt(nt ? xhi - xlo + 1 : 1, 0);
        for (uint64_t j = 0; j < nt; ++j) wt[stencil_start(s2[j].x, S.half) - xlo] += 1;
        const std::vector<int> b = balance(wt, G);
        for (int k = 0; k <= G; ++k) Mo[k] = xlo + b[k];
    }
    S.M0.resize(G);
    S.M1.resize(G);
    for (int k = 0; k < G; ++k) {
        S.M0[k] = Mo[k] - 1;
        S.M1[k] = Mo[k + 1] + w;
    }

    // ---- exchange layouts (complex counts)
    for (auto& c : S.cnt) c.assign(G, 0);
    for (int k = 0; k < G; ++k) {
        S.cnt[0][k] = (uint64_t)S.ncol(k) * S.rows(h);   // send0: k's window of my rows
        S.cnt[1][k] = (uint64_t)S.ncol(h) * S.rows(k);   // recv0: my window of k's rows
        S.cnt[2][k] = (uint64_t)S.nrow(k) * S.ncs(h);    // send1: k's rows of my columns
        S.cnt[3][k] = (uint64_t)S.nrow(h) * S.ncs(k);    // recv1: my rows of k's columns
    }
    for (int e = 0; e < 4; ++e) {
        S.off[e].assign(G + 1, 0);
        for (int k = 0; k < G; ++k) S.off[e][k + 1] = S.off[e][k] + S.cnt[e][k];
    }

    // ---- stage A buffers
    S.bsrc.alloc(std::max<uint64_t>(ns, 1));
    const size_t ra = (size_t)std::max(S.rows(h), 1) * n2;
    S.A.alloc(ra);
    ck(cudaMemsetAsync(S.A.p, 0, S.A.bytes(), st), "slab A");  // columns outside the spread stay zero
    S.A2.alloc(ra);
    plan_fft(S.fftA, n2, S.rows(h), "slab rows A");

    // ---- stage B: nodes in the Z order of their shifted fwd_in coordinates
    const int nc = std::max(S.ncol(h), 1);
    S.T.alloc((size_t)nc * n1);
    ck(cudaMemsetAsync(S.T.p, 0, S.T.bytes(), st), "slab T");  // rows outside the populated ones stay zero
    S.U.alloc((size_t)nc * n1);
    plan_fft(S.fftT, n1, S.ncol(h), "slab cols T");
    {
        std::vector<double> dyl(nc, 0.0);
        const std::vector<double> dy1 = download(P1.dy, n2, st);
        ck(cudaStreamSynchronize(st), "slab");
        for (int l = 0; l < S.ncol(h); ++l) dyl[l] = dy1[((S.J0[h] + l) % n2 + n2) % n2];
        S.dy_loc.upload(dyl.data(), nc, st);
    }
    const uint64_t nn = std::max<uint64_t>(S.n_need, 1);
    {
        std::vector<double2> ns_(nn), np_(nn), nk(nn), pt(nn);
        for (uint64_t i = 0; i < S.n_need; ++i) {
            const uint32_t v = need[i];
            const uint32_t k = pos1[v];
            ns_[i] = make_double2(s1[k].x, s1[k].y - (double)S.J0[h]);
            np_[i] = post1[k];
            nk[i] = kap[k];
            pt[i] = t2[v];
        }
        DevBuf<double2> a(nn), b(nn), c(nn);
        a.upload(ns_.data(), nn, st);
        b.upload(np_.data(), nn, st);
        c.upload(nk.data(), nn, st);
        S.pts_t.upload(pt.data(), nn, st);
        S.spec.alloc(nn);
        if (S.n_need) {
            DevBuf<uint32_t> keys(S.n_need), idx(S.n_need);
            S.need_shift = std::max(n1, nc) / 2 + w + 2;
            launch_morton_keys(a.p, S.n_need, S.half, S.need_shift, keys.p, st);
            launch_iota(idx.p, S.n_need, st);
            sort_by_key(keys.p, idx.p, S.n_need, st);
            build_tile_starts(keys.p, S.n_need, 10, S.need_tiles, S.need_ntiles, st);
            S.need_s.alloc(S.n_need);
            S.need_post.alloc(S.n_need);
            S.need_kappa.alloc(S.n_need);
            launch_gather(a.p, idx.p, S.need_s.p, S.n_need, st);
            launch_gather(b.p, idx.p, S.need_post.p, S.n_need, st);
            launch_gather(c.p, idx.p, S.need_kappa.p, S.n_need, st);
            S.need_dst = std::move(idx);  // Z position -> position in the spread's point arrays
        }
        ck(cudaStreamSynchronize(st), "slab nodes");
    }
    // the slab's spread: P2's tile rows, the slab's columns
    S.tgB = P2.tg;
    S.tgB.clo = S.C[h];
    S.tgB.nby = std::max((S.ncs(h) + kTileC - 1) / kTileC, 0);
    S.tgB.chi = S.C[h + 1];
    S.tgB.pitch = 0;
    if (S.n_need && S.tgB.nby) build_region_lists(S.pts_t.p, S.n_need, w, S.tgB, 0u, 0u, S.rl_s, S.rl_e, st);
    const int ncsh = std::max(S.ncs(h), 1);
    S.Bt.alloc((size_t)ncsh * m1);
    ck(cudaMemsetAsync(S.Bt.p, 0, S.Bt.bytes(), st), "slab B");  // rows outside the spread stay zero
    S.V.alloc((size_t)ncsh * m1);
    plan_fft(S.fftB, m1, S.ncs(h), "slab cols B");

    // ---- stage C: owned targets (Z order kept), their rows of D, windows
    const int nr = std::max(S.nrow(h), 1);
    S.Wr.alloc((size_t)nr * m2);
    ck(cudaMemsetAsync(S.Wr.p, 0, S.Wr.bytes(), st), "slab W");  // columns outside the slabs stay zero
    S.X.alloc((size_t)nr * m2);
    plan_fft(S.fftW, m2, S.nrow(h), "slab rows W");
    {
        std::vector<double> dxl(nr, 0.0);
        const std::vector<double> dx2 = download(P2.dx, m1, st);
        ck(cudaStreamSynchronize(st), "slab");
        for (int r = 0; r < S.nrow(h); ++r) dxl[r] = dx2[((S.M0[h] + r) % m1 + m1) % m1];
        S.dx_loc.upload(dxl.data(), nr, st);
    }
    std::vector<uint32_t> own;
    for (uint64_t j = 0; j < nt; ++j) {
        const int ix = stencil_start(s2[j].x, S.half);
        if (ix >= Mo[h] && ix < Mo[h + 1]) own.push_back((uint32_t)j);
    }
    S.n_own = own.size();
    const uint64_t no = std::max<uint64_t>(S.n_own, 1);
    {
        std::vector<double2> ts(no), tp(no);
        std::vector<uint32_t> td(no);
        for (uint64_t i = 0; i < S.n_own; ++i) {
            const uint32_t j = own[i];
            ts[i] = make_double2(s2[j].x - (double)S.M0[h], s2[j].y);
            tp[i] = post2[j];
            td[i] = p2.empty() ? j : p2[j];
        }
        S.tgt_s.upload(ts.data(), no, st);
        S.tgt_post.upload(tp.data(), no, st);
        S.tgt_dst.upload(td.data(), no, st);
        // rows of D for the owned targets (caller order), columns renumbered to
        // fwd_in's sorted source order (the order f_sorted is gathered in)
        std::vector<uint32_t> ps = download(P1.perm_t, ns, st);
        ck(cudaStreamSynchronize(st), "slab");
        std::vector<uint32_t> inv(ns);
        for (uint64_t i = 0; i < ns; ++i) inv[ps.empty() ? i : ps[i]] = (uint32_t)i;
        std::vector<uint64_t> r(no + 1, 0);
        for (uint64_t i = 0; i < S.n_own; ++i) {
            const uint32_t t = td[i];
            r[i + 1] = r[i] + (op.d.row_offsets[t + 1] - op.d.row_offsets[t]);
        }
        const uint64_t nz = std::max<uint64_t>(r[S.n_own], 1);
        std::vector<uint32_t> c2(nz, 0);
        std::vector<double> v2(2 * nz, 0.0);
        for (uint64_t i = 0; i < S.n_own; ++i) {
            const uint32_t t = td[i];
            uint64_t o = r[i];
            for (uint64_t e = op.d.row_offsets[t]; e < op.d.row_offsets[t + 1]; ++e, ++o) {
                c2[o] = inv[op.d.cols[e]];
                v2[2 * o] = op.d.values[2 * e];
                v2[2 * o + 1] = op.d.values[2 * e + 1];
            }
        }
        S.ro.upload(r.data(), no + 1, st);
        S.cols.upload(c2.data(), nz, st);
        S.vals.upload(reinterpret_cast<const double2*>(v2.data()), nz, st);
        S.f_sorted.alloc(std::max<uint64_t>(ns, 1));
        S.qs.alloc(no);
        ck(cudaStreamSynchronize(st), "slab targets");
    }
}

// stage A: f -> exchange-0 send buffer
void stage_a(sbd_slab& S, const double2* f, double2* send0, cudaStream_t st) {
    sbd_op& op = *S.op;
    const Plan& P1 = *op.fwd_in;
    const int G = S.world, h = S.rank, n2 = P1.ay.n;
    launch_gather_mul(f, P1.perm_t.n ? P1.perm_t.p : nullptr, P1.pre.p, S.bsrc.p, nullptr, op.d.n_src(), st);
    if (S.rows(h) > 0) {
        SpreadOut so;
        so.mode = 0;
        so.pitch = (size_t)n2;
        so.r0 = S.R[h];
        so.c0 = 0;
        so.rend = S.R[h + 1];
        so.cend = P1.chi;
        so.nby_run = P1.tg.nby;
        so.lists = P1.lists(false);
        so.cx0 = S.Q[h];
        so.ncx_run = S.Q[h + 1] - S.Q[h];
        const GridGeom g{P1.ax.n, n2, S.half};
        launch_spread_tiles(S.w, P1.win, g, P1.tg, nullptr, S.bsrc.p, P1.t.p, S.A.p, st, nullptr, nullptr, &so,
                            &so.lists, 0);
        ckfft(cufftSetStream(S.fftA, st), "cufftSetStream");
        ckfft(cufftExecZ2Z(S.fftA, reinterpret_cast<cufftDoubleComplex*>(S.A.p),
                           reinterpret_cast<cufftDoubleComplex*>(S.A2.p), CUFFT_INVERSE),
              "slab rows A");
        count_launch();
    }
    for (int k = 0; k < G; ++k)
        launch_wrap_transpose(S.A2.p, (size_t)n2, n2, S.J0[k], S.ncol(k), S.rows(h), send0 + S.off[0][k],
                              (size_t)S.rows(h), st);
}

// stage B: exchange-0 receive buffer -> exchange-1 send buffer
void stage_b(sbd_slab& S, const double2* recv0, double2* send1, cudaStream_t st) {
    sbd_op& op = *S.op;
    const Plan& P1 = *op.fwd_in;
    const Plan& P2 = *op.fwd_out;
    const int G = S.world, h = S.rank, n1 = P1.ax.n, m1 = P2.ax.n;
    if (S.ncol(h) > 0) {
        for (int k = 0; k < G; ++k)
            if (S.rows(k) > 0)
                ck(cudaMemcpy2DAsync(S.T.p + S.R[k], (size_t)n1 * 16, recv0 + S.off[1][k], (size_t)S.rows(k) * 16,
                                     (size_t)S.rows(k) * 16, (size_t)S.ncol(h), cudaMemcpyDeviceToDevice, st),
                   "slab unpack 0");
        ckfft(cufftSetStream(S.fftT, st), "cufftSetStream");
        ckfft(cufftExecZ2Z(S.fftT, reinterpret_cast<cufftDoubleComplex*>(S.T.p),
                           reinterpret_cast<cufftDoubleComplex*>(S.U.p), CUFFT_INVERSE),
              "slab cols T");
        count_launch();
    }
    if (S.n_need) {
        InterpTiles it;
        it.start = S.need_tiles.p;
        it.n = S.need_ntiles;
        it.shift = S.need_shift;
        it.out_lo = 0;
        const GridGeom g{n1, S.ncol(h), S.half};
        launch_interp(S.w, P1.win, g, S.n_need, S.need_s.p, S.need_post.p, S.need_kappa.p, P1.dx.p, S.dy_loc.p,
                      S.U.p, S.need_dst.p, S.spec.p, 0, 0, st, nullptr, /*transposed=*/true, &it, nullptr, 1);
    }
    if (S.ncs(h) > 0) {
        if (S.n_need && S.tgB.nby) {
            SpreadOut so;
            so.mode = 2;
            so.pitch = (size_t)m1;
            so.r0 = 0;
            so.c0 = S.C[h];
            so.rend = P2.rhi;
            so.cend = S.C[h + 1];
            so.nby_run = S.tgB.nby;
            so.lists.s1 = S.rl_s.p;
            so.lists.e1 = S.rl_e.p;
            so.lists.ncy = (S.tgB.nby + 1) / 2;
            const GridGeom g{m1, P2.ay.n, S.half};
            launch_spread_tiles(S.w, P2.win, g, S.tgB, nullptr, S.spec.p, S.pts_t.p, S.Bt.p, st, nullptr, nullptr,
                                &so, &so.lists, 0);
        }
        ckfft(cufftSetStream(S.fftB, st), "cufftSetStream");
        ckfft(cufftExecZ2Z(S.fftB, reinterpret_cast<cufftDoubleComplex*>(S.Bt.p),
                           reinterpret_cast<cufftDoubleComplex*>(S.V.p), CUFFT_INVERSE),
              "slab cols B");
        count_launch();
    }
    for (int k = 0; k < G; ++k)
        launch_wrap_transpose(S.V.p, (size_t)m1, m1, S.M0[k], S.nrow(k), S.ncs(h), send1 + S.off[2][k],
                              (size_t)S.ncs(h), st);
}

// stage C: exchange-1 receive buffer + f -> q at this rank's targets
void stage_c(sbd_slab& S, const double2* recv1, const double2* f, double2* q, cudaStream_t st) {
    sbd_op& op = *S.op;
    const Plan& P1 = *op.fwd_in;
    const Plan& P2 = *op.fwd_out;
    const int G = S.world, h = S.rank, m2 = P2.ay.n;
    if (S.nrow(h) <= 0 || !S.n_own) return;
    for (int k = 0; k < G; ++k)
        if (S.ncs(k) > 0)
            ck(cudaMemcpy2DAsync(S.Wr.p + S.C[k], (size_t)m2 * 16, recv1 + S.off[3][k], (size_t)S.ncs(k) * 16,
                                 (size_t)S.ncs(k) * 16, (size_t)S.nrow(h), cudaMemcpyDeviceToDevice, st),
               "slab unpack 1");
    ckfft(cufftSetStream(S.fftW, st), "cufftSetStream");
    ckfft(cufftExecZ2Z(S.fftW, reinterpret_cast<cufftDoubleComplex*>(S.Wr.p),
                       reinterpret_cast<cufftDoubleComplex*>(S.X.p), CUFFT_INVERSE),
          "slab rows W");
    count_launch();
    launch_gather(f, P1.perm_t.n ? P1.perm_t.p : nullptr, S.f_sorted.p, op.d.n_src(), st);
    launch_spmv_vec(S.n_own, S.ro.p, S.cols.p, S.vals.p, S.f_sorted.p, S.qs.p, st);
    const GridGeom g{S.nrow(h), m2, S.half};
    launch_interp(S.w, P2.win, g, S.n_own, S.tgt_s.p, S.tgt_post.p, nullptr, S.dx_loc.p, P2.dy.p, S.X.p,
                  S.tgt_dst.p, q, 0, 0, st, S.qs.p, false, nullptr, nullptr, 3);
}

template <typename F>
int guarded_slab(F&& f) {
    try {
        f();
        return SBD_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SBD_ERR_RUNTIME;
    }
}

} // namespace

extern "C" {

int sbd_slab_create(sbd_op* op, int rank, int world, sbd_slab** out) {
    return guarded_slab([&] {
        if (!op || !out || world < 1 || rank < 0 || rank >= world)
            throw Error(SBD_ERR_INVALID_ARGUMENT, "slab_create: bad argument");
        if (!op->fused) throw Error(SBD_ERR_RUNTIME, "slab decomposition needs both NUFFTs on the gridded path");
        std::lock_guard<std::recursive_mutex> lk(op->mu);
        DeviceGuard g(op->device);
        op->ensure_node_arrays(op->stream);  // a procedural operator: the slab plan reads the per-node arrays
        auto s = std::make_unique<sbd_slab>();
        s->op = op;
        s->rank = rank;
        s->world = world;
        s->device = op->device;
        build(*s, op->stream);
        *out = s.release();
    });
}

int sbd_slab_destroy(sbd_slab* s) {
    return guarded_slab([&] {
        if (!s) return;
        DeviceGuard g(s->device);
        delete s;
    });
}

int sbd_slab_counts(const sbd_slab* s, int exchange, uint64_t* send_counts, uint64_t* recv_counts) {
    return guarded_slab([&] {
        if (!s || (exchange != 0 && exchange != 1)) throw Error(SBD_ERR_INVALID_ARGUMENT, "slab_counts: bad argument");
        for (int k = 0; k < s->world; ++k) {
            if (send_counts) send_counts[k] = s->cnt[2 * exchange][k];
            if (recv_counts) recv_counts[k] = s->cnt[2 * exchange + 1][k];
        }
    });
}

int sbd_slab_stage(sbd_slab* s, int stage, const double* d_in, const double* d_f, double* d_out, void* stream) {
    return guarded_slab([&] {
        if (!s || stage < 0 || stage > 2) throw Error(SBD_ERR_INVALID_ARGUMENT, "slab_stage: bad argument");
        std::lock_guard<std::recursive_mutex> lk(s->op->mu);
        DeviceGuard g(s->device);
        cudaStream_t st = (cudaStream_t)stream;
        s->op->order_begin(st);
        auto* out = reinterpret_cast<double2*>(d_out);
        if (stage == 0) stage_a(*s, reinterpret_cast<const double2*>(d_f), out, st);
        if (stage == 1) stage_b(*s, reinterpret_cast<const double2*>(d_in), out, st);
        if (stage == 2)
            stage_c(*s, reinterpret_cast<const double2*>(d_in), reinterpret_cast<const double2*>(d_f), out, st);
        ck(cudaGetLastError(), "slab stage");
        s->op->order_end(st);
    });
}

} // extern "C"
