// op_internal.h -- the operator object behind the C ABI (sbd_op), shared by
// op.cpp (single-device apply, adjoint, sharded halves, C ABI) and slab.cpp
// (slab decomposition of one apply over several devices). Not public.
#pragma once

#include <algorithm>
#include <cstdio>
#include <memory>
#include <mutex>
#include <vector>

#include "../../include/sbd_b200.h"
#include "opdata.h"
#include "sbd_internal.h"

namespace sbdgpu {
// the thread-local message of sbd_last_error()
void set_last_error(const std::string& m);

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        ck(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};
} // namespace sbdgpu

using namespace sbdgpu;

struct sbd_op {
    OpData d;
    sbd_op_options opt;
    int device = 0;
    cudaStream_t stream = nullptr;
    std::unique_ptr<Plan> fwd_in, fwd_out;
    std::vector<uint32_t> perm_xi; // sorted xi position -> file index
    DevBuf<double2> w_sorted;      // omega-hat in sorted (canonical) xi order
    DevBuf<double2> w_in;          // omega-hat in fwd_in's output (interpolation) order
    DevBuf<uint64_t> ro;
    DevBuf<uint32_t> cols;
    DevBuf<double2> vals;
    FftWork work;
    DevBuf<double2> spec;
    DevBuf<double2> hf, hq; // staging for the host-buffer API
    // Pipelined host-buffer API (sbd_op_apply_async): two staging slots, the
    // H2D of f on cp_in, the apply on `stream`, the D2H of q on cp_out, so
    // the copies of one call overlap the device work of its neighbours.
    struct Slot {
        DevBuf<double2> f, q;
        cudaEvent_t h2d = nullptr, comp = nullptr, d2h = nullptr;
        bool used = false;
    } slot[2];
    cudaStream_t cp_in = nullptr, cp_out = nullptr;
    uint64_t tickets = 0;
    // Fused forward path (both plans gridded): D renumbered to (sorted target
    // row, sorted source column) so its f gathers are spatially local, and
    // kappa = omega-hat * fwd_out prephase so the xi interpolation emits the
    // xi spread's coefficients directly.
    bool fused = false;
    DevBuf<uint64_t> ro_s;
    DevBuf<uint32_t> cols_s;
    DevBuf<double2> vals_s;
    // Re(D') alone: for a real f, Im(D) only feeds Im(q) (Re(q) is bitwise the
    // complex product's), and a real-input apply of a real-omega-hat operator
    // returns a real q -- as the half split already does for the far field
    // (the reference's Im(D) is its NUFFT's window asymmetry, <= 2e-10 |D|)
    DevBuf<double> vals_sr;

    // rows [lo, hi) of the renumbered D' times f_sorted into qs
    // (real_f: the caller vouches for a real f, and f_sorted_re holds Re(f_sorted))
    DevBuf<double> f_sorted_re;
    void spmv_sorted(uint64_t lo, uint64_t hi, cudaStream_t st, bool real_f = false) {
        if (vals_sr.n && (real_f || !vals_s.n))
            launch_spmv_vec_real(hi - lo, ro_s.p + lo, cols_s.p, vals_sr.p, f_sorted.p, qs.p + lo, st,
                                 real_f && f_sorted_re.n ? f_sorted_re.p : nullptr);
        else
            launch_spmv_vec(hi - lo, ro_s.p + lo, cols_s.p, vals_s.p, f_sorted.p, qs.p + lo, st);
    }
    DevBuf<double2> kappa, f_sorted, qs;
    // Real-input half split: with real omega-hat and
    // antipodally paired rings, a real f has spectrum(-xi) = conj(spectrum(xi)),
    // so only the tag-0 half of each pair is interpolated and spread and the
    // far field is 2 Re(.). The device flag is set per apply and cleared by the
    // input gather when f has a nonzero imaginary part (no host round trip).
    bool herm_ok = false;
    uint64_t n_half = 0;           // tag-0 xi nodes (sorted positions [0, n_half))
    DevBuf<double2> kappa_h;       // kappa with self-conjugate nodes halved
    DevBuf<int> herm_flag;
    // Hermitian-FFT mode on top of the half split (Plan::enable_hfft): needs
    // the host to know f is real (host buffers are scanned, device buffers
    // checked with one reduction + sync)
    bool hfft_ok = false;
    DevBuf<int> imag_flag;
    StageTimer tm;
    // Every entry point holds `mu` for its whole call (host copies included),
    // so calls from several host threads are serialised (conv_operator.hpp:33-36:
    // apply is const and thread-safe). The device work of successive calls
    // shares this operator's scratch; `done` (recorded after each call's work)
    // orders it when consecutive calls use different streams.
    std::recursive_mutex mu;
    cudaEvent_t done = nullptr;
    cudaStream_t last_stream = nullptr;
    bool have_last = false;

    // Procedural ring nodes (sbd_op_options::procedural_rings; SURVEY 8f item
    // 3): the ring table and the node ids in the three orders the xi-side
    // kernels run in; the per-node arrays are then released and rebuilt by
    // ensure_node_arrays() for the paths that still read them.
    bool procedural = false;      // the xi-side kernels regenerate the nodes
    bool nodes_released = false;  // ... and the per-node arrays are not resident
    DevBuf<RingRow> ring_rows;
    DevBuf<uint32_t> id_sorted;   // canonical (fwd_out point) order
    DevBuf<uint32_t> id_z;        // fwd_in output (interpolation) order, bit 31 = halved under the split
    NodeGen node_gen(const uint32_t* ids) const {
        NodeGen g;
        g.id = ids;
        g.rings = ring_rows.p;
        g.ox = fwd_in->ax;
        g.oy = fwd_in->ay;
        g.osgn = (double)fwd_in->sign;
        g.ocxy = fwd_in->out_cxy();
        g.px = fwd_out->ax;
        g.py = fwd_out->ay;
        g.pbeta = fwd_out->beta;
        return g;
    }

    // Ring table and per-node ids (file order) when every ring of the file is
    // M equal-weight nodes rho (cos, sin)(2 pi j / M) -- what
    // build_ring_quadrature (ring_quadrature.cpp:51-66) writes: checked here on
    // the weights and sizes, and on the device against the file's coordinates.
    bool ring_table(std::vector<RingRow>& rows, std::vector<uint32_t>& ids) const {
        const uint64_t nx = d.n_xi();
        const size_t nr = d.ring_offsets.size() < 2 ? 0 : d.ring_offsets.size() - 1;
        if (!nx || !nr || nr >= (1u << (31 - kRingJBits)) || d.ring_offsets.front() != 0 ||
            (uint64_t)d.ring_offsets.back() != nx)
            return false;
        rows.resize(nr);
        ids.resize(nx);
        for (size_t r = 0; r < nr; ++r) {
            const uint64_t a = (uint64_t)d.ring_offsets[r], b = (uint64_t)d.ring_offsets[r + 1];
            if (b <= a || b - a >= (1ull << kRingJBits)) return false;
            const uint64_t m = b - a;
            // node 0 sits at angle 0: (rho, 0) exactly
            if (d.freqs[2 * a + 1] != 0.0 || !(d.freqs[2 * a] >= 0.0)) return false;
            rows[r].rho = d.freqs[2 * a];
            rows[r].two_over_m = 2.0 / (double)m;
            rows[r].wre = d.weights[2 * a];
            rows[r].wim = d.weights[2 * a + 1];
            for (uint64_t j = 0; j < m; ++j) {
                if (d.weights[2 * (a + j)] != rows[r].wre || d.weights[2 * (a + j) + 1] != rows[r].wim) return false;
                ids[a + j] = (uint32_t)(r << kRingJBits) | (uint32_t)j;
            }
        }
        return true;
    }

    // Rebuild the per-node arrays a procedural operator released (adjoint,
    // slab and unfused paths read them). Same device functions as the kernels.
    void ensure_node_arrays(cudaStream_t st) {
        if (!nodes_released) return;
        const uint64_t nx = d.n_xi();
        const NodeGen gs = node_gen(id_sorted.p), gz = node_gen(id_z.p);
        fwd_out->t.alloc(nx);
        fwd_out->pre.alloc(nx);
        launch_ring_point_arrays(gs, nx, fwd_out->t.p, fwd_out->pre.p, st);
        fwd_in->s.alloc(nx);
        fwd_in->post.alloc(nx);
        kappa.alloc(nx);
        if (herm_ok) kappa_h.alloc(nx);
        launch_ring_output_arrays(gz, nx, fwd_in->s.p, fwd_in->post.p, kappa.p, herm_ok ? kappa_h.p : nullptr, st);
        w_sorted.alloc(nx);
        launch_ring_nodes(id_sorted.p, nx, ring_rows.p, nullptr, w_sorted.p, st);
        w_in.alloc(nx);
        launch_ring_nodes(id_z.p, nx, ring_rows.p, nullptr, w_in.p, st);
        if (fwd_out->hrole == 2 && fwd_out->n0_pts) {
            // mirror images in their tile order: hv_t[k] = mirror(t[hv_src[k]])
            DevBuf<double2> m(fwd_out->n0_pts);
            launch_mirror_points(fwd_out->t.p, fwd_out->n0_pts, fwd_out->ax.n, fwd_out->ay.n, fwd_out->w, m.p, st);
            fwd_out->hv_t.alloc(fwd_out->n0_pts);
            launch_gather(m.p, fwd_out->hv_src.p, fwd_out->hv_t.p, fwd_out->n0_pts, st);
            ck(cudaStreamSynchronize(st), "node arrays");
        }
        ck(cudaStreamSynchronize(st), "node arrays");
        nodes_released = false;
        if (opt.verbose) std::fprintf(stderr, "[sbd] procedural rings: per-node arrays rebuilt\n");
    }

    // After the plans, the fused arrays and the half split exist: hand the ids
    // to the plans and drop the per-node arrays the forward path no longer reads.
    void enable_procedural(const std::vector<uint32_t>& ids_file, const std::vector<uint64_t>& halve) {
        const uint64_t nx = d.n_xi();
        if (!fused || !fwd_in->n_out_tiles || fwd_out->opts.spread_kernel != 0 || !fwd_out->rl1_s.n) {
            if (opt.verbose) std::fprintf(stderr, "[sbd] procedural rings off: needs the fused staged path\n");
            return;
        }
        std::vector<uint32_t> hs(nx);
        for (uint64_t i = 0; i < nx; ++i) hs[i] = ids_file[perm_xi[i]];
        id_sorted.upload(hs.data(), nx, stream);
        // fwd_in's output order: position v holds canonical node perm_s[v]
        std::vector<uint32_t> ps(nx);
        if (fwd_in->perm_s.n)
            ck(cudaMemcpyAsync(ps.data(), fwd_in->perm_s.p, nx * 4, cudaMemcpyDeviceToHost, stream), "perm");
        else
            for (uint64_t i = 0; i < nx; ++i) ps[i] = (uint32_t)i;
        ck(cudaStreamSynchronize(stream), "perm");
        std::vector<uint32_t> hz(nx);
        for (uint64_t v = 0; v < nx; ++v) hz[v] = hs[ps[v]];
        if (herm_ok && !halve.empty()) {
            std::vector<uint32_t> inv_xi(nx), pos_of(nx);
            for (uint64_t i = 0; i < nx; ++i) inv_xi[perm_xi[i]] = (uint32_t)i;
            for (uint64_t v = 0; v < nx; ++v) pos_of[ps[v]] = (uint32_t)v;
            for (uint64_t f : halve) hz[pos_of[inv_xi[f]]] |= kRingHalve;
        }
        id_z.upload(hz.data(), nx, stream);
        ck(cudaStreamSynchronize(stream), "node ids");
        fwd_out->gen_pts = node_gen(id_sorted.p);
        fwd_in->gen_out = node_gen(id_z.p);
        procedural = true;
        // release: the nodes as fwd_out's points and fwd_in's outputs, the
        // mirror images, omega-hat and kappa in both orders
        fwd_out->t = DevBuf<double2>();
        fwd_out->pre = DevBuf<double2>();
        fwd_out->pts = DevBuf<double2>();
        fwd_out->hv_t = DevBuf<double2>();
        fwd_in->s = DevBuf<double2>();
        fwd_in->post = DevBuf<double2>();
        fwd_in->frq = DevBuf<double2>();
        kappa = DevBuf<double2>();
        kappa_h = DevBuf<double2>();
        w_sorted = DevBuf<double2>();
        w_in = DevBuf<double2>();
        nodes_released = true;
        if (opt.verbose)
            std::fprintf(stderr, "[sbd] procedural rings on: %zu rings, per-node arrays released\n",
                         (size_t)ring_rows.n);
    }

    sbd_op() { sbd_op_options_default(&opt); }
    ~sbd_op() {
        for (Slot& sl : slot)
            for (cudaEvent_t e : {sl.h2d, sl.comp, sl.d2h})
                if (e) cudaEventDestroy(e);
        if (cp_in) cudaStreamDestroy(cp_in);
        if (cp_out) cudaStreamDestroy(cp_out);
        if (done) cudaEventDestroy(done);
        if (stream) cudaStreamDestroy(stream);
    }

    static bool capturing(cudaStream_t st) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
    }
    // before enqueueing a call's work on st: wait for the previous call's work
    // if it went to another stream
    void order_begin(cudaStream_t st) {
        if (have_last && last_stream != st && done && !capturing(st))
            ck(cudaStreamWaitEvent(st, done, 0), "operator order");
    }
    void order_end(cudaStream_t st) {
        if (capturing(st)) return;  // inside a graph capture the stream order is the graph's
        if (!done) ck(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "operator event");
        ck(cudaEventRecord(done, st), "operator order");
        last_stream = st;
        have_last = true;
    }

    // CompressedOperator::Impl::build_forward_plans (conv_operator.cpp:162-167)
    // plus the device upload.
    void build() {
        DeviceGuard g(device);
        ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
        tm.stream = stream;
        NufftOpts o;
        o.tol = d.nufft_tol;
        o.direct_threshold = d.direct_threshold;
        o.max_grid_bytes = d.max_grid_bytes;
        o.radix = opt.radix_first_pass < 0 ? -1 : (opt.radix_first_pass ? 1 : 0);
        o.spread_kernel = opt.spread_kernel;
        o.interp_kernel = opt.interp_kernel;
        const double* tgt = d.single ? d.src.data() : d.tgt.data();
        std::vector<uint8_t> tag;
        std::vector<uint64_t> halve;
        const bool split = herm_pairs(tag, halve);
        // procedural rings: the nodes both plans are built from are generated
        // on the device (file order) and must agree with the file's to rounding
        std::vector<uint32_t> ids_file;
        DevBuf<double2> xi_gen;
        bool proc = false;
        if (opt.procedural_rings) {
            std::vector<RingRow> rows;
            if (ring_table(rows, ids_file)) {
                const uint64_t nx = d.n_xi();
                ring_rows.upload(rows.data(), rows.size(), stream);
                DevBuf<uint32_t> idf;
                idf.upload(ids_file.data(), nx, stream);
                DevBuf<double2> xi_file;
                xi_file.upload(reinterpret_cast<const double2*>(d.freqs.data()), nx, stream);
                xi_gen.alloc(nx);
                launch_ring_nodes(idf.p, nx, ring_rows.p, xi_gen.p, nullptr, stream);
                const double dev = node_deviation(xi_file.p, xi_gen.p, nx, stream);
                proc = dev <= 1e-13;
                if (opt.verbose)
                    std::fprintf(stderr, "[sbd] procedural rings: generated nodes within %.2e of the file's\n", dev);
            } else if (opt.verbose) {
                std::fprintf(stderr, "[sbd] procedural rings off: the file's nodes are not equal-weight rings\n");
            }
        }
        // fwd_out = Plan(xi, tgt, +): xi take this plan's sorted order.
        fwd_out = std::make_unique<Plan>(d.freqs.data(), d.n_xi(), tgt, d.n_tgt(), +1, o, device,
                                         true, true, stream, split ? tag.data() : nullptr, nullptr,
                                         proc ? xi_gen.p : nullptr);
        perm_xi = fwd_out->adopt_point_order(stream);
        std::vector<double> xi_sorted(2 * d.n_xi()), w_host(2 * d.n_xi());
        for (uint64_t i = 0; i < d.n_xi(); ++i) {
            const uint32_t j = perm_xi[i];
            xi_sorted[2 * i] = d.freqs[2 * j];
            xi_sorted[2 * i + 1] = d.freqs[2 * j + 1];
            w_host[2 * i] = d.weights[2 * j];
            w_host[2 * i + 1] = d.weights[2 * j + 1];
        }
        // fwd_in = Plan(src, xi, -): its outputs (the xi nodes, in the canonical
        // order above) get their own Z-order for the interpolation; its perm_s
        // maps back, so the spectrum is written in the canonical order.
        std::vector<uint8_t> tag_sorted;
        if (split) {
            tag_sorted.resize(d.n_xi());
            for (uint64_t i = 0; i < d.n_xi(); ++i) tag_sorted[i] = tag[perm_xi[i]];
        }
        DevBuf<double2> xi_gen_sorted;
        if (proc) {
            // the generated nodes in the canonical order
            DevBuf<uint32_t> pd;
            pd.upload(perm_xi.data(), d.n_xi(), stream);
            xi_gen_sorted.alloc(d.n_xi());
            launch_gather(xi_gen.p, pd.p, xi_gen_sorted.p, d.n_xi(), stream);
            ck(cudaStreamSynchronize(stream), "generated nodes");
        }
        fwd_in = std::make_unique<Plan>(d.src.data(), d.n_src(), xi_sorted.data(), d.n_xi(), -1, o,
                                        device, true, true, stream,
                                        nullptr, split ? tag_sorted.data() : nullptr, nullptr,
                                        proc ? xi_gen_sorted.p : nullptr);
        w_sorted.upload(reinterpret_cast<const double2*>(w_host.data()), d.n_xi(), stream);
        w_in.alloc(std::max<uint64_t>(d.n_xi(), 1));
        if (fwd_in->perm_s.n)
            launch_gather(w_sorted.p, fwd_in->perm_s.p, w_in.p, d.n_xi(), stream);
        else
            ck(cudaMemcpyAsync(w_in.p, w_sorted.p, d.n_xi() * 16, cudaMemcpyDeviceToDevice, stream), "w_in");
        ro.upload(d.row_offsets.data(), d.row_offsets.size(), stream);
        cols.upload(d.cols.data(), d.cols.size(), stream);
        vals.upload(reinterpret_cast<const double2*>(d.values.data()), d.nnz(), stream);
        fwd_in->ensure_work(work, stream);
        fwd_out->ensure_work(work, stream);
        spec.alloc(std::max<uint64_t>(d.n_xi(), 1));
        ck(cudaStreamSynchronize(stream), "operator upload");
        build_fused();
        if (split) build_half(halve);
        if (herm_ok) build_hfft();
        if (proc) enable_procedural(ids_file, halve);
    }

    void build_hfft() {
        if (!opt.hermitian_fft) return;
        if (!fwd_in->enable_hfft(1, stream)) return;
        if (!fwd_out->enable_hfft(2, stream)) {
            fwd_in->hrole = 0;
            return;
        }
        // the spread reads the mirror images' values as conjugates of their
        // partners (Plan::hv_src); check that the computed outputs of fwd_in are
        // exactly the tag-0 points of fwd_out
        const uint64_t nx = d.n_xi(), n0 = n_half;
        std::vector<uint32_t> ps(nx);
        if (fwd_in->perm_s.n)
            ck(cudaMemcpyAsync(ps.data(), fwd_in->perm_s.p, nx * 4, cudaMemcpyDeviceToHost, stream), "perm");
        else
            for (uint64_t i = 0; i < nx; ++i) ps[i] = (uint32_t)i;
        ck(cudaStreamSynchronize(stream), "perm");
        for (uint64_t v = 0; v < n0; ++v)
            if (ps[v] >= n0) return;  // tag-0 outputs must map to tag-0 nodes
        imag_flag.alloc(1);
        ck(cudaStreamSynchronize(stream), "hfft");
        hfft_ok = true;
        if (opt.verbose) std::fprintf(stderr, "[sbd] Hermitian FFT mode on\n");
    }

    // 1 if f (n entries, device) is real; one reduction and a stream sync
    int device_real(const double2* f, uint64_t n, cudaStream_t st) {
        if (!imag_flag.n) imag_flag.alloc(1);
        launch_any_imag(f, n, imag_flag.p, st);
        int any = 1;
        ck(cudaMemcpyAsync(&any, imag_flag.p, sizeof(int), cudaMemcpyDeviceToHost, st), "imag flag");
        ck(cudaStreamSynchronize(st), "imag flag");
        return any ? 0 : 1;
    }

    // Antipodal pairing of the ring quadrature (ring_quadrature.cpp:51-66: ring
    // p holds M_p (even) nodes at angles 2 pi j / M_p, so node j + M_p/2 is -xi_j
    // up to rounding; a one-node ring is the zero frequency). tag 0 = computed,
    // 1 = taken as the conjugate of its partner. A pair whose rounded
    // coordinates put the partner's stencil somewhere other than the mirror of
    // the node's (an axis node with an even width, say: the window is 1, not 0,
    // at its edge) is computed on both nodes instead. `halve` lists the tag-0
    // nodes that enter 2 Re(.) with weight 1/2 (self-conjugate nodes and both
    // nodes of such pairs). False when omega-hat is not real or the pairing
    // does not hold to 1e-12 relative.
    bool herm_pairs(std::vector<uint8_t>& tag, std::vector<uint64_t>& halve) const {
        if (!opt.real_input_split) return false;
        const uint64_t nx = d.n_xi();
        if (nx < 2 || d.ring_offsets.size() < 2 || d.ring_offsets.front() != 0 ||
            (uint64_t)d.ring_offsets.back() != nx)
            return false;
        for (uint64_t i = 0; i < nx; ++i)
            if (d.weights[2 * i + 1] != 0.0) return false;
        // stencil geometry of the two plans (Plan(src, xi, -), Plan(xi, tgt, +))
        const int w = width_for_tol(d.nufft_tol);
        const double* tgt = d.single ? d.src.data() : d.tgt.data();
        const double* xi = d.freqs.data();
        const Axis inx = plan_axis(d.src.data(), d.n_src(), xi, nx, 0, -1.0, w);
        const Axis iny = plan_axis(d.src.data(), d.n_src(), xi, nx, 1, -1.0, w);
        const Axis outx = plan_axis(xi, nx, tgt, d.n_tgt(), 0, 1.0, w);
        const Axis outy = plan_axis(xi, nx, tgt, d.n_tgt(), 1, 1.0, w);
        auto mirrored = [&](uint64_t j, uint64_t q) {
            const double jx = xi[2 * j], jy = xi[2 * j + 1], qx = xi[2 * q], qy = xi[2 * q + 1];
            const bool in_ok =
                stencil_start_output(inx, qx, -1.0, w) == -(stencil_start_output(inx, jx, -1.0, w) + w - 1) &&
                stencil_start_output(iny, qy, -1.0, w) == -(stencil_start_output(iny, jy, -1.0, w) + w - 1);
            const bool out_ok =
                stencil_start_point(outx, qx, w) == outx.n - (stencil_start_point(outx, jx, w) + w - 1) &&
                stencil_start_point(outy, qy, w) == outy.n - (stencil_start_point(outy, jy, w) + w - 1);
            return in_ok && out_ok;
        };
        tag.assign(nx, 0);
        halve.clear();
        for (size_t r = 0; r + 1 < d.ring_offsets.size(); ++r) {
            const uint64_t a = (uint64_t)d.ring_offsets[r], b = (uint64_t)d.ring_offsets[r + 1];
            const uint64_t m = b - a;
            if (m == 1) {
                if (xi[2 * a] != 0.0 || xi[2 * a + 1] != 0.0) return false;
                halve.push_back(a);
                continue;
            }
            if (m == 0 || (m & 1)) return false;
            for (uint64_t j = a; j < a + m / 2; ++j) {
                const uint64_t q = j + m / 2;
                const double px = xi[2 * j], py = xi[2 * j + 1];
                const double sx = px + xi[2 * q], sy = py + xi[2 * q + 1];
                const double mag = std::sqrt(px * px + py * py);
                if (std::sqrt(sx * sx + sy * sy) > 1e-12 * mag || d.weights[2 * j] != d.weights[2 * q])
                    return false;
                if (mirrored(j, q)) {
                    // compute the node with xi_y <= 0: the source-side NUFFT (sign -1)
                    // then reads mostly the stored, non-negative band columns
                    tag[xi[2 * j + 1] > 0.0 ? j : q] = 1;
                } else {
                    halve.push_back(j);
                    halve.push_back(q);
                }
            }
        }
        return true;
    }

    void build_half(const std::vector<uint64_t>& halve) {
        if (!fused || !fwd_out->tagged_pts || !fwd_in->tagged_out || fwd_out->n0_pts != fwd_in->n0_out) {
            if (opt.verbose)
                std::fprintf(stderr, "[sbd] half split off: fused %d tagged %d %d n0 %llu %llu\n", (int)fused,
                             (int)fwd_out->tagged_pts, (int)fwd_in->tagged_out,
                             (unsigned long long)fwd_out->n0_pts, (unsigned long long)fwd_in->n0_out);
            return;
        }
        const uint64_t nx = d.n_xi();
        n_half = fwd_out->n0_pts;
        kappa_h.alloc(nx);
        ck(cudaMemcpyAsync(kappa_h.p, kappa.p, nx * 16, cudaMemcpyDeviceToDevice, stream), "kappa_h");
        if (!halve.empty()) {
            // position of each halved node in fwd_in's output order
            std::vector<uint32_t> inv_xi(nx);
            for (uint64_t i = 0; i < nx; ++i) inv_xi[perm_xi[i]] = (uint32_t)i;
            std::vector<uint32_t> pos_of(nx);
            if (fwd_in->perm_s.n) {
                std::vector<uint32_t> ps(nx);
                ck(cudaMemcpyAsync(ps.data(), fwd_in->perm_s.p, nx * 4, cudaMemcpyDeviceToHost, stream), "perm");
                ck(cudaStreamSynchronize(stream), "perm");
                for (uint64_t i = 0; i < nx; ++i) pos_of[ps[i]] = (uint32_t)i;
            } else {
                for (uint64_t i = 0; i < nx; ++i) pos_of[i] = (uint32_t)i;
            }
            std::vector<double2> kh(nx);
            ck(cudaMemcpyAsync(kh.data(), kappa_h.p, nx * 16, cudaMemcpyDeviceToHost, stream), "kappa_h");
            ck(cudaStreamSynchronize(stream), "kappa_h");
            for (uint64_t f : halve) {
                double2& v = kh[pos_of[inv_xi[f]]];
                v.x *= 0.5;
                v.y *= 0.5;
            }
            ck(cudaMemcpyAsync(kappa_h.p, kh.data(), nx * 16, cudaMemcpyHostToDevice, stream), "kappa_h");
        }
        if (opt.verbose)
            std::fprintf(stderr, "[sbd] half split: %zu nodes at weight 1/2\n", halve.size());
        herm_flag.alloc(1);
        ck(cudaStreamSynchronize(stream), "half split");
        herm_ok = true;
        if (opt.verbose)
            std::fprintf(stderr, "[sbd] real-input half split: %llu of %llu xi nodes\n",
                         (unsigned long long)n_half, (unsigned long long)nx);
    }

    void build_fused() {
        fused = fwd_in->pruned && fwd_out->pruned && fwd_in->perm_t.n == d.n_src() &&
                fwd_out->perm_s.n == d.n_tgt() && opt.fused;
        if (!fused) return;
        const uint64_t ns = d.n_src(), nt = d.n_tgt(), nx = d.n_xi();
        // kappa = w_sorted * pre_out (conv_operator.cpp:305 then nufft.cpp:233)
        {
            DevBuf<double2> kc(nx);  // canonical order, then fwd_in's output order
            ck(cudaMemcpyAsync(kc.p, w_sorted.p, nx * 16, cudaMemcpyDeviceToDevice, stream), "kappa");
            launch_mul(kc.p, fwd_out->pre.p, nx, stream);
            kappa.alloc(nx);
            if (fwd_in->perm_s.n)
                launch_gather(kc.p, fwd_in->perm_s.p, kappa.p, nx, stream);
            else
                ck(cudaMemcpyAsync(kappa.p, kc.p, nx * 16, cudaMemcpyDeviceToDevice, stream), "kappa");
            ck(cudaStreamSynchronize(stream), "kappa");
        }
        f_sorted.alloc(ns);
        qs.alloc(nt);
        // D' rows in target-sorted order, columns renumbered to source-sorted positions
        std::vector<uint32_t> ps(ns), pt(nt), inv(ns);
        ck(cudaMemcpyAsync(ps.data(), fwd_in->perm_t.p, ns * 4, cudaMemcpyDeviceToHost, stream), "perm");
        ck(cudaMemcpyAsync(pt.data(), fwd_out->perm_s.p, nt * 4, cudaMemcpyDeviceToHost, stream), "perm");
        ck(cudaStreamSynchronize(stream), "perm");
        for (uint64_t i = 0; i < ns; ++i) inv[ps[i]] = (uint32_t)i;
        std::vector<uint64_t> ro2(nt + 1, 0);
        for (uint64_t r = 0; r < nt; ++r) ro2[r + 1] = ro2[r] + (d.row_offsets[pt[r] + 1] - d.row_offsets[pt[r]]);
        std::vector<uint32_t> c2(d.nnz());
        std::vector<double> v2(2 * d.nnz());
#pragma omp parallel for schedule(static, 4096)
        for (int64_t r = 0; r < (int64_t)nt; ++r) {
            const uint64_t a = d.row_offsets[pt[r]], b = d.row_offsets[pt[r] + 1];
            uint64_t o = ro2[r];
            for (uint64_t i = a; i < b; ++i, ++o) {
                c2[o] = inv[d.cols[i]];
                v2[2 * o] = d.values[2 * i];
                v2[2 * o + 1] = d.values[2 * i + 1];
            }
        }
        ro_s.upload(ro2.data(), nt + 1, stream);
        cols_s.upload(c2.data(), c2.size(), stream);
        // D exactly real: only the real values; else both (the real copy is
        // used for real f when omega-hat is real, i.e. the half split applies)
        bool dreal = true;
        for (uint64_t i = 0; i < d.nnz() && dreal; ++i) dreal = v2[2 * i + 1] == 0.0;
        bool wreal = true;
        for (uint64_t i = 0; i < d.n_xi() && wreal; ++i) wreal = d.weights[2 * i + 1] == 0.0;
        if (dreal || wreal) {
            std::vector<double> vr(d.nnz());
            for (uint64_t i = 0; i < d.nnz(); ++i) vr[i] = v2[2 * i];
            vals_sr.upload(vr.data(), d.nnz(), stream);
        }
        if (!dreal) vals_s.upload(reinterpret_cast<const double2*>(v2.data()), d.nnz(), stream);
        ck(cudaStreamSynchronize(stream), "fused upload");
    }

    // conv_operator.cpp:301-309 on device buffers, one right-hand side.
    // real_hint: 1 = f is real (the Hermitian-FFT mode and the Re(D) pass
    // apply), 0 = complex, -1 = unknown. Never a host round trip: the half
    // split's device flag (cleared by the input gather when f has an imaginary
    // part) covers the unknown case.

    // Batched right-hand sides: D f for all columns in one
    // pass over D (k_spmm: the values and columns are read once for up to 8
    // right-hand sides), then the far field per column with qs_pre as addend.
    DevBuf<double2> fs_all, qs_all;
    void apply_batch(const double2* f, double2* q, int nrhs, cudaStream_t st, const int* real_hint) {
        const uint64_t ns = d.n_src(), nt = d.n_tgt();
        std::vector<int> real(nrhs);
        for (int r = 0; r < nrhs; ++r) real[r] = herm_ok && real_hint && real_hint[r] == 1 ? 1 : 0;
        if (fs_all.n < ns * nrhs) fs_all.alloc(ns * nrhs);
        if (qs_all.n < nt * nrhs) qs_all.alloc(nt * nrhs);
        for (int r = 0; r < nrhs; ++r)
            launch_gather(f + (size_t)r * ns, fwd_in->perm_t.p, fs_all.p + (size_t)r * ns, ns, st);
        if (tm.on) tm.start("spmv");
        for (int pass = 0; pass < 2; ++pass) {  // real columns (Re(D) when kept), then the others
            const bool rd = pass == 0 && vals_sr.n;
            SpmmCols cs;
            auto flush = [&]() {
                if (!cs.n) return;
                launch_spmm(nt, ro_s.p, cols_s.p, vals_s.p, rd || !vals_s.n ? vals_sr.p : nullptr, fs_all.p, ns,
                            qs_all.p, nt, cs, st);
                cs.n = 0;
            };
            for (int r = 0; r < nrhs; ++r) {
                const bool mine = pass == 0 ? (real[r] && vals_sr.n) : !(real[r] && vals_sr.n);
                if (!mine) continue;
                cs.idx[cs.n++] = r;
                if (cs.n == kSpmmMax) flush();
            }
            flush();
        }
        if (tm.on) tm.stop();
        for (int r = 0; r < nrhs; ++r)
            apply_one(f + (size_t)r * ns, q + (size_t)r * nt, st, real_hint ? real_hint[r] : -1,
                      qs_all.p + (size_t)r * nt);
    }

    void apply_one(const double2* f, double2* q, cudaStream_t st, int real_hint = -1,
                   const double2* qs_pre = nullptr) {
        if (fused) {
            HermArgs hin, hout;
            const bool real_f = herm_ok && real_hint == 1;
            const bool hfft_now = hfft_ok && real_f;
            if (herm_ok) {
                ck(cudaMemsetAsync(herm_flag.p, 1, sizeof(int), st), "half flag");
                hin.flag = hout.flag = herm_flag.p;
                hin.n = n_half;
                hin.mult = kappa_h.p;
                hin.clear = true;
                hout.n = ~0ull;
                hout.two_re = true;
                if (real_f) {
                    if (!f_sorted_re.n) f_sorted_re.alloc(d.n_src());
                    hin.raw_re = f_sorted_re.p;
                }
                if (hfft_now) {
                    hin.hfft = hout.hfft = true;
                    hin.hcols = fwd_in->hcols;

                }
            }
            // spectrum_b = NUFFT-(f) * w * pre_out, with f_sorted kept for the CSR pass
            fwd_in->apply_pruned(f, false, f_sorted.p, spec.p, kappa.p, nullptr, work, st, &tm,
                                 "spread_src", "fft_in", "interp_xi", 0, ~0ull, 0, ~0ull,
                                 herm_ok ? &hin : nullptr);
            // (a second stream for the CSR pass beside the xi spread and the
            // second FFT was measured: no gain on config 4 -- the overlapped
            // kernels slow down by the CSR pass's time)
            if (!qs_pre) {  // else D f was formed by the batched pass
                if (tm.on) tm.start("spmv");
                spmv_sorted(0, d.n_tgt(), st, real_f);
                if (tm.on) tm.stop();
            }
            // q = NUFFT+(spectrum) + D f, scattered to the caller's target order
            fwd_out->apply_pruned(spec.p, true, nullptr, q, nullptr, qs_pre ? qs_pre : qs.p, work, st, &tm,
                                  "spread_xi", "fft_out", "interp_tgt", 0, ~0ull, 0, ~0ull,
                                  herm_ok ? &hout : nullptr);
            return;
        }
        fwd_in->apply(f, spec.p, work, st, &tm, w_in.p, "spread_src", "fft_in", "interp_xi");
        fwd_out->apply(spec.p, q, work, st, &tm, nullptr, "spread_xi", "fft_out", "interp_tgt");
        if (tm.on) tm.start("spmv");
        launch_spmv(d.n_tgt(), ro.p, cols.p, vals.p, f, q, st);
        if (tm.on) tm.stop();
    }

    // Sharded forward half (multi-GPU): the kappa-weighted
    // spectrum of the sources in sorted range [lo, hi). Summing it over a
    // partition of the sources gives exactly the single-device spectrum.
    // The real-input half split applies to the sharded halves too: for a real
    // f only the computed half of the spectrum ([0, n_half) in this order) is
    // formed, reduced and read. shard_real keeps the decision for the
    // backward half (same f on every rank, so every rank decides alike).
    int shard_real = 0;

    uint64_t spectrum_length(const double2* f, cudaStream_t st) {
        shard_real = herm_ok ? device_real(f, d.n_src(), st) : 0;
        return shard_real ? n_half : d.n_xi();
    }

    HermArgs shard_herm(bool forward, cudaStream_t st) {
        HermArgs h;
        ck(cudaMemsetAsync(herm_flag.p, 1, sizeof(int), st), "half flag");
        h.flag = herm_flag.p;
        h.hfft = hfft_ok;
        if (forward) {
            h.n = n_half;
            h.mult = kappa_h.p;
            h.clear = true;
            if (hfft_ok) h.hcols = fwd_in->hcols;  // conjugates are rebuilt after the reduction
        } else {
            h.n = ~0ull;
            h.two_re = true;

        }
        return h;
    }

    void forward_spectrum(const double2* f, uint64_t lo, uint64_t hi, double2* spec_out,
                          cudaStream_t st) {
        if (!fused) throw Error(SBD_ERR_RUNTIME, "sharded apply needs both NUFFTs on the gridded path");
        // shard_real: decided by the spectrum_length call for this f
        HermArgs h;
        if (shard_real) h = shard_herm(true, st);
        fwd_in->apply_pruned(f, false, f_sorted.p, spec_out, kappa.p, nullptr, work, st, &tm,
                             "spread_src", "fft_in", "interp_xi", lo, hi, 0, ~0ull, shard_real ? &h : nullptr);
    }

    // Sharded backward half: q at the targets in sorted range [lo, hi)
    // (written at their caller indices) = NUFFT+(spectrum) + D f on those rows.
    void backward_targets(const double2* spec_in, const double2* f, uint64_t lo, uint64_t hi,
                          double2* q, cudaStream_t st) {
        if (!fused) throw Error(SBD_ERR_RUNTIME, "sharded apply needs both NUFFTs on the gridded path");
        hi = std::min<uint64_t>(hi, d.n_tgt());
        lo = std::min(lo, hi);
        if (shard_real && !f_sorted_re.n) f_sorted_re.alloc(d.n_src());
        launch_gather_mul(f, fwd_in->perm_t.p, fwd_in->pre.p, work.bbuf.p, f_sorted.p, d.n_src(), st, 0, 0, nullptr,
                          shard_real ? f_sorted_re.p : nullptr);
        if (tm.on) tm.start("spmv");
        spmv_sorted(lo, hi, st, shard_real);
        if (tm.on) tm.stop();
        HermArgs h;
        if (shard_real) {
            h = shard_herm(false, st);
        }
        fwd_out->apply_pruned(spec_in, true, nullptr, q, nullptr, qs.p, work, st, &tm, "spread_xi",
                              "fft_out", "interp_tgt", 0, ~0ull, lo, hi, shard_real ? &h : nullptr);
    }

    // D^H as its own CSR (values conjugated), built on the first adjoint: the
    // near-field part of the adjoint becomes a gather SpMV like the forward
    // one instead of a scatter with fp64 atomics (point_cloud.cpp:125-132).
    // On the fused path it is renumbered like D': rows = sources in fwd_in's
    // sorted order, columns = targets in fwd_out's sorted order (entries
    // sorted), so its u gathers are spatially local, and D^H u enters the
    // source-side gather as its addend.
    DevBuf<uint64_t> roT;
    DevBuf<uint32_t> colsT;
    DevBuf<double2> valsT, u_sorted, qsT;
    bool dT_ready = false;
    void build_adjoint_csr(cudaStream_t st) {
        const uint64_t ns = d.n_src(), nt = d.n_tgt(), nnz = d.nnz();
        std::vector<uint64_t> r(ns + 1, 0);
        for (uint64_t i = 0; i < nnz; ++i) ++r[d.cols[i] + 1];
        for (uint64_t c = 0; c < ns; ++c) r[c + 1] += r[c];
        std::vector<uint64_t> pos(r.begin(), r.end() - 1);
        std::vector<uint32_t> c2(nnz);
        std::vector<double> v2(2 * nnz);
        for (uint64_t t = 0; t < nt; ++t)
            for (uint64_t i = d.row_offsets[t]; i < d.row_offsets[t + 1]; ++i) {
                const uint64_t o = pos[d.cols[i]]++;
                c2[o] = (uint32_t)t;
                v2[2 * o] = d.values[2 * i];
                v2[2 * o + 1] = -d.values[2 * i + 1];
            }
        if (fused) {
            std::vector<uint32_t> ps(ns), pt(nt), inv_t(nt);
            ck(cudaMemcpyAsync(ps.data(), fwd_in->perm_t.p, ns * 4, cudaMemcpyDeviceToHost, st), "perm");
            ck(cudaMemcpyAsync(pt.data(), fwd_out->perm_s.p, nt * 4, cudaMemcpyDeviceToHost, st), "perm");
            ck(cudaStreamSynchronize(st), "perm");
            for (uint64_t j = 0; j < nt; ++j) inv_t[pt[j]] = (uint32_t)j;
            std::vector<uint64_t> r2(ns + 1, 0);
            for (uint64_t k = 0; k < ns; ++k) r2[k + 1] = r2[k] + (r[ps[k] + 1] - r[ps[k]]);
            std::vector<uint32_t> c3(nnz);
            std::vector<double> v3(2 * nnz);
#pragma omp parallel for schedule(dynamic, 4096)
            for (int64_t k = 0; k < (int64_t)ns; ++k) {
                const uint64_t a = r[ps[k]], e = r[ps[k] + 1], o = r2[k];
                std::vector<std::pair<uint32_t, uint64_t>> row;
                row.reserve(e - a);
                for (uint64_t i = a; i < e; ++i) row.emplace_back(inv_t[c2[i]], i);
                std::sort(row.begin(), row.end());
                for (uint64_t q = 0; q < row.size(); ++q) {
                    c3[o + q] = row[q].first;
                    v3[2 * (o + q)] = v2[2 * row[q].second];
                    v3[2 * (o + q) + 1] = v2[2 * row[q].second + 1];
                }
            }
            r.swap(r2);
            c2.swap(c3);
            v2.swap(v3);
            u_sorted.alloc(std::max<uint64_t>(nt, 1));
            qsT.alloc(std::max<uint64_t>(ns, 1));
        }
        roT.upload(r.data(), ns + 1, st);
        colsT.upload(c2.data(), nnz, st);
        valsT.upload(reinterpret_cast<const double2*>(v2.data()), nnz, st);
        ck(cudaStreamSynchronize(st), "adjoint CSR");
        dT_ready = true;
    }

    // conv_operator.cpp:311-324: A^H u = conj(fwd_in^T (w . fwd_out^T conj(u))) + D^H u
    void apply_adjoint_one(const double2* u, double2* q, cudaStream_t st) {
        ensure_node_arrays(st);
        if (!dT_ready) build_adjoint_csr(st);
        if (fused) {
            if (tm.on) tm.start("spmv_adjoint");
            launch_gather(u, fwd_out->perm_s.p, u_sorted.p, d.n_tgt(), st);
            launch_spmv_vec(d.n_src(), roT.p, colsT.p, valsT.p, u_sorted.p, qsT.p, st);
            if (tm.on) tm.stop();
            fwd_out->apply_transpose(u, spec.p, work, st, &tm, w_sorted.p, /*conj_in=*/1, 0);
            fwd_in->apply_transpose(spec.p, q, work, st, &tm, nullptr, 0, /*conj_out=*/1, qsT.p);
            return;
        }
        fwd_out->apply_transpose(u, spec.p, work, st, &tm, w_sorted.p, /*conj_in=*/1, 0);
        fwd_in->apply_transpose(spec.p, q, work, st, &tm, nullptr, 0, /*conj_out=*/1);
        if (tm.on) tm.start("spmv_adjoint");
        launch_spmv_vec(d.n_src(), roT.p, colsT.p, valsT.p, u, q, st, /*accumulate=*/true);
        if (tm.on) tm.stop();
    }

    size_t device_bytes() const {
        return fwd_in->device_bytes() + fwd_out->device_bytes() + w_sorted.bytes() + w_in.bytes() + ro.bytes() +
               ro_s.bytes() + cols_s.bytes() + vals_s.bytes() + vals_sr.bytes() + fs_all.bytes() + qs_all.bytes() + kappa.bytes() + f_sorted.bytes() +
               qs.bytes() + work.bbuf.bytes() +
               cols.bytes() + vals.bytes() + work.grid.bytes() + work.T.bytes() + work.band.bytes() +
               spec.bytes() + hf.bytes() + hq.bytes() + kappa_h.bytes() + roT.bytes() + colsT.bytes() +
               valsT.bytes() + u_sorted.bytes() + qsT.bytes() + id_sorted.bytes() + id_z.bytes() + ring_rows.bytes();
    }

    // conv_operator.cpp:338-353
    uint64_t ref_bytes() const {
        uint64_t b = 0;
        b += (d.n_src() + (d.single ? 0 : d.n_tgt())) * 16;
        b += d.n_xi() * 16 * 2;
        b += d.ring_offsets.size() * 4;
        b += d.row_offsets.size() * 8 + d.cols.size() * 4 + d.nnz() * 16;
        const uint64_t per = 32;
        if (fwd_in->fast) b += (d.n_src() + d.n_xi()) * per;
        if (fwd_out->fast) b += (d.n_xi() + d.n_tgt()) * per;
        return b;
    }
};
