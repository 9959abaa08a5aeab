// op.cpp -- the compressed operator on one B200 (reference CompressedOperator,
// /root/reference/proj/src/conv_operator.cpp) and the C ABI of
// include/sbd_b200.h.
//
// Layout on the device:
//   xi nodes are stored ONCE, sorted by the fwd_out spread tile; the spectrum
//   lives in that order between the two NUFFTs, and omega-hat is pre-permuted
//   to it, so the conv_operator.cpp:305 multiply is fused into the xi-side
//   interpolation. Sources/targets keep the caller's order at the boundary;
//   each plan carries its own tile permutation internally.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <fstream>
#include <mutex>

#include "../../include/sbd_b200.h"
#include "assemble_gpu.h"
#include "bessel_host.h"
#include "opdata.h"
#include "sbd_internal.h"

namespace sbdgpu {

namespace {
thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
} // namespace
thread_local bool g_verbose = false;

[[noreturn]] void throw_cuda(cudaError_t e, const char* what) {
    throw Error(SBD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
[[noreturn]] void throw_cufft(cufftResult r, const char* what) {
    throw Error(SBD_ERR_CUDA, std::string(what) + ": cuFFT error " + std::to_string((int)r));
}
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

template <typename T>
void wr(std::ostream& os, const T& v) {
    os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
void wrv(std::ostream& os, const std::vector<T>& v, size_t elem_per) {
    const uint64_t n = v.size() / elem_per;
    wr(os, n);
    os.write(reinterpret_cast<const char*>(v.data()), (std::streamsize)(v.size() * sizeof(T)));
}
template <typename T>
void rd(std::istream& is, T& v) {
    is.read(reinterpret_cast<char*>(&v), sizeof(T));
}
template <typename T>
void rdv(std::istream& is, std::vector<T>& v, size_t elem_per) {
    uint64_t n = 0;
    rd(is, n);
    if (!is || n > (uint64_t(1) << 40)) throw Error(SBD_ERR_RUNTIME, "load: truncated operator file");
    v.resize(n * elem_per);
    is.read(reinterpret_cast<char*>(v.data()), (std::streamsize)(v.size() * sizeof(T)));
}

const char kMagic[8] = {'S', 'B', 'D', 'O', 'P', 'v', '1', '\0'};

// CSR and ring invariants every kernel relies on (a foreign or corrupt file
// must fail here, before anything reaches the device): row_offsets starts at
// 0, never decreases and ends at nnz; every column is a source index;
// ring_offsets never decrease and stay within the node count.
void validate(const OpData& d, const std::string& path) {
    auto bad = [&](const char* what) {
        throw Error(SBD_ERR_RUNTIME, std::string("load: inconsistent operator file ") + path + " (" + what + ")");
    };
    const auto& ro = d.row_offsets;
    if (ro.empty() || ro.front() != 0 || ro.back() != d.cols.size()) bad("row offsets do not span the values");
    for (size_t i = 1; i < ro.size(); ++i)
        if (ro[i] < ro[i - 1]) bad("row offsets decrease");
    const uint64_t ns = d.n_src();
    for (uint32_t c : d.cols)
        if (c >= ns) bad("column index out of range");
    const auto& rg = d.ring_offsets;
    for (size_t i = 0; i < rg.size(); ++i)
        if (rg[i] < 0 || (uint64_t)rg[i] > d.n_xi() || (i && rg[i] < rg[i - 1])) bad("ring offsets");
}

// conv_operator.cpp:449-490
OpData read_sbdop(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw Error(SBD_ERR_RUNTIME, "load: cannot open " + path);
    char magic[8];
    is.read(magic, 8);
    if (!is || std::memcmp(magic, kMagic, 8) != 0)
        throw Error(SBD_ERR_RUNTIME, "load: not an operator file (bad magic)");
    OpData d;
    uint8_t single = 0;
    rd(is, d.kind);
    rd(is, d.k);
    rd(is, single);
    d.single = single != 0;
    rd(is, d.eps);
    rd(is, d.alpha);
    rd(is, d.a);
    rd(is, d.dmin);
    rd(is, d.dmax);
    rd(is, d.nufft_tol);
    rdv(is, d.src, 2);
    rd(is, d.src_diam);
    if (!d.single) {
        rdv(is, d.tgt, 2);
        rd(is, d.tgt_diam);
    }
    rdv(is, d.freqs, 2);
    rdv(is, d.weights, 2);
    rdv(is, d.ring_offsets, 1);
    rd(is, d.total_error_budget);
    rdv(is, d.row_offsets, 1);
    rdv(is, d.cols, 1);
    rdv(is, d.values, 2);
    SbdRecord& s = d.sbd;
    rd(is, s.a);
    rd(is, s.P);
    rd(is, s.constant_offset);
    rd(is, s.achieved_error);
    rd(is, s.radial_scale);
    rd(is, s.bc);
    rd(is, s.H);
    rdv(is, s.coeffs, 1);
    rdv(is, s.roots, 1);
    rdv(is, s.norm_constants, 1);
    if (!is) throw Error(SBD_ERR_RUNTIME, "load: truncated operator file " + path);
    if (d.weights.size() != d.freqs.size() || d.row_offsets.size() != d.n_tgt() + 1 ||
        d.values.size() != 2 * d.cols.size())
        throw Error(SBD_ERR_RUNTIME, "load: inconsistent operator file " + path);
    validate(d, path);
    return d;
}

// conv_operator.cpp:357-397
void write_sbdop(const OpData& d, const std::string& path) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw Error(SBD_ERR_RUNTIME, "save: cannot open " + path);
    os.write(kMagic, 8);
    wr(os, d.kind);
    wr(os, d.k);
    wr(os, (uint8_t)(d.single ? 1 : 0));
    wr(os, d.eps);
    wr(os, d.alpha);
    wr(os, d.a);
    wr(os, d.dmin);
    wr(os, d.dmax);
    wr(os, d.nufft_tol);
    wrv(os, d.src, 2);
    wr(os, d.src_diam);
    if (!d.single) {
        wrv(os, d.tgt, 2);
        wr(os, d.tgt_diam);
    }
    wrv(os, d.freqs, 2);
    wrv(os, d.weights, 2);
    wrv(os, d.ring_offsets, 1);
    wr(os, d.total_error_budget);
    wrv(os, d.row_offsets, 1);
    wrv(os, d.cols, 1);
    wrv(os, d.values, 2);
    const SbdRecord& s = d.sbd;
    wr(os, s.a);
    wr(os, s.P);
    wr(os, s.constant_offset);
    wr(os, s.achieved_error);
    wr(os, s.radial_scale);
    wr(os, s.bc);
    wr(os, s.H);
    wrv(os, s.coeffs, 1);
    wrv(os, s.roots, 1);
    wrv(os, s.norm_constants, 1);
    if (!os) throw Error(SBD_ERR_RUNTIME, "save: write failed for " + path);
}

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
    void spmv_sorted(uint64_t lo, uint64_t hi, cudaStream_t st, bool real_f = false) {
        if (vals_sr.n && (real_f || !vals_s.n))
            launch_spmv_vec_real(hi - lo, ro_s.p + lo, cols_s.p, vals_sr.p, f_sorted.p, qs.p + lo, st);
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
        // fwd_out = Plan(xi, tgt, +): xi take this plan's sorted order.
        fwd_out = std::make_unique<Plan>(d.freqs.data(), d.n_xi(), tgt, d.n_tgt(), +1, o, device,
                                         true, true, stream, split ? tag.data() : nullptr);
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
        fwd_in = std::make_unique<Plan>(d.src.data(), d.n_src(), xi_sorted.data(), d.n_xi(), -1, o,
                                        device, true, true, stream,
                                        nullptr, split ? tag_sorted.data() : nullptr);
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
        launch_gather_mul(f, fwd_in->perm_t.p, fwd_in->pre.p, work.bbuf.p, f_sorted.p, d.n_src(), st, 0, 0);
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
               valsT.bytes() + u_sorted.bytes() + qsT.bytes();
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

struct sbd_nufft {
    std::unique_ptr<Plan> plan;
    int device = 0;
    cudaStream_t stream = nullptr;
    FftWork work;
    DevBuf<double2> in, out;
    ~sbd_nufft() {
        if (stream) cudaStreamDestroy(stream);
    }
};

// ------------------------------------------------------------------ C ABI
namespace {
template <typename F>
int guarded(F&& f) {
    try {
        f();
        return SBD_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_err = "out of host memory";
        return SBD_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SBD_ERR_RUNTIME;
    }
}
} // namespace


extern "C" {

const char* sbd_last_error(void) { return g_err.c_str(); }
const char* sbd_version(void) { return "sbd_b200 0.1.0 (sm_100a)"; }
uint64_t sbd_kernel_launch_count(void) { return g_launches.load(); }

double sbd_bessel(int which, double x) {
    try {
        switch (which) {
            case 0: return bessel_j0(x);
            case 1: return bessel_j1(x);
            case 2: return bessel_y0(x);
            case 3: return bessel_y1(x);
        }
    } catch (const std::exception&) {
    }
    return std::nan("");
}

double sbd_window_fit_error(int w, double beta) {
    double err = -1.0;
    if (w < 4 || w > kMaxW) return err;
    fit_window(w, beta, &err);
    return err;
}

void sbd_assemble_options_default(sbd_assemble_options* o) {
    o->eps = 1e-6;
    o->alpha = 0.0;
    o->a_override = 0.0;
    o->small_k_factor = 0.5;
    o->nufft_direct_threshold = uint64_t(1) << 20;
    o->max_grid_bytes = uint64_t(4) << 30;
    o->device = 0;
    sbd_op_options_default(&o->pipeline);
}

void sbd_op_options_default(sbd_op_options* o) {
    o->real_input_split = 1;
    o->hermitian_fft = 1;
    o->radix_first_pass = -1;
    o->spread_kernel = 0;
    o->interp_kernel = 0;
    o->fused = 1;
    o->verbose = 0;
}

static void check_options(const sbd_op_options& o) {
    if (o.radix_first_pass < -1 || o.radix_first_pass > 1 || o.spread_kernel < 0 || o.spread_kernel > 3 ||
        o.interp_kernel < 0 || o.interp_kernel > 3)
        throw Error(SBD_ERR_INVALID_ARGUMENT, "options: value out of range");
}

int sbd_op_load(const char* path, int device, uint64_t max_grid_bytes, sbd_op** out) {
    return sbd_op_load_ex(path, device, max_grid_bytes, nullptr, out);
}

int sbd_op_load_ex(const char* path, int device, uint64_t max_grid_bytes, const sbd_op_options* options,
                   sbd_op** out) {
    return guarded([&] {
        if (!path || !out) throw Error(SBD_ERR_INVALID_ARGUMENT, "load: null argument");
        auto op = std::make_unique<sbd_op>();
        if (options) {
            check_options(*options);
            op->opt = *options;
        }
        op->d = read_sbdop(path);
        if (max_grid_bytes) op->d.max_grid_bytes = max_grid_bytes;
        op->device = device;
        op->build();
        *out = op.release();
    });
}

int sbd_op_assemble(int kind, double k, const double* src_xy, uint64_t n_src, const double* tgt_xy,
                    uint64_t n_tgt, const sbd_assemble_options* opts, sbd_op** out) {
    return guarded([&] {
        if (!out || (n_src && !src_xy)) throw Error(SBD_ERR_INVALID_ARGUMENT, "assemble: null argument");
        sbd_assemble_options o;
        sbd_assemble_options_default(&o);
        if (opts) o = *opts;
        check_options(o.pipeline);
        g_verbose = o.pipeline.verbose != 0;
        auto op = std::make_unique<sbd_op>();
        op->opt = o.pipeline;
        assemble_opdata(kind, k, src_xy, n_src, tgt_xy, n_tgt, o, op->d);
        op->d.direct_threshold = o.nufft_direct_threshold;
        op->d.max_grid_bytes = o.max_grid_bytes;
        op->device = o.device;
        op->build();
        *out = op.release();
    });
}

int sbd_op_save(const sbd_op* op, const char* path) {
    return guarded([&] {
        if (!op || !path) throw Error(SBD_ERR_INVALID_ARGUMENT, "save: null argument");
        write_sbdop(op->d, path);
    });
}

int sbd_op_destroy(sbd_op* op) {
    return guarded([&] {
        if (!op) return;
        DeviceGuard g(op->device);
        delete op;
    });
}

int sbd_op_info(const sbd_op* op, sbd_op_info_t* info) {
    return guarded([&] {
        if (!op || !info) throw Error(SBD_ERR_INVALID_ARGUMENT, "info: null argument");
        const OpData& d = op->d;
        std::memset(info, 0, sizeof(*info));
        info->n_src = d.n_src();
        info->n_tgt = d.n_tgt();
        info->n_xi = d.n_xi();
        info->nnz = d.nnz();
        info->single_cloud = d.single;
        info->kind = d.kind;
        info->k = d.k;
        info->eps = d.eps;
        info->alpha = d.alpha;
        info->a = d.a;
        info->delta_min = d.dmin;
        info->delta_max = d.dmax;
        info->nufft_tol = d.nufft_tol;
        info->P = d.sbd.P;
        const Plan& pi = *op->fwd_in;
        const Plan& po = *op->fwd_out;
        info->w = pi.fast ? pi.w : po.w;
        info->beta = pi.fast ? pi.beta : po.beta;
        info->fast_in = pi.fast;
        info->fast_out = po.fast;
        info->n1_in = pi.ax.n;
        info->n2_in = pi.ay.n;
        info->n1_out = po.ax.n;
        info->n2_out = po.ay.n;
        info->bytes = op->ref_bytes();
        info->device_bytes = op->device_bytes();
    });
}

int sbd_op_get(const sbd_op* op, int which, void* dst, uint64_t* count) {
    return guarded([&] {
        if (!op) throw Error(SBD_ERR_INVALID_ARGUMENT, "get: null operator");
        const OpData& d = op->d;
        const void* src = nullptr;
        uint64_t n = 0, esz = 8;
        const std::vector<double>& tgt = d.single ? d.src : d.tgt;
        switch (which) {
            case 0: src = d.src.data(); n = d.src.size(); break;
            case 1: src = tgt.data(); n = tgt.size(); break;
            case 2: src = d.freqs.data(); n = d.freqs.size(); break;
            case 3: src = d.weights.data(); n = d.weights.size(); break;
            case 4: src = d.row_offsets.data(); n = d.row_offsets.size(); break;
            case 5: src = d.cols.data(); n = d.cols.size(); esz = 4; break;
            case 6: src = d.values.data(); n = d.values.size(); break;
            case 7: src = d.ring_offsets.data(); n = d.ring_offsets.size(); esz = 4; break;
            case 8: src = d.sbd.coeffs.data(); n = d.sbd.coeffs.size(); break;
            case 9: src = d.sbd.roots.data(); n = d.sbd.roots.size(); break;
            case 10: src = d.sbd.norm_constants.data(); n = d.sbd.norm_constants.size(); break;
            default: throw Error(SBD_ERR_INVALID_ARGUMENT, "get: unknown array");
        }
        if (count) *count = n;
        if (dst && n) std::memcpy(dst, src, n * esz);
    });
}

static void apply_device_rhs(sbd_op* op, const double* d_f, double* d_q, int nrhs, cudaStream_t st,
                             const int* real_hint) {
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    op->tm.stream = st;
    op->order_begin(st);
    const auto* f = reinterpret_cast<const double2*>(d_f);
    auto* q = reinterpret_cast<double2*>(d_q);
    if (op->fused && nrhs > 1) {
        op->apply_batch(f, q, nrhs, st, real_hint);
    } else {
        for (int r = 0; r < nrhs; ++r)
            op->apply_one(f + (size_t)r * op->d.n_src(), q + (size_t)r * op->d.n_tgt(), st,
                          real_hint ? real_hint[r] : -1);
    }
    ck(cudaGetLastError(), "apply");
    op->order_end(st);
}

int sbd_op_apply_device(sbd_op* op, const double* d_f, double* d_q, int nrhs, void* stream) {
    return guarded([&] {
        if (!op || !d_f || !d_q || nrhs < 1) throw Error(SBD_ERR_INVALID_ARGUMENT, "apply: bad argument");
        apply_device_rhs(op, d_f, d_q, nrhs, (cudaStream_t)stream, nullptr);
    });
}

int sbd_op_apply_device_ex(sbd_op* op, const double* d_f, double* d_q, int nrhs, void* stream,
                           const int* f_is_real) {
    return guarded([&] {
        if (!op || !d_f || !d_q || nrhs < 1) throw Error(SBD_ERR_INVALID_ARGUMENT, "apply: bad argument");
        apply_device_rhs(op, d_f, d_q, nrhs, (cudaStream_t)stream, f_is_real);
    });
}

int sbd_op_apply_adjoint_device(sbd_op* op, const double* d_u, double* d_q, int nrhs,
                                void* stream) {
    return guarded([&] {
        if (!op || !d_u || !d_q || nrhs < 1) throw Error(SBD_ERR_INVALID_ARGUMENT, "apply_adjoint: bad argument");
        std::lock_guard<std::recursive_mutex> lk(op->mu);
        DeviceGuard g(op->device);
        cudaStream_t st = (cudaStream_t)stream;
        op->tm.stream = st;
        op->order_begin(st);
        const auto* u = reinterpret_cast<const double2*>(d_u);
        auto* q = reinterpret_cast<double2*>(d_q);
        for (int r = 0; r < nrhs; ++r)
            op->apply_adjoint_one(u + (size_t)r * op->d.n_tgt(), q + (size_t)r * op->d.n_src(), st);
        ck(cudaGetLastError(), "apply_adjoint");
        op->order_end(st);
    });
}

int sbd_op_shard_bounds(const sbd_op* op, int side, int nshards, uint64_t* bounds) {
    return guarded([&] {
        if (!op || !bounds || nshards < 1 || (side != 0 && side != 1))
            throw Error(SBD_ERR_INVALID_ARGUMENT, "shard_bounds: bad argument");
        const uint64_t n = side == 0 ? op->d.n_src() : op->d.n_tgt();
        for (int i = 0; i <= nshards; ++i) bounds[i] = n * (uint64_t)i / (uint64_t)nshards;
    });
}

int sbd_op_spectrum_length(sbd_op* op, const double* d_f, void* stream, uint64_t* n) {
    return guarded([&] {
        if (!op || !d_f || !n) throw Error(SBD_ERR_INVALID_ARGUMENT, "spectrum_length: null argument");
        std::lock_guard<std::recursive_mutex> lk(op->mu);
        DeviceGuard g(op->device);
        op->order_begin((cudaStream_t)stream);
        *n = op->spectrum_length(reinterpret_cast<const double2*>(d_f), (cudaStream_t)stream);
    });
}

int sbd_op_forward_spectrum(sbd_op* op, const double* d_f, uint64_t src_lo, uint64_t src_hi,
                            double* d_spec, void* stream) {
    return guarded([&] {
        if (!op || !d_f || !d_spec) throw Error(SBD_ERR_INVALID_ARGUMENT, "forward_spectrum: null argument");
        std::lock_guard<std::recursive_mutex> lk(op->mu);
        DeviceGuard g(op->device);
        op->tm.stream = (cudaStream_t)stream;
        op->order_begin((cudaStream_t)stream);
        op->forward_spectrum(reinterpret_cast<const double2*>(d_f), src_lo, src_hi,
                             reinterpret_cast<double2*>(d_spec), (cudaStream_t)stream);
        ck(cudaGetLastError(), "forward_spectrum");
        op->order_end((cudaStream_t)stream);
    });
}

int sbd_op_backward_targets(sbd_op* op, const double* d_spec, const double* d_f, uint64_t tgt_lo,
                            uint64_t tgt_hi, double* d_q, void* stream) {
    return guarded([&] {
        if (!op || !d_spec || !d_f || !d_q) throw Error(SBD_ERR_INVALID_ARGUMENT, "backward_targets: null argument");
        std::lock_guard<std::recursive_mutex> lk(op->mu);
        DeviceGuard g(op->device);
        op->tm.stream = (cudaStream_t)stream;
        op->order_begin((cudaStream_t)stream);
        op->backward_targets(reinterpret_cast<const double2*>(d_spec), reinterpret_cast<const double2*>(d_f),
                             tgt_lo, tgt_hi, reinterpret_cast<double2*>(d_q), (cudaStream_t)stream);
        ck(cudaGetLastError(), "backward_targets");
        op->order_end((cudaStream_t)stream);
    });
}

static int host_apply(sbd_op* op, const double* in, double* out, int nrhs, bool adjoint) {
    return guarded([&] {
        if (!op || !in || !out || nrhs < 1) throw Error(SBD_ERR_INVALID_ARGUMENT, "apply: bad argument");
        // the lock spans the staging copies, the apply and the copy back: the
        // staging buffers hf / hq are the operator's (concurrent
        // host calls must not interleave their copies)
        std::lock_guard<std::recursive_mutex> lk(op->mu);
        DeviceGuard g(op->device);
        const uint64_t nin = adjoint ? op->d.n_tgt() : op->d.n_src();
        const uint64_t nout = adjoint ? op->d.n_src() : op->d.n_tgt();
        op->order_begin(op->stream);
        if (op->hf.n < nin * nrhs) op->hf.alloc(nin * nrhs);
        if (op->hq.n < nout * nrhs) op->hq.alloc(nout * nrhs);
        ck(cudaMemcpyAsync(op->hf.p, in, nin * nrhs * 16, cudaMemcpyHostToDevice, op->stream), "H2D f");
        if (adjoint) {
            const int rc = sbd_op_apply_adjoint_device(op, (double*)op->hf.p, (double*)op->hq.p, nrhs, op->stream);
            if (rc) throw Error(rc, g_err);
        } else {
            // real right-hand sides, decided on the host copy while the H2D runs
            std::vector<int> real(nrhs, 1);
            for (int r = 0; r < nrhs; ++r) {
                const double* x = in + (size_t)r * nin * 2;
                int any = 0;
#pragma omp parallel for reduction(| : any) schedule(static)
                for (int64_t i = 0; i < (int64_t)nin; ++i) any |= x[2 * i + 1] != 0.0;
                real[r] = !any;
            }
            apply_device_rhs(op, (double*)op->hf.p, (double*)op->hq.p, nrhs, op->stream, real.data());
        }
        ck(cudaMemcpyAsync(out, op->hq.p, nout * nrhs * 16, cudaMemcpyDeviceToHost, op->stream), "D2H q");
        ck(cudaStreamSynchronize(op->stream), "apply sync");
        op->order_end(op->stream);
    });
}

int sbd_op_apply_async(sbd_op* op, const double* f, double* q, int nrhs, uint64_t* ticket) {
    return guarded([&] {
        if (!op || !f || !q || nrhs < 1 || !ticket) throw Error(SBD_ERR_INVALID_ARGUMENT, "apply_async: bad argument");
        std::lock_guard<std::recursive_mutex> lk(op->mu);
        DeviceGuard g(op->device);
        const uint64_t nin = op->d.n_src(), nout = op->d.n_tgt();
        if (!op->cp_in) {
            ck(cudaStreamCreateWithFlags(&op->cp_in, cudaStreamNonBlocking), "stream");
            ck(cudaStreamCreateWithFlags(&op->cp_out, cudaStreamNonBlocking), "stream");
            for (auto& sl : op->slot)
                for (cudaEvent_t* e : {&sl.h2d, &sl.comp, &sl.d2h})
                    ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
        }
        const uint64_t t = op->tickets++;
        sbd_op::Slot& sl = op->slot[t & 1];
        if (sl.f.n < nin * nrhs || sl.q.n < nout * nrhs) {
            // (re)allocating a slot's buffers: its previous call must be done
            if (sl.used) ck(cudaEventSynchronize(sl.d2h), "apply_async slot");
            if (sl.f.n < nin * nrhs) sl.f.alloc(nin * nrhs);
            if (sl.q.n < nout * nrhs) sl.q.alloc(nout * nrhs);
        }
        // realness per column, on the host while earlier calls run
        std::vector<int> real(nrhs, 1);
        for (int r = 0; r < nrhs; ++r) {
            const double* x = f + (size_t)r * nin * 2;
            int any = 0;
#pragma omp parallel for reduction(| : any) schedule(static)
            for (int64_t i = 0; i < (int64_t)nin; ++i) any |= x[2 * i + 1] != 0.0;
            real[r] = !any;
        }
        // H2D of f once the slot's previous apply has consumed its input
        if (sl.used) ck(cudaStreamWaitEvent(op->cp_in, sl.comp, 0), "wait");
        ck(cudaMemcpyAsync(sl.f.p, f, nin * nrhs * 16, cudaMemcpyHostToDevice, op->cp_in), "H2D f");
        ck(cudaEventRecord(sl.h2d, op->cp_in), "event");
        // the apply once f is in and the slot's previous q has left
        ck(cudaStreamWaitEvent(op->stream, sl.h2d, 0), "wait");
        if (sl.used) ck(cudaStreamWaitEvent(op->stream, sl.d2h, 0), "wait");
        apply_device_rhs(op, (const double*)sl.f.p, (double*)sl.q.p, nrhs, op->stream, real.data());
        ck(cudaEventRecord(sl.comp, op->stream), "event");
        // D2H of q
        ck(cudaStreamWaitEvent(op->cp_out, sl.comp, 0), "wait");
        ck(cudaMemcpyAsync(q, sl.q.p, nout * nrhs * 16, cudaMemcpyDeviceToHost, op->cp_out), "D2H q");
        ck(cudaEventRecord(sl.d2h, op->cp_out), "event");
        sl.used = true;
        *ticket = t;
    });
}

int sbd_op_wait(sbd_op* op, uint64_t ticket) {
    return guarded([&] {
        if (!op) throw Error(SBD_ERR_INVALID_ARGUMENT, "wait: null operator");
        cudaEvent_t e = nullptr;
        {
            std::lock_guard<std::recursive_mutex> lk(op->mu);
            if (ticket >= op->tickets) throw Error(SBD_ERR_INVALID_ARGUMENT, "wait: unknown ticket");
            // a slot's event is re-recorded by the call two tickets later, which
            // completes after this one: waiting on it is waiting long enough
            e = op->slot[ticket & 1].d2h;
        }
        DeviceGuard g(op->device);
        ck(cudaEventSynchronize(e), "wait");
    });
}

int sbd_op_apply(sbd_op* op, const double* f, double* q, int nrhs) {
    return host_apply(op, f, q, nrhs, false);
}

int sbd_op_apply_adjoint(sbd_op* op, const double* u, double* q, int nrhs) {
    return host_apply(op, u, q, nrhs, true);
}

int sbd_op_set_profiling(sbd_op* op, int enable) {
    return guarded([&] {
        if (!op) throw Error(SBD_ERR_INVALID_ARGUMENT, "null operator");
        std::lock_guard<std::recursive_mutex> lk(op->mu);
        op->tm.reset();
        op->tm.on = enable != 0;
    });
}

int sbd_op_stage_times(sbd_op* op, double* ms, const char** names, int cap) {
    if (!op) return -1;
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    return op->tm.read(ms, names, cap);
}

int sbd_op_stage_times_reset(sbd_op* op) {
    return guarded([&] {
        if (!op) throw Error(SBD_ERR_INVALID_ARGUMENT, "null operator");
        std::lock_guard<std::recursive_mutex> lk(op->mu);
        op->tm.reset();
    });
}

double sbd_cloud_diameter(const double* xy, uint64_t n) {
    try {
        return cloud_diameter(xy, n);
    } catch (const std::exception&) {
        return std::nan("");
    }
}

int sbd_nufft_create(const double* points, uint64_t np, const double* freqs, uint64_t nf, int sign,
                     double tol, int mode, uint64_t direct_threshold, uint64_t max_grid_bytes,
                     int device, sbd_nufft** out) {
    return guarded([&] {
        if (!out) throw Error(SBD_ERR_INVALID_ARGUMENT, "nufft: null argument");
        auto p = std::make_unique<sbd_nufft>();
        p->device = device;
        DeviceGuard g(device);
        ck(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking), "stream");
        NufftOpts o;
        o.tol = tol;
        o.mode = mode;
        o.direct_threshold = direct_threshold;
        o.max_grid_bytes = max_grid_bytes ? max_grid_bytes : (uint64_t(4) << 30);
        p->plan = std::make_unique<Plan>(points, np, freqs, nf, sign, o, device, true, true, p->stream);
        p->plan->ensure_work(p->work, p->stream);
        *out = p.release();
    });
}

static int nufft_run(sbd_nufft* p, const double* in, double* out, bool transpose) {
    return guarded([&] {
        if (!p || !in || !out) throw Error(SBD_ERR_INVALID_ARGUMENT, "nufft apply: null argument");
        DeviceGuard g(p->device);
        const uint64_t nin = transpose ? p->plan->nf : p->plan->np;
        const uint64_t nout = transpose ? p->plan->np : p->plan->nf;
        p->in.upload(reinterpret_cast<const double2*>(in), nin, p->stream);
        if (p->out.n < nout) p->out.alloc(std::max<uint64_t>(nout, 1));
        if (transpose)
            p->plan->apply_transpose(p->in.p, p->out.p, p->work, p->stream, nullptr);
        else
            p->plan->apply(p->in.p, p->out.p, p->work, p->stream, nullptr);
        ck(cudaMemcpyAsync(out, p->out.p, nout * 16, cudaMemcpyDeviceToHost, p->stream), "D2H");
        ck(cudaStreamSynchronize(p->stream), "nufft sync");
    });
}

int sbd_nufft_apply(sbd_nufft* p, const double* coeffs, double* out) {
    return nufft_run(p, coeffs, out, false);
}
int sbd_nufft_apply_transpose(sbd_nufft* p, const double* values, double* out) {
    return nufft_run(p, values, out, true);
}

int sbd_nufft_info(const sbd_nufft* p, int* fast, int* w, int* n1, int* n2) {
    return guarded([&] {
        if (!p) throw Error(SBD_ERR_INVALID_ARGUMENT, "null plan");
        if (fast) *fast = p->plan->fast;
        if (w) *w = p->plan->w;
        if (n1) *n1 = p->plan->ax.n;
        if (n2) *n2 = p->plan->ay.n;
    });
}

int sbd_nufft_destroy(sbd_nufft* p) {
    return guarded([&] {
        if (!p) return;
        DeviceGuard g(p->device);
        delete p;
    });
}

int sbd_ndft_direct(const double* points, uint64_t np, const double* freqs, uint64_t nf,
                    const double* coeffs, int sign, int device, double* out) {
    return guarded([&] {
        DeviceGuard g(device);
        cudaStream_t st;
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        DevBuf<double2> p, f, c, o(std::max<uint64_t>(nf, 1));
        p.upload(reinterpret_cast<const double2*>(points), np, st);
        f.upload(reinterpret_cast<const double2*>(freqs), nf, st);
        c.upload(reinterpret_cast<const double2*>(coeffs), np, st);
        launch_ndft(p.p, np, f.p, nf, c.p, sign, o.p, st);
        ck(cudaMemcpyAsync(out, o.p, nf * 16, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "ndft sync");
        cudaStreamDestroy(st);
    });
}

int sbd_choose_parameters(uint64_t n, double eps, double alpha, double* a, int* p_hint) {
    return guarded([&] {
        // conv_operator.cpp:121-133
        if (!(eps > 0.0 && eps < 1.0)) throw Error(SBD_ERR_DOMAIN, "choose_parameters: eps must lie in (0, 1)");
        if (alpha < 0.0 || alpha > 1.0 / 6.0 + 1e-12)
            throw Error(SBD_ERR_DOMAIN, "choose_parameters: alpha must lie in [0, 1/6]");
        const double log_eps = std::fabs(std::log(eps));
        if (!((double)n > log_eps)) throw Error(SBD_ERR_DOMAIN, "choose_parameters: requires N_z > |log eps|");
        double av = std::pow(log_eps, 2.0 / 3.0) / std::pow((double)n, 2.0 / 3.0 - alpha);
        av = std::min(av, 0.5);
        if (a) *a = av;
        if (p_hint) *p_hint = (int)std::ceil(0.30 * log_eps / av);
    });
}

} // extern "C"
