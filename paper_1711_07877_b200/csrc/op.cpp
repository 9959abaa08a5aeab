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
#include "op_internal.h"

namespace sbdgpu {

namespace {
thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
} // namespace
thread_local bool g_verbose = false;
void set_last_error(const std::string& m) { g_err = m; }

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


} // namespace sbdgpu

using namespace sbdgpu;


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
    o->procedural_rings = 0;
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
        info->procedural_rings = op->procedural ? 1 : 0;
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
