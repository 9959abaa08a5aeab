// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver over the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see oracle/Makefile; output oracle/_ref/libsbdref.so).
// It is the "reference" arm of the parity tests and of `bench.py --impl reference`,
// and the generator of reference operator files / golden vectors. It never links
// into the product, and the product never calls it.
//
// Entry points map 1:1 onto the reference's public API:
//   ref_assemble_save  -> make_cloud + CompressedOperator::assemble + save
//                         (reference proj/src/conv_operator.cpp:244-294, 357-397)
//   ref_op_load/apply  -> CompressedOperator::load / apply / apply_adjoint
//                         (conv_operator.cpp:449-490, 301-309, 311-324)
//   ref_raw_*          -> the same four apply stages driven through the public
//                         NufftPlan / SparsePairMatrix API with a caller-chosen
//                         max_grid_bytes (load() pins it to the 4 GiB default,
//                         nufft.hpp:23, which config 4's 5.4 GB grid exceeds)
//   ref_nufft          -> NufftPlan(points, freqs, sign, opts).apply / apply_transpose
//   ref_bessel         -> bessel.hpp functions
#include <cstdint>
#include <cstring>
#include <fstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sbd/bessel.hpp"
#include "sbd/conv_operator.hpp"
#include "sbd/nufft.hpp"
#include "sbd/point_cloud.hpp"
#include "sbd/ring_quadrature.hpp"

using namespace sbd;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
    if (dynamic_cast<const std::domain_error*>(&e)) return 2;
    return 3;
}

std::vector<Vec2> to_points(const double* xy, std::uint64_t n) {
    std::vector<Vec2> p(n);
    for (std::uint64_t i = 0; i < n; ++i) p[i] = {xy[2 * i], xy[2 * i + 1]};
    return p;
}

std::vector<cplx> to_cplx(const double* v, std::uint64_t n) {
    std::vector<cplx> c(n);
    for (std::uint64_t i = 0; i < n; ++i) c[i] = {v[2 * i], v[2 * i + 1]};
    return c;
}

void from_cplx(const std::vector<cplx>& c, double* out) {
    for (std::size_t i = 0; i < c.size(); ++i) {
        out[2 * i] = c[i].real();
        out[2 * i + 1] = c[i].imag();
    }
}

// SBDOPv1 reader (layout of conv_operator.cpp:357-447) for the raw driver.
struct RawOp {
    int kind = 0;
    double k = 0.0;
    bool single = false;
    double eps = 0, alpha = 0, a = 0, dmin = 0, dmax = 0, nufft_tol = 0;
    std::vector<Vec2> src, tgt;
    FrequencyQuadrature quad;
    SparsePairMatrix D;
    std::unique_ptr<NufftPlan> fwd_in, fwd_out;
};

template <typename T>
void rd(std::istream& is, T& v) {
    is.read(reinterpret_cast<char*>(&v), sizeof(T));
}
template <typename T>
void rdv(std::istream& is, std::vector<T>& v) {
    std::uint64_t n = 0;
    rd(is, n);
    v.resize(n);
    is.read(reinterpret_cast<char*>(v.data()), (std::streamsize)(n * sizeof(T)));
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_assemble_save(int kind, double k, const double* src_xy, std::uint64_t n_src,
                      const double* tgt_xy, std::uint64_t n_tgt, double eps, double alpha,
                      double a_override, double small_k_factor, std::uint64_t max_grid_bytes,
                      const char* path, double* info) {
    try {
        KernelSpec ks = kind == 1 ? kernel_helmholtz(k) : kernel_laplace();
        AssembleOptions o;
        o.eps = eps;
        o.alpha = alpha;
        o.a_override = a_override;
        o.small_k_factor = small_k_factor;
        if (max_grid_bytes) o.max_grid_bytes = max_grid_bytes;
        PointCloud s = make_cloud(to_points(src_xy, n_src));
        CompressedOperator op = tgt_xy ? CompressedOperator::assemble(
                                             ks, s, make_cloud(to_points(tgt_xy, n_tgt)), o)
                                       : CompressedOperator::assemble(ks, s, o);
        op.save(path);
        if (info) {
            info[0] = op.annulus_a();
            info[1] = op.delta_min();
            info[2] = op.delta_max();
            info[3] = (double)op.decomposition().P;
            info[4] = (double)op.quadrature().size();
            info[5] = (double)op.close_matrix().nnz();
            info[6] = (double)op.bytes();
            info[7] = op.decomposition().achieved_error;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void* ref_op_load(const char* path) {
    try {
        return new CompressedOperator(CompressedOperator::load(path));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_op_free(void* h) { delete static_cast<CompressedOperator*>(h); }

int ref_op_apply(void* h, const double* f, std::uint64_t n, double* q) {
    try {
        const auto* op = static_cast<CompressedOperator*>(h);
        from_cplx(op->apply(to_cplx(f, n)), q);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_op_apply_adjoint(void* h, const double* u, std::uint64_t n, double* q) {
    try {
        const auto* op = static_cast<CompressedOperator*>(h);
        from_cplx(op->apply_adjoint(to_cplx(u, n)), q);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void* ref_raw_open(const char* path, std::uint64_t max_grid_bytes) {
    try {
        std::ifstream is(path, std::ios::binary);
        if (!is) throw std::runtime_error(std::string("cannot open ") + path);
        char magic[8];
        is.read(magic, 8);
        if (std::memcmp(magic, "SBDOPv1", 8) != 0) throw std::runtime_error("bad magic");
        auto op = std::make_unique<RawOp>();
        std::int32_t kind = 0;
        std::uint8_t single = 0;
        rd(is, kind);
        rd(is, op->k);
        rd(is, single);
        op->kind = kind;
        op->single = single != 0;
        rd(is, op->eps);
        rd(is, op->alpha);
        rd(is, op->a);
        rd(is, op->dmin);
        rd(is, op->dmax);
        rd(is, op->nufft_tol);
        double diam = 0.0;
        rdv(is, op->src);
        rd(is, diam);
        if (!op->single) {
            rdv(is, op->tgt);
            rd(is, diam);
        } else {
            op->tgt = op->src;
        }
        rdv(is, op->quad.freqs);
        rdv(is, op->quad.weights);
        rdv(is, op->quad.ring_offsets);
        rd(is, op->quad.total_error_budget);
        rdv(is, op->D.row_offsets);
        rdv(is, op->D.cols);
        rdv(is, op->D.values);
        if (!is) throw std::runtime_error("truncated operator file");
        NufftOptions no;
        no.tol = op->nufft_tol;
        if (max_grid_bytes) no.max_grid_bytes = max_grid_bytes;
        // Same plan pair as CompressedOperator::Impl::build_forward_plans
        // (conv_operator.cpp:162-167).
        op->fwd_in = std::make_unique<NufftPlan>(op->src, op->quad.freqs, NufftSign::Minus, no);
        op->fwd_out = std::make_unique<NufftPlan>(op->quad.freqs, op->tgt, NufftSign::Plus, no);
        return op.release();
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_raw_free(void* h) { delete static_cast<RawOp*>(h); }

// stage 0: full apply (conv_operator.cpp:301-309); 1: fwd_in only -> spectrum
// (before the weights); 2: fwd_out only (input = weighted spectrum); 3: q += D f.
int ref_raw_stage(void* h, int stage, const double* in, std::uint64_t n_in, double* out) {
    try {
        auto* op = static_cast<RawOp*>(h);
        const std::vector<cplx> x = to_cplx(in, n_in);
        if (stage == 0) {
            std::vector<cplx> spectrum = op->fwd_in->apply(x);
            for (int v = 0; v < op->quad.size(); ++v) spectrum[v] *= op->quad.weights[v];
            std::vector<cplx> q = op->fwd_out->apply(spectrum);
            op->D.accumulate_apply(x, q);
            from_cplx(q, out);
        } else if (stage == 1) {
            from_cplx(op->fwd_in->apply(x), out);
        } else if (stage == 2) {
            from_cplx(op->fwd_out->apply(x), out);
        } else if (stage == 3) {
            std::vector<cplx> q = to_cplx(out, op->tgt.size());
            op->D.accumulate_apply(x, q);
            from_cplx(q, out);
        } else {
            throw std::invalid_argument("bad stage");
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_nufft(const double* pts, std::uint64_t np, const double* frq, std::uint64_t nf, int sign,
              double tol, int mode, std::uint64_t max_grid_bytes, int transpose, const double* in,
              double* out, int* meta) {
    try {
        NufftOptions o;
        o.tol = tol;
        o.mode = mode == 1 ? NufftOptions::Mode::Direct
                           : (mode == 2 ? NufftOptions::Mode::Fast : NufftOptions::Mode::Auto);
        if (max_grid_bytes) o.max_grid_bytes = max_grid_bytes;
        NufftPlan plan(to_points(pts, np), to_points(frq, nf),
                       sign > 0 ? NufftSign::Plus : NufftSign::Minus, o);
        if (meta) {
            meta[0] = plan.fast_path() ? 1 : 0;
            meta[1] = plan.kernel_width();
        }
        if (in && out) {
            if (transpose)
                from_cplx(plan.apply_transpose(to_cplx(in, nf)), out);
            else
                from_cplx(plan.apply(to_cplx(in, np)), out);
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

double ref_bessel(int which, int n, double x) {
    try {
        switch (which) {
            case 0: return bessel_j0(x);
            case 1: return bessel_j1(x);
            case 2: return bessel_jn(n, x);
            case 3: return bessel_y0(x);
            case 4: return bessel_y1(x);
            case 5: return bessel_i0(x);
        }
    } catch (const std::exception& e) {
        fail(e);
    }
    return 0.0 / 0.0;
}

double ref_cloud_diameter(const double* xy, std::uint64_t n) { return cloud_diameter(to_points(xy, n)); }

int ref_choose_parameters(std::uint64_t n, double eps, double alpha, double* a, int* p_hint) {
    try {
        const ChosenParameters p = choose_parameters(n, eps, alpha);
        *a = p.a;
        *p_hint = p.P_hint;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

} // extern "C"
