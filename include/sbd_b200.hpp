// sbd_b200.hpp -- header-only C++ mirror of the reference operator API over
// the C ABI in sbd_b200.h. A user of the reference library
// (/root/reference/proj/include/sbd/conv_operator.hpp, kernels.hpp,
// nufft.hpp) switches by replacing `sbd::` with `sbd_b200::` and linking
// libsbd_b200.so; signatures, argument meaning and exception types match:
//
//   reference                                         here
//   ------------------------------------------------  -----------------------------------------
//   sbd::CompressedOperator::assemble(k, src, tgt, o)  sbd_b200::CompressedOperator::assemble(...)
//   sbd::CompressedOperator::assemble(k, cloud, o)     (same, single cloud)
//   sbd::CompressedOperator::load(path) / save(path)   load(path[, device, max_grid_bytes]) / save
//   op.apply(f) / op.apply_adjoint(u)                  op.apply(f) / op.apply_adjoint(u)
//   op.eps() / delta_min() / delta_max() / bytes()...  same accessors
//   sbd::NufftPlan(points, freqs, sign, opts)          sbd_b200::NufftPlan(...)
//   std::invalid_argument / domain_error / runtime_error / SbdConvergenceError   same
//
// Points are sbd_b200::Vec2 (two doubles, the layout of sbd::Vec2), values
// std::complex<double>. Everything runs on the GPU selected by `device`.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sbd_b200.h"

namespace sbd_b200 {

using cplx = std::complex<double>;

struct Vec2 {
    double x = 0.0, y = 0.0;
};
static_assert(sizeof(Vec2) == 16, "Vec2 must be two packed doubles");
static_assert(sizeof(cplx) == 16, "complex<double> must be interleaved re, im");

struct SbdConvergenceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc) {
    if (rc == SBD_OK) return;
    const std::string msg = sbd_last_error();
    switch (rc) {
        case SBD_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SBD_ERR_DOMAIN: throw std::domain_error(msg);
        case SBD_ERR_CONVERGENCE: throw SbdConvergenceError(msg);
        default: throw std::runtime_error(msg);
    }
}
} // namespace detail

// kernels.hpp:59-72
struct KernelSpec {
    enum class Kind { Laplace = SBD_KERNEL_LAPLACE, Helmholtz = SBD_KERNEL_HELMHOLTZ };
    Kind kind = Kind::Laplace;
    double k = 0.0;
    bool is_complex() const { return kind == Kind::Helmholtz; }
};
inline KernelSpec kernel_laplace() { return {}; }
inline KernelSpec kernel_helmholtz(double k) {
    if (!(k > 0.0)) throw std::domain_error("kernel_helmholtz: k must be positive");
    return {KernelSpec::Kind::Helmholtz, k};
}

// conv_operator.hpp:24-31 (+ device)
struct AssembleOptions {
    double eps = 1e-6;
    double alpha = 0.0;
    double a_override = 0.0;
    double small_k_factor = 0.5;
    std::uint64_t nufft_direct_threshold = std::uint64_t(1) << 20;
    std::uint64_t max_grid_bytes = std::uint64_t(4) << 30;
    int device = 0;
};

inline double cloud_diameter(const std::vector<Vec2>& pts) {
    return sbd_cloud_diameter(reinterpret_cast<const double*>(pts.data()), pts.size());
}

// conv_operator.hpp:37-79
class CompressedOperator {
  public:
    static CompressedOperator assemble(const KernelSpec& kernel, const std::vector<Vec2>& source,
                                       const std::vector<Vec2>& target, const AssembleOptions& o) {
        const bool single = source.size() == target.size() &&
                            std::equal(source.begin(), source.end(), target.begin(),
                                       [](const Vec2& a, const Vec2& b) { return a.x == b.x && a.y == b.y; });
        return assemble_impl(kernel, source, single ? nullptr : &target, o);
    }
    static CompressedOperator assemble(const KernelSpec& kernel, const std::vector<Vec2>& cloud,
                                       const AssembleOptions& o) {
        return assemble_impl(kernel, cloud, nullptr, o);
    }
    static CompressedOperator load(const std::string& path, int device = 0,
                                   std::uint64_t max_grid_bytes = 0) {
        sbd_op* h = nullptr;
        detail::check(sbd_op_load(path.c_str(), device, max_grid_bytes, &h));
        return CompressedOperator(h);
    }

    CompressedOperator(CompressedOperator&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    CompressedOperator& operator=(CompressedOperator&& o) noexcept {
        if (this != &o) {
            reset();
            h_ = std::exchange(o.h_, nullptr);
        }
        return *this;
    }
    CompressedOperator(const CompressedOperator&) = delete;
    CompressedOperator& operator=(const CompressedOperator&) = delete;
    ~CompressedOperator() { reset(); }

    // q = NUFFT+[target](w * NUFFT-[source](f)) + D f  (conv_operator.cpp:301-309)
    std::vector<cplx> apply(const std::vector<cplx>& f) const {
        const sbd_op_info_t i = info();
        if (f.size() != i.n_src) throw std::invalid_argument("apply: input size mismatch");
        std::vector<cplx> q(i.n_tgt);
        detail::check(sbd_op_apply(h_, reinterpret_cast<const double*>(f.data()),
                                   reinterpret_cast<double*>(q.data()), 1));
        return q;
    }
    // conv_operator.cpp:311-324
    std::vector<cplx> apply_adjoint(const std::vector<cplx>& u) const {
        const sbd_op_info_t i = info();
        if (u.size() != i.n_tgt) throw std::invalid_argument("apply_adjoint: input size mismatch");
        std::vector<cplx> q(i.n_src);
        detail::check(sbd_op_apply_adjoint(h_, reinterpret_cast<const double*>(u.data()),
                                           reinterpret_cast<double*>(q.data()), 1));
        return q;
    }
    // Device buffers on a caller stream (no reference analogue).
    void apply_device(const cplx* d_f, cplx* d_q, int nrhs = 1, void* stream = nullptr) const {
        detail::check(sbd_op_apply_device(h_, reinterpret_cast<const double*>(d_f),
                                          reinterpret_cast<double*>(d_q), nrhs, stream));
    }
    // f_is_real: nrhs flags (1 real, 0 complex, -1 unknown); lets real columns
    // take the Hermitian-FFT mode without a host round trip
    void apply_device(const cplx* d_f, cplx* d_q, int nrhs, void* stream, const int* f_is_real) const {
        detail::check(sbd_op_apply_device_ex(h_, reinterpret_cast<const double*>(d_f),
                                             reinterpret_cast<double*>(d_q), nrhs, stream, f_is_real));
    }

    void save(const std::string& path) const { detail::check(sbd_op_save(h_, path.c_str())); }

    sbd_op_info_t info() const {
        sbd_op_info_t i;
        detail::check(sbd_op_info(h_, &i));
        return i;
    }
    bool single_cloud() const { return info().single_cloud != 0; }
    double eps() const { return info().eps; }
    double delta_min() const { return info().delta_min; }
    double delta_max() const { return info().delta_max; }
    double annulus_a() const { return info().a; }
    std::uint64_t bytes() const { return info().bytes; }
    std::vector<Vec2> source() const { return get<Vec2>(0, 2); }
    std::vector<Vec2> target() const { return get<Vec2>(1, 2); }
    std::vector<Vec2> frequencies() const { return get<Vec2>(2, 2); }
    std::vector<cplx> weights() const { return get<cplx>(3, 2); }
    sbd_op* handle() const { return h_; }

  private:
    explicit CompressedOperator(sbd_op* h) : h_(h) {}
    void reset() {
        if (h_) sbd_op_destroy(h_);
        h_ = nullptr;
    }
    static CompressedOperator assemble_impl(const KernelSpec& kernel, const std::vector<Vec2>& src,
                                            const std::vector<Vec2>* tgt, const AssembleOptions& o) {
        sbd_assemble_options c;
        sbd_assemble_options_default(&c);
        c.eps = o.eps;
        c.alpha = o.alpha;
        c.a_override = o.a_override;
        c.small_k_factor = o.small_k_factor;
        c.nufft_direct_threshold = o.nufft_direct_threshold;
        c.max_grid_bytes = o.max_grid_bytes;
        c.device = o.device;
        sbd_op* h = nullptr;
        detail::check(sbd_op_assemble((int)kernel.kind, kernel.k, reinterpret_cast<const double*>(src.data()),
                                      src.size(), tgt ? reinterpret_cast<const double*>(tgt->data()) : nullptr,
                                      tgt ? tgt->size() : 0, &c, &h));
        return CompressedOperator(h);
    }
    template <typename T>
    std::vector<T> get(int which, int doubles_per) const {
        std::uint64_t n = 0;
        detail::check(sbd_op_get(h_, which, nullptr, &n));
        std::vector<T> v(n / doubles_per);
        detail::check(sbd_op_get(h_, which, v.data(), &n));
        return v;
    }
    sbd_op* h_ = nullptr;
};

// nufft.hpp:18-56
enum class NufftSign : int { Plus = +1, Minus = -1 };
struct NufftOptions {
    double tol = 1e-9;
    enum class Mode { Auto, Direct, Fast } mode = Mode::Auto;
    std::uint64_t direct_threshold = std::uint64_t(1) << 20;
    std::uint64_t max_grid_bytes = std::uint64_t(4) << 30;
    int device = 0;
};

class NufftPlan {
  public:
    NufftPlan(const std::vector<Vec2>& points, const std::vector<Vec2>& freqs, NufftSign sign,
              NufftOptions o = {})
        : np_(points.size()), nf_(freqs.size()) {
        detail::check(sbd_nufft_create(reinterpret_cast<const double*>(points.data()), np_,
                                       reinterpret_cast<const double*>(freqs.data()), nf_, (int)sign,
                                       o.tol, (int)o.mode, o.direct_threshold, o.max_grid_bytes,
                                       o.device, &h_));
    }
    NufftPlan(NufftPlan&& o) noexcept : h_(std::exchange(o.h_, nullptr)), np_(o.np_), nf_(o.nf_) {}
    NufftPlan(const NufftPlan&) = delete;
    NufftPlan& operator=(const NufftPlan&) = delete;
    ~NufftPlan() {
        if (h_) sbd_nufft_destroy(h_);
    }
    std::vector<cplx> apply(const std::vector<cplx>& c) const {
        if (c.size() != np_) throw std::invalid_argument("nufft apply: coefficient count mismatch");
        std::vector<cplx> out(nf_);
        detail::check(sbd_nufft_apply(h_, reinterpret_cast<const double*>(c.data()),
                                      reinterpret_cast<double*>(out.data())));
        return out;
    }
    std::vector<cplx> apply_transpose(const std::vector<cplx>& v) const {
        if (v.size() != nf_) throw std::invalid_argument("nufft apply_transpose: value count mismatch");
        std::vector<cplx> out(np_);
        detail::check(sbd_nufft_apply_transpose(h_, reinterpret_cast<const double*>(v.data()),
                                                reinterpret_cast<double*>(out.data())));
        return out;
    }
    bool fast_path() const {
        int fast = 0;
        detail::check(sbd_nufft_info(h_, &fast, nullptr, nullptr, nullptr));
        return fast != 0;
    }
    int kernel_width() const {
        int w = 0;
        detail::check(sbd_nufft_info(h_, nullptr, &w, nullptr, nullptr));
        return w;
    }

  private:
    sbd_nufft* h_ = nullptr;
    std::uint64_t np_ = 0, nf_ = 0;
};

} // namespace sbd_b200
