// sbd_internal.h -- internal types shared by the host C++ and the sm_100a
// kernels of the B200 SBD apply path. Not part of the public ABI
// (include/sbd_b200.h is).
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace sbdgpu {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void throw_cuda(cudaError_t e, const char* what);
[[noreturn]] void throw_cufft(cufftResult r, const char* what);
inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw_cuda(e, what);
}
inline void ckfft(cufftResult r, const char* what) {
    if (r != CUFFT_SUCCESS) throw_cufft(r, what);
}
void count_launch(int n = 1);
// setup diagnostics on stderr for the calling thread's current entry point
// (sbd_op_options::verbose; no environment switches)
extern thread_local bool g_verbose;

// ---------------------------------------------------------------- buffers
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p; n = o.n; o.p = nullptr; o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) ck(cudaMalloc(&p, count * sizeof(T) + 64), "cudaMalloc");
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
    void upload(const T* h, size_t count, cudaStream_t s) {
        if (count > n) alloc(count);
        if (count) ck(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
    }
};

// ---------------------------------------------------------------- window
// Kaiser-Bessel window phi(z) = I0(beta sqrt(1 - z^2)) (reference
// nufft.cpp:28-32) restated per tap as a polynomial in v = 2u - 1 where
// u = ix0 - t + w/2 in [0, 1) is the (exactly computed) sub-cell offset.
// Tap i and tap w-1-i share one even/odd split: P_i(v) = E_i(v^2) + v O_i(v^2),
// P_{w-1-i}(v) = E_i(v^2) - v O_i(v^2). Degree 15 (8 + 8 coefficients) keeps
// the sup-norm error ~1e-16 of the window peak for every w the reference can
// choose (4..17); see window.cpp.
constexpr int kMaxW = 17;
constexpr int kPairs = (kMaxW + 1) / 2;
constexpr int kHorner = 8;
struct WindowPoly {
    double e[kPairs][kHorner];
    double o[kPairs][kHorner];
};
WindowPoly fit_window(int w, double beta, double* max_rel_err = nullptr);
double kb_window_host(double beta, double z);     // exact reference formula (long double I0)
double kb_window_hat_host(double beta, double w); // nufft.cpp:34-45

// ---------------------------------------------------------------- geometry
// Per-axis plan geometry, restated from nufft.cpp:65-72 / 139-155.
struct Axis {
    double center = 0.0, fcenter = 0.0, gamma = 1.0;
    int n = 0;
    double alpha1 = 0.0, alpha2 = 0.0;
};

// Plan geometry of one axis (nufft.cpp:127-154), exactly as Plan computes it,
// and the stencil start ceil(c - w/2) of a point / an output on that axis as
// k_plan_points / k_plan_outputs + the spread / interpolation compute it.
Axis plan_axis(const double* pts_xy, uint64_t np, const double* frq_xy, uint64_t nf, int comp,
               double sg, int w);
int stencil_start_point(const Axis& a, double p, int w);
int stencil_start_output(const Axis& a, double f, double sg, int w);

struct NufftOpts {
    double tol = 1e-9;
    int mode = 0; // 0 auto, 1 direct, 2 fast
    uint64_t direct_threshold = uint64_t(1) << 20;
    uint64_t max_grid_bytes = uint64_t(4) << 30;
    // kernel / pipeline selection (sbd_op_options in include/sbd_b200.h; every
    // choice stays within the parity bar)
    int radix = -1;        // radix first pass folded into the untangle/pack: -1 auto (n > 4096), 0 off, 1 force
    int spread_kernel = 0; // 0 CTA spread over region lists, 1 CTA over bins, 2 per-warp DMMA, 3 scalar tiles
    int interp_kernel = 0; // 0 auto, 1 staged DMMA tiles, 2 DMMA per warp, 3 scalar
};

int width_for_tol(double tol);  // nufft.cpp:47-52
int next_fast_even(int n);      // nufft.cpp:55-63

// Timing of the apply stages with CUDA events (only when profiling).
struct StageTimer {
    bool on = false;
    cudaStream_t stream = nullptr;
    std::vector<std::string> names;
    std::vector<cudaEvent_t> begin, end;
    void reset();
    void start(const char* name, cudaStream_t on_stream = nullptr);  // nullptr: `stream`
    void stop(cudaStream_t on_stream = nullptr);
    int read(double* ms, const char** nm, int cap);
    ~StageTimer();
};

// Grid / FFT scratch of one or more plans of equal grid size. The pruned
// forward path keeps the invariant "grid and T are zero outside the recorded
// dirty rectangles", so no full-grid memset is needed per apply.
struct FftWork {
    DevBuf<double2> grid, T, band;
    DevBuf<double2> T1, bandT; // transposed band columns before / after the column transform
    int tt_r0 = 0, tt_r1 = 0;  // rows (x) possibly nonzero in every Tt row (cuFFT-T path) ...
    int tt_pitch = 0, tt_rows = 0; // ... for a Tt of this pitch (n1) and row count (bc)
    DevBuf<double2> bbuf; // spread coefficients b = c * prephase, sorted point order
    int n1 = 0, n2 = 0, bc = 0;
    int gr0 = 0, gr1 = 0, gc0 = 0, gc1 = 0; // grid cells possibly nonzero ...
    int g_pitch = 0;                        // ... in a row-major layout of this pitch
    int tr0 = 0, tr1 = 0;                   // rows of T possibly nonzero ...
    int t_pitch = 0;                        // ... at this pitch
    void ensure(int n1_, int n2_, int bc_, cudaStream_t st);
};

// Spread tiles of the pruned forward path: one warp owns kTileR x kTileC
// grid cells (lanes = columns, rows in registers).
constexpr int kTileR = 16;
constexpr int kTileC = 16;
struct TileGeom {
    int rlo, clo, nbx, nby;
    int tr;              // rows per tile (8 or 16)
    int pitch;           // 0: write the full n1 x n2 grid; else compact region layout
    int rhi, chi;        // region end (writes clipped here)
};

// A type-III NUFFT plan on one device (reference NufftPlan, nufft.hpp:30-56).
// Point side ("t": spread in apply, gather in apply_transpose) and output side
// ("s": gather in apply, spread in apply_transpose) are stored in a sorted
// order chosen for locality; perm_* map sorted position -> caller index (empty
// when the caller's order is kept).


// Plan-time region lists of the CTA spread: for each 32 x 32 region (row-major,
// ncy regions per row) the entries (point index | 0x80000000 for the second
// point arrays) of the points whose stencil overlaps it; list 2 is skipped
// while the device half-split flag is set.
struct SpreadLists {
    const uint32_t *s1 = nullptr, *e1 = nullptr, *s2 = nullptr, *e2 = nullptr;
    int ncy = 0;
};

struct HermArgs;

// Procedural ring nodes (ring_quadrature.cpp:24-69): node j
// of ring p is rho_p (cos, sin)(2 pi j / M_p) with weight w_p, so the xi-side
// kernels can regenerate a node's plan arrays (grid / mode coordinates,
// prephase, postphase, omega-hat) from a 4-byte id instead of streaming them.
// id = ring << kRingJBits | j; bit 31: the node enters the real-input half
// split with weight 1/2 (op_internal.h herm_pairs).
constexpr int kRingJBits = 17;
constexpr uint32_t kRingHalve = 0x80000000u;
struct RingRow {
    double rho, two_over_m, wre, wim;
};
struct NodeGen {
    const uint32_t* id = nullptr;  // ids in the consuming kernel's node order
    const RingRow* rings = nullptr;
    Axis ox, oy;                   // the nodes as a plan's outputs (fwd_in): mode coordinates, postphase
    double osgn = 1.0, ocxy = 1.0;
    Axis px, py;                   // the nodes as a plan's points (fwd_out): grid coordinates, prephase
    double pbeta = 0.0;
};

class Plan {
  public:
    // pt_tag / out_tag (optional, caller order, 0/1): sort tag-0 entries before
    // tag-1 entries on that side (the real-input half split, op.cpp)
    // dev_pts / dev_frq (optional, device, caller order): the values the
    // per-point / per-output arrays are computed from instead of the uploaded
    // host copies (procedural ring nodes: generated on the device, so that the
    // xi-side kernels regenerate them bitwise; the geometry still comes from
    // the host arrays)
    Plan(const double* pts_xy, uint64_t np, const double* frq_xy, uint64_t nf, int sign,
         const NufftOpts& opts, int device, bool sort_points, bool sort_outputs, cudaStream_t st,
         const uint8_t* pt_tag = nullptr, const uint8_t* out_tag = nullptr,
         const double2* dev_pts = nullptr, const double2* dev_frq = nullptr);
    ~Plan();
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;

    bool fast = false;
    int sign = 1;
    int device = 0;
    int w = 0;
    double beta = 0.0;
    Axis ax, ay;
    uint64_t np = 0, nf = 0;
    WindowPoly win{};
    NufftOpts opts;

    // direct path (and point/freq sets kept for it)
    DevBuf<double2> pts, frq;
    // fast path, sorted
    DevBuf<uint32_t> perm_t, perm_s;
    DevBuf<double2> t, pre;  // point side: grid coords (cells), prephase
    DevBuf<double2> s, post; // output side: mode coords, postphase
    DevBuf<double> dx, dy;   // deconvolution per FFT index (nufft.cpp:194-205)
    mutable cufftHandle fft = 0; // full 2D transform (transpose path), created lazily

    // Pruned forward path (apply): points binned by kTileR x kTileC tiles of
    // the populated region; row FFTs over the populated rows only, column FFTs
    // over the band columns only (the only modes the interpolation reads).
    bool pruned = false;
    int rlo = 0, rhi = 0, clo = 0, chi = 0; // region written by the spread tiles
    TileGeom tg{};
    DevBuf<uint32_t> bin_start;
    // tagged sides: tag-0 entries are sorted positions [0, n0_*); the points'
    // tile bins of the tag-1 entries are in bin_start2
    bool tagged_pts = false, tagged_out = false;
    uint64_t n0_pts = 0, n0_out = 0;
    DevBuf<uint32_t> bin_start2;
    DevBuf<uint32_t> out_tiles;  // Z-order block starts of the sorted outputs
    uint32_t n_out_tiles = 0;
    int out_shift = 0;
    int band2 = 0, bc = 0;
    DevBuf<double> dy_band;
    cufftHandle fft_row = 0;
    cufftHandle fft_colT = 0;  // contiguous transforms of the transposed band columns
    // radix first passes of the complex pipeline's two transforms in our own
    // kernels (k_dif_rows / k_band_transpose_dif), cuFFT on contiguous
    // length-n/r passes: 1 = cuFFT's own full-length transform
    int crad_row = 1, crad_col = 1;
    cufftHandle fft_row_m = 0, fft_colT_m = 0;
    DevBuf<double2> ctw_row, ctw_col;

    // Hermitian-FFT mode for a real input (op.cpp). Role 1 (fwd_in): the
    // spread grid is real; its rows are packed in pairs into complex rows ->
    // Z2Z rows -> untangle + transpose of the columns 0..n2/4 -> Z2Z columns;
    // the xi interpolation reads the negative columns by conjugate symmetry.
    // Role 2 (fwd_out): the tag-0 points plus their mirror images (conjugate
    // values) make the spread grid Hermitian; only the columns m2 <= n2/2 are
    // spread (transposed) -> Z2Z columns -> band rows, two per complex row ->
    // Z2Z rows give the real band for the target interpolation.
    int hrole = 0;
    cufftHandle hp1 = 0, hp2 = 0;
    int hrad = 1;                    // radix of the first pass folded into untangle (role 1, columns)
                                     // or pack (role 2, rows); 1: none
    DevBuf<double2> htw;             // its twiddles e^{+2 pi i m / n}
    int hrad0 = 1;                   // radix of the first pass of the other (first) transform, as
                                     // its own kernel (k_dif_rows) before a length n / hrad0 cuFFT pass
    DevBuf<double2> htw0;
    mutable DevBuf<double2> hA, hB, hC, hD;
    int hnm = 0, hnby = 0, hb1 = 0, hB1 = 0, hcols = 0;
    DevBuf<double2> hv_t;             // role 2: mirrored tag-0 points, sorted by tile
    DevBuf<uint32_t> hv_bins, hv_of;  // their bins; tag-0 sorted position -> mirrored position
    DevBuf<uint32_t> hv_src;          // mirrored position -> tag-0 sorted position
    // region lists of the CTA spread: set 1 (tag-0 or all points), set 2
    // (tag-1 points), mirror images (role 2)
    DevBuf<uint32_t> rl1_s, rl1_e, rl2_s, rl2_e, rlh_s, rlh_e;
    SpreadLists lists(bool mirror) const {
        SpreadLists l;
        l.s1 = rl1_s.p;
        l.e1 = rl1_e.p;
        l.s2 = mirror ? rlh_s.p : rl2_s.p;
        l.e2 = mirror ? rlh_e.p : rl2_e.p;
        l.ncy = (tg.nby + 1) / 2;
        return l;
    }
    DevBuf<double> hdx_band;          // role 2: deconvolution of the band rows
    bool enable_hfft(int role, cudaStream_t st);

    // Procedural sides (op_internal.h): with gen_*.id set the pruned forward
    // path regenerates the side's arrays in its kernels, and t / pre / pts /
    // hv_t (points) or s / post / frq (outputs) may be released; every other
    // path needs them materialised again (sbd_op::ensure_node_arrays).
    NodeGen gen_pts, gen_out;
    double out_cxy() const;  // postphase scale (nufft.cpp:183-184)

    uint64_t cells() const { return fast ? (uint64_t)ax.n * (uint64_t)ay.n : 0; }
    size_t device_bytes() const;

    // Enqueue apply / apply_transpose on stream `st`. in/out in caller order.
    // `grid` must hold cells() complex values. `extra` (optional) multiplies
    // the outputs elementwise in SORTED output order (used for omega-hat).
    void apply(const double2* in, double2* out, FftWork& wk, cudaStream_t st,
               StageTimer* tm, const double2* mult = nullptr, const char* tag_spread = "spread",
               const char* tag_fft = "fft", const char* tag_interp = "interp") const;
    // Pruned forward path with the operator's fused inputs/outputs:
    //  in_is_b: `in` already holds b = c * prephase in this plan's sorted point
    //           order (else b is formed from caller-order `in`, and the sorted
    //           copy of `in` is written to raw_sorted when given);
    //  addend:  per sorted output, added after mult before the scatter.
    //  herm:    real-input half split (HermArgs), nullptr = off
    //  before_interp: the interpolation waits for this event (work on another stream)
    void apply_pruned(const double2* in, bool in_is_b, double2* raw_sorted, double2* out,
                      const double2* mult, const double2* addend, FftWork& wk, cudaStream_t st,
                      StageTimer* tm, const char* tag_spread, const char* tag_fft,
                      const char* tag_interp, uint64_t in_lo = 0, uint64_t in_hi = ~0ull,
                      uint64_t out_lo = 0, uint64_t out_hi = ~0ull,
                      const HermArgs* herm = nullptr, cudaEvent_t before_interp = nullptr) const;
    // addend (optional, pruned path): added per SORTED point after conj_out
    void apply_transpose(const double2* in, double2* out, FftWork& wk, cudaStream_t st,
                         StageTimer* tm, const double2* mult = nullptr, int conj_in = 0,
                         int conj_out = 0, const double2* addend = nullptr) const;
    // Pruned transposed path (nufft.cpp:295-367 restricted to what is nonzero
    // and read), built on first use: tile-owned spread of the output side at
    // its mode coordinates into a compact region, fold with the deconvolution
    // into the transposed band, column transforms, untranspose into the
    // populated rows, row transforms, gather at the point side.
    struct TransposeWork {
        bool ready = false;
        TileGeom tg{};
        DevBuf<uint32_t> rl_s, rl_e;
        DevBuf<double2> b, Z, V, Wt, Tz, G;  // G: full n1 x n2, zero outside the populated rows
        // dense point side (>= 0.25 per band cell): the gather runs the staged
        // tensor-core interpolation over a Z order of the points
        bool morton = false;
        uint32_t m_ntiles = 0;
        int m_shift = 0;
        DevBuf<uint32_t> m_tiles, m_src, m_dst;  // Z position -> sorted point / output index
        DevBuf<double2> m_t, m_phase;            // positions, prephase x mult in Z order
        const double2* m_mult_of = nullptr;      // the mult m_phase was formed with
    };
    mutable TransposeWork tpw;
    void apply_transpose_pruned(const double2* in, double2* out, cudaStream_t st, StageTimer* tm,
                                const double2* mult, int conj_in, int conj_out, const double2* addend) const;
    void ensure_work(FftWork& wk, cudaStream_t st) const;
    // In-place unnormalised e^{+2 pi i} 2D transform of a full n1 x n2 grid
    // (FFTW_BACKWARD, nufft.cpp:207-213, 252).
    void full_transform(double2* grid, cudaStream_t st) const;
    // Drop the point-side permutation: the caller promises to pass point-side
    // data in this plan's sorted order from now on. Returns the permutation
    // (sorted position -> caller index) on the host.
    std::vector<uint32_t> adopt_point_order(cudaStream_t st);
};

// Real-input half split (op.cpp): when the device flag is nonzero at kernel
// time, the xi-side interpolation computes only the first `n` sorted outputs
// (the tag-0 half of the antipodal pairs) with multiplier `mult`, the xi-side
// spread reads only the tag-0 points, and the target-side interpolation
// returns 2 Re(.). `clear`: the input gather zeroes the flag when an input has
// a nonzero imaginary part.
struct HermArgs {
    int* flag = nullptr;
    uint64_t n = 0;
    const double2* mult = nullptr;
    bool two_re = false;
    bool clear = false;
    // Hermitian-FFT mode (Plan::enable_hfft): the xi interpolation reads a
    // band stored for columns [0, hcols) only (the rest by conjugate symmetry)
    // and also writes conj(value) to out2[perm2[v]] (the mirrored spread's input)
    int hcols = 0;
    double2* out2 = nullptr;
    const uint32_t* perm2 = nullptr;
    bool hfft = false;  // take the Hermitian-FFT pipelines in apply_pruned
    double* raw_re = nullptr;  // the input gather also writes Re(sorted input) here (the real CSR pass reads it)
};

// Output of the tile-owned spread: mode 0 = complex grid[(row-r0)*pitch +
// col-c0]; 1 = real parts into rgrid rows (same indexing); 2 = transposed
// complex grid[(col-c0)*pitch + row-r0]. Rows < rend and columns < cend are
// written; only the first nby_run tile columns run. pos2/b2: the point
// arrays of the second bin set (nullptr: the first set's arrays).
struct SpreadOut {
    int mode = 0;  // 3 = real rows packed in pairs (row 2k -> Re, 2k+1 -> Im of row k)
    double* rgrid = nullptr;
    size_t pitch = 0;
    int r0 = 0, c0 = 0, rend = 0, cend = 0;
    int nby_run = 0;
    const double2* pos2 = nullptr;
    const double2* b2 = nullptr;
    const uint32_t* src2 = nullptr;  // mirror image -> tag-0 partner (b2 = conj(b[src2]))
    SpreadLists lists;
    int cx0 = 0, ncx_run = 0;  // CTA spread: run region rows [cx0, cx0 + ncx_run) only (0: all)
    NodeGen gen;               // gen.id != nullptr: procedural points (pos / pos2 are not read)
};

// ---------------------------------------------------------------- kernels
// Launchers (kernels.cu). n1/n2 grid sizes, half = w/2.
struct GridGeom {
    int n1, n2;
    double half;
    // rows stored in radix-r first-pass order (k_untangle_dif): mode j at
    // (j mod rad) rad_m + j / rad; rad_magic = ceil(2^32 / rad)
    int rad = 1, rad_m = 0;
    unsigned rad_magic = 0;
};

// procedural ring nodes: xi / w (either may be null) of the ids; the largest
// |a - b| / |a| over n nodes; the plan arrays of ids in a kernel's order
void launch_ring_nodes(const uint32_t* id, uint64_t n, const RingRow* rings, double2* xi, double2* w,
                       cudaStream_t st);
double node_deviation(const double2* a, const double2* b, uint64_t n, cudaStream_t st);
void launch_ring_point_arrays(const NodeGen& gen, uint64_t n, double2* t, double2* pre, cudaStream_t st);
void launch_ring_output_arrays(const NodeGen& gen, uint64_t n, double2* s, double2* post, double2* kappa,
                               double2* kappa_h, cudaStream_t st);
void launch_plan_points(const double2* pts, uint64_t n, Axis ax, Axis ay, double beta,
                        double2* t, double2* pre, cudaStream_t st);
void launch_plan_outputs(const double2* frq, uint64_t n, Axis ax, Axis ay, double sgn,
                         double2* s, double2* post, cudaStream_t st);
void launch_deconv_tables(Axis a, double beta, double* d, cudaStream_t st);
void launch_bin_keys(const double2* pos, uint64_t n, GridGeom g, int tile, uint32_t* keys,
                     cudaStream_t st);
// min/max of the stencil starts ceil(t - w/2): ext = {ixmin, ixmax, iymin, iymax}
void launch_stencil_extent(const double2* pos, uint64_t n, double half, int* ext, cudaStream_t st);
// tag (optional, 0/1 per entry) becomes key bit 31 (Morton keys then use 15
// bits per axis)
void launch_morton_keys(const double2* pos, uint64_t n, double half, int shift, uint32_t* keys,
                        cudaStream_t st, const uint8_t* tag = nullptr);
void launch_tile_keys(const double2* pos, uint64_t n, double half, TileGeom tg, uint32_t* keys,
                      cudaStream_t st, const uint8_t* tag = nullptr);
// start[b] = base + first i with ((key[i] & mask) >> 5) >= b
void launch_bin_bounds(const uint32_t* sorted_keys, uint64_t n, uint32_t nbins, uint32_t* start,
                       cudaStream_t st, uint32_t base = 0, uint32_t mask = 0xffffffffu);
// Tile-owned spread: writes every cell of the tiles (no atomics, no memset).
// bin_start2 (optional): a second bin set over the same tiles (tag-1 points),
// skipped when *herm is nonzero
// variant: NufftOpts::spread_kernel
void launch_spread_tiles(int w, const WindowPoly& win, GridGeom g, TileGeom tg,
                         const uint32_t* bin_start, const double2* b, const double2* pos,
                         double2* grid, cudaStream_t st, const uint32_t* bin_start2 = nullptr,
                         const int* herm = nullptr, const SpreadOut* out = nullptr,
                         const SpreadLists* lists = nullptr, int variant = 0);
// SpreadLists of n points (tile-geometry grid coordinates), entries (base + k) | tagbit
void build_region_lists(const double2* pos, uint64_t n, int w, TileGeom tg, uint32_t base, uint32_t tagbit,
                        DevBuf<uint32_t>& start, DevBuf<uint32_t>& ent, cudaStream_t st);
// Tt[c * n1 + r] = T[(r - rin0) * n2 + m(c)] for r in [r0, r1), c < B,
// m(c) = c (c <= b) else n2 - B + c
// rin > 1: the rows of T are in the (j mod rin) n2/rin + j/rin order a radix-rin first
// pass (launch_dif_rows) + length n2/rin transforms leave
void launch_band_transpose(const double2* T, int n2, int r0, int r1, int b, int B, double2* Tt,
                           int n1, cudaStream_t st, int rin0 = 0, int conj_out = 0, int rin = 1);
// the same with the radix-R first pass of the length n1 column transform folded in:
// Tt[c n1 + s n1/R + k], rows of T counted from r0; tw[m] = e^{+2 pi i m / n1}
void launch_band_transpose_dif(const double2* T, int n2, int r0, int r1, int b, int B, double2* Tt, int n1, int R,
                               const double2* tw, cudaStream_t st, int rin = 1);
void launch_mirror_points(const double2* t, uint64_t n, int n1, int n2, int w, double2* out,
                          cudaStream_t st);
// b[k] = (conj_in ? conj : id)(in[perm ? perm[k] : k]) * phase[k]
void launch_gather_conj_mul(const double2* in, const uint32_t* perm, const double2* phase, int conj_in,
                            double2* b, uint64_t n, cudaStream_t st);
// V[c n1 + (jx mod n1)] = Z[(jx - rlo) pz + (jy - clo)] dx[jx mod n1] dy[jy mod n2] for the band
// modes |jx| <= b1, jy = c (c <= b2) or c - B (else), zero where Z has no cell
void launch_band_fold(const double2* Z, int pz, int rlo, int rhi, int clo, int chi, int b1, int n1, int b2,
                      int B, int n2, const double* dx, const double* dy, double2* V, cudaStream_t st);
// Tz[(r - r0) n2 + m(c)] = Wt[c n1 + r] for r in [r0, r1), c < B (inverse of launch_band_transpose)
void launch_band_untranspose(const double2* Wt, int n1, int r0, int r1, int b, int B, double2* Tz, int n2,
                             cudaStream_t st, int rin = 1);  // rin: Wt's columns in a radix first pass's order
// out[l opitch + q] = in[q ipitch + ((j0 + l) mod nin)] for l < L, q < Q (a
// transposing gather with a wrapped column window; the slab exchanges' packing)
void launch_wrap_transpose(const double2* in, size_t ipitch, int nin, int j0, int L, int Q, double2* out,
                           size_t opitch, cudaStream_t st);
// out[idx[k]] = conj(in[k]) for k < n
void launch_conj_scatter(const double2* in, uint64_t n, const uint32_t* idx, double2* out, cudaStream_t st);
// *flag = 1 if some x[k] has a nonzero imaginary part, else 0
void launch_any_imag(const double2* x, uint64_t n, int* flag, cudaStream_t st);
// packed real rows -> untangled, transposed half band (see kernels.cu)
void launch_untangle_transpose(const double2* T, int n2, int nr, int B, double2* Tt, int n1, int r0,
                               cudaStream_t st);
// the same untangle with the radix-R (3, 5, 9) first pass of the length
// n1 = R M column transform folded in; tw[m] = e^{+2 pi i m / n1}
void launch_untangle_dif(const double2* T, int n2, int nr, int B, double2* Tt, int n1, int r0, int R,
                         const double2* tw, cudaStream_t st, const double* colf = nullptr, int rin = 1);
// radix-R first pass of `rows` contiguous length-n transforms (X -> Y, mode j
// then at (j mod R) n/R + j/R after a batched length n/R pass); columns outside
// [c_lo, c_hi) of X are zero and not read. tw[m] = e^{+2 pi i m / n}
void launch_dif_rows(const double2* X, int rows, int n, int R, int c_lo, int c_hi, const double2* tw, double2* Y,
                     cudaStream_t st);
// Hermitian band rows from half-plane columns -> pairs packed into full rows
void launch_pack_rows(const double2* Y, int n1, int m0, int n2, int b1, int B1, double2* Z, cudaStream_t st);
// the same packing with the radix-R first pass of the length n2 = R M row
// transform folded in (rows in (j mod R) M + j / R order); tw[m] = e^{+2 pi i m / n2}
void launch_pack_dif(const double2* Y, int n1, int m0, int n2, int b1, int B1, double2* Z, int R,
                     const double2* tw, cudaStream_t st, int rin = 1);


// interpolation from a real band grid whose rows are packed in pairs (row r =
// component r & 1 of complex row r >> 1, complex pitch g.n2):
// out[perm?perm[k]:k] = Re(sum taps * dx dy * grid * phase[k]) + addend[k]
void launch_interp_real(int w, const WindowPoly& win, GridGeom g, uint64_t n, const double2* pos,
                        const double2* phase, const double* dx, const double* dy, const double* grid,
                        const uint32_t* perm, const double2* addend, double2* out, cudaStream_t st,
                        const struct InterpTiles* tiles = nullptr, int variant = 0);
// b[k] = in[perm[k]] phase[k] for k in [lo, hi) (zero elsewhere); raw[k] = in[perm[k]].
// clear (optional): set to 0 when some in[k] has a nonzero imaginary part.
void launch_gather_mul(const double2* in, const uint32_t* perm, const double2* phase, double2* b,
                       double2* raw, uint64_t n, cudaStream_t st, uint64_t lo = 0,
                       uint64_t hi = ~0ull, int* clear = nullptr, double* raw_re = nullptr);  // raw_re[k] = Re(in[perm[k]])
void launch_spmv_vec(uint64_t rows, const uint64_t* ro, const uint32_t* cols, const double2* vals,
                     const double2* f, double2* qs, cudaStream_t st, bool accumulate = false);
// f_re (optional): Re(f) as its own array for an f known to be real (q exactly real)
void launch_spmv_vec_real(uint64_t rows, const uint64_t* ro, const uint32_t* cols, const double* vals,
                          const double2* f, double2* qs, cudaStream_t st, const double* f_re = nullptr);
// D' times up to kSpmmMax right-hand sides in one pass over D': column j of
// the set is f + idx[j] * ldf -> qs + idx[j] * ldq. vals_r (Re(D')) replaces
// vals when given.
constexpr int kSpmmMax = 8;
struct SpmmCols {
    int n = 0;
    int idx[kSpmmMax] = {};
};
void launch_spmm(uint64_t rows, const uint64_t* ro, const uint32_t* cols, const double2* vals,
                 const double* vals_r, const double2* f, uint64_t ldf, double2* qs, uint64_t ldq,
                 const SpmmCols& cs, cudaStream_t st);
void sort_by_key(uint32_t* keys, uint32_t* vals, uint64_t n, cudaStream_t st);
void launch_iota(uint32_t* v, uint64_t n, cudaStream_t st);
template <typename T>
void launch_gather(const T* src, const uint32_t* perm, T* dst, uint64_t n, cudaStream_t st);

// spread: grid[...] += (in[perm?perm[k]:k] * phase[k] (* mult[k])) * taps,
// with optional deconv factors folded into the taps.
void launch_spread(int w, const WindowPoly& win, GridGeom g, uint64_t n, const uint32_t* perm,
                   const double2* in, const double2* pos, const double2* phase,
                   const double2* mult, const double* dx, const double* dy, double2* grid,
                   int conj_in, cudaStream_t st);
// interp: out[perm?perm[k]:k] (+)= sum taps * (dx dy) * grid * phase[k] (* mult[k])
// Z-ordered outputs grouped by 32 x 32 stencil-cell block (k_interp_tile):
// block t = sorted positions [start[t], start[t+1]); out_lo = the absolute
// sorted index of the call's first output
struct InterpTiles {
    const uint32_t* start = nullptr;
    uint32_t n = 0;
    int shift = 0;
    uint64_t out_lo = 0;
};
void launch_interp(int w, const WindowPoly& win, GridGeom g, uint64_t n, const double2* pos,
                   const double2* phase, const double2* mult, const double* dx, const double* dy,
                   const double2* grid, const uint32_t* perm, double2* out, int accumulate,
                   int conj_out, cudaStream_t st, const double2* addend = nullptr,
                   bool transposed = false, const InterpTiles* tiles = nullptr,
                   const HermArgs* herm = nullptr, int variant = 0,  // variant: NufftOpts::interp_kernel
                   const NodeGen* gen = nullptr);  // procedural outputs (staged transposed path)
// map[new] = old sorted position: outputs of each Z-order block dealt round-robin
// over the shared-memory banks of the staged real target interpolation
void bank_interleave_outputs(const uint32_t* tile_start, uint32_t ntiles, const double2* pos, uint64_t n, int w,
                             int shift, DevBuf<uint32_t>& map, cudaStream_t st);
// sorted keys -> starts of the runs of equal key >> bits
void build_tile_starts(const uint32_t* sorted_keys, uint64_t n, int bits, DevBuf<uint32_t>& start,
                       uint32_t& ntiles, cudaStream_t st);
// direct sum out[v] = sum_k c_k e^{i sign z_k . f_v}
void launch_ndft(const double2* pts, uint64_t np, const double2* frq, uint64_t nf,
                 const double2* c, int sign, double2* out, cudaStream_t st);
void launch_mul(double2* x, const double2* m, uint64_t n, cudaStream_t st);
void launch_conj(const double2* in, double2* out, uint64_t n, cudaStream_t st);
void launch_spmv(uint64_t rows, const uint64_t* ro, const uint32_t* cols, const double2* vals,
                 const double2* f, double2* q, cudaStream_t st);
void launch_spmv_adjoint(uint64_t rows, const uint64_t* ro, const uint32_t* cols,
                         const double2* vals, const double2* u, double2* q, cudaStream_t st);

} // namespace sbdgpu
