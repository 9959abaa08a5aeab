/*
 * sbd_b200.h -- C ABI of the B200-native Sparse Bessel Decomposition apply path.
 *
 * Drop-in boundary for the reference C++ library's online path (reference:
 * /root/reference/proj/include/sbd/conv_operator.hpp and nufft.hpp). Plain
 * pointers and sizes only; complex arrays are interleaved (re, im) float64
 * exactly like std::complex<double> (reference vec2.hpp:8), points are (x, y)
 * float64 pairs exactly like sbd::Vec2 (vec2.hpp:10-23).
 *
 * Every entry point returns an int status (SBD_OK = 0). On failure the
 * thread-local message is available from sbd_last_error(). The C++ wrapper in
 * sbd_b200.hpp maps the codes back onto the exception types the reference
 * throws (conv_operator.cpp:246-247, 265, 303; nufft.cpp:158-160, 387-388).
 *
 * Entry point                     replaces (reference file:line)
 * ------------------------------  -----------------------------------------------
 * sbd_op_assemble                 CompressedOperator::assemble  conv_operator.cpp:244-294
 * sbd_op_load / sbd_op_save       CompressedOperator::load/save conv_operator.cpp:449-490 / 357-397
 * sbd_op_apply                    CompressedOperator::apply     conv_operator.cpp:301-309
 * sbd_op_apply_adjoint            CompressedOperator::apply_adjoint conv_operator.cpp:311-324
 * sbd_op_apply_device[_adjoint]   (same, device buffers on a caller stream; no reference analogue)
 * sbd_op_info / sbd_op_get        accessors + bytes()           conv_operator.hpp:56-70
 * sbd_nufft_create/apply/...      NufftPlan ctor/apply/apply_transpose nufft.cpp:369-398
 * sbd_ndft_direct                 ndft_direct                   nufft.cpp:76-93
 * sbd_choose_parameters           choose_parameters             conv_operator.cpp:121-133
 */
#ifndef SBD_B200_H
#define SBD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum sbd_status {
    SBD_OK = 0,
    SBD_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    SBD_ERR_DOMAIN = 2,           /* std::domain_error */
    SBD_ERR_RUNTIME = 3,          /* std::runtime_error */
    SBD_ERR_CUDA = 4,             /* CUDA / cuFFT failure (no reference analogue) */
    SBD_ERR_CONVERGENCE = 5       /* SbdConvergenceError (sbd.hpp:31-38) */
};

enum sbd_kernel_kind { SBD_KERNEL_LAPLACE = 0, SBD_KERNEL_HELMHOLTZ = 1 };

typedef struct sbd_op sbd_op;
typedef struct sbd_nufft sbd_nufft;

/* Pipeline options of an operator (no reference analogue: the reference has
 * one CPU code path). Every combination computes the same operator within
 * the parity bar; the defaults are the fastest path. They replace the
 * process-wide environment switches of earlier builds. */
typedef struct sbd_op_options {
    int real_input_split;  /* 1: for real f on an operator with real omega-hat and antipodally
                              paired rings, compute one node of each pair (q = 2 Re(.)). Default 1 */
    int hermitian_fft;     /* 1: on top of the split, transform half the grid (real f known on the
                              host, or passed as a hint). Default 1 */
    int radix_first_pass;  /* -1: fold a radix-3/5/9 first FFT pass into our kernels when n > 4096
                              (default); 0: never; 1: whenever n factorises (tests) */
    int spread_kernel;     /* 0: CTA spread over plan-time region lists (default); 1: CTA spread
                              over the tile bins; 2: per-warp DMMA spread; 3: scalar tiles */
    int interp_kernel;     /* 0: automatic (default); 1: staged DMMA tiles; 2: DMMA per warp;
                              3: scalar */
    int fused;             /* 1: fused forward path (renumbered D, omega-hat folded into the
                              xi interpolation). Default 1 */
    int verbose;           /* 1: setup diagnostics on stderr. Default 0 */
    int procedural_rings;  /* 1: the xi nodes are regenerated inside the xi-side kernels from
                              (rho_p, M_p, weight_p, j) (ring_quadrature.cpp:24-69) and their
                              per-node arrays (coordinates, phases, omega-hat: ~170 B per node)
                              are not kept in HBM; needs ring-generated nodes (else stays off,
                              see sbd_op_info_t.procedural_rings) and the fused path. The other
                              paths (adjoint, sharded, slab) rebuild the arrays on first use.
                              Default 0: the kernels are issue-bound, not HBM-bound, so the
                              regeneration costs time; the mode trades it for capacity */
} sbd_op_options;

void sbd_op_options_default(sbd_op_options* o);

/* AssembleOptions (conv_operator.hpp:24-31) plus the device ordinal and the
 * pipeline options. */
typedef struct sbd_assemble_options {
    double eps;                      /* 1e-6 */
    double alpha;                    /* 0 */
    double a_override;               /* 0: N-based rule (conv_operator.cpp:263-269) */
    double small_k_factor;           /* 0.5 */
    uint64_t nufft_direct_threshold; /* 2^20 */
    uint64_t max_grid_bytes;         /* 4 GiB */
    int device;                      /* CUDA ordinal */
    sbd_op_options pipeline;         /* sbd_op_options_default */
} sbd_assemble_options;

typedef struct sbd_op_info_t {
    uint64_t n_src, n_tgt, n_xi, nnz;
    int single_cloud, kind;
    double k, eps, alpha, a, delta_min, delta_max, nufft_tol;
    int P;                           /* SBD order */
    int w;                           /* NUFFT kernel width (both plans) */
    double beta;                     /* KB shape parameter */
    int n1_in, n2_in, n1_out, n2_out; /* oversampled grids (0 on the direct path) */
    int fast_in, fast_out;           /* fast (gridded) vs direct path per plan */
    uint64_t bytes;                  /* CompressedOperator::bytes() (conv_operator.cpp:338-353) */
    uint64_t device_bytes;           /* HBM actually held by this operator */
    int procedural_rings;            /* 1: the xi-side kernels regenerate the ring nodes */
} sbd_op_info_t;

const char* sbd_last_error(void);
const char* sbd_version(void);

void sbd_assemble_options_default(sbd_assemble_options* o);

/* ---- operator lifecycle ---- */
int sbd_op_assemble(int kind, double k, const double* src_xy, uint64_t n_src,
                    const double* tgt_xy /* NULL: single cloud */, uint64_t n_tgt,
                    const sbd_assemble_options* opts, sbd_op** out);
int sbd_op_load(const char* path, int device, uint64_t max_grid_bytes /* 0: 4 GiB */,
                sbd_op** out);
/* The same with pipeline options (NULL: defaults). Rejects files whose CSR or
 * ring arrays are inconsistent (SBD_ERR_RUNTIME) before anything is uploaded. */
int sbd_op_load_ex(const char* path, int device, uint64_t max_grid_bytes,
                   const sbd_op_options* options, sbd_op** out);
int sbd_op_save(const sbd_op* op, const char* path);
int sbd_op_destroy(sbd_op* op);
int sbd_op_info(const sbd_op* op, sbd_op_info_t* info);

/* Copies an operator array to host memory. which: 0 src points (2*n_src),
 * 1 tgt points (2*n_tgt), 2 freqs (2*n_xi), 3 weights (2*n_xi),
 * 4 D row_offsets (u64, n_tgt+1), 5 D cols (u32, nnz), 6 D values (2*nnz),
 * 7 ring_offsets (i32), 8 SBD coeffs, 9 SBD roots, 10 SBD norm constants.
 * With dst == NULL only *count (elements of the natural type) is written. */
int sbd_op_get(const sbd_op* op, int which, void* dst, uint64_t* count);

/* ---- the hot path ---- */
/* Concurrency: calls on one operator from several host threads are safe
 * (reference conv_operator.hpp:33-36); they are serialised, and device work
 * of successive calls is ordered across streams by an operator event. */
/* q = A f for nrhs right-hand sides stored back to back (f: nrhs x n_src,
 * q: nrhs x n_tgt, interleaved complex). Host buffers; the H2D of f and the
 * D2H of q are inside the call (synchronous: use sbd_op_apply_async to overlap
 * them with neighbouring applies); realness of f is detected on the host. */
int sbd_op_apply(sbd_op* op, const double* f, double* q, int nrhs);
int sbd_op_apply_adjoint(sbd_op* op, const double* u, double* q, int nrhs);
/* Pipelined host-buffer apply (no reference analogue): enqueues the H2D of f,
 * the apply and the D2H of q, and returns a ticket; sbd_op_wait(ticket) blocks
 * until q is in host memory. Consecutive calls overlap the copies of one call
 * with the device work of its neighbours (two staging slots, two copy
 * streams). f must stay unchanged and q untouched until the wait; pinned
 * host memory gives asynchronous copies. */
int sbd_op_apply_async(sbd_op* op, const double* f, double* q, int nrhs, uint64_t* ticket);
int sbd_op_wait(sbd_op* op, uint64_t ticket);
/* Same on device buffers, enqueued on `stream` (a cudaStream_t; NULL is the
 * legacy default stream, as everywhere in CUDA). Returns without
 * synchronising (and is CUDA-graph capturable). Whether f is real is decided
 * on the device, so the Hermitian-FFT mode (which needs it on the host) is
 * not used; sbd_op_apply_device_ex takes the caller's knowledge instead. */
int sbd_op_apply_device(sbd_op* op, const double* d_f, double* d_q, int nrhs, void* stream);
/* f_is_real: nrhs entries, 1 = column is real (must be: an imaginary part is
 * then ignored), 0 = complex, -1 = unknown (decided on the device); NULL = all
 * unknown. Never synchronises. */
int sbd_op_apply_device_ex(sbd_op* op, const double* d_f, double* d_q, int nrhs, void* stream,
                           const int* f_is_real);
int sbd_op_apply_adjoint_device(sbd_op* op, const double* d_u, double* d_q, int nrhs,
                                void* stream);

/* ---- multi-GPU building blocks (north_star scheme) ----
 * One apply split over G devices, each holding the same operator:
 *   spec_r = sbd_op_forward_spectrum(f, source shard r)   (sources sharded)
 *   spec   = sum_r spec_r                                  (one allreduce of n_xi complex)
 *   q[T_r] = sbd_op_backward_targets(spec, f, target shard r)  (targets + D rows sharded)
 * Shards are ranges of the operator's spatially sorted source / target
 * orders; sbd_op_shard_bounds returns an even split (side 0 sources, 1
 * targets) as nshards+1 bounds. `spec` has n_xi complex entries in the
 * operator's internal xi order and already carries omega-hat and the
 * second NUFFT's prephase. Requires both NUFFTs on the gridded path. */
int sbd_op_shard_bounds(const sbd_op* op, int side, int nshards, uint64_t* bounds);
/* Number n of leading spectrum entries that sbd_op_forward_spectrum writes
 * and sbd_op_backward_targets reads for this (device) f: n_xi, or, for a real
 * f on an operator with real omega-hat and antipodally paired rings, the
 * computed half of the pairs (the real-input half split; the all-reduce then
 * moves n complex values). Runs one reduction over f and syncs `stream` (the
 * only host round trip of a sharded apply); the decision is kept for the
 * following forward/backward calls on this f. */
int sbd_op_spectrum_length(sbd_op* op, const double* d_f, void* stream, uint64_t* n);
int sbd_op_forward_spectrum(sbd_op* op, const double* d_f, uint64_t src_lo, uint64_t src_hi,
                            double* d_spec, void* stream);
int sbd_op_backward_targets(sbd_op* op, const double* d_spec, const double* d_f, uint64_t tgt_lo,
                            uint64_t tgt_hi, double* d_q, void* stream);

/* ---- slab decomposition of one apply over `world` devices ----
 * No stage is replicated: rank r spreads the sources into its row slab of the
 * first grid, exchanges band columns (all-to-all 0), interpolates the xi
 * nodes of its slab of the second grid and spreads them, exchanges band rows
 * (all-to-all 1), and evaluates its targets. Per apply:
 *   stage 0: d_f (all sources, caller order)    -> d_out = send buffer of exchange 0
 *   (all-to-all 0: send counts/offsets from sbd_slab_counts(s, 0, ...))
 *   stage 1: d_in = receive buffer of exchange 0 -> d_out = send buffer of exchange 1
 *   (all-to-all 1)
 *   stage 2: d_in = receive buffer of exchange 1, d_f -> d_out = q (caller order; only
 *            this rank's targets are written)
 * Counts are complex elements per peer (send[k]: to rank k; recv[k]: from rank k);
 * buffers hold them back to back in rank order. Complex pipeline (every xi node).
 * Requires both NUFFTs on the gridded path. */
typedef struct sbd_slab sbd_slab;
int sbd_slab_create(sbd_op* op, int rank, int world, sbd_slab** out);
int sbd_slab_destroy(sbd_slab* s);
int sbd_slab_counts(const sbd_slab* s, int exchange, uint64_t* send_counts, uint64_t* recv_counts);
int sbd_slab_stage(sbd_slab* s, int stage, const double* d_in, const double* d_f, double* d_out, void* stream);

/* Per-stage CUDA-event timing of every apply since profiling was enabled (or
 * since the last reset). names: "spread_src", "fft_in", "interp_xi",
 * "spread_xi", "fft_out", "interp_tgt", "spmv", ... ms[i] in milliseconds.
 * Returns the number of records. */
int sbd_op_set_profiling(sbd_op* op, int enable);
int sbd_op_stage_times(sbd_op* op, double* ms, const char** names, int cap);
int sbd_op_stage_times_reset(sbd_op* op);

/* Exact diameter of a point cloud (make_cloud, point_cloud.cpp:13-65). */
double sbd_cloud_diameter(const double* xy, uint64_t n);

/* ---- standalone type-III NUFFT (NufftPlan) ---- */
/* mode: 0 Auto, 1 Direct, 2 Fast (nufft.hpp:18-24). */
int sbd_nufft_create(const double* points, uint64_t np, const double* freqs, uint64_t nf, int sign,
                     double tol, int mode, uint64_t direct_threshold, uint64_t max_grid_bytes,
                     int device, sbd_nufft** out);
int sbd_nufft_apply(sbd_nufft* p, const double* coeffs, double* out);
int sbd_nufft_apply_transpose(sbd_nufft* p, const double* values, double* out);
/* fast, w, n1, n2 (n1 = n2 = 0 on the direct path) */
int sbd_nufft_info(const sbd_nufft* p, int* fast, int* w, int* n1, int* n2);
int sbd_nufft_destroy(sbd_nufft* p);

int sbd_ndft_direct(const double* points, uint64_t np, const double* freqs, uint64_t nf,
                    const double* coeffs, int sign, int device, double* out);

/* choose_parameters (conv_operator.cpp:121-133). */
int sbd_choose_parameters(uint64_t n, double eps, double alpha, double* a, int* p_hint);

/* Number of CUDA kernels this library launched since load (process-wide). */
uint64_t sbd_kernel_launch_count(void);

/* Diagnostics: sup-norm error of the device Kaiser-Bessel window polynomials
 * for width w and shape beta, relative to the window peak I0(beta). */
double sbd_window_fit_error(int w, double beta);

/* Diagnostics: the host Bessel functions of the offline assembly.
 * which: 0 J0, 1 J1, 2 Y0, 3 Y1. NaN on a domain error. */
double sbd_bessel(int which, double x);

#ifdef __cplusplus
}
#endif

#endif
