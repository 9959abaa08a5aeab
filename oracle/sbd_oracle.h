/*
 * oracle/sbd_oracle.h -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference's online apply path (CompressedOperator::apply, reference
 * proj/src/conv_operator.cpp:301-309) and of its type-III NUFFT
 * (proj/src/nufft.cpp). Used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the CHECKER only; the product never links it.
 *
 * Parity pinned against: the unmodified reference compiled into
 * oracle/_ref/libsbdref.so (tests/test_oracle.py) and the golden fixtures in
 * tests/golden/ generated from it by tests/golden/make_golden.py.
 *
 * Complex arrays are interleaved (re, im) doubles; points are (x, y) pairs.
 * Functions return 0 on success, nonzero on error (orc_last_error()).
 */
#ifndef SBD_ORACLE_H
#define SBD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_plan orc_plan;
typedef struct orc_op orc_op;

const char* orc_last_error(void);

double orc_bessel_i0(double r);
double orc_kb_window(double beta, double z);
double orc_kb_window_hat(double beta, double w);

/* mode: 0 auto, 1 direct, 2 fast (NufftOptions::Mode, nufft.hpp:18-24). */
orc_plan* orc_plan_create(const double* points, uint64_t np, const double* freqs, uint64_t nf,
                          int sign, double tol, int mode, uint64_t direct_threshold,
                          uint64_t max_grid_bytes);
void orc_plan_free(orc_plan* p);
int orc_plan_apply(const orc_plan* p, const double* coeffs, double* out);
int orc_plan_apply_transpose(const orc_plan* p, const double* values, double* out);
/* geom[0..11] = fast, w, beta, n1, n2, cx, cy, fcx, fcy, gx, gy, cells */
void orc_plan_geometry(const orc_plan* p, double* geom);
int orc_ndft_direct(const double* points, uint64_t np, const double* freqs, uint64_t nf,
                    const double* coeffs, int sign, double* out);

/* SBDOPv1 operator (reference conv_operator.cpp:357-490). */
orc_op* orc_op_open(const char* path, uint64_t max_grid_bytes);
void orc_op_free(orc_op* op);
/* info[0..9] = n_src, n_tgt, n_xi, nnz, single, kind, k, nufft_tol, eps, dmax */
void orc_op_info(const orc_op* op, double* info);
int orc_op_apply(const orc_op* op, const double* f, double* q);
int orc_op_apply_adjoint(const orc_op* op, const double* u, double* q);
/* stage 1: fwd_in(f) -> spectrum (unweighted); 2: fwd_out(spectrum) -> q;
 * 3: q += D f. */
int orc_op_stage(const orc_op* op, int stage, const double* in, double* out);
/* omega-hat (2*n_xi doubles, file order) */
void orc_op_weights(const orc_op* op, double* w);

#ifdef __cplusplus
}
#endif

#endif
