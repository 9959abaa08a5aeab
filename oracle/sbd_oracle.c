/*
 * oracle/sbd_oracle.c -- TEST INFRASTRUCTURE ONLY. Plain-C restatement of the
 * reference's apply path; see sbd_oracle.h for the contract. Each function
 * cites the reference file:line it restates (paths under /root/reference/proj).
 */
#define _POSIX_C_SOURCE 200809L
#include "sbd_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fft235.h"

static _Thread_local char g_err[256];

static int seterr(const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return 1;
}

const char* orc_last_error(void) { return g_err; }

static const double kPi = 3.14159265358979323846;
static const double kSigma = 2.0; /* nufft.cpp:19 */

/* bessel.cpp:216-227 -- power series, all terms positive. */
double orc_bessel_i0(double r) {
    r = fabs(r);
    const double q = 0.25 * r * r;
    double term = 1.0, sum = 1.0;
    for (int m = 1; m < 128; ++m) {
        term *= q / ((double)m * (double)m);
        sum += term;
        if (term < 1e-17 * sum) break;
    }
    return sum;
}

/* nufft.cpp:28-32 */
double orc_kb_window(double beta, double z) {
    const double s = 1.0 - z * z;
    if (s <= 0.0) return s == 0.0 ? 1.0 : 0.0;
    return orc_bessel_i0(beta * sqrt(s));
}

/* nufft.cpp:34-45 */
double orc_kb_window_hat(double beta, double w) {
    const double s2 = beta * beta - w * w;
    if (s2 > 1e-12) {
        const double s = sqrt(s2);
        return 2.0 * sinh(s) / s;
    }
    if (s2 < -1e-12) {
        const double s = sqrt(-s2);
        return 2.0 * sin(s) / s;
    }
    return 2.0 * (1.0 + s2 / 6.0);
}

/* nufft.cpp:47-52 */
static int width_for_tol(double tol) {
    const double digits = -log10(tol > 1e-15 ? tol : 1e-15);
    int w = (int)ceil(digits) + 2;
    return w < 4 ? 4 : (w > 17 ? 17 : w);
}

/* nufft.cpp:55-63 */
static int next_fast_even(int n) {
    n += n & 1;
    for (;; n += 2) {
        int m = n;
        while (m % 2 == 0) m /= 2;
        while (m % 3 == 0) m /= 3;
        while (m % 5 == 0) m /= 5;
        if (m == 1) return n;
    }
}

typedef struct {
    double center, fcenter, gamma;
    int n;
    double alpha1, alpha2;
} axis_t; /* nufft.cpp:65-72 */

struct orc_plan {
    int sign, fast;
    uint64_t np, nf;
    double *points, *freqs; /* direct path copies */
    int w;
    double beta;
    axis_t ax, ay;
    double *tx, *ty, *pre;   /* pre: interleaved complex */
    double *sx, *sy, *post;  /* post: interleaved complex */
    double *dx, *dy;         /* deconvolution factors */
};

/* nufft.cpp:76-93 */
int orc_ndft_direct(const double* points, uint64_t np, const double* freqs, uint64_t nf,
                    const double* coeffs, int sign, double* out) {
    const double s = sign > 0 ? 1.0 : -1.0;
    for (uint64_t v = 0; v < nf; ++v) {
        const double fx = s * freqs[2 * v], fy = s * freqs[2 * v + 1];
        double ar = 0.0, ai = 0.0;
        for (uint64_t k = 0; k < np; ++k) {
            const double phase = points[2 * k] * fx + points[2 * k + 1] * fy;
            const double c = cos(phase), sn = sin(phase);
            const double cr = coeffs[2 * k], ci = coeffs[2 * k + 1];
            ar += cr * c - ci * sn;
            ai += cr * sn + ci * c;
        }
        out[2 * v] = ar;
        out[2 * v + 1] = ai;
    }
    return 0;
}

static void span(const double* v, uint64_t n, int comp, double s, double* lo, double* hi) {
    *lo = 1e300;
    *hi = -1e300;
    for (uint64_t i = 0; i < n; ++i) {
        const double x = s * v[2 * i + comp];
        if (x < *lo) *lo = x;
        if (x > *hi) *hi = x;
    }
    if (n == 0) *lo = *hi = 0.0;
}

/* nufft.cpp:139-155 */
static void setup_axis(orc_plan* p, axis_t* a, int comp) {
    double plo, phi, flo, fhi;
    span(p->points, p->np, comp, 1.0, &plo, &phi);
    span(p->freqs, p->nf, comp, (double)p->sign, &flo, &fhi);
    a->center = 0.5 * (plo + phi);
    a->fcenter = 0.5 * (flo + fhi);
    double X = 0.5 * (phi - plo), Xf = 1e-8 * (1.0 + fabs(a->center));
    double S = 0.5 * (fhi - flo), Sf = 1e-8 * (1.0 + fabs(a->fcenter));
    if (Xf > X) X = Xf;
    if (Sf > S) S = Sf;
    a->gamma = kSigma * X / kPi;
    a->n = next_fast_even((int)ceil(2.0 * kSigma * (a->gamma * S + 0.5 * p->w + 1.0)));
    a->alpha1 = kPi * p->w / a->n;
    a->alpha2 = 0.5 * p->w / a->gamma;
}

/* nufft.cpp:194-205 */
static double* make_deconv(const orc_plan* p, const axis_t* a) {
    double* d = (double*)calloc((size_t)a->n, sizeof(double));
    const int band = a->n / (int)(2.0 * kSigma);
    for (int m = 0; m < a->n; ++m) {
        const int j = m <= a->n / 2 ? m : m - a->n;
        if (abs(j) > band) continue;
        const double psi1 = a->alpha1 * orc_kb_window_hat(p->beta, a->alpha1 * j);
        d[m] = ((j & 1) ? -1.0 : 1.0) / psi1;
    }
    return d;
}

/* nufft.cpp:127-216 (build_fast) */
static int build_fast(orc_plan* p, double tol, uint64_t max_grid_bytes) {
    p->w = width_for_tol(tol);
    p->beta = 2.3562 * p->w;
    setup_axis(p, &p->ax, 0);
    setup_axis(p, &p->ay, 1);
    const uint64_t cells = (uint64_t)p->ax.n * (uint64_t)p->ay.n;
    if (cells * 16u > max_grid_bytes) return seterr("nufft: oversampled grid exceeds the memory limit");

    p->tx = (double*)malloc(sizeof(double) * (p->np + 1));
    p->ty = (double*)malloc(sizeof(double) * (p->np + 1));
    p->pre = (double*)malloc(sizeof(double) * 2 * (p->np + 1));
    for (uint64_t k = 0; k < p->np; ++k) {
        const double px = p->points[2 * k] - p->ax.center;
        const double py = p->points[2 * k + 1] - p->ay.center;
        const double ux = px / p->ax.gamma, uy = py / p->ay.gamma;
        p->tx[k] = (ux + kPi) * p->ax.n / (2.0 * kPi);
        p->ty[k] = (uy + kPi) * p->ay.n / (2.0 * kPi);
        const double phase = px * p->ax.fcenter + py * p->ay.fcenter;
        const double dec = (p->ax.alpha2 * orc_kb_window_hat(p->beta, p->ax.alpha2 * px)) *
                           (p->ay.alpha2 * orc_kb_window_hat(p->beta, p->ay.alpha2 * py));
        /* cplx(cos, sin) / dec  (std::complex / double divides each part) */
        p->pre[2 * k] = cos(phase) / dec;
        p->pre[2 * k + 1] = sin(phase) / dec;
    }
    p->sx = (double*)malloc(sizeof(double) * (p->nf + 1));
    p->sy = (double*)malloc(sizeof(double) * (p->nf + 1));
    p->post = (double*)malloc(sizeof(double) * 2 * (p->nf + 1));
    const double cx = 2.0 * kPi / (p->ax.n * p->ax.gamma);
    const double cy = 2.0 * kPi / (p->ay.n * p->ay.gamma);
    const double s = (double)p->sign;
    for (uint64_t v = 0; v < p->nf; ++v) {
        const double fx = s * p->freqs[2 * v], fy = s * p->freqs[2 * v + 1];
        p->sx[v] = p->ax.gamma * (fx - p->ax.fcenter);
        p->sy[v] = p->ay.gamma * (fy - p->ay.fcenter);
        const double phase = p->ax.center * fx + p->ay.center * fy;
        p->post[2 * v] = cos(phase) * (cx * cy);
        p->post[2 * v + 1] = sin(phase) * (cx * cy);
    }
    p->dx = make_deconv(p, &p->ax);
    p->dy = make_deconv(p, &p->ay);
    p->fast = 1;
    return 0;
}

/* nufft.cpp:369-380 (ctor + Auto/Direct/Fast decision) */
orc_plan* orc_plan_create(const double* points, uint64_t np, const double* freqs, uint64_t nf,
                          int sign, double tol, int mode, uint64_t direct_threshold,
                          uint64_t max_grid_bytes) {
    orc_plan* p = (orc_plan*)calloc(1, sizeof(orc_plan));
    p->sign = sign > 0 ? 1 : -1;
    p->np = np;
    p->nf = nf;
    p->points = (double*)malloc(sizeof(double) * 2 * (np + 1));
    p->freqs = (double*)malloc(sizeof(double) * 2 * (nf + 1));
    if (np) memcpy(p->points, points, sizeof(double) * 2 * np);
    if (nf) memcpy(p->freqs, freqs, sizeof(double) * 2 * nf);
    const uint64_t work = np * nf;
    const int direct = mode == 1 || (mode == 0 && work <= direct_threshold);
    if (!direct && build_fast(p, tol, max_grid_bytes) != 0) {
        orc_plan_free(p);
        return NULL;
    }
    return p;
}

void orc_plan_free(orc_plan* p) {
    if (!p) return;
    free(p->points); free(p->freqs);
    free(p->tx); free(p->ty); free(p->pre);
    free(p->sx); free(p->sy); free(p->post);
    free(p->dx); free(p->dy);
    free(p);
}

void orc_plan_geometry(const orc_plan* p, double* g) {
    g[0] = p->fast; g[1] = p->w; g[2] = p->beta;
    g[3] = p->ax.n; g[4] = p->ay.n;
    g[5] = p->ax.center; g[6] = p->ay.center;
    g[7] = p->ax.fcenter; g[8] = p->ay.fcenter;
    g[9] = p->ax.gamma; g[10] = p->ay.gamma;
    g[11] = (double)p->ax.n * (double)p->ay.n;
}

static inline int wrap(int i, int n) { return ((i % n) + n) % n; }

/* Spread: nufft.cpp:229-250 (also :308-326 with the roles of the two sides
 * swapped). b_k = c_k * phase_k; separable KB taps with periodic wrap. */
static void spread(const orc_plan* p, uint64_t count, const double* c, const double* phase,
                   const double* t1, const double* t2, double* g) {
    const int w = p->w, n1 = p->ax.n, n2 = p->ay.n;
    const double half = 0.5 * w;
    double wx[32], wy[32];
    for (uint64_t k = 0; k < count; ++k) {
        const double br = c[2 * k] * phase[2 * k] - c[2 * k + 1] * phase[2 * k + 1];
        const double bi = c[2 * k] * phase[2 * k + 1] + c[2 * k + 1] * phase[2 * k];
        if (br == 0.0 && bi == 0.0) continue;
        const int ix0 = (int)ceil(t1[k] - half), iy0 = (int)ceil(t2[k] - half);
        for (int i = 0; i < w; ++i) {
            wx[i] = orc_kb_window(p->beta, (ix0 + i - t1[k]) / half);
            wy[i] = orc_kb_window(p->beta, (iy0 + i - t2[k]) / half);
        }
        for (int i = 0; i < w; ++i) {
            const int mx = wrap(ix0 + i, n1);
            const double bxr = br * wx[i], bxi = bi * wx[i];
            double* row = g + 2 * (size_t)mx * n2;
            for (int j = 0; j < w; ++j) {
                const int my = wrap(iy0 + j, n2);
                row[2 * my] += bxr * wy[j];
                row[2 * my + 1] += bxi * wy[j];
            }
        }
    }
}

/* Interpolate: nufft.cpp:262-283 (row partial first, then x weight). */
static void interp(const orc_plan* p, uint64_t count, const double* s1, const double* s2,
                   const double* phase, const double* g, double* out) {
    const int w = p->w, n1 = p->ax.n, n2 = p->ay.n;
    const double half = 0.5 * w;
    double wx[32], wy[32];
    for (uint64_t v = 0; v < count; ++v) {
        const int jx0 = (int)ceil(s1[v] - half), jy0 = (int)ceil(s2[v] - half);
        for (int i = 0; i < w; ++i) {
            wx[i] = orc_kb_window(p->beta, (jx0 + i - s1[v]) / half);
            wy[i] = orc_kb_window(p->beta, (jy0 + i - s2[v]) / half);
        }
        double ar = 0.0, ai = 0.0;
        for (int i = 0; i < w; ++i) {
            const int mx = wrap(jx0 + i, n1);
            const double* row = g + 2 * (size_t)mx * n2;
            double rr = 0.0, ri = 0.0;
            for (int j = 0; j < w; ++j) {
                const int my = wrap(jy0 + j, n2);
                rr += row[2 * my] * wy[j];
                ri += row[2 * my + 1] * wy[j];
            }
            ar += rr * wx[i];
            ai += ri * wx[i];
        }
        out[2 * v] = ar * phase[2 * v] - ai * phase[2 * v + 1];
        out[2 * v + 1] = ar * phase[2 * v + 1] + ai * phase[2 * v];
    }
}

/* Deconvolution: nufft.cpp:254-260 (forward: out-of-band rows left alone) and
 * :328-335 (transpose: out-of-band rows zeroed). */
static void deconv(const orc_plan* p, double* g, int zero_out_of_band) {
    const int n1 = p->ax.n, n2 = p->ay.n;
    for (int mx = 0; mx < n1; ++mx) {
        const double dx = p->dx[mx];
        double* row = g + 2 * (size_t)mx * n2;
        if (dx == 0.0) {
            if (zero_out_of_band) memset(row, 0, sizeof(double) * 2 * (size_t)n2);
            continue;
        }
        for (int my = 0; my < n2; ++my) {
            const double f = dx * p->dy[my];
            row[2 * my] *= f;
            row[2 * my + 1] *= f;
        }
    }
}

/* nufft.cpp:218-290 */
int orc_plan_apply(const orc_plan* p, const double* coeffs, double* out) {
    if (!p->fast) return orc_ndft_direct(p->points, p->np, p->freqs, p->nf, coeffs, p->sign, out);
    const size_t cells = (size_t)p->ax.n * p->ay.n;
    double* g = (double*)calloc(2 * cells, sizeof(double));
    if (!g) return seterr("oracle: grid allocation failed");
    spread(p, p->np, coeffs, p->pre, p->tx, p->ty, g);
    fft235_2d_inplace(p->ax.n, p->ay.n, +1, g);
    deconv(p, g, 0);
    interp(p, p->nf, p->sx, p->sy, p->post, g, out);
    free(g);
    return 0;
}

/* nufft.cpp:295-367 */
int orc_plan_apply_transpose(const orc_plan* p, const double* values, double* out) {
    if (!p->fast) return orc_ndft_direct(p->freqs, p->nf, p->points, p->np, values, p->sign, out);
    const size_t cells = (size_t)p->ax.n * p->ay.n;
    double* g = (double*)calloc(2 * cells, sizeof(double));
    if (!g) return seterr("oracle: grid allocation failed");
    spread(p, p->nf, values, p->post, p->sx, p->sy, g);
    deconv(p, g, 1);
    fft235_2d_inplace(p->ax.n, p->ay.n, +1, g);
    interp(p, p->np, p->tx, p->ty, p->pre, g, out);
    free(g);
    return 0;
}

/* ---------------- operator (conv_operator.cpp) ---------------- */

struct orc_op {
    int kind, single;
    double k, eps, alpha, a, dmin, dmax, nufft_tol;
    uint64_t n_src, n_tgt, n_xi, nnz;
    double *src, *tgt, *freqs, *weights;
    uint64_t* row_offsets;
    uint32_t* cols;
    double* values;
    orc_plan *fwd_in, *fwd_out;
};

static int rd(FILE* f, void* dst, size_t bytes) { return fread(dst, 1, bytes, f) == bytes ? 0 : 1; }

static void* rdvec(FILE* f, size_t elem, uint64_t* count, int* bad) {
    uint64_t n = 0;
    if (rd(f, &n, 8)) { *bad = 1; return NULL; }
    void* p = malloc(elem * n + 16);
    if (!p || (n && rd(f, p, elem * n))) { *bad = 1; free(p); return NULL; }
    if (count) *count = n;
    return p;
}

/* conv_operator.cpp:449-490 (load) + :162-167 (build_forward_plans). */
orc_op* orc_op_open(const char* path, uint64_t max_grid_bytes) {
    FILE* f = fopen(path, "rb");
    if (!f) { seterr("load: cannot open"); return NULL; }
    char magic[8];
    int bad = rd(f, magic, 8) || memcmp(magic, "SBDOPv1", 8) != 0;
    if (bad) { fclose(f); seterr("load: not an operator file (bad magic)"); return NULL; }
    orc_op* op = (orc_op*)calloc(1, sizeof(orc_op));
    int32_t kind = 0;
    uint8_t single = 0;
    double diam;
    bad |= rd(f, &kind, 4) | rd(f, &op->k, 8) | rd(f, &single, 1);
    op->kind = kind;
    op->single = single;
    bad |= rd(f, &op->eps, 8) | rd(f, &op->alpha, 8) | rd(f, &op->a, 8) | rd(f, &op->dmin, 8) |
           rd(f, &op->dmax, 8) | rd(f, &op->nufft_tol, 8);
    op->src = (double*)rdvec(f, 16, &op->n_src, &bad);
    bad |= rd(f, &diam, 8);
    if (!single) {
        op->tgt = (double*)rdvec(f, 16, &op->n_tgt, &bad);
        bad |= rd(f, &diam, 8);
    } else {
        op->n_tgt = op->n_src;
    }
    op->freqs = (double*)rdvec(f, 16, &op->n_xi, &bad);
    uint64_t nw = 0, nr = 0, nrow = 0, nc = 0, nv = 0;
    op->weights = (double*)rdvec(f, 16, &nw, &bad);
    free(rdvec(f, 4, &nr, &bad)); /* ring_offsets: not needed by apply */
    double budget;
    bad |= rd(f, &budget, 8);
    op->row_offsets = (uint64_t*)rdvec(f, 8, &nrow, &bad);
    op->cols = (uint32_t*)rdvec(f, 4, &nc, &bad);
    op->values = (double*)rdvec(f, 16, &nv, &bad);
    op->nnz = nv;
    fclose(f);
    if (bad || nw != op->n_xi || nrow != op->n_tgt + 1 || nc != nv) {
        orc_op_free(op);
        seterr("load: truncated operator file");
        return NULL;
    }
    const double* tgt = op->single ? op->src : op->tgt;
    const uint64_t direct_threshold = (uint64_t)1 << 20;
    if (!max_grid_bytes) max_grid_bytes = (uint64_t)4 << 30;
    op->fwd_in = orc_plan_create(op->src, op->n_src, op->freqs, op->n_xi, -1, op->nufft_tol, 0,
                                 direct_threshold, max_grid_bytes);
    op->fwd_out = orc_plan_create(op->freqs, op->n_xi, tgt, op->n_tgt, +1, op->nufft_tol, 0,
                                  direct_threshold, max_grid_bytes);
    if (!op->fwd_in || !op->fwd_out) {
        orc_op_free(op);
        return NULL;
    }
    return op;
}

void orc_op_free(orc_op* op) {
    if (!op) return;
    orc_plan_free(op->fwd_in);
    orc_plan_free(op->fwd_out);
    free(op->src); free(op->tgt); free(op->freqs); free(op->weights);
    free(op->row_offsets); free(op->cols); free(op->values);
    free(op);
}

void orc_op_info(const orc_op* op, double* info) {
    info[0] = (double)op->n_src; info[1] = (double)op->n_tgt; info[2] = (double)op->n_xi;
    info[3] = (double)op->nnz; info[4] = op->single; info[5] = op->kind; info[6] = op->k;
    info[7] = op->nufft_tol; info[8] = op->eps; info[9] = op->dmax;
}

/* point_cloud.cpp:116-123 */
static void spmv(const orc_op* op, const double* f, double* q) {
    for (uint64_t k = 0; k < op->n_tgt; ++k) {
        double ar = 0.0, ai = 0.0;
        for (uint64_t i = op->row_offsets[k]; i < op->row_offsets[k + 1]; ++i) {
            const double vr = op->values[2 * i], vi = op->values[2 * i + 1];
            const double fr = f[2 * (size_t)op->cols[i]], fi = f[2 * (size_t)op->cols[i] + 1];
            ar += vr * fr - vi * fi;
            ai += vr * fi + vi * fr;
        }
        q[2 * k] += ar;
        q[2 * k + 1] += ai;
    }
}

/* point_cloud.cpp:125-132 */
static void spmv_adjoint(const orc_op* op, const double* u, double* q) {
    for (uint64_t k = 0; k < op->n_tgt; ++k) {
        const double ur = u[2 * k], ui = u[2 * k + 1];
        for (uint64_t i = op->row_offsets[k]; i < op->row_offsets[k + 1]; ++i) {
            const double vr = op->values[2 * i], vi = -op->values[2 * i + 1];
            const size_t c = op->cols[i];
            q[2 * c] += vr * ur - vi * ui;
            q[2 * c + 1] += vr * ui + vi * ur;
        }
    }
}

static void weight(const orc_op* op, double* s) {
    for (uint64_t v = 0; v < op->n_xi; ++v) {
        const double sr = s[2 * v], si = s[2 * v + 1];
        const double wr = op->weights[2 * v], wi = op->weights[2 * v + 1];
        s[2 * v] = sr * wr - si * wi;
        s[2 * v + 1] = sr * wi + si * wr;
    }
}

/* conv_operator.cpp:301-309 */
int orc_op_apply(const orc_op* op, const double* f, double* q) {
    double* s = (double*)malloc(sizeof(double) * 2 * (op->n_xi + 1));
    int rc = orc_plan_apply(op->fwd_in, f, s);
    if (!rc) {
        weight(op, s);
        rc = orc_plan_apply(op->fwd_out, s, q);
    }
    if (!rc) spmv(op, f, q);
    free(s);
    return rc;
}

/* conv_operator.cpp:311-324 */
int orc_op_apply_adjoint(const orc_op* op, const double* u, double* q) {
    const uint64_t nt = op->n_tgt, ns = op->n_src;
    double* ub = (double*)malloc(sizeof(double) * 2 * (nt + 1));
    for (uint64_t i = 0; i < nt; ++i) { ub[2 * i] = u[2 * i]; ub[2 * i + 1] = -u[2 * i + 1]; }
    double* s = (double*)malloc(sizeof(double) * 2 * (op->n_xi + 1));
    int rc = orc_plan_apply_transpose(op->fwd_out, ub, s);
    if (!rc) {
        weight(op, s);
        rc = orc_plan_apply_transpose(op->fwd_in, s, q);
    }
    if (!rc) {
        for (uint64_t i = 0; i < ns; ++i) q[2 * i + 1] = -q[2 * i + 1];
        spmv_adjoint(op, u, q);
    }
    free(ub);
    free(s);
    return rc;
}

void orc_op_weights(const orc_op* op, double* w) {
    memcpy(w, op->weights, sizeof(double) * 2 * op->n_xi);
}

int orc_op_stage(const orc_op* op, int stage, const double* in, double* out) {
    switch (stage) {
        case 1: return orc_plan_apply(op->fwd_in, in, out);
        case 2: return orc_plan_apply(op->fwd_out, in, out);
        case 3: spmv(op, in, out); return 0;
    }
    return seterr("bad stage");
}
