/*
 * oracle/fft235.c -- TEST INFRASTRUCTURE ONLY. See fft235.h.
 *
 * Recursive decimation-in-time mixed-radix FFT (radices 4, 2, 3, 5, generic).
 * Twiddles are computed in long double and rounded once, so the transform is
 * accurate to a few ulps times log(n): far below the 1e-9 parity bar the
 * oracle is used for ("the shim FFT changes results only
 * at rounding level").
 */
#include "fft235.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

struct fft235_plan1d {
    int n;
    int sign;
    int nfac;
    int fac[64];
    double* tw; /* 2n doubles: exp(sign*2*pi*i*k/n), k = 0..n-1 */
    double* scratch;
};

static void factorize(int n, int* fac, int* nfac) {
    int k = 0;
    while (n % 4 == 0) { fac[k++] = 4; n /= 4; }
    while (n % 2 == 0) { fac[k++] = 2; n /= 2; }
    for (int r = 3; r * r <= n; r += 2)
        while (n % r == 0) { fac[k++] = r; n /= r; }
    if (n > 1) fac[k++] = n;
    *nfac = k;
}

fft235_plan1d* fft235_plan1d_create(int n, int sign) {
    if (n < 1) return NULL;
    fft235_plan1d* p = (fft235_plan1d*)calloc(1, sizeof(*p));
    p->n = n;
    p->sign = sign >= 0 ? 1 : -1;
    factorize(n, p->fac, &p->nfac);
    p->tw = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (int k = 0; k < n; ++k) {
        /* Exact symmetric reduction keeps cos/sin arguments in [0, pi/4]-ish range. */
        long double ang = two_pi * (long double)k / (long double)n;
        p->tw[2 * k] = (double)cosl(ang);
        p->tw[2 * k + 1] = (double)(p->sign * sinl(ang));
    }
    p->scratch = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    return p;
}

void fft235_plan1d_destroy(fft235_plan1d* p) {
    if (!p) return;
    free(p->tw);
    free(p->scratch);
    free(p);
}

/* out[0..n) = DFT_n of in[0], in[s], in[2s], ...; twiddle table stride tws
 * (w_n^j = tw[j*tws]). */
static void rec(const fft235_plan1d* P, const double* in, double* out, int n, size_t s,
                const int* fac, size_t tws) {
    if (n == 1) {
        out[0] = in[0];
        out[1] = in[1];
        return;
    }
    const int r = fac[0];
    const int m = n / r;
    for (int q = 0; q < r; ++q) rec(P, in + 2 * q * s, out + 2 * (size_t)q * m, m, s * r, fac + 1, tws * r);

    const double* tw = P->tw;
    const size_t N = (size_t)P->n;
    if (r == 2) {
        for (int k = 0; k < m; ++k) {
            double* a = out + 2 * k;
            double* b = out + 2 * (k + m);
            const double wr = tw[2 * ((k * tws) % N)], wi = tw[2 * ((k * tws) % N) + 1];
            const double br = b[0] * wr - b[1] * wi, bi = b[0] * wi + b[1] * wr;
            const double ar = a[0], ai = a[1];
            a[0] = ar + br; a[1] = ai + bi;
            b[0] = ar - br; b[1] = ai - bi;
        }
        return;
    }
    if (r == 4) {
        const double sg = (double)P->sign; /* w_4 = sign * i */
        for (int k = 0; k < m; ++k) {
            double x[4][2];
            for (int q = 0; q < 4; ++q) {
                const double* v = out + 2 * (k + (size_t)q * m);
                const size_t j = ((size_t)q * k * tws) % N;
                const double wr = tw[2 * j], wi = tw[2 * j + 1];
                x[q][0] = v[0] * wr - v[1] * wi;
                x[q][1] = v[0] * wi + v[1] * wr;
            }
            const double t0r = x[0][0] + x[2][0], t0i = x[0][1] + x[2][1];
            const double t1r = x[0][0] - x[2][0], t1i = x[0][1] - x[2][1];
            const double t2r = x[1][0] + x[3][0], t2i = x[1][1] + x[3][1];
            const double t3r = x[1][0] - x[3][0], t3i = x[1][1] - x[3][1];
            /* (sign*i) * t3 */
            const double u3r = -sg * t3i, u3i = sg * t3r;
            double* o0 = out + 2 * k;
            double* o1 = out + 2 * (k + (size_t)m);
            double* o2 = out + 2 * (k + 2 * (size_t)m);
            double* o3 = out + 2 * (k + 3 * (size_t)m);
            o0[0] = t0r + t2r; o0[1] = t0i + t2i;
            o2[0] = t0r - t2r; o2[1] = t0i - t2i;
            o1[0] = t1r + u3r; o1[1] = t1i + u3i;
            o3[0] = t1r - u3r; o3[1] = t1i - u3i;
        }
        return;
    }
    /* Generic radix r (3, 5, and any leftover prime): O(r^2) butterfly. */
    double xs[2 * 64];
    double* x = r <= 64 ? xs : (double*)malloc(sizeof(double) * 2 * (size_t)r);
    const size_t twr = N / (size_t)r; /* w_r^j = tw[j * N/r] */
    for (int k = 0; k < m; ++k) {
        for (int q = 0; q < r; ++q) {
            const double* v = out + 2 * (k + (size_t)q * m);
            const size_t j = ((size_t)q * k * tws) % N;
            const double wr = tw[2 * j], wi = tw[2 * j + 1];
            x[2 * q] = v[0] * wr - v[1] * wi;
            x[2 * q + 1] = v[0] * wi + v[1] * wr;
        }
        for (int pq = 0; pq < r; ++pq) {
            double accr = 0.0, acci = 0.0;
            for (int q = 0; q < r; ++q) {
                const size_t j = (((size_t)q * pq) % r) * twr;
                const double wr = tw[2 * j], wi = tw[2 * j + 1];
                accr += x[2 * q] * wr - x[2 * q + 1] * wi;
                acci += x[2 * q] * wi + x[2 * q + 1] * wr;
            }
            double* o = out + 2 * (k + (size_t)pq * m);
            o[0] = accr;
            o[1] = acci;
        }
    }
    if (x != xs) free(x);
}

void fft235_exec1d(const fft235_plan1d* p, const double* in, double* out) {
    rec(p, in, out, p->n, 1, p->fac, 1);
}

void fft235_2d_inplace(int n0, int n1, int sign, double* data) {
    fft235_plan1d* p1 = fft235_plan1d_create(n1, sign);
    fft235_plan1d* p0 = n0 == n1 ? p1 : fft235_plan1d_create(n0, sign);
    const int nmax = n0 > n1 ? n0 : n1;
    double* a = (double*)malloc(sizeof(double) * 2 * (size_t)nmax);
    double* b = (double*)malloc(sizeof(double) * 2 * (size_t)nmax);
    for (int i = 0; i < n0; ++i) {
        double* row = data + 2 * (size_t)i * n1;
        memcpy(a, row, sizeof(double) * 2 * (size_t)n1);
        fft235_exec1d(p1, a, row);
    }
    for (int j = 0; j < n1; ++j) {
        for (int i = 0; i < n0; ++i) {
            a[2 * i] = data[2 * ((size_t)i * n1 + j)];
            a[2 * i + 1] = data[2 * ((size_t)i * n1 + j) + 1];
        }
        fft235_exec1d(p0, a, b);
        for (int i = 0; i < n0; ++i) {
            data[2 * ((size_t)i * n1 + j)] = b[2 * i];
            data[2 * ((size_t)i * n1 + j) + 1] = b[2 * i + 1];
        }
    }
    free(a);
    free(b);
    if (p0 != p1) fft235_plan1d_destroy(p0);
    fft235_plan1d_destroy(p1);
}
