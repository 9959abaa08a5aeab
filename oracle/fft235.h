/*
 * oracle/fft235.h -- TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * A small, accurate, unnormalised mixed-radix complex FFT used by
 *   (1) the FFTW shim (oracle/shim/fftw3.h) that lets the unmodified reference
 *       sources under /root/reference/proj/src compile into oracle/_ref, and
 *   (2) the plain-C restatement of the apply path (oracle/sbd_oracle.c).
 *
 * Convention (FFTW's): out[k] = sum_j in[j] * exp(sign * 2*pi*i*j*k/n), no scaling.
 * The reference only ever requests FFTW_BACKWARD (sign = +1) 2D transforms of
 * 2/3/5-smooth even sizes (reference proj/src/nufft.cpp:55-63, :207-213), but any
 * n is accepted (prime factors > 5 fall back to an O(r^2) generic butterfly).
 */
#ifndef SBD_ORACLE_FFT235_H
#define SBD_ORACLE_FFT235_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fft235_plan1d fft235_plan1d;

fft235_plan1d* fft235_plan1d_create(int n, int sign);
void fft235_plan1d_destroy(fft235_plan1d* p);
/* in and out are interleaved complex (re, im) arrays of length n; in != out. */
void fft235_exec1d(const fft235_plan1d* p, const double* in, double* out);

/* In-place 2D transform of a row-major n0 x n1 interleaved complex array. */
void fft235_2d_inplace(int n0, int n1, int sign, double* data);

#ifdef __cplusplus
}
#endif

#endif
