/*
 * oracle/shim/fftw_shim.c -- TEST-ONLY implementation of the FFTW3 subset in
 * oracle/shim/fftw3.h, on top of oracle/fft235.c. Never part of the product.
 */
#define _POSIX_C_SOURCE 200112L
#include "fftw3.h"

#include <stdlib.h>
#include <string.h>

#include "../fft235.h"

struct sbd_shim_fftw_plan_s {
    int n0, n1, sign;
    fftw_complex* in;
    fftw_complex* out;
};

fftw_complex* fftw_alloc_complex(size_t n) {
    void* p = NULL;
    if (posix_memalign(&p, 64, n * sizeof(fftw_complex) + 64) != 0) return NULL;
    return (fftw_complex*)p;
}

void fftw_free(void* p) { free(p); }

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
    (void)flags;
    if (n0 < 1 || n1 < 1) return NULL;
    fftw_plan p = (fftw_plan)calloc(1, sizeof(*p));
    p->n0 = n0;
    p->n1 = n1;
    p->sign = sign;
    p->in = in;
    p->out = out;
    return p;
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    const size_t cells = (size_t)p->n0 * (size_t)p->n1;
    if (in != out) memcpy(out, in, cells * sizeof(fftw_complex));
    fft235_2d_inplace(p->n0, p->n1, p->sign, (double*)out);
}

void fftw_execute(const fftw_plan p) { fftw_execute_dft(p, p->in, p->out); }

void fftw_destroy_plan(fftw_plan p) { free(p); }
