/*
 * oracle/shim/fftw3.h -- TEST-ONLY stand-in for the FFTW3 subset the reference
 * uses (FFTW3 is not installed in this image).
 *
 * Call sites in the reference: proj/src/nufft.cpp:118-119, 207-213, 224, 252,
 * 287, 301, 338, 364. Only FFTW_BACKWARD (+1) 2D complex transforms are used.
 * Backed by oracle/fft235.c. Never part of the product.
 */
#ifndef SBD_ORACLE_FFTW3_SHIM_H
#define SBD_ORACLE_FFTW3_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct sbd_shim_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)

fftw_complex* fftw_alloc_complex(size_t n);
void fftw_free(void* p);
fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
