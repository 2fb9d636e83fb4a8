/* oracle/shim/fftw3.h — TEST INFRASTRUCTURE ONLY (see oracle/README.md).
 *
 * Minimal FFTW3 API subset so the UNCHANGED reference core
 * (/root/reference/proj/src/core/spectral.cpp) compiles in this image, where
 * FFTW3 is absent. Only the surface the reference touches is provided:
 *   fftw_complex, fftw_plan, fftw_plan_dft_2d, fftw_execute_dft,
 *   FFTW_FORWARD / FFTW_BACKWARD / FFTW_ESTIMATE / FFTW_UNALIGNED
 * (call sites: reference spectral.cpp:32 plan, spectral.cpp:47 execute).
 *
 * Semantics follow the published FFTW3 contract: unnormalised 2-D DFT with
 * exponent sign `sign` (FFTW_FORWARD = -1), row-major n0 x n1 arrays, the
 * plan may be executed on any arrays of the planned shape. The arithmetic is
 * an fp64 radix-2 (power-of-two) / direct-DFT (other sizes) row-column
 * transform; tests/test_oracle.py pins it against numpy.fft to 1e-12.
 */
#ifndef GT_SHIM_FFTW3_H
#define GT_SHIM_FFTW3_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct gt_shim_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
