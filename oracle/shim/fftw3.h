/* ORACLE TEST INFRASTRUCTURE — not product code.
 *
 * Minimal stand-in for the subset of the FFTW3 API that the reference's
 * FFT engine calls (reference: proj/core/src/fft.cpp:3,16-26,41-48):
 *   fftw_plan_dft(rank, n, in, out, sign, flags)   (fft.cpp:21-22)
 *   fftw_execute_dft(plan, in, out)                (fft.cpp:47)
 * FFTW itself (version unpinned in the reference: bare find_library(fftw3),
 * core/CMakeLists.txt:3-4) is not installed in this image.  Semantics kept:
 * row-major multi-dimensional complex DFT, any in/out pointer at execute
 * time (new-array interface), sign -1 forward / +1 backward, unnormalised.
 * The reference only ever plans power-of-two shapes (fft.cpp:58-70); the
 * shim rejects anything else by returning a null plan, which the reference
 * turns into std::runtime_error (fft.cpp:23).
 */
#ifndef PCB_ORACLE_FFTW3_SHIM_H
#define PCB_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct pcb_shim_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign,
                        unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
