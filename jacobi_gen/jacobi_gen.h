/* jacobi_gen.h — seeded, counter-based, row-addressable synthetic linear systems.
 *
 * This module is the ONLY code shared between the CPU oracle (oracle/) and the
 * CUDA path (paper_1403_5805_b200/): it builds INPUTS (A, b, x*) and holds none
 * of the Jacobi method's arithmetic.  The recipe (DESIGN.md §4 "Input recipe")
 * follows BASELINE.json configs and SURVEY.md §8(d):
 *
 *   off-diagonal a_ij  = k_ij * 2^-abits,  k_ij = (int32)(h(seed,0,i*n+j) >> 32) >> (31-abits)
 *                        abits = 31 for fp64 storage, 23 for fp32 storage, so every value is
 *                        exact in the storage type and uniform on [-1, 1).
 *   x*_i               = kx_i * 2^-31,     kx_i = (int32)(h(seed,2,i) >> 32)          (U[-1,1))
 *   rowabs_i           = sum_{j!=i} |a_ij|, computed EXACTLY as an int64 sum of |k_ij|
 *   diag (mode ADD)    = fl(rowabs_i + (1 + (h(seed,1,i) >> 12) * 2^-52))           (rowabs + U[1,2))
 *   diag (mode SCALE)  = fl(scale * rowabs_i)                                        (1.05 or 1.2 x rowabs)
 *   fp32 storage       = a_ii stored as (float)diag, and the fp64 diag used below is that float
 *   b_i                = fl( fl(S_i * 2^-(abits+31)) + fl(a_ii * x*_i) ),  S_i = sum_{j!=i} k_ij*kx_j
 *                        computed EXACTLY in 128-bit integers, so b is independent of any
 *                        summation order and the host and device twins agree bit for bit.
 *   x0 = 0 (the caller fills it).
 *
 * h(seed, stream, idx) = mix64(key(seed, stream) + (idx + 1) * 0x9E3779B97F4A7C15), with
 * mix64 the splitmix64 finaliser and key(seed, stream) = mix64(seed ^ (stream << 56) ^ 0xD1B54A32D192ED03).
 *
 * A is written row-major with leading dimension lda (elements), rows r0..r1-1 of the system,
 * i.e. A_rows[(r - r0) * lda + j] = a_rj for j < n; padding columns j in [n, lda) are written 0.
 */
#ifndef JACOBI_GEN_H
#define JACOBI_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { JGEN_F64 = 0, JGEN_F32 = 1 };
enum { JGEN_DIAG_ADD = 0, JGEN_DIAG_SCALE = 1 };

typedef struct {
  int64_t n;          /* system dimension, >= 1 */
  uint64_t seed;      /* BASELINE.json: seed 0 for every config */
  int a_dtype;        /* JGEN_F64 or JGEN_F32 (storage of A) */
  int diag_mode;      /* JGEN_DIAG_ADD (rowabs + U[1,2)) or JGEN_DIAG_SCALE (scale * rowabs) */
  double diag_scale;  /* used when diag_mode == JGEN_DIAG_SCALE */
} jgen_cfg;

/* Host generator (multithreaded; bitwise independent of nthreads).  Returns 0 or -1 on bad args.
 * A_rows: (r1-r0) x lda elements of a_dtype; b_rows: r1-r0 doubles (nullable); */
int jgen_host_rows(const jgen_cfg* cfg, int64_t r0, int64_t r1, void* A_rows, int64_t lda,
                   double* b_rows, int nthreads);
/* x*: n doubles. */
int jgen_host_xstar(const jgen_cfg* cfg, double* xstar);
/* Only the diagonal entries of rows r0..r1-1 and b (no A storage): O((r1-r0) * n) work. */
int jgen_host_diag_b(const jgen_cfg* cfg, int64_t r0, int64_t r1, double* diag_rows, double* b_rows,
                     int nthreads);

/* Device twin (CUDA).  All pointers are device pointers; stream is a cudaStream_t (nullable).
 * Enqueues the work and returns 0, or a negative value on bad args / CUDA launch error. */
int jgen_device_rows(const jgen_cfg* cfg, int64_t r0, int64_t r1, void* dA_rows, int64_t lda,
                     double* d_b_rows, void* stream);
int jgen_device_xstar(const jgen_cfg* cfg, double* d_xstar, void* stream);

#ifdef __cplusplus
}
#endif
#endif
