/* gen_common.h — the counter-based draws of jacobi_gen.h, written once for host and device.
 * Input construction only (see jacobi_gen.h); no Jacobi arithmetic lives here. */
#ifndef JACOBI_GEN_COMMON_H
#define JACOBI_GEN_COMMON_H
#include <stdint.h>

#ifdef __CUDACC__
#define JG_HD __host__ __device__ __forceinline__
#else
#define JG_HD static inline
#endif

JG_HD uint64_t jg_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
JG_HD uint64_t jg_key(uint64_t seed, uint64_t stream) {
  return jg_mix64(seed ^ (stream << 56) ^ 0xD1B54A32D192ED03ull);
}
JG_HD uint64_t jg_draw(uint64_t key, uint64_t idx) {
  return jg_mix64(key + (idx + 1) * 0x9E3779B97F4A7C15ull);
}
/* stream 0: integer numerator of a_ij (j != i); value = k * 2^-abits */
JG_HD int32_t jg_ka(uint64_t key0, uint64_t idx, int abits) {
  return ((int32_t)(jg_draw(key0, idx) >> 32)) >> (31 - abits);
}
/* stream 2: integer numerator of x*_i; value = kx * 2^-31 */
JG_HD int32_t jg_kx(uint64_t key2, uint64_t i) { return (int32_t)(jg_draw(key2, i) >> 32); }
/* stream 1: 1 + U[0,1) with 52 fractional bits (exact in fp64) */
JG_HD double jg_extra(uint64_t key1, uint64_t i) {
  return 1.0 + (double)(jg_draw(key1, i) >> 12) * 0x1p-52;
}

/* Correctly rounded conversion of a signed 128-bit integer (given as hi:lo two's complement)
 * times 2^-scale to double.  The top 64 significant bits are kept with a sticky bit so that the
 * single uint64 -> double round-to-nearest conversion equals the exact rounding. */
JG_HD double jg_i128_to_double(int64_t hi, uint64_t lo, int scale) {
  int neg = hi < 0;
  uint64_t uh = (uint64_t)hi, ul = lo;
  if (neg) { ul = ~ul + 1; uh = ~uh + (ul == 0); }
  if (uh == 0 && ul == 0) return 0.0;
  int e;  /* value = top * 2^e */
  uint64_t top;
  if (uh == 0) { top = ul; e = 0; }
  else {
    int lz = 0; uint64_t t = uh; while (!(t & 0x8000000000000000ull)) { t <<= 1; ++lz; }
    top = (uh << lz) | (lz ? (ul >> (64 - lz)) : 0);
    uint64_t rest = lz ? (ul << lz) : ul;
    if (rest) top |= 1;
    e = 64 - lz;
  }
#ifdef __CUDA_ARCH__
  double d = __ull2double_rn(top);
#else
  double d = (double)top;
#endif
  /* exact scaling by a power of two (no overflow/underflow for the ranges used here) */
  int s = e - scale;
  while (s > 0) { int q = s > 60 ? 60 : s; d *= (double)(1ull << q); s -= q; }
  while (s < 0) { int q = -s > 60 ? 60 : -s; d /= (double)(1ull << q); s += q; }
  return neg ? -d : d;
}

#endif
