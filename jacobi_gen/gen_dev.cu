// Device twin of the host generator (jacobi_gen.h): bitwise-identical A, b and x*.
// One CTA per row; integer sums are exact, so the block reduction order is irrelevant.
#include "jacobi_gen.h"
#include "gen_common.h"
#include <cuda_runtime.h>

namespace {

constexpr int kThreads = 256;

template <typename T, int ABITS>
__global__ void __launch_bounds__(kThreads) k_gen_rows(jgen_cfg c, int64_t r0, T* __restrict__ A,
                                                     int64_t lda, double* __restrict__ b) {
  const int64_t i = r0 + blockIdx.x;
  const int64_t n = c.n;
  const uint64_t k0 = jg_key(c.seed, 0), k1 = jg_key(c.seed, 1), k2 = jg_key(c.seed, 2);
  T* row = A + (int64_t)blockIdx.x * lda;
  int64_t sabs = 0;
  unsigned __int128 acc = 0;
  for (int64_t j = threadIdx.x; j < lda; j += kThreads) {
    if (j >= n) { row[j] = T(0); continue; }
    if (j == i) continue;
    int32_t k = jg_ka(k0, (uint64_t)i * (uint64_t)n + (uint64_t)j, ABITS);
    row[j] = ABITS == 23 ? (T)((float)k * 0x1p-23f) : (T)((double)k * 0x1p-31);
    sabs += k < 0 ? -(int64_t)k : (int64_t)k;
    acc += (unsigned __int128)(__int128)((int64_t)k * (int64_t)jg_kx(k2, (uint64_t)j));
  }
  __shared__ int64_t s_abs[kThreads];
  __shared__ unsigned __int128 s_acc[kThreads];
  s_abs[threadIdx.x] = sabs;
  s_acc[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      s_abs[threadIdx.x] += s_abs[threadIdx.x + s];
      s_acc[threadIdx.x] += s_acc[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double rowabs = (double)s_abs[0];
    rowabs = ABITS == 23 ? __dmul_rn(rowabs, 0x1p-23) : __dmul_rn(rowabs, 0x1p-31);
    double diag = c.diag_mode == JGEN_DIAG_SCALE ? __dmul_rn(c.diag_scale, rowabs)
                                                 : __dadd_rn(rowabs, jg_extra(k1, (uint64_t)i));
    if (ABITS == 23) diag = (double)__double2float_rn(diag);
    row[i] = (T)diag;
    double xs = __dmul_rn((double)jg_kx(k2, (uint64_t)i), 0x1p-31);
    unsigned __int128 a = s_acc[0];
    double off = jg_i128_to_double((int64_t)(uint64_t)(a >> 64), (uint64_t)a, ABITS + 31);
    if (b) b[blockIdx.x] = __dadd_rn(off, __dmul_rn(diag, xs));
  }
}

__global__ void k_gen_xstar(jgen_cfg c, double* xs) {
  const uint64_t k2 = jg_key(c.seed, 2);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.n; i += (int64_t)gridDim.x * blockDim.x)
    xs[i] = __dmul_rn((double)jg_kx(k2, (uint64_t)i), 0x1p-31);
}

}  // namespace

extern "C" int jgen_device_rows(const jgen_cfg* c, int64_t r0, int64_t r1, void* dA, int64_t lda,
                                double* db, void* stream) {
  if (!c || c->n < 1 || r0 < 0 || r1 > c->n || r0 > r1 || !dA || lda < c->n) return -1;
  if (r1 == r0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  // grid.x is limited to 2^31-1 rows per launch; chunk anyway to keep launches modest.
  const int64_t chunk = 1 << 20;
  for (int64_t a = r0; a < r1; a += chunk) {
    int64_t e = a + chunk < r1 ? a + chunk : r1;
    unsigned nb = (unsigned)(e - a);
    if (c->a_dtype == JGEN_F32)
      k_gen_rows<float, 23><<<nb, kThreads, 0, s>>>(*c, a, (float*)dA + (a - r0) * lda, lda, db ? db + (a - r0) : nullptr);
    else
      k_gen_rows<double, 31><<<nb, kThreads, 0, s>>>(*c, a, (double*)dA + (a - r0) * lda, lda, db ? db + (a - r0) : nullptr);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int jgen_device_xstar(const jgen_cfg* c, double* dxs, void* stream) {
  if (!c || c->n < 1 || !dxs) return -1;
  k_gen_xstar<<<592, 256, 0, (cudaStream_t)stream>>>(*c, dxs);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
