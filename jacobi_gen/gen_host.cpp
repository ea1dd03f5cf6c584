// Host generator (jacobi_gen.h).  Rows are independent, so threads split rows and the output
// does not depend on the thread count.  Compiled with -ffp-contract=off: the two roundings in
// b_i = fl(fl(S) + fl(a_ii * x*_i)) must stay separate to match the device twin.
#include "jacobi_gen.h"
#include "gen_common.h"
#include <thread>
#include <vector>
#include <cstring>

namespace {

struct RowOut { double diag; double b; };

// Everything about row i except the A storage: rowabs, diag and b (see jacobi_gen.h).
template <typename StoreFn>
RowOut gen_row(const jgen_cfg* c, int64_t i, StoreFn store) {
  const int abits = c->a_dtype == JGEN_F32 ? 23 : 31;
  const uint64_t k0 = jg_key(c->seed, 0), k1 = jg_key(c->seed, 1), k2 = jg_key(c->seed, 2);
  const int64_t n = c->n;
  int64_t sabs = 0;
  unsigned __int128 acc = 0;  // two's complement accumulation of sum k_ij * kx_j, j != i
  for (int64_t j = 0; j < n; ++j) {
    if (j == i) continue;
    int32_t k = jg_ka(k0, (uint64_t)i * (uint64_t)n + (uint64_t)j, abits);
    store(j, k);
    sabs += k < 0 ? -(int64_t)k : (int64_t)k;
    __int128 p = (__int128)((int64_t)k * (int64_t)jg_kx(k2, (uint64_t)j));
    acc += (unsigned __int128)p;
  }
  double rowabs = (double)sabs;
  rowabs = abits == 23 ? rowabs * 0x1p-23 : rowabs * 0x1p-31;
  double diag = c->diag_mode == JGEN_DIAG_SCALE ? c->diag_scale * rowabs : rowabs + jg_extra(k1, (uint64_t)i);
  if (c->a_dtype == JGEN_F32) diag = (double)(float)diag;
  double xs = (double)jg_kx(k2, (uint64_t)i) * 0x1p-31;
  double off = jg_i128_to_double((int64_t)(uint64_t)(acc >> 64), (uint64_t)acc, abits + 31);
  double dx = diag * xs;
  RowOut r{diag, off + dx};
  return r;
}

template <typename F>
void parallel_rows(int64_t r0, int64_t r1, int nthreads, F f) {
  if (nthreads < 1) nthreads = 1;
  int64_t rows = r1 - r0;
  if (nthreads > rows) nthreads = (int)(rows > 0 ? rows : 1);
  if (nthreads == 1) { for (int64_t r = r0; r < r1; ++r) f(r); return; }
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t) {
    int64_t a = r0 + rows * t / nthreads, b = r0 + rows * (t + 1) / nthreads;
    th.emplace_back([=] { for (int64_t r = a; r < b; ++r) f(r); });
  }
  for (auto& t : th) t.join();
}

bool bad(const jgen_cfg* c) {
  return !c || c->n < 1 || (c->a_dtype != JGEN_F64 && c->a_dtype != JGEN_F32) ||
         (c->diag_mode != JGEN_DIAG_ADD && c->diag_mode != JGEN_DIAG_SCALE);
}

}  // namespace

extern "C" int jgen_host_rows(const jgen_cfg* c, int64_t r0, int64_t r1, void* A_rows, int64_t lda,
                              double* b_rows, int nthreads) {
  if (bad(c) || r0 < 0 || r1 > c->n || r0 > r1 || !A_rows || lda < c->n) return -1;
  const int f32 = c->a_dtype == JGEN_F32;
  parallel_rows(r0, r1, nthreads, [&](int64_t i) {
    RowOut ro;
    if (f32) {
      float* row = (float*)A_rows + (i - r0) * lda;
      ro = gen_row(c, i, [&](int64_t j, int32_t k) { row[j] = (float)k * 0x1p-23f; });
      row[i] = (float)ro.diag;
      for (int64_t j = c->n; j < lda; ++j) row[j] = 0.0f;
    } else {
      double* row = (double*)A_rows + (i - r0) * lda;
      ro = gen_row(c, i, [&](int64_t j, int32_t k) { row[j] = (double)k * 0x1p-31; });
      row[i] = ro.diag;
      for (int64_t j = c->n; j < lda; ++j) row[j] = 0.0;
    }
    if (b_rows) b_rows[i - r0] = ro.b;
  });
  return 0;
}

extern "C" int jgen_host_diag_b(const jgen_cfg* c, int64_t r0, int64_t r1, double* diag_rows,
                                double* b_rows, int nthreads) {
  if (bad(c) || r0 < 0 || r1 > c->n || r0 > r1) return -1;
  parallel_rows(r0, r1, nthreads, [&](int64_t i) {
    RowOut ro = gen_row(c, i, [](int64_t, int32_t) {});
    if (diag_rows) diag_rows[i - r0] = ro.diag;
    if (b_rows) b_rows[i - r0] = ro.b;
  });
  return 0;
}

extern "C" int jgen_host_xstar(const jgen_cfg* c, double* xs) {
  if (bad(c) || !xs) return -1;
  const uint64_t k2 = jg_key(c->seed, 2);
  for (int64_t i = 0; i < c->n; ++i) xs[i] = (double)jg_kx(k2, (uint64_t)i) * 0x1p-31;
  return 0;
}
