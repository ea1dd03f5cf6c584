/* oracle.c — plain, slow, obviously correct CPU Jacobi (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  It shares no code with the CUDA path (paper_1403_5805_b200/) and includes
 * none of its headers.  Compile: gcc -O2 -ffp-contract=off (no -ffast-math): every product and
 * sum is rounded separately, in ascending j, exactly as written below.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, a text extraction of arXiv:1403.5805):
 *   - PAPER.md:55 (§2, component equation):
 *       x_i^(k) = (1/a_ii) { sum_{j=1, j!=i}^n (-a_ij x_j^(k-1)) + b_i }
 *     written as (b_i - s_i) / a_ii with s_i = sum_{j!=i} a_ij x_j^(k-1) (reading R9:
 *     one correctly rounded division; the pseudocode's sign flip at PAPER.md:63 is a typo, R6).
 *   - PAPER.md:59-66 (§2, pseudocode): k = 1; while k <= L: (a) update every component from X^t;
 *     (b) if ||X - X^t|| < tol return X; (c) k = k + 1; (d) X^t = X.  "Terminate the procedure if
 *     the iteration limit has been reached" -> return X^(L).
 *   - The distance is the max norm max_i |x_i^(k) - x_i^(k-1)| (BASELINE.json north_star and
 *     configs; PAPER.md:51/94 say Euclidean — reading R1), NaN-sticky (reading R12), compared
 *     with strict "<" (R2), checked after every sweep including the first (R3).  The paper's own
 *     Euclidean distance sqrt(sum_i (x_i^(k+1) - x_i^(k))^2) of PAPER.md:94 is the norm = 1 option
 *     of oracle_jacobi_norm (NEXT-2 row), summed in ascending i.
 *   - PAPER.md:53: "the algorithm will fail if a_ii = 0" -> status EZERODIAG with the lowest i.
 *   - Gaussian elimination with partial pivoting (oracle_ge_solve): the textbook direct solve used
 *     only to pin the converged Jacobi value (north_star: "checked on tiny systems against a direct
 *     Gaussian-elimination solve").
 *
 * Pins (tests/test_oracle_pins.py): closed-form 2x2 iterates (P1), exact rational 3x3 iterates
 * from tests/golden (P2), first sweep = b / diag bitwise (P3), diagonal systems (P4), integer
 * fixed point (P5), power-of-two row scaling invariance (P6), GE + numpy.linalg.solve (P7),
 * planted solution (P8), contraction (P9), exact-rational brute force (P10), split runs (P11),
 * thread-count invariance (P13), divergent paper regime (P14).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Status values (numerically equal to the C-ABI's; defined here independently). */
#define OR_CONVERGED 0
#define OR_MAX_ITER 1
#define OR_EINVAL (-1)
#define OR_EZERODIAG (-2)
#define OR_ENONFINITE (-3)
#define OR_ENOMEM (-4)

/* a_ij read from row-major storage of either precision (fp32 values widen exactly). */
static double a_at(const void* A, int a_f32, int64_t lda, int64_t i, int64_t j) {
  if (a_f32) return (double)((const float*)A)[i * lda + j];
  return ((const double*)A)[i * lda + j];
}

/* One application of PAPER.md:55 to rows [r0, r1) of the system: x_new[i - r0] from x_old (length n).
 * A_rows holds those rows (row r at A_rows[(r - r0) * lda]). */
void oracle_sweep_rows(int64_t n, int a_f32, const void* A_rows, int64_t lda, int64_t r0, int64_t r1,
                       const double* b_rows, const double* x_old, double* x_new_rows) {
  for (int64_t i = r0; i < r1; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      double p = a_at(A_rows, a_f32, lda, i - r0, j) * x_old[j];
      s = s + p;
    }
    double aii = a_at(A_rows, a_f32, lda, i - r0, i);
    x_new_rows[i - r0] = (b_rows[i - r0] - s) / aii;
  }
}

/* Euclidean distance of PAPER.md:94 (§3.1): sqrt( sum_i (u_i - v_i)^2 ), ascending i (NEXT-2 row). */
double oracle_l2_dist(int64_t n, const double* u, const double* v) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double t = u[i] - v[i];
    double t2 = t * t;
    s = s + t2;
  }
  return sqrt(s);
}

/* max_i |u_i - v_i|, NaN-sticky: once a NaN difference is seen the result is NaN (R12). */
double oracle_maxnorm_dist(int64_t n, const double* u, const double* v) {
  double d = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double t = fabs(u[i] - v[i]);
    if (isnan(t)) return t;
    if (t > d) d = t;
  }
  return d;
}

typedef struct {
  int64_t n, lda, r0, r1;
  int a_f32;
  const void* A;
  const double* b;
  const double** xo;
  double** xn;
  pthread_barrier_t* bar;
  volatile int* stop;
} worker_t;

static void* worker(void* p) {
  worker_t* w = (worker_t*)p;
  for (;;) {
    pthread_barrier_wait(w->bar);              /* sweep start (or stop) */
    if (*w->stop) break;
    oracle_sweep_rows(w->n, w->a_f32, (const char*)w->A + (size_t)w->r0 * w->lda * (w->a_f32 ? 4 : 8),
                      w->lda, w->r0, w->r1, w->b + w->r0, *w->xo, *w->xn + w->r0);
    pthread_barrier_wait(w->bar);              /* sweep done */
  }
  return NULL;
}

static int all_finite(int64_t cnt, const double* v) {
  for (int64_t i = 0; i < cnt; ++i) if (!isfinite(v[i])) return 0;
  return 1;
}

/* The serial algorithm of PAPER.md:59-66 (rows of step (a) split over nthreads; each row's
 * arithmetic is identical, so the result is bitwise independent of nthreads).
 * hist (nullable, length >= max_iter) receives d_k for k = 1..iters.
 * Validation order: EINVAL, then EZERODIAG (lowest i), then ENONFINITE.
 * x_out / iters_out are written only when the status is >= 0; x_out may alias x0. */
int oracle_jacobi_norm(int64_t n, int a_f32, const void* A, int64_t lda, const double* b, const double* x0,
                       int64_t max_iter, double tol, double* x_out, int64_t* iters_out, double* hist,
                       int nthreads, int norm) {
  if (n < 1 || !A || !b || !x0 || !x_out || !iters_out || lda < n || max_iter < 0 || isnan(tol) || tol < 0 ||
      (norm != 0 && norm != 1))
    return OR_EINVAL;
  for (int64_t i = 0; i < n; ++i)
    if (a_at(A, a_f32, lda, i, i) == 0.0) return OR_EZERODIAG;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j)
      if (!isfinite(a_at(A, a_f32, lda, i, j))) return OR_ENONFINITE;
  if (!all_finite(n, b) || !all_finite(n, x0)) return OR_ENONFINITE;

  double* xt = (double*)malloc((size_t)n * sizeof(double)); /* X^t */
  double* x = (double*)malloc((size_t)n * sizeof(double));  /* X   */
  if (!xt || !x) { free(xt); free(x); return OR_ENOMEM; }
  memcpy(xt, x0, (size_t)n * sizeof(double));               /* input (c): X^t = X^0 */

  if (nthreads < 1) nthreads = 1;
  if (nthreads > n) nthreads = (int)n;
  pthread_barrier_t bar;
  volatile int stop = 0;
  const double* xo_ptr = xt;
  double* xn_ptr = x;
  worker_t* ws = NULL;
  pthread_t* th = NULL;
  if (nthreads > 1) {
    pthread_barrier_init(&bar, NULL, (unsigned)nthreads + 1);
    ws = (worker_t*)calloc((size_t)nthreads, sizeof(worker_t));
    th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
      ws[t] = (worker_t){n, lda, n * t / nthreads, n * (t + 1) / nthreads, a_f32, A, b, &xo_ptr, &xn_ptr, &bar, &stop};
      pthread_create(&th[t], NULL, worker, &ws[t]);
    }
  }

  int status = OR_MAX_ITER;
  int64_t k = 1;                                             /* step 1: k = 1 */
  while (k <= max_iter) {                                    /* step 2: while k <= L */
    xo_ptr = xt; xn_ptr = x;
    if (nthreads > 1) { pthread_barrier_wait(&bar); pthread_barrier_wait(&bar); }
    else oracle_sweep_rows(n, a_f32, A, lda, 0, n, b, xt, x); /* (a) */
    double d = norm ? oracle_l2_dist(n, x, xt)                 /* (b) ||X - X^t||: Euclidean */
                    : oracle_maxnorm_dist(n, x, xt);           /*     or max norm (north_star, R1) */
    if (hist) hist[k - 1] = d;
    if (d < tol) { status = OR_CONVERGED; break; }             /*     < tol: return X */
    k = k + 1;                                                 /* (c) */
    double* t = xt; xt = x; x = t;                             /* (d) X^t = X */
  }
  /* On convergence X is in x; on exhaustion X^(L) is in xt after the final (d). */
  const double* res = (status == OR_CONVERGED) ? x : xt;
  int64_t iters = (status == OR_CONVERGED) ? k : max_iter;

  if (nthreads > 1) {
    stop = 1;
    pthread_barrier_wait(&bar);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    pthread_barrier_destroy(&bar);
    free(ws); free(th);
  }
  memmove(x_out, res, (size_t)n * sizeof(double));
  *iters_out = iters;
  free(xt); free(x);
  return status;
}

/* Max-norm entry point (the north star's stop rule). */
int oracle_jacobi(int64_t n, int a_f32, const void* A, int64_t lda, const double* b, const double* x0,
                  int64_t max_iter, double tol, double* x_out, int64_t* iters_out, double* hist, int nthreads) {
  return oracle_jacobi_norm(n, a_f32, A, lda, b, x0, max_iter, tol, x_out, iters_out, hist, nthreads, 0);
}

/* Gaussian elimination with partial pivoting on a copy of A (fp64, row-major, lda = n).
 * Returns 0, OR_EINVAL, OR_ENOMEM, or OR_EZERODIAG when a pivot column is exactly zero (singular). */
int oracle_ge_solve(int64_t n, const double* A, const double* b, double* x) {
  if (n < 1 || !A || !b || !x) return OR_EINVAL;
  double* M = (double*)malloc((size_t)n * (size_t)n * sizeof(double));
  double* r = (double*)malloc((size_t)n * sizeof(double));
  if (!M || !r) { free(M); free(r); return OR_ENOMEM; }
  memcpy(M, A, (size_t)n * (size_t)n * sizeof(double));
  memcpy(r, b, (size_t)n * sizeof(double));
  for (int64_t c = 0; c < n; ++c) {
    int64_t p = c;
    for (int64_t i = c + 1; i < n; ++i) if (fabs(M[i * n + c]) > fabs(M[p * n + c])) p = i;
    if (M[p * n + c] == 0.0) { free(M); free(r); return OR_EZERODIAG; }
    if (p != c) {
      for (int64_t j = 0; j < n; ++j) { double t = M[c * n + j]; M[c * n + j] = M[p * n + j]; M[p * n + j] = t; }
      double t = r[c]; r[c] = r[p]; r[p] = t;
    }
    for (int64_t i = c + 1; i < n; ++i) {
      double f = M[i * n + c] / M[c * n + c];
      for (int64_t j = c; j < n; ++j) M[i * n + j] = M[i * n + j] - f * M[c * n + j];
      r[i] = r[i] - f * r[c];
    }
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = r[i];
    for (int64_t j = i + 1; j < n; ++j) s = s - M[i * n + j] * x[j];
    x[i] = s / M[i * n + i];
  }
  free(M); free(r);
  return 0;
}
