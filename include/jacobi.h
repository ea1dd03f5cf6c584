/* jacobi.h — C-ABI of the B200-native dense Jacobi sweep.
 *
 * Method: Margaris, Souravlas & Roumeliotis, "Parallel implementations of the Jacobi linear
 * algebraic systems solver" (arXiv:1403.5805); citations are lines of /root/reference/PAPER.md.
 *
 *   Sweep (§2 component equation; matrix form X^(k) = T X^(k-1) + C):
 *       x_i^(k) = ( b_i - sum_{j != i} a_ij x_j^(k-1) ) / a_ii        (one IEEE division)
 *   Distance (stop test):  d_k = max_i |x_i^(k) - x_i^(k-1)|   (max norm: BASELINE.json north_star;
 *       PAPER.md:51/94 use the Euclidean norm — DESIGN.md reading R1).  NaN-sticky.
 *   Loop (§2 pseudocode): k = 1..max_iter; stop after sweep k when d_k < tol
 *       (strict) -> JACOBI_CONVERGED, iters = k; else after max_iter sweeps -> JACOBI_MAX_ITER,
 *       iters = max_iter, x = X^(max_iter).  max_iter = 0 returns x0 (MAX_ITER, iters 0).
 *       tol = 0 is the fixed-iteration mode (never converges).
 *   Precondition a_ii != 0: violated -> JACOBI_EZERODIAG (lowest such i).
 *   Row-block distribution (§3 / §3.1): rank r of P owns rows [r*n/P, (r+1)*n/P);
 *       P must divide n.  Every sweep ends with an allgather of x (the MPI_Allgather variant of
 *       §3.1, done with NCCL over NVLink) and a one-scalar max allreduce of d_k — or, after
 *       jacobi_plan_ipc_attach, with the fused exchange: the sweep kernel itself stores its new x
 *       rows into every peer's buffer over NVLink and signals their arrival counters (§3.3 one-sided
 *       puts; overlapping transfer and compute).
 *   Single-GPU solver path (chosen per plan from measured crossovers, same results bit for bit):
 *       small n: one thread-block-cluster launch with A in shared memory; mid-size A (<= 148 MB
 *       fp64 / 300 MB fp32): persistent cooperative launches with a grid barrier per sweep; larger
 *       A: CUDA graphs of sweep kernels.  jacobi_plan_info reports which.
 *
 * Conventions (all functions):
 *   - Sizes are int64_t.  A is row-major: a_ij = A[i*lda + j], lda >= n (elements).  b, x0, x_out
 *     are fp64 of length n (b: length m = rows owned, for the distributed plan).
 *   - A is fp64 (JACOBI_F64) or fp32 (JACOBI_F32: values are widened exactly; all arithmetic fp64).
 *   - Ownership: the caller owns every buffer it passes.  A, b, x0 are read-only and are consumed
 *     before x_out is written, so x_out may alias x0.  A device-resident A passed to a plan
 *     (a_on_device = 1) is BORROWED: it must stay valid and unmodified until jacobi_plan_destroy
 *     (it is copied only when its pointer is not 32-byte aligned or lda is not a multiple of 8).
 *     The library owns its own device allocations and frees them in jacobi_plan_destroy (or before
 *     jacobi_solve returns).
 *   - Outputs (x_out, iters_out, dist_hist) are written only when the status is >= 0 — except the
 *     DEVICE history of jacobi_plan_solve_device, which the kernels fill while the solve runs
 *     (d_dist_hist[k-1] once d_k is known), so a failed device solve may leave it partly written.
 *   - Validation order: JACOBI_EINVAL (n < 1, NULL pointer, lda < n, max_iter < 0, tol < 0 or NaN,
 *     bad dtype) before any CUDA call; then JACOBI_EINDIVISIBLE (distributed, P does not divide n);
 *     then JACOBI_EZERODIAG (lowest i, across ranks); then JACOBI_ENONFINITE (any non-finite value
 *     in A, b or x0).
 *   - Errors: every negative status sets a thread-local message readable with jacobi_last_error().
 *     There is no CPU fallback: without a usable CUDA device the status is JACOBI_ECUDA.
 *   - Determinism: results are bitwise reproducible run to run and bitwise independent of the
 *     number of ranks / row blocks (the per-row summation order depends only on column indices).
 *   - Threading: a plan is used by one host thread at a time; distinct plans are independent.
 *   - Streams: cuda_stream (a cudaStream_t, may be NULL) is the stream every kernel, copy and NCCL
 *     call of the plan is issued on; NULL makes the plan create its own stream, a blocking one
 *     (ordered with the legacy default stream, where device inputs written on stream 0 — torch's
 *     default stream — are complete before the plan reads them).  Device inputs written on any
 *     other stream must be complete, or ordered before the call on cuda_stream, by the caller.
 *     Functions return after the work they enqueue has completed: its results are written and
 *     visible to the host and to any stream.  They synchronize the stream, except a small-n device
 *     solve (one cluster launch), which returns when the kernel's completion record — written after
 *     every result store, behind a system-scope fence — reaches host memory (the kernel may still be
 *     retiring; later work on the stream is ordered after it as usual).
 */
#ifndef JACOBI_H
#define JACOBI_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  JACOBI_CONVERGED = 0,     /* some k <= max_iter had d_k < tol; iters_out = k            */
  JACOBI_MAX_ITER = 1,      /* max_iter sweeps done without d_k < tol (not an error)      */
  JACOBI_EINVAL = -1,       /* bad argument                                               */
  JACOBI_EZERODIAG = -2,    /* a_ii == 0 for some i (message names the lowest i)          */
  JACOBI_ENONFINITE = -3,   /* NaN or Inf in A, b or x0                                   */
  JACOBI_ENOMEM = -4,       /* device or pinned host allocation failed                    */
  JACOBI_ECUDA = -5,        /* CUDA runtime error (message has the CUDA error string)     */
  JACOBI_ENCCL = -6,        /* NCCL error                                                 */
  JACOBI_EINDIVISIBLE = -7  /* distributed: nranks does not divide n                      */
};

enum { JACOBI_F64 = 0, JACOBI_F32 = 1 };
/* Distance of the stop test: the north star's max norm (default) or the paper's Euclidean norm
 * sqrt(sum_i (x_i^(k) - x_i^(k-1))^2) of PAPER.md:94 (summed in a fixed order: trees over blocks of
 * 256 rows, then the block sums; bitwise independent of the rank count when 256 divides n/P). */
enum { JACOBI_NORM_MAX = 0, JACOBI_NORM_L2 = 1 };

typedef struct jacobi_plan jacobi_plan;

/* One-shot solve on the current CUDA device with HOST pointers (A: n x n, lda = n).
 * Copies A, b, x0 to the device, runs the sweeps, copies x back. */
int jacobi_solve(int64_t n, const double* A, const double* b, const double* x0, int64_t max_iter,
                 double tol, double* x_out, int64_t* iters_out);
/* Same with A stored as fp32 (values widened exactly; fp64 accumulation, fp64 x and b). */
int jacobi_solve_f32a(int64_t n, const float* A, const double* b, const double* x0, int64_t max_iter,
                      double tol, double* x_out, int64_t* iters_out);

/* Plan API: uploads (or borrows) A once, validates it (EZERODIAG, ENONFINITE) and keeps the
 * device state, so repeated solves (and timing) exclude the upload.
 *   dtype: JACOBI_F64 / JACOBI_F32;  A: n rows of lda elements, host (a_on_device = 0) or device. */
int jacobi_plan_create(jacobi_plan** out, int64_t n, int dtype, const void* A, int64_t lda,
                       int a_on_device, void* cuda_stream);
/* Solve with HOST pointers: b (n, or m for a distributed plan), x0 (n), x_out (n),
 * dist_hist (nullable; receives d_1..d_iters, needs max_iter entries). */
int jacobi_plan_solve(jacobi_plan* plan, const double* b, const double* x0, int64_t max_iter, double tol,
                      double* x_out, int64_t* iters_out, double* dist_hist);
/* Same contract with DEVICE pointers (b, x0, x_out, dist_hist on the plan's device); only the
 * 48-byte stop state crosses PCIe.  x_out may alias x0.  d_dist_hist (nullable) must hold max_iter
 * doubles — the library cannot check a device pointer's extent (the Python binding does) — and is
 * written by the kernels during the solve (see Outputs above). */
int jacobi_plan_solve_device(jacobi_plan* plan, const double* d_b, const double* d_x0, int64_t max_iter,
                             double tol, double* d_x_out, int64_t* iters_out, double* d_dist_hist);
void jacobi_plan_destroy(jacobi_plan* plan);

/* Test hook for SURVEY.md pin P12(a): run each sweep of a single-GPU plan as `nblocks` row-block
 * launches (nblocks must divide the plan's rows).  Results must be bitwise identical to 1. */
int jacobi_plan_set_row_blocks(jacobi_plan* plan, int nblocks);
/* Select the stop-test norm (JACOBI_NORM_MAX or JACOBI_NORM_L2) for subsequent solves. */
int jacobi_plan_set_norm(jacobi_plan* plan, int norm);
/* Sweeps per captured CUDA graph batch (multiple of 4, 4..1024; default 32).  A tol > 0 solve on a
 * plan without NCCL runs the batches as the body of a device-side while loop (a conditional graph
 * node: one graph launch per solve, the loop condition set by the device's stop decision after each
 * batch; JACOBI_GRAPH_WHILE=0 disables it); fixed-iteration solves and distributed plans launch
 * batches from the host and poll the stop state once per batch.  Sweeps of the batch after the stop
 * decision are no-op launches, so tol runs favour short batches. */
int jacobi_plan_set_batch(jacobi_plan* plan, int sweeps_per_batch);

typedef struct {
  int64_t n, lda, rows, row0;   /* global size, A leading dimension, owned rows, first owned row */
  int dtype, rank, nranks;
  int chunk_cols;               /* column chunk width of the sweep kernel (depends on n only)   */
  int rows_per_warp;            /* rows a warp streams together (x reuse factor)               */
  int grid_ctas, threads_per_cta;
  int a_borrowed;               /* 1 if the caller's device A is used in place                 */
  int64_t sweeps_launched;      /* sweep kernels launched by the last solve (incl. no-ops)     */
  double bytes_per_sweep;       /* algorithmic HBM bytes per sweep: rows*n*s_A + 8n + 16*rows  */
  int variant;                  /* sweep kernel variant in use (JACOBI_SWEEP_VARIANT overrides)  */
  int num_variants;             /* variants compiled in (all give bitwise-identical results)    */
  int cluster_ctas;             /* > 0: small-n plan, each solve runs in one thread-block-cluster
                                   launch with A resident in shared memory (same bits); 0: graph
                                   of sweep kernels.  JACOBI_SMALL_N=0 in the environment disables */
  int persistent_ctas;          /* > 0: mid-size plan, each solve runs as cooperative launches of
                                   this many CTAs (all sweeps of a launch, grid barrier between
                                   sweeps; same bits); JACOBI_PERSIST=0/1 disables / forces it
                                   where it applies (1 GPU, row blocks, max norm)                 */
  int l2_keep_permille;         /* share of each CTA's rows loaded with L2::evict_last (kept in L2
                                   across sweeps; whole 8-row tiles for fp64); 0: A streams with
                                   evict_first.  Changes no result bit.  JACOBI_L2_KEEP overrides  */
} jacobi_plan_info_t;
int jacobi_plan_info(const jacobi_plan* plan, jacobi_plan_info_t* info);

/* Per-sweep kernel timing (CUDA events around each sweep kernel, launched without a graph on the
 * plan's stream): runs `sweeps` fixed sweeps from the given DEVICE b / x0 and writes each kernel's
 * duration in ms.  For roofline measurements; the solve path itself uses CUDA graphs. */
int jacobi_plan_time_sweeps(jacobi_plan* plan, const double* d_b, const double* d_x0, int sweeps,
                            float* ms_out);
/* Per-GPU shard measurement (SURVEY.md §8(e); PAPER.md:72 row blocks, :84-90 per-rank partial
 * products): on a 1-GPU row-wise plan, times `sweeps` (1..4096) fixed sweeps of ONLY rows
 * [rank*n/nranks, (rank+1)*n/nranks) — the work rank `rank` of an nranks-rank row-block plan does per
 * sweep — with the kernel variant, grid and L2-resident share that rank's plan would choose (they depend
 * on the m x n block's shape only), and no exchange.  mode 0: a CUDA graph of sweep kernels (the
 * graph path); 1: the persistent grid solver on the shard; 2: the persistent fused-exchange kernel
 * (k_solve_gridsync_push) with its peer set reduced to this GPU (pushes, remote atomics and arrival
 * counters all local); 3: rank `rank`'s column slab of an nranks-rank column-wise plan (NEXT-4,
 * the n x m slab of columns [rank*m, (rank+1)*m) writing all n row sums, then the
 * epilogue on the rank's m rows; m must be a multiple of 8).  d_b (n) and d_x0 (n) are device vectors.  Writes the average ms per sweep
 * (CUDA events around one warm launch of all sweeps) and, if variant_out is non-NULL, the sweep
 * variant (-1 / -2 for modes 1 / 2; the slab kernel's variant for mode 3).  Rows outside the shard keep x0, so the iterates are not the
 * system's: a measurement hook, not a solver.  Errors: EINVAL (distributed / emulating plan,
 * nranks does not divide n, bad arguments, persistent mode unsupported for this shape, mode 3 with
 * n / nranks not a multiple of 8), ENOMEM (mode 3: no room for the slab copy), ECUDA. */
int jacobi_plan_time_shard(jacobi_plan* plan, int nranks, int rank, const double* d_b, const double* d_x0,
                           int sweeps, int mode, float* ms_per_sweep, int* variant_out);

/* ------------------------------------------------------------------ distributed (NCCL) */
/* Row-block partition of PAPER.md:72: rows [rank*m, (rank+1)*m), m = n/nranks. */
int jacobi_partition(int64_t n, int nranks, int rank, int64_t* row0, int64_t* rows);
/* 128-byte NCCL unique id (rank 0 creates it; the caller broadcasts it, e.g. via torch.distributed). */
int jacobi_nccl_unique_id(void* out128);
/* One process per GPU: rank passes its own row block A_rows (rows x lda, rows = n/nranks).
 * Collective over the nranks processes (all must call it).  Solve then takes b of length rows,
 * x0 and x_out of length n (every rank receives the full solution). */
int jacobi_dist_plan_create(jacobi_plan** out, const void* uid128, int rank, int nranks, int64_t n,
                            int dtype, const void* A_rows, int64_t lda, int a_on_device,
                            void* cuda_stream);

/* Column-wise distribution (§3.2; NEXT-4 comparison scheme): rank r passes the
 * n x m column slab A_cols (rows 0..n-1, columns [r*m, (r+1)*m), lda >= m).  Each sweep computes the
 * slab's partial row sums for all n rows from the rank's own x slice, a reduce-scatter (sum, the
 * "MPI_Allreduce ... MPI_SUM" of PAPER.md:100 restricted to the rows each rank finalizes) gives rank
 * r the sums of rows [r*m, (r+1)*m), and the epilogue updates that slice — the only part of x the
 * rank needs next sweep, so x is allgathered once, at the end.  The rank-sum order is NCCL's, so
 * results are NOT bitwise independent of P (they are within the parity tolerance).  For nranks > 1,
 * m = n / nranks must be a multiple of 8 (32-byte aligned slab columns), else JACOBI_EINVAL. */
int jacobi_dist_plan_create_colwise(jacobi_plan** out, const void* uid128, int rank, int nranks, int64_t n,
                                    int dtype, const void* A_cols, int64_t lda, int a_on_device,
                                    void* cuda_stream);
/* Test hook: emulate a P-slab column-wise sweep on one GPU (P | n, n/P a multiple of 8 when P > 1): P slab launches write row sums,
 * and the epilogue adds the P partials in slab order.  Exercises the slab kernels with col0 > 0. */
int jacobi_plan_set_col_blocks(jacobi_plan* plan, int nblocks);

/* Fused exchange (the non-blocking overlap of PAPER.md:82 and the one-sided
 * put/get of PAPER.md:118-148): instead of NCCL collectives after each sweep, the sweep kernel's
 * epilogue stores every new x_i into every rank's x buffer over NVLink, folds max|dx| into every rank's
 * distance slot with remote atomics, and after a system-scope fence each CTA bumps every rank's
 * arrival counter; the next sweep's prologue waits for its own counter (acquire).  Max norm only.
 *   jacobi_plan_ipc_export: 256 bytes of CUDA IPC handles of this rank's x buffers, slots, counters.
 *   jacobi_plan_ipc_attach: all ranks' 256-byte blocks (rank order) -> peer mappings; enables the mode.
 * Both are called on every rank of a row-wise distributed plan (the caller gathers the handles). */
int jacobi_plan_ipc_export(jacobi_plan* plan, void* out256);
int jacobi_plan_ipc_attach(jacobi_plan* plan, const void* all_handles);
/* Test hook: the fused exchange with P ranks emulated on one GPU (P | n, P <= 8): per-rank x copies,
 * slots and counters; the ranks' sweep kernels run as P sequential launches, so no launch ever waits
 * on a concurrently running one.  Results equal the plain plan bit for bit. */
int jacobi_plan_set_p2p_emulation(jacobi_plan* plan, int P);

/* ------------------------------------------------------------------ measurement */
/* Read-only HBM ceiling: streams `nbytes` of device memory with the sweep kernel's load flavour
 * (256-bit, L1::no_allocate) and returns the best GB/s of `reps` timed passes. */
int jacobi_bwprobe(int64_t nbytes, int reps, double* best_gbs);

const char* jacobi_last_error(void);
int jacobi_version(void); /* 100 * major + minor */
/* Name of a sweep-kernel variant ("k_sweep_cta R4 U1", ...; jacobi_plan_info_t.variant), or NULL
 * when 0 <= variant < num_variants does not hold.  Static storage, never freed.  No CUDA call. */
const char* jacobi_variant_name(int variant);
/* Bounds-checked build (libjacobi_check.so, make lib-check): returns 1 and writes the mask of bounds
 * violations the sweep kernels recorded since the last reset (bit 0/1: A below/past its block, 2: past
 * the row pitch, 3: x read past its buffer, 4: x ring copy, 5: epilogue row); reset != 0 clears it.
 * The release library returns 0 and writes 0.  Debug aid replacing compute-sanitizer on this pool. */
int jacobi_debug_bounds_check(unsigned long long* violations, int reset);

#ifdef __cplusplus
}
#endif
#endif
