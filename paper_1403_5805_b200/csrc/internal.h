// internal.h — plan layout, device stop state and kernel launchers shared by the C-ABI sources.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <string>
#include <vector>
#include "jacobi.h"

namespace jacobi {

// Device-resident stop state of one solve.  Written by the host at solve start,
// then only by the first CTA of a sweep kernel's prologue and by k_advance.
struct State {
  int64_t kbase;      // sweeps of earlier graph batches; sweep k = kbase + j + 1
  int64_t max_iter;   // L of PAPER.md:59
  double tol;         // tol of PAPER.md:59 (strict "<", max norm)
  double* hist;       // d_k history (device, nullable), hist[k-1] = d_k
  int32_t done;       // stop decided
  int32_t status;     // JACOBI_CONVERGED / JACOBI_MAX_ITER once done
  int64_t iters;      // sweeps performed once done
  int32_t nonfinite;  // b or x0 held NaN/Inf (set by k_prepare): every sweep is a no-op, solve -> ENONFINITE
  int32_t fault;      // fused exchange: a peer's signal did not arrive within kPeerWaitNs (JACOBI_ECUDA)
};

// Completion record of a one-launch small-n device solve, written by the kernel into mapped pinned
// host memory (seq last, after a system fence): the host polls it instead of a state copy + stream
// synchronisation.
struct HostDone {
  int32_t status;
  int32_t nonfinite;
  int64_t iters;
  unsigned long long seq;
};

// NEXT-1 fused exchange: every rank's x buffers, distance slots and arrival counters (peer-mapped
// pointers over NVLink, or copies on one GPU when P ranks are emulated).  Device-resident.
enum { kMaxPeers = 8 };
struct PeerArgs {
  int P, rank;
  unsigned long long total_ctas;             // sweep-kernel CTAs over all ranks (arrivals per sweep)
  unsigned long long wait_ns;                // bound on one wait for the peers' signals (then fault)
  double* x0[kMaxPeers];
  double* x1[kMaxPeers];
  unsigned long long* dslot[kMaxPeers];
  unsigned long long* flags[kMaxPeers];      // [2] arrival counters per parity of k
};

// Everything a sweep kernel needs; fixed for the life of a plan (captured into CUDA graphs).
struct SweepArgs {
  const void* A;            // owned rows, row-major, lda elements per row (fp64 or fp32)
  int64_t lda;
  int64_t n;                // global columns
  int64_t m;                // rows handled by this launch
  int64_t row0;             // global index of the launch's first row (diagonal position)
  const double* diag;       // a_ii of the launch's rows (fp64)
  const double* b;          // b of the launch's rows
  double* x0buf;            // full-length x ping-pong buffers: sweep k reads x[(k-1)&1], writes x[k&1]
  double* x1buf;
  double* part;             // partial row sums, part[c * m + r]
  unsigned* cnt;            // per row-tile arrival counters (reset by the finalizing warp)
  unsigned* dyn;            // dynamic tile assignment (variants with DYN): dyn[0] is the launch's
                            // tile-claim counter, dyn[1] counts CTAs that finished their claims; the
                            // last CTA to finish resets both for the next launch (k_prepare zeroes
                            // them per solve).  This needs every CTA of a launch to reach the end of
                            // cta_sweep, i.e. all CTAs agree on s_go (they read the same stop state:
                            // the bounds-checked build checks, in the last CTA, that the claims
                            // add up to ncta * 4 + tiles, i.e. the launch began from zero)
  unsigned long long* dslot;// 4-slot ring of max|dx| bit patterns; sweep k uses slot k & 3
  State* st;
  int64_t col0, cend;       // column range of A held here: [0, n) row-wise; a slab column-wise (NEXT-4)
  double* rsum;             // non-null: write the row sums over [col0, cend) to rsum[row] (column-wise
                            // partial products) instead of applying the epilogue
  double* sq;               // norm == L2: (x_i^(k) - x_i^(k-1))^2 of the launch's rows
  const PeerArgs* peers;    // non-null: fused exchange (NEXT-1) — CTA kernel only
  int norm;                 // JACOBI_NORM_MAX / JACOBI_NORM_L2
  int chunk;                // columns per work item (multiple of 512, depends on n only)
  int nchunks;              // ceil(n / chunk)
  int tiles;                // ceil(m / R)
  int l2_keep_pm;           // per-mille of the work units loaded with L2 evict_last (variants with POL)
  const void* a_base;       // the stored block's allocation and its extent in elements, and the
  int64_t a_elems, x_len;   // x buffers' length: checked by the JACOBI_BOUNDS_CHECK build only
};
// Bounds-checked build (make lib-check -> libjacobi_check.so): every tile's A rows and columns, the
// x range it reads and the rows it writes are checked against the allocations; a violation sets a
// bit in a device flag that jacobi_debug_bounds_check() reports.  The release build compiles the
// checks out.
unsigned long long bounds_violations(bool reset);

// Launchers (sweep.cu).  Return cudaGetLastError() of the launch.
cudaError_t launch_sweep(int dtype, int variant, const SweepArgs& a, int j, int grid, cudaStream_t s);
cudaError_t launch_advance(State* st, unsigned long long* dslot, int K, cudaStream_t s);
cudaError_t launch_advance_while(State* st, unsigned long long* dslot, int K, cudaGraphConditionalHandle h,
                                 cudaStream_t s);
cudaError_t launch_setup_diag(int dtype, const void* A, int64_t lda, int64_t m, int64_t row0,
                              double* diag, unsigned long long* zero_min, cudaStream_t s);
cudaError_t launch_scan_nonfinite_A(int dtype, const void* A, int64_t lda, int64_t m, int64_t n,
                                    int* flag, cudaStream_t s);
cudaError_t launch_prepare(State* st, int64_t max_iter, double tol, double* hist, unsigned long long* dslot,
                           unsigned* cnt, int64_t ncnt, double* b, const double* b_src, int64_t m, double* x0,
                           const double* x0_src, int64_t n, unsigned long long* flags, unsigned long long* gbar,
                           cudaStream_t s);
cudaError_t launch_finalize(const State* st, const double* x0buf, const double* x1buf, double* dst, int64_t n,
                            cudaStream_t s);
cudaError_t launch_copy_pitched(int dtype, const void* src, int64_t src_ld, void* dst, int64_t dst_ld,
                                int64_t rows, int64_t n, cudaStream_t s);
int num_variants();
const char* variant_name(int variant);
int default_variant(int dtype, int nchunks, int chunk, bool l2_keep, int64_t rows, int num_sms);
int slab_variant(int dtype, int nchunks, int chunk, int fallback);  // column slabs (ncols < n)
bool variant_is_cta(int variant);
bool variant_is_push(int variant);
int push_variant(int dtype, int64_t rows, int num_sms);
bool variant_fits(int variant, int nchunks, int dtype, int chunk);
int variant_rows_dt(int variant, int dtype);
int variant_rows(int variant);
int variant_threads(int variant);
int sweep_grid(int dtype, int variant, int num_sms, int nchunks, int chunk);
int chunk_for(int64_t n, int dtype);
// Column-wise epilogue (NEXT-4): s_i = sum over nb partial blocks (ascending), then x_i^(k), |dx|.
cudaError_t launch_colsum_epilogue(const double* rsum, int nb, int64_t stride, int64_t rows, int64_t row0,
                                   const double* b, const double* diag, double* x0buf, double* x1buf,
                                   unsigned long long* dslot, double* sq, int norm, State* st, int j,
                                   cudaStream_t s);
// cluster.cu (NEXT-3 small-n solver)
int cluster_plan(int64_t n, int dtype, size_t* smem);
cudaError_t launch_solve_cluster(int dtype, int C, size_t smem, const void* A, int64_t lda, int64_t n, int chunk,
                                 int norm, const double* diag, const double* b, double* x0buf, double* x1buf,
                                 State* st, int64_t k0, int64_t k1, cudaStream_t s, const double* x0_src = nullptr,
                                 double* x_out = nullptr, int64_t max_iter = 0, double tol = 0.0,
                                 double* hist = nullptr, HostDone* done = nullptr, unsigned long long seq = 0);
enum { kMaxSweepsPerLaunch = 4096 };
enum { kL2Block = 256 };  // rows per L2 partial sum (P-invariant when it divides the rows per rank)
cudaError_t launch_l2_partials(const double* sq, int64_t m, double* blk, const State* st, cudaStream_t s);
cudaError_t launch_l2_final(const double* blk, int64_t nblk, unsigned long long* dslot, State* st, int j,
                            cudaStream_t s);
double bwprobe(int64_t nbytes, int reps);
// Persistent grid solver (NEXT-3, mid-size n): sweeps k0..k1 in one cooperative launch.  With the
// Euclidean rule every CTA reduces all rows' dx^2 itself, for at most kGridMaxL2Rows rows.
enum : int64_t { kGridMaxL2Rows = 64 * kL2Block };
int gridsync_plan(int dtype, int nchunks, int num_sms, size_t* smem);
cudaError_t launch_solve_gridsync(int dtype, const SweepArgs& a, unsigned long long* gbar, int64_t k0, int64_t k1,
                                  int grid, size_t smem, cudaStream_t s);
// ... and over P ranks with the fused exchange (the launch holds nvr virtual ranks when emulated).
int gridsync_push_plan(int dtype, int nchunks, int num_sms, size_t* smem);
cudaError_t launch_solve_gridsync_push(int dtype, const SweepArgs* ranks_dev, int nvr, int64_t k0, int64_t k1,
                                       int grid, size_t smem, cudaStream_t s);

}  // namespace jacobi

// The opaque plan of jacobi.h.
struct jacobi_plan {
  int64_t n = 0, lda = 0, m = 0, row0 = 0;
  int64_t a_rows = 0, a_cols = 0;  // stored block of A: m x n (row-wise) or n x m (column slab)
  int dtype = JACOBI_F64, rank = 0, nranks = 1;
  int device = 0, num_sms = 0, grid = 0;
  int nblocks = 1;               // P12(a) row-block emulation
  bool colwise = false;          // NEXT-4: this rank holds the n x m column slab [row0, row0 + m)
  int colblocks = 1;             // 1-GPU emulation of a P-slab column-wise sweep (test hook)
  double* rsum = nullptr;        // column-wise row sums: colblocks x n (emulation) or n (distributed)
  double* rs_own = nullptr;      // distributed column-wise: reduce-scatter output (m)
  int gemv_variant = 0, gemv_grid = 0;  // kernel for the emulated column slabs
  // NEXT-1 fused exchange
  int p2p = 0;                   // 0 off; >= 1: number of ranks (peer-mapped, or emulated on one GPU)
  bool p2p_emul = false;         // P ranks emulated on this GPU (sequential row-block launches)
  int p2p_drop = -1;             // fault injection (JACOBI_P2P_EMUL_DROP): virtual rank never launched
  jacobi::PeerArgs* peers_dev = nullptr;  // one PeerArgs per (virtual) rank
  unsigned long long* flags = nullptr;    // own arrival counters [2]
  double* ex_x = nullptr;        // emulation: x copies of virtual ranks 1..P-1 (2 buffers each)
  unsigned long long* ex_dslot = nullptr;
  unsigned long long* ex_flags = nullptr;
  std::vector<void*> ipc_open;   // opened peer mappings (closed at destroy)
  // persistent fused-exchange solver (k_solve_gridsync_push): one SweepArgs per (virtual) rank of
  // the launch; emulation uses its own PeerArgs (total_ctas = the one grid's CTAs)
  int push_G = 0;
  size_t push_smem = 0;
  jacobi::SweepArgs* push_ranks_dev = nullptr;
  jacobi::PeerArgs* push_peers_dev = nullptr;
  int variant = 0;               // sweep kernel variant (R, U, threads); default per dtype, JACOBI_SWEEP_VARIANT overrides
  int batch = 32;                // sweeps per graph batch
  int l2_keep_pm = 0;            // per-mille of A's work units kept L2-resident (evict_last) by the POL variants
  int grid_G = 0;                // persistent grid solver: CTAs (0 = not used)
  size_t grid_smem = 0;
  unsigned long long* gbar = nullptr;  // its grid-barrier counter (zeroed per solve)
  int norm = JACOBI_NORM_MAX;    // distance of the stop test
  int cluster_C = 0;             // > 0: small-n solves run in one cluster launch (cluster.cu)
  size_t cluster_smem = 0;
  double* sq = nullptr;          // per-row squared change (L2)
  double* blk = nullptr;         // local L2 block partials (ceil(m / kL2Block))
  double* blk_all = nullptr;     // all ranks' block partials (distributed L2)
  int64_t nblk = 0;
  bool own_stream = false, a_borrowed = false;
  cudaStream_t stream = nullptr;
  const void* dA = nullptr;      // device A (owned or borrowed)
  void* dA_owned = nullptr;
  double* diag = nullptr;
  double* b = nullptr;           // owned copy of b (rows)
  double* x[2] = {nullptr, nullptr};   // full-length ping-pong (x_len doubles each)
  int64_t x_len = 0;
  double* part = nullptr;
  unsigned* cnt = nullptr;
  unsigned long long* dslot = nullptr;
  jacobi::State* st = nullptr;   // device
  jacobi::State* st_host = nullptr;   // pinned mirror
  jacobi::HostDone* done_host = nullptr;  // mapped pinned completion record (one-launch small-n solves)
  jacobi::HostDone* done_dev = nullptr;   // its device address
  unsigned long long done_seq = 0;
  double* hist_dev = nullptr;    // device history buffer for host-pointer solves
  int64_t hist_cap = 0;
  int* flag_dev = nullptr;       // scratch: non-finite flag / zero-diag min index
  unsigned long long* zmin_dev = nullptr;
  ncclComm_t comm = nullptr;     // distributed plans only
  // [0]: a batch of sweeps launched and polled from the host; [1]: a device-side while loop over
  // batches (conditional graph node) used for tol runs; each with the configuration it was built for
  cudaGraphExec_t graphs[2] = {nullptr, nullptr};
  int gkey[2][4] = {{0, 0, -1, 0}, {0, 0, -1, 0}};  // batch, nblocks, norm, colblocks
  int64_t sweeps_launched = 0;
  int chunk = 0;
};

// Error helpers (plan.cu)
int jacobi_set_error(int code, const std::string& msg);
#define JCUDA(call)                                                                             \
  do {                                                                                          \
    cudaError_t _e = (call);                                                                    \
    if (_e != cudaSuccess)                                                                      \
      return jacobi_set_error(_e == cudaErrorMemoryAllocation ? JACOBI_ENOMEM : JACOBI_ECUDA,   \
                              std::string(#call) + ": " + cudaGetErrorString(_e));              \
  } while (0)
#define JRC(call)                                                                               \
  do {                                                                                          \
    int _rc = (call);                                                                           \
    if (_rc) return _rc;                                                                        \
  } while (0)
#define JNCCL(call)                                                                             \
  do {                                                                                          \
    ncclResult_t _r = (call);                                                                   \
    if (_r != ncclSuccess)                                                                      \
      return jacobi_set_error(JACOBI_ENCCL, std::string(#call) + ": " + ncclGetErrorString(_r));\
  } while (0)

// Shared by plan.cu / dist.cu
int plan_init_common(jacobi_plan* p, int64_t n, int64_t m, int64_t row0, int dtype, const void* A,
                     int64_t a_rows, int64_t a_cols, int64_t lda, int a_on_device, void* stream);
int plan_validate_A(jacobi_plan* p, unsigned long long* zero_row, int* nonfinite);
