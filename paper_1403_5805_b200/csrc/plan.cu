// plan.cu — the C-ABI of include/jacobi.h: plans, validation, CUDA-graph sweep batches, stop polling.
//
// Solve loop (PAPER.md:59-66 on the device).  A solve captures, once per plan, a CUDA graph of K
// sweep kernels (+ the exchange collectives for distributed plans) followed by k_advance.  The host
// launches batches with a look-ahead of two and polls the 48-byte device stop state (copied to
// pinned memory behind each batch); sweeps after the device's stop decision exit in their prologue.
// No batch is issued beyond ceil(max_iter / K), so tol = 0 runs never wait on a poll.
#include "internal.h"
#include <atomic>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX: ranges cost nothing unless a tracing tool is attached
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace {
thread_local std::string g_err;
constexpr int kLookahead = 2;

// NVTX range for tracing tools (Nsight Systems / ncu --nvtx): plan setup, solve phases.
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
  Range(const Range&) = delete;
  Range& operator=(const Range&) = delete;
};
// Path choice by size (profiles/size_sweep_r01.jsonl, per-sweep µs, 400-sweep solves):
// - the persistent grid solver removes the ~8 µs per-sweep floor of the graph of sweep kernels
//   (fp64 n = 768-3584: 8.6-20.5 -> 5.2-17.3 µs; c2 4096: 21.8 -> 20.9; fp32 up to n = 8192 / 268 MB:
//   52.0 -> 49.7) and ties or loses beyond (fp64 6144: 53.9 vs 52.9; 12288: 192.6 vs 186.0);
// - the cluster solver (A in shared memory of 16 SMs, conflict-free vector smem loads) beats the
//   persistent solver's ~4 µs floor for small n (cluster vs persistent, JACOBI_CLUSTER_MAXN sweep,
//   profiles/cluster_r01.jsonl: fp64 256: 1.52 vs 4.2, 512: 3.23 vs 4.22, 576: 5.16 vs 4.11; fp32
//   512: 3.14 vs 3.84, 576: 5.21 vs 3.95 — more than 32 rows per CTA puts 3 rows on a warp).
// fp64 limit re-measured with the whole-tile L2 keep (persistent / graph µs per sweep): n = 4224 (143 MB)
// 24.2 / 25.5, 4352 (152 MB) 28.5 / 28.0, 4608 (170 MB) 30.5 / 29.5.
constexpr double kPersistMaxBytesF64 = 148e6, kPersistMaxBytesF32 = 300e6;
constexpr int64_t kClusterPreferMaxN_F64 = 512, kClusterPreferMaxN_F32 = 512;

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }
}  // namespace

int jacobi_set_error(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

extern "C" const char* jacobi_last_error(void) { return g_err.c_str(); }
extern "C" int jacobi_version(void) { return 100; }
extern "C" const char* jacobi_variant_name(int variant) { return jacobi::variant_name(variant); }
extern "C" int jacobi_debug_bounds_check(unsigned long long* violations, int reset) {
#ifdef JACOBI_BOUNDS_CHECK
  if (violations) *violations = jacobi::bounds_violations(reset != 0);
  return 1;
#else
  (void)reset;
  if (violations) *violations = 0;
  return 0;
#endif
}

// Frees everything the plan owns.  Every release is checked; the first failure is reported through
// jacobi_last_error (destroy itself cannot return a status) and the runtime's error state is cleared.
static int plan_free(jacobi_plan* p) {
  if (!p) return 0;
  std::string first;
  auto chk = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && first.empty()) first = std::string(what) + ": " + cudaGetErrorString(e);
  };
  for (cudaGraphExec_t g : p->graphs)
    if (g) chk(cudaGraphExecDestroy(g), "cudaGraphExecDestroy");
  if (p->comm) ncclCommDestroy(p->comm);
  void* dev[] = {p->dA_owned, p->diag, p->b, p->x[0], p->x[1], p->part, p->cnt, p->dslot, p->st,
                 p->hist_dev, p->flag_dev, p->zmin_dev, p->sq, p->blk, p->blk_all, p->rsum, p->rs_own,
                 p->flags, p->ex_x, p->ex_dslot, p->ex_flags, p->peers_dev, p->gbar, p->push_ranks_dev,
                 p->push_peers_dev};
  const char* names[] = {"A", "diag", "b", "x0", "x1", "part", "cnt", "dslot", "state", "hist", "flag", "zmin",
                         "sq", "blk", "blk_all", "rsum", "rs_own", "flags", "ex_x", "ex_dslot", "ex_flags", "peers",
                         "gbar", "push_ranks", "push_peers"};
  for (void* q : p->ipc_open) chk(cudaIpcCloseMemHandle(q), "cudaIpcCloseMemHandle");
  for (size_t i = 0; i < sizeof(dev) / sizeof(dev[0]); ++i)
    if (dev[i]) chk(cudaFree(dev[i]), names[i]);
  if (p->st_host) chk(cudaFreeHost(p->st_host), "cudaFreeHost(state)");
  if (p->done_host) chk(cudaFreeHost(p->done_host), "cudaFreeHost(done)");
  if (p->own_stream && p->stream) chk(cudaStreamDestroy(p->stream), "cudaStreamDestroy");
  delete p;
  cudaGetLastError();
  if (!first.empty()) return jacobi_set_error(JACOBI_ECUDA, "plan release: " + first);
  return 0;
}

// Attribute a pending (asynchronously reported) CUDA error to the step that produced it.
static int check_last(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return jacobi_set_error(JACOBI_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}
#define JLAST(what)                  \
  do {                               \
    int _rc = check_last(what);      \
    if (_rc) return _rc;             \
  } while (0)

// L2-resident share of A (sweep variants with POL), per mille of the stored block's work units: a
// budget of 55 % of the L2 (per-unit Weyl keep walked per warp, µs per sweep at budget 0.45 / 0.55 /
// 0.6 / 0.65: c2 17.4 / 16.7 / 17.0 / 16.5, c3 P = 8 shard graph 35.5 / 34.6 / 34.8 / 36.1, P = 4 72.0 /
// 72.5 / 73.8 / 74.6, profiles/keep_budget*_r02.txt) is kept across sweeps
// with evict_last loads and the rest streams with evict_first, whenever that budget is at least 2 % of
// the block (a smaller share is not worth giving up the dynamic-tile kernel of large blocks).  Each CTA
// keeps that share of its own (tile, chunk) units (keep_unit in sweep.cu), so the kept bytes stay within
// the budget at any row length.  A function of the block's shape only: a P-rank plan's rank applies it
// to its m x n block (c2 keeps 54 %; c3 at P = 1/2/4/8 keeps 3.3 / 6.7 / 13.5 / 27 % of the block; c4 and
// c5 blocks are too large).  JACOBI_L2_KEEP (per mille) and JACOBI_L2_BUDGET (fraction of the L2) override.
static int l2_keep_for(int l2, int64_t a_rows, int64_t a_cols, int dtype, int num_sms) {
  (void)num_sms;
  const double a_bytes = (double)a_rows * (double)a_cols * (dtype == JACOBI_F32 ? 4.0 : 8.0);
  double budget = 0.55;
  if (const char* e = getenv("JACOBI_L2_BUDGET")) budget = atof(e);
  int keep = (l2 > 0 && a_bytes > 0) ? (int)std::min(1000.0, std::floor(1000.0 * budget * l2 / a_bytes)) : 0;
  if (keep < 20) keep = 0;
  if (const char* e = getenv("JACOBI_L2_KEEP")) keep = std::max(0, std::min(1000, atoi(e)));
  return keep;
}

// Sweep-kernel variant for a GEMV over `ncols` columns and `rows` rows per launch (default from
// measurements; the JACOBI_SWEEP_VARIANT override is honoured when the variant can tile the chunking).
static void choose_variant_for(const jacobi_plan* p, int64_t ncols, int64_t rows, int l2_keep_pm, int* variant,
                               int* grid, bool compact_slab = false) {
  const int nch = (int)((ncols + p->chunk - 1) / p->chunk);
  int v = jacobi::default_variant(p->dtype, nch, p->chunk, l2_keep_pm > 0, rows, p->num_sms);
  // a rank's compact column slab (NEXT-4; the 1-GPU P-slab emulation reads strided slabs of the whole A
  // and keeps the default: 380 vs 390 µs per c3 sweep as 8 slabs)
  if (compact_slab && ncols < p->n) v = jacobi::slab_variant(p->dtype, nch, p->chunk, v);
  if (const char* e = getenv("JACOBI_SWEEP_VARIANT")) {  // tuning override (all variants: same bits)
    const int vi = atoi(e);
    if (vi >= 0 && vi < jacobi::num_variants() && !jacobi::variant_is_push(vi) &&
        jacobi::variant_fits(vi, nch, p->dtype, p->chunk))
      v = vi;
  }
  *variant = v;
  *grid = jacobi::sweep_grid(p->dtype, v, p->num_sms, nch, p->chunk);
}
static void choose_variant(const jacobi_plan* p, int64_t ncols, int* variant, int* grid) {
  choose_variant_for(p, ncols, p->colwise ? p->n : p->m / p->nblocks, p->l2_keep_pm, variant, grid,
                     p->colwise && ncols == p->m);
}

// Common plan setup.  The stored block of A is a_rows x a_cols (row-major, lda): the m x n row block
// (row-wise) or the n x m column slab [row0, row0 + m) (column-wise, NEXT-4).
int plan_init_common(jacobi_plan* p, int64_t n, int64_t m, int64_t row0, int dtype, const void* A, int64_t a_rows,
                     int64_t a_cols, int64_t lda, int a_on_device, void* stream) {
  Range nvtx_range("jacobi: plan setup (A upload)");
  JLAST("pending CUDA error before plan creation");
  p->n = n;
  p->m = m;
  p->row0 = row0;
  p->dtype = dtype;
  p->a_rows = a_rows;
  p->a_cols = a_cols;
  JCUDA(cudaGetDevice(&p->device));
  JCUDA(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, p->device));
  int major = 0;
  JCUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, p->device));
  if (major != 10) return jacobi_set_error(JACOBI_ECUDA, "device is not sm_100 (B200); this build targets sm_100a only");
  if (stream) {
    p->stream = (cudaStream_t)stream;
  } else {
    // A blocking stream: ordered with the legacy default stream, so device buffers the caller filled
    // there (e.g. torch's default stream, handle 0) are complete before the plan reads them.
    JCUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamDefault));
    p->own_stream = true;
  }
  const int64_t elt = dtype == JACOBI_F32 ? 4 : 8;
  const int64_t lda_dev = round_up(a_cols, 8);
  if (a_on_device && ((uintptr_t)A % 32 == 0) && lda % 8 == 0) {
    p->dA = A;
    p->lda = lda;
    p->a_borrowed = true;
  } else {
    JCUDA(cudaMalloc(&p->dA_owned, (size_t)(a_rows * lda_dev * elt)));
    p->lda = lda_dev;
    p->dA = p->dA_owned;
    if (a_on_device) {
      JCUDA(jacobi::launch_copy_pitched(dtype, A, lda, p->dA_owned, lda_dev, a_rows, a_cols, p->stream));
    } else if (lda == lda_dev) {
      JCUDA(cudaMemcpyAsync(p->dA_owned, A, (size_t)(a_rows * lda * elt), cudaMemcpyHostToDevice, p->stream));
    } else {
      JCUDA(cudaMemsetAsync(p->dA_owned, 0, (size_t)(a_rows * lda_dev * elt), p->stream));
      JCUDA(cudaMemcpy2DAsync(p->dA_owned, (size_t)(lda_dev * elt), A, (size_t)(lda * elt), (size_t)(a_cols * elt),
                              (size_t)a_rows, cudaMemcpyHostToDevice, p->stream));
    }
  }
  JLAST("A upload");
  p->chunk = jacobi::chunk_for(n, dtype);
  {
    int l2 = 0;
    JCUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, p->device));
    p->l2_keep_pm = l2_keep_for(l2, a_rows, a_cols, dtype, p->num_sms);
  }
  choose_variant(p, a_cols, &p->variant, &p->grid);
  JLAST("sweep kernel occupancy query");
  p->x_len = round_up(n, 256) + 256;
  const int64_t nchunks = (a_cols + p->chunk - 1) / p->chunk;
  JCUDA(cudaMalloc(&p->diag, (size_t)m * 8));
  JCUDA(cudaMalloc(&p->b, (size_t)m * 8));
  JCUDA(cudaMalloc(&p->x[0], (size_t)p->x_len * 8));
  JCUDA(cudaMalloc(&p->x[1], (size_t)p->x_len * 8));
  JCUDA(cudaMalloc(&p->part, (size_t)(nchunks * a_rows) * 8));
  JCUDA(cudaMalloc(&p->cnt, (size_t)a_rows * 4 * 5));  // + 4 dynamic-tile counters per row block
  p->nblk = (m + jacobi::kL2Block - 1) / jacobi::kL2Block;
  JCUDA(cudaMalloc(&p->sq, (size_t)m * 2 * 8));  // two halves: the persistent solver double-buffers dx^2
  JCUDA(cudaMalloc(&p->blk, (size_t)p->nblk * 8));
  JCUDA(cudaMalloc(&p->dslot, 4 * 8));
  JCUDA(cudaMalloc(&p->gbar, 8));
  JCUDA(cudaMalloc(&p->flags, 2 * 8));
  JCUDA(cudaMemsetAsync(p->flags, 0, 2 * 8, p->stream));
  JCUDA(cudaMalloc(&p->st, sizeof(jacobi::State)));
  JCUDA(cudaMalloc(&p->flag_dev, 16));
  JCUDA(cudaMalloc(&p->zmin_dev, 8));
  JCUDA(cudaMallocHost(&p->st_host, kLookahead * sizeof(jacobi::State)));
  JCUDA(cudaHostAlloc(&p->done_host, sizeof(jacobi::HostDone), cudaHostAllocMapped));
  p->done_host->seq = 0;
  JCUDA(cudaHostGetDevicePointer(&p->done_dev, p->done_host, 0));
  JCUDA(cudaMemsetAsync(p->x[0], 0, (size_t)p->x_len * 8, p->stream));
  JCUDA(cudaMemsetAsync(p->x[1], 0, (size_t)p->x_len * 8, p->stream));
  JCUDA(cudaMemsetAsync(p->cnt, 0, (size_t)a_rows * 4 * 5, p->stream));
  JLAST("plan buffers");
  return 0;
}

// Setup kernels: diag gather + lowest zero-diagonal row + non-finite scan of A.
int plan_validate_A(jacobi_plan* p, unsigned long long* zero_row, int* nonfinite) {
  JCUDA(cudaMemsetAsync(p->zmin_dev, 0xff, 8, p->stream));
  JCUDA(cudaMemsetAsync(p->flag_dev, 0, 4, p->stream));
  // a_ii of the owned rows: row block -> A[r][row0 + r]; column slab -> A[row0 + r][r].
  const size_t esz = p->dtype == JACOBI_F32 ? 4 : 8;
  const void* dbase = p->colwise ? (const char*)p->dA + (size_t)(p->row0 * p->lda - p->row0) * esz : p->dA;
  JCUDA(jacobi::launch_setup_diag(p->dtype, dbase, p->lda, p->m, p->row0, p->diag, p->zmin_dev, p->stream));
  JCUDA(jacobi::launch_scan_nonfinite_A(p->dtype, p->dA, p->lda, p->a_rows, p->a_cols, p->flag_dev, p->stream));
  if (p->comm) {
    JNCCL(ncclAllReduce(p->zmin_dev, p->zmin_dev, 1, ncclUint64, ncclMin, p->comm, p->stream));
    JNCCL(ncclAllReduce(p->flag_dev, p->flag_dev, 1, ncclInt32, ncclMax, p->comm, p->stream));
  }
  JCUDA(cudaMemcpyAsync(zero_row, p->zmin_dev, 8, cudaMemcpyDeviceToHost, p->stream));
  JCUDA(cudaMemcpyAsync(nonfinite, p->flag_dev, 4, cudaMemcpyDeviceToHost, p->stream));
  JCUDA(cudaStreamSynchronize(p->stream));
  return 0;
}

static int validate_result(unsigned long long zero_row, int nonfinite) {
  if (zero_row != ~0ull)
    return jacobi_set_error(JACOBI_EZERODIAG, "a_ii == 0 at i = " + std::to_string(zero_row) +
                                                  " (PAPER.md:53: the method needs a_ii != 0)");
  if (nonfinite) return jacobi_set_error(JACOBI_ENONFINITE, "A contains NaN or Inf");
  return 0;
}

extern "C" int jacobi_plan_create(jacobi_plan** out, int64_t n, int dtype, const void* A, int64_t lda,
                                  int a_on_device, void* cuda_stream) {
  if (!out || !A || n < 1 || lda < n || (dtype != JACOBI_F64 && dtype != JACOBI_F32))
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_create: bad argument (out/A NULL, n < 1, lda < n or dtype)");
  jacobi_plan* p = new jacobi_plan();
  int rc = plan_init_common(p, n, n, 0, dtype, A, n, n, lda, a_on_device, cuda_stream);
  if (rc == 0) {
    const char* e = getenv("JACOBI_SMALL_N");
    if (!(e && e[0] == '0')) p->cluster_C = jacobi::cluster_plan(n, dtype, &p->cluster_smem);
    rc = check_last("small-n cluster setup");
  }
  if (rc == 0) {  // persistent grid solver where it applies (NEXT-3, mid-size n)
    const char* e = getenv("JACOBI_PERSIST");
    const double a_bytes = (double)n * (double)n * (dtype == JACOBI_F32 ? 4.0 : 8.0);
    const bool want = e ? e[0] == '1' : a_bytes <= (dtype == JACOBI_F32 ? kPersistMaxBytesF32 : kPersistMaxBytesF64);
    if (want && n >= p->num_sms)
      p->grid_G = jacobi::gridsync_plan(dtype, (int)((n + p->chunk - 1) / p->chunk), p->num_sms, &p->grid_smem);
    cudaGetLastError();  // an unsupported configuration only leaves the path off
  }
  unsigned long long zr = 0;
  int nf = 0;
  if (rc == 0) rc = plan_validate_A(p, &zr, &nf);
  if (rc == 0) rc = validate_result(zr, nf);
  if (rc != 0) {
    std::string keep = g_err;
    plan_free(p);
    g_err = keep;
    return rc;
  }
  *out = p;
  return 0;
}

extern "C" void jacobi_plan_destroy(jacobi_plan* p) {
  if (p && p->stream) cudaStreamSynchronize(p->stream);
  int rc = plan_free(p);
  if (rc && getenv("JACOBI_DEBUG")) fprintf(stderr, "jacobi_plan_destroy: %s\n", jacobi_last_error());
}

extern "C" int jacobi_plan_set_row_blocks(jacobi_plan* p, int nblocks) {
  if (!p || nblocks < 1 || p->m % nblocks != 0 || p->comm || p->p2p)
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_set_row_blocks: nblocks must divide the rows of a 1-GPU plan");
  p->nblocks = nblocks;
  return 0;
}

extern "C" int jacobi_plan_set_col_blocks(jacobi_plan* p, int nblocks) {
  if (!p || nblocks < 1 || p->n % nblocks != 0 || p->comm || p->colwise || p->p2p ||
      (nblocks > 1 && (p->n / nblocks) % 8 != 0))
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_set_col_blocks: nblocks must divide n of a 1-GPU plan "
                                           "into slabs of a multiple of 8 columns (32-byte aligned loads)");
  if (nblocks > 1) {
    cudaFree(p->rsum);
    p->rsum = nullptr;
    JCUDA(cudaMalloc(&p->rsum, (size_t)(nblocks * p->n) * 8));
    choose_variant(p, p->n / nblocks, &p->gemv_variant, &p->gemv_grid);
    JLAST("column-block setup");
  }
  p->colblocks = nblocks;
  return 0;
}

// NEXT-1 helpers --------------------------------------------------------------------------------
// Bound on one wait for the peers' sweep signals: 10 s, or JACOBI_PEER_WAIT_MS.
static unsigned long long peer_wait_ns() {
  const char* e = getenv("JACOBI_PEER_WAIT_MS");
  const long long ms = e ? atoll(e) : 10000;
  return (unsigned long long)std::max(1ll, ms) * 1000000ull;
}

static int p2p_pick_variant(jacobi_plan* p, int64_t rows_per_rank) {
  const int nch = (int)((p->n + p->chunk - 1) / p->chunk);
  int v = jacobi::push_variant(p->dtype, rows_per_rank, p->num_sms);
  if (!jacobi::variant_fits(v, nch, p->dtype, p->chunk)) v = jacobi::push_variant(p->dtype, 0, p->num_sms);
  if (!jacobi::variant_fits(v, nch, p->dtype, p->chunk))
    return jacobi_set_error(JACOBI_EINVAL, "fused exchange needs the CTA sweep kernel (n with >= 16 chunks)");
  p->variant = v;
  p->grid = jacobi::sweep_grid(p->dtype, v, p->num_sms, nch, p->chunk);
  return check_last("fused-exchange variant");
}

extern "C" int jacobi_plan_set_p2p_emulation(jacobi_plan* p, int P) {
  if (!p || P < 1 || P > jacobi::kMaxPeers || p->comm || p->colwise || p->colblocks > 1 || p->m % P != 0 ||
      p->norm != JACOBI_NORM_MAX || p->p2p)
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_set_p2p_emulation: 1-GPU max-norm plan, P in [1, 8] dividing n, once");
  JRC(p2p_pick_variant(p, p->m / P));
  if (P > 1) {
    JCUDA(cudaMalloc(&p->ex_x, (size_t)(P - 1) * 2 * p->x_len * 8));
    JCUDA(cudaMemsetAsync(p->ex_x, 0, (size_t)(P - 1) * 2 * p->x_len * 8, p->stream));
    JCUDA(cudaMalloc(&p->ex_dslot, (size_t)(P - 1) * 4 * 8));
    JCUDA(cudaMalloc(&p->ex_flags, (size_t)(P - 1) * 2 * 8));
  }
  std::vector<jacobi::PeerArgs> pa(P);
  for (int r = 0; r < P; ++r) {
    jacobi::PeerArgs& a = pa[r];
    std::memset(&a, 0, sizeof(a));
    a.P = P;
    a.rank = r;
    a.total_ctas = (unsigned long long)P * p->grid;
    a.wait_ns = peer_wait_ns();
    for (int q = 0; q < P; ++q) {
      a.x0[q] = q == 0 ? p->x[0] : p->ex_x + (size_t)(q - 1) * 2 * p->x_len;
      a.x1[q] = q == 0 ? p->x[1] : a.x0[q] + p->x_len;
      a.dslot[q] = q == 0 ? p->dslot : p->ex_dslot + (size_t)(q - 1) * 4;
      a.flags[q] = q == 0 ? p->flags : p->ex_flags + (size_t)(q - 1) * 2;
    }
  }
  JCUDA(cudaMalloc(&p->peers_dev, sizeof(jacobi::PeerArgs) * P));
  JCUDA(cudaMemcpyAsync(p->peers_dev, pa.data(), sizeof(jacobi::PeerArgs) * P, cudaMemcpyHostToDevice, p->stream));
  JCUDA(cudaStreamSynchronize(p->stream));
  p->p2p = P;
  p->p2p_emul = true;
  p->nblocks = P;
  if (const char* e = getenv("JACOBI_P2P_EMUL_DROP")) p->p2p_drop = atoi(e);  // fault-injection test hook
  return 0;
}

extern "C" int jacobi_plan_ipc_export(jacobi_plan* p, void* out256) {
  if (!p || !out256 || !p->comm || p->colwise)
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_ipc_export: row-wise distributed plan and a 256-byte buffer");
  cudaIpcMemHandle_t h[4];
  JCUDA(cudaIpcGetMemHandle(&h[0], p->x[0]));
  JCUDA(cudaIpcGetMemHandle(&h[1], p->x[1]));
  JCUDA(cudaIpcGetMemHandle(&h[2], p->dslot));
  JCUDA(cudaIpcGetMemHandle(&h[3], p->flags));
  static_assert(sizeof(h) == 256, "4 IPC handles");
  std::memcpy(out256, h, sizeof(h));
  return 0;
}

extern "C" int jacobi_plan_ipc_attach(jacobi_plan* p, const void* all_handles) {
  if (!p || !all_handles || !p->comm || p->colwise || p->nranks > jacobi::kMaxPeers || p->norm != JACOBI_NORM_MAX ||
      p->p2p)
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_ipc_attach: row-wise max-norm distributed plan, <= 8 ranks, once");
  JRC(p2p_pick_variant(p, p->m));
  jacobi::PeerArgs a;
  std::memset(&a, 0, sizeof(a));
  a.P = p->nranks;
  a.rank = p->rank;
  a.total_ctas = (unsigned long long)p->nranks * p->grid;  // same device type on every rank
  a.wait_ns = peer_wait_ns();
  const cudaIpcMemHandle_t* h = static_cast<const cudaIpcMemHandle_t*>(all_handles);
  for (int q = 0; q < p->nranks; ++q) {
    if (q == p->rank) {
      a.x0[q] = p->x[0];
      a.x1[q] = p->x[1];
      a.dslot[q] = p->dslot;
      a.flags[q] = p->flags;
      continue;
    }
    void* ptr[4];
    for (int i = 0; i < 4; ++i) JCUDA(cudaIpcOpenMemHandle(&ptr[i], h[q * 4 + i], cudaIpcMemLazyEnablePeerAccess));
    a.x0[q] = static_cast<double*>(ptr[0]);
    a.x1[q] = static_cast<double*>(ptr[1]);
    a.dslot[q] = static_cast<unsigned long long*>(ptr[2]);
    a.flags[q] = static_cast<unsigned long long*>(ptr[3]);
    p->ipc_open.push_back(ptr[0]);
    p->ipc_open.push_back(ptr[1]);
    p->ipc_open.push_back(ptr[2]);
    p->ipc_open.push_back(ptr[3]);
  }
  JCUDA(cudaMalloc(&p->peers_dev, sizeof(a)));
  JCUDA(cudaMemcpyAsync(p->peers_dev, &a, sizeof(a), cudaMemcpyHostToDevice, p->stream));
  JCUDA(cudaStreamSynchronize(p->stream));
  p->p2p = p->nranks;
  return 0;
}

extern "C" int jacobi_plan_set_norm(jacobi_plan* p, int norm) {
  if (!p || (norm != JACOBI_NORM_MAX && norm != JACOBI_NORM_L2))
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_set_norm: norm must be JACOBI_NORM_MAX or JACOBI_NORM_L2");
  if (norm == JACOBI_NORM_L2 && p->p2p)
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_set_norm: the fused exchange supports the max norm only");
  if (norm == JACOBI_NORM_L2 && p->comm && !p->blk_all) {
    JCUDA(cudaMalloc(&p->blk_all, (size_t)(p->nblk * p->nranks) * 8));
  }
  p->norm = norm;
  return 0;
}

extern "C" int jacobi_plan_set_batch(jacobi_plan* p, int K) {
  if (!p || K < 4 || K > 1024 || K % 4 != 0)
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_set_batch: K must be a multiple of 4 in [4, 1024]");
  p->batch = K;
  return 0;
}

// The persistent grid solver applies to 1-GPU row-block plans (the Euclidean rule up to
// kGridMaxL2Rows rows); the cluster solver (both norms) to 1-GPU plans whose A fits its shared
// memory.  Where both apply, the cluster solver is preferred only for small n (the measured
// crossover above) unless JACOBI_PERSIST=1 forces the grid solver.
static bool grid_applies(const jacobi_plan* p) {
  return p->grid_G > 0 && p->nblocks == 1 && p->colblocks == 1 && !p->comm && !p->p2p && !p->colwise &&
         (p->norm == JACOBI_NORM_MAX || p->m <= (int64_t)jacobi::kGridMaxL2Rows);
}
static bool use_cluster(const jacobi_plan* p) {
  if (!(p->cluster_C && p->nblocks == 1 && p->colblocks == 1 && !p->comm && !p->p2p)) return false;
  const char* e = getenv("JACOBI_PERSIST");
  const bool force_grid = e && e[0] == '1';
  int64_t prefer = p->dtype == JACOBI_F32 ? kClusterPreferMaxN_F32 : kClusterPreferMaxN_F64;
  if (const char* m = getenv("JACOBI_CLUSTER_MAXN")) prefer = atoll(m);  // tuning override
  return !grid_applies(p) || (!force_grid && p->n <= prefer);
}
static bool use_grid(const jacobi_plan* p) { return grid_applies(p) && !use_cluster(p); }
// Persistent fused-exchange solver: opt-in (JACOBI_PERSIST=1) on a fused-exchange plan.
static bool use_grid_push(const jacobi_plan* p) {
  const char* e = getenv("JACOBI_PERSIST");
  return p->p2p && e && e[0] == '1' && p->norm == JACOBI_NORM_MAX && p->colblocks == 1 && !p->colwise;
}


extern "C" int jacobi_plan_info(const jacobi_plan* p, jacobi_plan_info_t* info) {
  if (!p || !info) return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_info: NULL argument");
  info->n = p->n;
  info->lda = p->lda;
  info->rows = p->m;
  info->row0 = p->row0;
  info->dtype = p->dtype;
  info->rank = p->rank;
  info->nranks = p->nranks;
  info->chunk_cols = p->chunk;
  info->rows_per_warp = jacobi::variant_rows_dt(p->variant, p->dtype);
  info->grid_ctas = p->grid;
  info->threads_per_cta = jacobi::variant_threads(p->variant);
  info->a_borrowed = p->a_borrowed ? 1 : 0;
  info->sweeps_launched = p->sweeps_launched;
  const double sA = p->dtype == JACOBI_F32 ? 4.0 : 8.0;
  info->bytes_per_sweep = (double)p->m * (double)p->n * sA + 8.0 * (double)p->n + 16.0 * (double)p->m;
  info->variant = p->variant;
  info->num_variants = jacobi::num_variants();
  info->cluster_ctas = use_cluster(p) ? p->cluster_C : 0;
  info->persistent_ctas = use_grid(p) ? p->grid_G : (use_grid_push(p) ? p->num_sms : 0);
  info->l2_keep_permille = p->l2_keep_pm;
  return 0;
}

static jacobi::SweepArgs sweep_args(const jacobi_plan* p, int blk) {
  const int64_t mb = p->m / p->nblocks;
  const int64_t esz = p->dtype == JACOBI_F32 ? 4 : 8;
  jacobi::SweepArgs a;
  a.A = (const char*)p->dA + (size_t)(blk * mb * p->lda * esz);
  a.lda = p->lda;
  a.n = p->n;
  a.m = mb;
  a.row0 = p->row0 + blk * mb;
  a.diag = p->diag + blk * mb;
  a.b = p->b + blk * mb;
  a.x0buf = p->x[0];
  a.x1buf = p->x[1];
  a.part = p->part;
  a.cnt = p->cnt;
  a.dyn = p->cnt + p->a_rows + 4 * blk;
  a.dslot = p->dslot;
  a.st = p->st;
  a.col0 = 0;
  a.cend = p->n;
  a.rsum = nullptr;
  a.peers = nullptr;
  a.sq = p->sq + blk * mb;
  a.norm = p->norm;
  a.chunk = p->chunk;
  a.nchunks = (int)((p->n + p->chunk - 1) / p->chunk);
  const int R = jacobi::variant_rows_dt(p->variant, p->dtype);
  a.tiles = (int)((mb + R - 1) / R);
  a.l2_keep_pm = p->l2_keep_pm;
  a.a_base = p->dA;
  a.a_elems = p->a_rows * p->lda;
  a.x_len = p->x_len;
#ifdef JACOBI_BOUNDS_CHECK
  if (getenv("JACOBI_CHECK_SELFTEST")) a.a_elems -= p->lda;  // checker self-test: the last row is "outside"
#endif
  return a;
}

// The sweep kernels of sweep j: row blocks (row-wise; P12a emulation when nblocks > 1), or column
// slabs writing row sums (column-wise NEXT-4: this rank's slab, or the 1-GPU P-slab emulation).
static int launch_gemv(jacobi_plan* p, int j) {
  if (p->p2p) {  // NEXT-1 fused exchange: (virtual) rank r's launch reads and signals its own copies
    const int nr = p->p2p_emul ? p->p2p : 1;
    for (int r = 0; r < nr; ++r) {
      if (p->p2p_emul && r == p->p2p_drop) continue;  // injected fault: this virtual rank never signals
      jacobi::SweepArgs a = sweep_args(p, p->p2p_emul ? r : 0);
      a.peers = p->peers_dev + r;
      if (p->p2p_emul && r > 0) {
        a.x0buf = p->ex_x + (size_t)(r - 1) * 2 * p->x_len;
        a.x1buf = a.x0buf + p->x_len;
        a.dslot = p->ex_dslot + (size_t)(r - 1) * 4;
      }
      JCUDA(jacobi::launch_sweep(p->dtype, p->variant, a, j, p->grid, p->stream));
    }
    return 0;
  }
  if (!p->colwise && p->colblocks == 1) {
    for (int blk = 0; blk < p->nblocks; ++blk)
      JCUDA(jacobi::launch_sweep(p->dtype, p->variant, sweep_args(p, blk), j, p->grid, p->stream));
    return 0;
  }
  const int nb = p->colwise ? 1 : p->colblocks;
  const int64_t w = p->colwise ? p->m : p->n / nb;  // slab width
  const size_t esz = p->dtype == JACOBI_F32 ? 4 : 8;
  const int v = p->colwise ? p->variant : p->gemv_variant;
  const int grid = p->colwise ? p->grid : p->gemv_grid;
  for (int q = 0; q < nb; ++q) {
    jacobi::SweepArgs a = sweep_args(p, 0);
    a.col0 = p->colwise ? p->row0 : q * w;
    a.cend = a.col0 + w;
    // pointer to column col0 of row 0 of the stored block (kernels index A by global column)
    a.A = p->colwise ? p->dA : (const char*)p->dA + (size_t)(q * w) * esz;
    a.m = p->n;  // every row of the system
    a.row0 = 0;
    a.rsum = p->rsum + (size_t)q * p->n;
    a.nchunks = (int)((w + p->chunk - 1) / p->chunk);
    const int R = jacobi::variant_rows_dt(v, p->dtype);
    a.tiles = (int)((p->n + R - 1) / R);
    JCUDA(jacobi::launch_sweep(p->dtype, v, a, j, grid, p->stream));
  }
  return 0;
}

// Enqueue sweep j of a batch plus, for distributed plans, the exchange:
// row-wise: in-place allgather of the new x slice and max-allreduce of d_k's bits; column-wise:
// reduce-scatter (sum) of the row sums, the epilogue on the owned rows, and the max-allreduce.
static int enqueue_sweep(jacobi_plan* p, int j) {
  JRC(launch_gemv(p, j));
  if (p->p2p) return 0;  // the exchange happened inside the sweep kernel
  if (p->colwise) {
    JNCCL(ncclReduceScatter(p->rsum, p->rs_own, (size_t)p->m, ncclDouble, ncclSum, p->comm, p->stream));
    JCUDA(jacobi::launch_colsum_epilogue(p->rs_own, 1, p->m, p->m, p->row0, p->b, p->diag, p->x[0], p->x[1],
                                         p->dslot, p->sq, p->norm, p->st, j, p->stream));
  } else if (p->colblocks > 1) {
    JCUDA(jacobi::launch_colsum_epilogue(p->rsum, p->colblocks, p->n, p->n, 0, p->b, p->diag, p->x[0], p->x[1],
                                         p->dslot, p->sq, p->norm, p->st, j, p->stream));
  }
  if (p->comm && p->colwise) {
    if (p->norm == JACOBI_NORM_MAX)
      JNCCL(ncclAllReduce(p->dslot + ((j + 1) & 3), p->dslot + ((j + 1) & 3), 1, ncclUint64, ncclMax, p->comm,
                          p->stream));
  } else if (p->comm) {
    // k = kbase + j + 1 with kbase a multiple of the batch size (a multiple of 4): parity is static.
    // One NCCL group: the allgather of x and the one-scalar max allreduce go out as one launch.
    double* xk = p->x[(j + 1) & 1];
    JNCCL(ncclGroupStart());
    JNCCL(ncclAllGather(xk + p->row0, xk, (size_t)p->m, ncclDouble, p->comm, p->stream));
    if (p->norm == JACOBI_NORM_MAX)
      JNCCL(ncclAllReduce(p->dslot + ((j + 1) & 3), p->dslot + ((j + 1) & 3), 1, ncclUint64, ncclMax, p->comm,
                          p->stream));
    JNCCL(ncclGroupEnd());
  }
  if (p->norm == JACOBI_NORM_L2) {  // PAPER.md:94 Euclidean distance, fixed-order reduction
    JCUDA(jacobi::launch_l2_partials(p->sq, p->m, p->blk, p->st, p->stream));
    const double* all = p->blk;
    int64_t nall = p->nblk;
    if (p->comm) {
      JNCCL(ncclAllGather(p->blk, p->blk_all, (size_t)p->nblk, ncclDouble, p->comm, p->stream));
      all = p->blk_all;
      nall = p->nblk * p->nranks;
    }
    JCUDA(jacobi::launch_l2_final(all, nall, p->dslot, p->st, j, p->stream));
  }
  return 0;
}

// Device-side loop (plans without NCCL): one graph whose only node is a conditional WHILE node; its
// body is a batch of K sweeps followed by k_advance_while, which settles the stop decision for the
// batch's last sweep and sets the loop condition, so a solve is one graph launch and one wait — no
// host polling and no look-ahead batches of no-op sweeps after the stop.  JACOBI_GRAPH_WHILE=0 falls
// back to host-polled batches (also used by distributed plans: NCCL is not captured into a
// conditional body).
static bool want_while_graph(const jacobi_plan* p) {
  const char* e = getenv("JACOBI_GRAPH_WHILE");
  return !p->comm && !(e && e[0] == '0');
}

static int build_while_graph(jacobi_plan* p) {
  cudaGraph_t g = nullptr;
  JCUDA(cudaGraphCreate(&g, 0));
  int rc = 0;
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNode_t node;
  cudaGraphNodeParams cp = {};
  if (e == cudaSuccess) {
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
  }
  if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(p->stream, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                          cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g);
    cudaGetLastError();
    return jacobi_set_error(JACOBI_ECUDA, std::string("while graph: ") + cudaGetErrorString(e));
  }
  for (int j = 0; j < p->batch && rc == 0; ++j) rc = enqueue_sweep(p, j);
  if (rc == 0) {
    cudaError_t ae = jacobi::launch_advance_while(p->st, p->dslot, p->batch, h, p->stream);
    if (ae != cudaSuccess) rc = jacobi_set_error(JACOBI_ECUDA, std::string("k_advance_while: ") + cudaGetErrorString(ae));
  }
  cudaGraph_t body = nullptr;
  cudaError_t ee = cudaStreamEndCapture(p->stream, &body);
  if (rc == 0 && ee != cudaSuccess) rc = jacobi_set_error(JACOBI_ECUDA, std::string("while body capture: ") + cudaGetErrorString(ee));
  if (rc == 0) {
    cudaError_t ie = cudaGraphInstantiate(&p->graphs[1], g, 0);
    if (ie != cudaSuccess) rc = jacobi_set_error(JACOBI_ECUDA, std::string("while graph instantiate: ") + cudaGetErrorString(ie));
  }
  cudaGraphDestroy(g);
  cudaGetLastError();
  return rc;
}

// The graph for a solve: the device-side while loop (wg) or a host-polled batch, built on first use
// for the plan's current configuration and cached.  Returns the slot used (0 or 1).
static int ensure_graph(jacobi_plan* p, bool wg, int* slot) {
  const int key[4] = {p->batch, p->nblocks, p->norm, p->colblocks};
  const int w = wg ? 1 : 0;
  *slot = w;
  if (p->graphs[w] && std::memcmp(p->gkey[w], key, sizeof(key)) == 0) return 0;
  if (p->graphs[w]) {
    cudaGraphExecDestroy(p->graphs[w]);
    p->graphs[w] = nullptr;
  }
  if (wg) {
    JRC(build_while_graph(p));
    std::memcpy(p->gkey[1], key, sizeof(key));
    return 0;
  }
  cudaGraph_t g = nullptr;
  JCUDA(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
  int rc = 0;
  for (int j = 0; j < p->batch && rc == 0; ++j) rc = enqueue_sweep(p, j);
  if (rc == 0) {
    cudaError_t e = jacobi::launch_advance(p->st, p->dslot, p->batch, p->stream);
    if (e != cudaSuccess) rc = jacobi_set_error(JACOBI_ECUDA, std::string("k_advance: ") + cudaGetErrorString(e));
  }
  cudaError_t ee = cudaStreamEndCapture(p->stream, &g);
  if (rc != 0) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (ee != cudaSuccess) return jacobi_set_error(JACOBI_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ee));
  cudaError_t ie = cudaGraphInstantiate(&p->graphs[0], g, 0);
  cudaGraphDestroy(g);
  if (ie != cudaSuccess) return jacobi_set_error(JACOBI_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
  std::memcpy(p->gkey[0], key, sizeof(key));
  return 0;
}

// Copies inputs in and resets the device stop state: two copies, one memset and k_prepare (which
// also scans b and x0 for NaN/Inf).  No host round trip: ENONFINITE is read with the stop state.
static int solve_prepare(jacobi_plan* p, const double* b, const double* x0, bool dev, int64_t max_iter, double tol,
                         double* hist_dev) {
  Range nvtx_range("jacobi: solve prepare");
  if (!dev) {  // host inputs: H2D copies; device inputs are copied by k_prepare itself
    JCUDA(cudaMemcpyAsync(p->b, b, (size_t)p->m * 8, cudaMemcpyHostToDevice, p->stream));
    JCUDA(cudaMemcpyAsync(p->x[0], x0, (size_t)p->n * 8, cudaMemcpyHostToDevice, p->stream));
  }
  JCUDA(cudaMemsetAsync(p->st, 0, sizeof(jacobi::State), p->stream));
  JCUDA(jacobi::launch_prepare(p->st, max_iter, tol, hist_dev, p->dslot, p->cnt, p->a_rows * 5, p->b, dev ? b : nullptr,
                               p->m, p->x[0], dev ? x0 : nullptr, p->n, p->p2p ? p->flags : nullptr, p->gbar,
                               p->stream));
  if (p->p2p_emul) {  // virtual ranks 1..P-1: their x^(0), slots and counters
    for (int r = 1; r < p->p2p; ++r)
      JCUDA(cudaMemcpyAsync(p->ex_x + (size_t)(r - 1) * 2 * p->x_len, p->x[0], (size_t)p->n * 8,
                            cudaMemcpyDeviceToDevice, p->stream));
    JCUDA(cudaMemsetAsync(p->ex_dslot, 0, (size_t)(p->p2p - 1) * 4 * 8, p->stream));
    JCUDA(cudaMemsetAsync(p->ex_flags, 0, (size_t)(p->p2p - 1) * 2 * 8, p->stream));
  }
  if (p->comm)
    JNCCL(ncclAllReduce(&p->st->nonfinite, &p->st->nonfinite, 1, ncclInt32, ncclMax, p->comm, p->stream));
  return 0;
}

static int nonfinite_error() { return jacobi_set_error(JACOBI_ENONFINITE, "b or x0 contains NaN or Inf"); }

// Runs graph batches until the device decides to stop.  Fills *fin with the final state.
static int solve_run(jacobi_plan* p, int64_t max_iter, double tol, jacobi::State* fin) {
  Range nvtx_range("jacobi: sweeps (CUDA graph batches)");
  // tol runs stop where the device decides: loop on the device (no polling, no look-ahead batches of
  // no-op sweeps).  Fixed runs know their batch count: host-launched batches cost nothing extra there,
  // and keep every sweep kernel visible to launch-level profilers.
  int w = 0;
  int rc = ensure_graph(p, tol > 0 && want_while_graph(p), &w);
  if (rc && w == 1) rc = ensure_graph(p, false, &w);  // no conditional nodes here: host-polled batches
  if (rc) return rc;
  const int64_t K = p->batch;
  cudaGraphExec_t graph = p->graphs[w];
  if (w == 1) {  // the whole solve: one launch of the device-side loop, one wait
    JCUDA(cudaGraphLaunch(graph, p->stream));
    JCUDA(cudaMemcpyAsync(&p->st_host[0], p->st, sizeof(jacobi::State), cudaMemcpyDeviceToHost, p->stream));
    cudaError_t se = cudaStreamSynchronize(p->stream);
    if (se != cudaSuccess) return jacobi_set_error(JACOBI_ECUDA, std::string("sweep loop: ") + cudaGetErrorString(se));
    const jacobi::State& s = p->st_host[0];
    if (s.nonfinite) return nonfinite_error();
    if (s.fault) return jacobi_set_error(JACOBI_ECUDA, "fused exchange: a peer's sweep signal did not arrive within the wait bound");
    if (!s.done) return jacobi_set_error(JACOBI_ECUDA, "internal: device loop ended without a stop decision");
    p->sweeps_launched = ((std::max<int64_t>(s.iters, 1) + K - 1) / K) * K * p->nblocks;  // batches run x K
    *fin = s;
    return 0;
  }
  const int64_t max_batches = (max_iter + K - 1) / K;  // the stop is decided within these
  cudaEvent_t ev[kLookahead];
  for (int i = 0; i < kLookahead; ++i) JCUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  int64_t issued = 0, waited = 0;
  bool done = false;
  p->sweeps_launched = 0;
  auto issue = [&]() -> int {
    const int slot = (int)(issued % kLookahead);
    JCUDA(cudaGraphLaunch(graph, p->stream));
    JCUDA(cudaMemcpyAsync(&p->st_host[slot], p->st, sizeof(jacobi::State), cudaMemcpyDeviceToHost, p->stream));
    JCUDA(cudaEventRecord(ev[slot], p->stream));
    ++issued;
    p->sweeps_launched += K * p->nblocks;
    return 0;
  };
  while (rc == 0 && issued < std::min<int64_t>(kLookahead, max_batches)) rc = issue();
  while (rc == 0 && !done) {
    const int slot = (int)(waited % kLookahead);
    cudaError_t e = cudaEventSynchronize(ev[slot]);
    if (e != cudaSuccess) { rc = jacobi_set_error(JACOBI_ECUDA, std::string("sweep batch: ") + cudaGetErrorString(e)); break; }
    if (p->comm) {
      ncclResult_t ar = ncclSuccess;
      ncclCommGetAsyncError(p->comm, &ar);
      if (ar != ncclSuccess && ar != ncclInProgress) { rc = jacobi_set_error(JACOBI_ENCCL, ncclGetErrorString(ar)); break; }
    }
    ++waited;
    if (p->st_host[slot].nonfinite) {
      rc = nonfinite_error();
      break;
    }
    if (p->st_host[slot].fault) {
      rc = jacobi_set_error(JACOBI_ECUDA, "fused exchange: a peer's sweep signal did not arrive within 10 s");
      break;
    }
    if (p->st_host[slot].done) {
      *fin = p->st_host[slot];
      done = true;
      break;
    }
    if (waited >= max_batches) {
      rc = jacobi_set_error(JACOBI_ECUDA, "internal: stop not decided after max_iter sweeps");
      break;
    }
    if (issued < max_batches) rc = issue();
  }
  cudaError_t se = cudaStreamSynchronize(p->stream);  // drain look-ahead no-op batches
  for (int i = 0; i < kLookahead; ++i) cudaEventDestroy(ev[i]);
  if (rc == 0 && se != cudaSuccess) rc = jacobi_set_error(JACOBI_ECUDA, std::string("sync: ") + cudaGetErrorString(se));
  return rc;
}

// Small-n path (NEXT-3): the whole solve in cluster launches of at most kMaxSweepsPerLaunch sweeps.
// dev_out (device solves): k_finalize copies x^(iters) there before the state is read back, so the
// solve needs one host synchronisation.
static int solve_cluster(jacobi_plan* p, int64_t max_iter, jacobi::State* fin, double* dev_out) {
  Range nvtx_range("jacobi: sweeps (cluster solver)");
  p->sweeps_launched = 0;
  for (int64_t k0 = 1;;) {
    const int64_t k1 = std::min<int64_t>(k0 + jacobi::kMaxSweepsPerLaunch - 1, max_iter);
    JCUDA(jacobi::launch_solve_cluster(p->dtype, p->cluster_C, p->cluster_smem, p->dA, p->lda, p->n, p->chunk,
                                       p->norm, p->diag, p->b, p->x[0], p->x[1], p->st, k0, k1, p->stream));
    if (dev_out) JCUDA(jacobi::launch_finalize(p->st, p->x[0], p->x[1], dev_out, p->n, p->stream));
    JCUDA(cudaMemcpyAsync(&p->st_host[0], p->st, sizeof(jacobi::State), cudaMemcpyDeviceToHost, p->stream));
    JCUDA(cudaStreamSynchronize(p->stream));
    p->sweeps_launched += 1;
    if (p->st_host[0].nonfinite) return nonfinite_error();
    if (p->st_host[0].done) {
      *fin = p->st_host[0];
      return 0;
    }
    if (k1 >= max_iter) return jacobi_set_error(JACOBI_ECUDA, "internal: small-n solve ended without a stop decision");
    k0 = k1 + 1;
  }
}

// Persistent path (NEXT-3, mid-size n): the solve in cooperative launches of at most
// kMaxSweepsPerLaunch sweeps.
static int solve_grid(jacobi_plan* p, int64_t max_iter, jacobi::State* fin, double* dev_out) {
  Range nvtx_range("jacobi: sweeps (persistent grid solver)");
  p->sweeps_launched = 0;
  const jacobi::SweepArgs a = sweep_args(p, 0);
  for (int64_t k0 = 1;;) {
    const int64_t k1 = std::min<int64_t>(k0 + jacobi::kMaxSweepsPerLaunch - 1, max_iter);
    JCUDA(jacobi::launch_solve_gridsync(p->dtype, a, p->gbar, k0, k1, p->grid_G, p->grid_smem, p->stream));
    if (dev_out) JCUDA(jacobi::launch_finalize(p->st, p->x[0], p->x[1], dev_out, p->n, p->stream));
    JCUDA(cudaMemcpyAsync(&p->st_host[0], p->st, sizeof(jacobi::State), cudaMemcpyDeviceToHost, p->stream));
    JCUDA(cudaStreamSynchronize(p->stream));
    p->sweeps_launched += 1;
    if (p->st_host[0].fault)
      return jacobi_set_error(JACOBI_ECUDA, "persistent solver: grid barrier wait timed out");
    if (p->st_host[0].nonfinite) return nonfinite_error();
    if (p->st_host[0].done) {
      *fin = p->st_host[0];
      return 0;
    }
    if (k1 >= max_iter) return jacobi_set_error(JACOBI_ECUDA, "internal: persistent solve ended without a stop decision");
    k0 = k1 + 1;
  }
}

// Persistent fused-exchange solver (opt-in with JACOBI_PERSIST=1 on a fused-exchange plan; validated
// with emulated ranks on one GPU): builds the per-rank launch arguments once, then runs the solve in
// cooperative launches of at most kMaxSweepsPerLaunch sweeps, like solve_grid.

static int grid_push_setup(jacobi_plan* p) {
  if (p->push_ranks_dev) return 0;
  const int nch = (int)((p->n + p->chunk - 1) / p->chunk);
  p->push_G = jacobi::gridsync_push_plan(p->dtype, nch, p->num_sms, &p->push_smem);
  cudaGetLastError();
  if (!p->push_G) return jacobi_set_error(JACOBI_EINVAL, "persistent fused exchange: configuration not supported");
  const int nvr = p->p2p_emul ? p->p2p : 1;
  std::vector<jacobi::SweepArgs> ra(nvr);
  std::vector<jacobi::PeerArgs> pa;
  if (p->p2p_emul) {  // the emulated ranks' PeerArgs, with the one grid's CTAs as the arrival count
    pa.resize(nvr);
    JCUDA(cudaMemcpy(pa.data(), p->peers_dev, sizeof(jacobi::PeerArgs) * nvr, cudaMemcpyDeviceToHost));
    for (auto& q : pa) q.total_ctas = (unsigned long long)p->push_G;
    JCUDA(cudaMalloc(&p->push_peers_dev, sizeof(jacobi::PeerArgs) * nvr));
    JCUDA(cudaMemcpy(p->push_peers_dev, pa.data(), sizeof(jacobi::PeerArgs) * nvr, cudaMemcpyHostToDevice));
  } else {
    jacobi::PeerArgs q;  // real ranks: every rank launches push_G CTAs
    JCUDA(cudaMemcpy(&q, p->peers_dev, sizeof(q), cudaMemcpyDeviceToHost));
    q.total_ctas = (unsigned long long)p->nranks * p->push_G;
    JCUDA(cudaMalloc(&p->push_peers_dev, sizeof(q)));
    JCUDA(cudaMemcpy(p->push_peers_dev, &q, sizeof(q), cudaMemcpyHostToDevice));
  }
  for (int r = 0; r < nvr; ++r) {
    jacobi::SweepArgs a = sweep_args(p, p->p2p_emul ? r : 0);
    a.peers = p->push_peers_dev + r;
    if (p->p2p_emul && r > 0) {
      a.x0buf = p->ex_x + (size_t)(r - 1) * 2 * p->x_len;
      a.x1buf = a.x0buf + p->x_len;
      a.dslot = p->ex_dslot + (size_t)(r - 1) * 4;
    }
    ra[r] = a;
  }
  JCUDA(cudaMalloc(&p->push_ranks_dev, sizeof(jacobi::SweepArgs) * nvr));
  JCUDA(cudaMemcpy(p->push_ranks_dev, ra.data(), sizeof(jacobi::SweepArgs) * nvr, cudaMemcpyHostToDevice));
  return 0;
}

static int solve_grid_push(jacobi_plan* p, int64_t max_iter, jacobi::State* fin, double* dev_out) {
  Range nvtx_range("jacobi: sweeps (persistent fused exchange)");
  JRC(grid_push_setup(p));
  p->sweeps_launched = 0;
  const int nvr = p->p2p_emul ? p->p2p : 1;
  for (int64_t k0 = 1;;) {
    const int64_t k1 = std::min<int64_t>(k0 + jacobi::kMaxSweepsPerLaunch - 1, max_iter);
    JCUDA(jacobi::launch_solve_gridsync_push(p->dtype, p->push_ranks_dev, nvr, k0, k1, p->push_G, p->push_smem,
                                             p->stream));
    if (dev_out) JCUDA(jacobi::launch_finalize(p->st, p->x[0], p->x[1], dev_out, p->n, p->stream));
    JCUDA(cudaMemcpyAsync(&p->st_host[0], p->st, sizeof(jacobi::State), cudaMemcpyDeviceToHost, p->stream));
    JCUDA(cudaStreamSynchronize(p->stream));
    p->sweeps_launched += 1;
    if (p->st_host[0].fault)
      return jacobi_set_error(JACOBI_ECUDA, "fused exchange: a peer's sweep signal did not arrive within the wait bound");
    if (p->st_host[0].nonfinite) return nonfinite_error();
    if (p->st_host[0].done) {
      *fin = p->st_host[0];
      return 0;
    }
    if (k1 >= max_iter) return jacobi_set_error(JACOBI_ECUDA, "internal: persistent solve ended without a stop decision");
    k0 = k1 + 1;
  }
}

static int solve_impl(jacobi_plan* p, const double* b, const double* x0, bool dev, int64_t max_iter, double tol,
                      double* x_out, int64_t* iters_out, double* hist) {
  Range nvtx_range("jacobi: solve");
  if (!p || !b || !x0 || !x_out || !iters_out || max_iter < 0 || std::isnan(tol) || tol < 0)
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_solve: bad argument (NULL pointer, max_iter < 0, tol < 0 or NaN)");
  JCUDA(cudaSetDevice(p->device));
  double* hist_dev = nullptr;
  if (hist && max_iter > 0) {
    if (dev) {
      hist_dev = hist;
    } else {
      if (p->hist_cap < max_iter) {
        cudaFree(p->hist_dev);
        p->hist_dev = nullptr;
        p->hist_cap = 0;
        JCUDA(cudaMalloc(&p->hist_dev, (size_t)max_iter * 8));
        p->hist_cap = max_iter;
      }
      hist_dev = p->hist_dev;
    }
  }
  if (dev && max_iter > 0 && max_iter <= jacobi::kMaxSweepsPerLaunch && use_cluster(p)) {
    // Small-n device solve in ONE launch: the cluster kernel initialises the stop state, scans b and
    // x0, reads them in place and writes x_out itself; one read-back of the state, one sync.
    Range nvtx_fused("jacobi: sweeps (cluster solver, fused start)");
    const unsigned long long seq = ++p->done_seq;
    JCUDA(jacobi::launch_solve_cluster(p->dtype, p->cluster_C, p->cluster_smem, p->dA, p->lda, p->n, p->chunk,
                                       p->norm, p->diag, b, p->x[0], p->x[1], p->st, 1, max_iter, p->stream, x0,
                                       x_out, max_iter, tol, hist_dev, p->done_dev, seq));
    p->sweeps_launched = 1;
    // Poll the mapped completion record (written after x_out is globally visible); every 256 polls
    // ask the stream, so a kernel that ended without writing it (an error) is caught by the
    // synchronising read-back below.
    volatile jacobi::HostDone* d = p->done_host;
    for (unsigned i = 1;; ++i) {
      if (d->seq == seq) {
        std::atomic_thread_fence(std::memory_order_acquire);
        if (d->nonfinite) return nonfinite_error();
        *iters_out = d->iters;
        return d->status;
      }
      if ((i & 255) == 0 && cudaStreamQuery(p->stream) != cudaErrorNotReady) break;
    }
    JCUDA(cudaMemcpyAsync(&p->st_host[0], p->st, sizeof(jacobi::State), cudaMemcpyDeviceToHost, p->stream));
    JCUDA(cudaStreamSynchronize(p->stream));
    JLAST("solve");
    if (p->st_host[0].nonfinite) return nonfinite_error();
    if (!p->st_host[0].done) return jacobi_set_error(JACOBI_ECUDA, "internal: small-n solve ended without a stop decision");
    *iters_out = p->st_host[0].iters;
    return p->st_host[0].status;
  }
  int rc = solve_prepare(p, b, x0, dev, max_iter, tol, hist_dev);
  if (rc < 0) return rc;
  jacobi::State fin{};
  bool finalized = false;  // x_out already written on the device (k_finalize, device solves)
  if (max_iter == 0) {  // X^0 (reading R14), once the inputs are known to be finite
    JCUDA(cudaMemcpyAsync(&p->st_host[0], p->st, sizeof(jacobi::State), cudaMemcpyDeviceToHost, p->stream));
    JCUDA(cudaStreamSynchronize(p->stream));
    if (p->st_host[0].nonfinite) return nonfinite_error();
    fin.status = JACOBI_MAX_ITER;
    fin.iters = 0;
  } else if (use_cluster(p)) {
    rc = solve_cluster(p, max_iter, &fin, dev ? x_out : nullptr);
    if (rc) return rc;
    finalized = dev;
  } else if (use_grid(p)) {
    rc = solve_grid(p, max_iter, &fin, dev ? x_out : nullptr);
    if (rc) return rc;
    finalized = dev;
  } else if (use_grid_push(p)) {
    rc = solve_grid_push(p, max_iter, &fin, dev ? x_out : nullptr);
    if (rc) return rc;
    finalized = dev;
  } else {
    rc = solve_run(p, max_iter, tol, &fin);
    if (rc) return rc;
  }
  if (p->colwise && fin.iters > 0) {  // column-wise ranks hold only their slice: assemble x^(iters)
    double* xf = p->x[fin.iters & 1];
    JNCCL(ncclAllGather(xf + p->row0, xf, (size_t)p->m, ncclDouble, p->comm, p->stream));
  }
  const cudaMemcpyKind kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (!finalized) JCUDA(cudaMemcpyAsync(x_out, p->x[fin.iters & 1], (size_t)p->n * 8, kind, p->stream));
  if (hist && !dev && fin.iters > 0)
    JCUDA(cudaMemcpyAsync(hist, hist_dev, (size_t)fin.iters * 8, cudaMemcpyDeviceToHost, p->stream));
  if (!finalized || (hist && !dev && fin.iters > 0)) JCUDA(cudaStreamSynchronize(p->stream));
  JLAST("solve");
  *iters_out = fin.iters;
  return fin.status;
}

extern "C" int jacobi_plan_solve(jacobi_plan* p, const double* b, const double* x0, int64_t max_iter, double tol,
                                 double* x_out, int64_t* iters_out, double* dist_hist) {
  return solve_impl(p, b, x0, false, max_iter, tol, x_out, iters_out, dist_hist);
}

extern "C" int jacobi_plan_solve_device(jacobi_plan* p, const double* b, const double* x0, int64_t max_iter,
                                        double tol, double* x_out, int64_t* iters_out, double* dist_hist) {
  return solve_impl(p, b, x0, true, max_iter, tol, x_out, iters_out, dist_hist);
}

extern "C" int jacobi_plan_time_sweeps(jacobi_plan* p, const double* d_b, const double* d_x0, int sweeps,
                                       float* ms_out) {
  if (!p || !d_b || !d_x0 || sweeps < 1 || !ms_out)
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_time_sweeps: bad argument");
  JCUDA(cudaSetDevice(p->device));
  int rc = solve_prepare(p, d_b, d_x0, true, sweeps, 0.0, nullptr);
  if (rc < 0) return rc;
  JCUDA(cudaMemcpyAsync(&p->st_host[0], p->st, sizeof(jacobi::State), cudaMemcpyDeviceToHost, p->stream));
  JCUDA(cudaStreamSynchronize(p->stream));
  if (p->st_host[0].nonfinite) return nonfinite_error();
  cudaEvent_t e0, e1;
  JCUDA(cudaEventCreate(&e0));
  JCUDA(cudaEventCreate(&e1));
  for (int j = 0; j < sweeps && rc == 0; ++j) {
    cudaEventRecord(e0, p->stream);
    rc = launch_gemv(p, j);  // the sweep kernel(s) alone are timed
    cudaEventRecord(e1, p->stream);
    if (rc == 0) rc = [&]() -> int {  // the rest of the sweep (exchange, column-wise epilogue)
      if (p->p2p) return 0;           // fused exchange: nothing outside the kernel
      if (p->colwise) {
        JNCCL(ncclReduceScatter(p->rsum, p->rs_own, (size_t)p->m, ncclDouble, ncclSum, p->comm, p->stream));
        JCUDA(jacobi::launch_colsum_epilogue(p->rs_own, 1, p->m, p->m, p->row0, p->b, p->diag, p->x[0], p->x[1],
                                             p->dslot, p->sq, JACOBI_NORM_MAX, p->st, j, p->stream));
      } else if (p->colblocks > 1) {
        JCUDA(jacobi::launch_colsum_epilogue(p->rsum, p->colblocks, p->n, p->n, 0, p->b, p->diag, p->x[0],
                                             p->x[1], p->dslot, p->sq, JACOBI_NORM_MAX, p->st, j, p->stream));
      }
      if (p->comm && !p->colwise) {
        double* xk = p->x[(j + 1) & 1];
        JNCCL(ncclAllGather(xk + p->row0, xk, (size_t)p->m, ncclDouble, p->comm, p->stream));
      }
      if (p->comm)
        JNCCL(ncclAllReduce(p->dslot + ((j + 1) & 3), p->dslot + ((j + 1) & 3), 1, ncclUint64, ncclMax, p->comm,
                            p->stream));
      return 0;
    }();
    cudaError_t se = cudaEventSynchronize(e1);
    if (se != cudaSuccess && rc == 0) rc = jacobi_set_error(JACOBI_ECUDA, cudaGetErrorString(se));
    if (rc == 0) cudaEventElapsedTime(&ms_out[j], e0, e1);
  }
  cudaStreamSynchronize(p->stream);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return rc;
}

// Per-GPU shard measurement (see jacobi.h): the sweeps rank `rank` of an nranks-rank row-block plan
// would run on its m x n block — the same kernel variant, grid and L2-resident share its plan would
// choose (they depend on the block's shape only) — timed on this GPU without the exchange.
extern "C" int jacobi_plan_time_shard(jacobi_plan* p, int nranks, int rank, const double* d_b, const double* d_x0,
                                      int sweeps, int mode, float* ms_per_sweep, int* variant_out) {
  if (!p || nranks < 1 || rank < 0 || rank >= nranks || !d_b || !d_x0 || sweeps < 1 ||
      sweeps > jacobi::kMaxSweepsPerLaunch || mode < 0 || mode > 3 || !ms_per_sweep || p->comm || p->colwise ||
      p->p2p || p->nblocks != 1 || p->colblocks != 1 || p->n % nranks != 0)
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_time_shard: 1-GPU row-wise plan, nranks | n, 0 <= rank < "
                                           "nranks, 1 <= sweeps <= 4096, mode 0/1/2/3");
  if (mode == 3 && (p->n / nranks) % 8 != 0)
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_time_shard: column slabs need n / nranks a multiple of 8");
  JCUDA(cudaSetDevice(p->device));
  const int64_t ms = p->n / nranks, r0 = (int64_t)rank * ms;
  int l2 = 0;
  JCUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, p->device));
  const int keep = l2_keep_for(l2, ms, p->n, p->dtype, p->num_sms);
  int v = 0, grid = 0;
  choose_variant_for(p, p->n, ms, keep, &v, &grid);
  JLAST("shard variant");
  const int64_t esz = p->dtype == JACOBI_F32 ? 4 : 8;
  jacobi::SweepArgs a = sweep_args(p, 0);
  a.A = (const char*)p->dA + (size_t)(r0 * p->lda * esz);
  a.m = ms;
  a.row0 = r0;
  a.diag = p->diag + r0;
  a.b = p->b + r0;
  a.sq = p->sq + r0;
  a.tiles = (int)((ms + jacobi::variant_rows_dt(v, p->dtype) - 1) / jacobi::variant_rows_dt(v, p->dtype));
  a.l2_keep_pm = keep;
  double* slab_rsum = nullptr;
  void* slab_A = nullptr;
  if (mode == 3) {  // NEXT-4: rank `rank`'s n x m column slab (columns [r0, r0 + m)) writing all n row sums,
    // stored as that rank stores it: a compact n x m block (lda = m), copied out of this plan's A
    const int keep3 = l2_keep_for(l2, p->n, ms, p->dtype, p->num_sms);
    choose_variant_for(p, ms, p->n, keep3, &v, &grid, true);
    JLAST("slab variant");
    a = sweep_args(p, 0);
    a.col0 = r0;
    a.cend = r0 + ms;
    cudaError_t e = cudaMalloc(&slab_A, (size_t)(p->n * ms * esz));
    if (e == cudaSuccess) e = cudaMalloc(&slab_rsum, (size_t)p->n * 8);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(slab_A, (size_t)(ms * esz), (const char*)p->dA + (size_t)(r0 * esz), (size_t)(p->lda * esz),
                            (size_t)(ms * esz), (size_t)p->n, cudaMemcpyDeviceToDevice, p->stream);
    if (e != cudaSuccess) {  // nothing else is allocated yet
      if (slab_A) cudaFree(slab_A);
      if (slab_rsum) cudaFree(slab_rsum);
      cudaGetLastError();
      return jacobi_set_error(e == cudaErrorMemoryAllocation ? JACOBI_ENOMEM : JACOBI_ECUDA,
                              std::string("jacobi_plan_time_shard (column slab): ") + cudaGetErrorString(e));
    }
    a.A = slab_A;  // kernels index A by global column: row i, column c at A[i * lda + c - col0]
    a.lda = ms;
    a.a_base = slab_A;
    a.a_elems = p->n * ms;
    a.m = p->n;
    a.row0 = 0;
    a.nchunks = (int)((ms + p->chunk - 1) / p->chunk);
    a.tiles = (int)((p->n + jacobi::variant_rows_dt(v, p->dtype) - 1) / jacobi::variant_rows_dt(v, p->dtype));
    a.l2_keep_pm = keep3;
    a.rsum = slab_rsum;
  }
  int rc = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaGraphExec_t gx = nullptr;
  jacobi::SweepArgs* ra = nullptr;
  jacobi::PeerArgs* pa = nullptr;
  size_t smem = 0;
  int G = 0;
  auto prepare = [&]() -> int {
    JRC(solve_prepare(p, d_b, d_x0, true, sweeps, 0.0, nullptr));
    JCUDA(cudaMemsetAsync(p->flags, 0, 2 * 8, p->stream));
    return 0;
  };
  auto launch = [&]() -> int {
    if (mode == 0 || mode == 3) {
      JCUDA(cudaGraphLaunch(gx, p->stream));
    } else if (mode == 1) {
      JCUDA(jacobi::launch_solve_gridsync(p->dtype, a, p->gbar, 1, sweeps, G, smem, p->stream));
    } else {
      JCUDA(jacobi::launch_solve_gridsync_push(p->dtype, ra, 1, 1, sweeps, G, smem, p->stream));
    }
    return 0;
  };
  rc = [&]() -> int {
    const int nch = (int)((p->n + p->chunk - 1) / p->chunk);
    if (mode == 0 || mode == 3) {  // a graph of `sweeps` sweep kernels, like the rank's graph minus the collectives
      cudaGraph_t g = nullptr;
      JCUDA(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
      int lrc = 0;
      for (int j = 0; j < sweeps && lrc == 0; ++j) {
        cudaError_t e = jacobi::launch_sweep(p->dtype, v, a, j, grid, p->stream);
        if (e == cudaSuccess && mode == 3)  // the rank's epilogue on its own m rows (after the reduce-scatter)
          e = jacobi::launch_colsum_epilogue(slab_rsum + r0, 1, ms, ms, r0, p->b + r0, p->diag + r0, p->x[0], p->x[1],
                                             p->dslot, p->sq, JACOBI_NORM_MAX, p->st, j, p->stream);
        if (e != cudaSuccess) lrc = jacobi_set_error(JACOBI_ECUDA, std::string("shard sweep: ") + cudaGetErrorString(e));
      }
      cudaError_t ee = cudaStreamEndCapture(p->stream, &g);
      if (lrc) { if (g) cudaGraphDestroy(g); return lrc; }
      JCUDA(ee);
      cudaError_t ie = cudaGraphInstantiate(&gx, g, 0);
      cudaGraphDestroy(g);
      JCUDA(ie);
    } else if (mode == 1) {  // the persistent grid solver restricted to the shard's rows
      G = jacobi::gridsync_plan(p->dtype, nch, p->num_sms, &smem);
      cudaGetLastError();
      if (!G) return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_time_shard: persistent solver not supported here");
      v = -1;
    } else {  // the persistent fused-exchange kernel of a rank, its peer set reduced to this GPU
      G = jacobi::gridsync_push_plan(p->dtype, nch, p->num_sms, &smem);
      cudaGetLastError();
      if (!G) return jacobi_set_error(JACOBI_EINVAL, "jacobi_plan_time_shard: persistent fused exchange not supported");
      jacobi::PeerArgs q;
      std::memset(&q, 0, sizeof(q));
      q.P = 1;
      q.rank = 0;
      q.total_ctas = (unsigned long long)G;
      q.wait_ns = peer_wait_ns();
      q.x0[0] = p->x[0];
      q.x1[0] = p->x[1];
      q.dslot[0] = p->dslot;
      q.flags[0] = p->flags;
      JCUDA(cudaMalloc(&pa, sizeof(q)));
      JCUDA(cudaMemcpy(pa, &q, sizeof(q), cudaMemcpyHostToDevice));
      a.peers = pa;
      JCUDA(cudaMalloc(&ra, sizeof(a)));
      JCUDA(cudaMemcpy(ra, &a, sizeof(a), cudaMemcpyHostToDevice));
      v = -2;
    }
    JCUDA(cudaEventCreate(&e0));
    JCUDA(cudaEventCreate(&e1));
    JRC(prepare());
    JRC(launch());  // warm-up (graph upload, L2 state)
    JRC(prepare());
    JCUDA(cudaEventRecord(e0, p->stream));
    JRC(launch());
    JCUDA(cudaEventRecord(e1, p->stream));
    JCUDA(cudaEventSynchronize(e1));
    float ms_tot = 0.f;
    JCUDA(cudaEventElapsedTime(&ms_tot, e0, e1));
    JCUDA(cudaMemcpy(&p->st_host[0], p->st, sizeof(jacobi::State), cudaMemcpyDeviceToHost));
    if (p->st_host[0].fault) return jacobi_set_error(JACOBI_ECUDA, "jacobi_plan_time_shard: wait timed out");
    *ms_per_sweep = ms_tot / (float)sweeps;
    if (variant_out) *variant_out = v;
    return 0;
  }();
  cudaStreamSynchronize(p->stream);
  if (gx) cudaGraphExecDestroy(gx);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (ra) cudaFree(ra);
  if (pa) cudaFree(pa);
  if (slab_rsum) cudaFree(slab_rsum);
  if (slab_A) cudaFree(slab_A);
  cudaGetLastError();
  return rc;
}

static int solve_oneshot(int64_t n, int dtype, const void* A, const double* b, const double* x0, int64_t max_iter,
                         double tol, double* x_out, int64_t* iters_out) {
  if (n < 1 || !A || !b || !x0 || !x_out || !iters_out || max_iter < 0 || std::isnan(tol) || tol < 0)
    return jacobi_set_error(JACOBI_EINVAL, "jacobi_solve: bad argument (n < 1, NULL pointer, max_iter < 0, tol < 0 or NaN)");
  jacobi_plan* p = nullptr;
  int rc = jacobi_plan_create(&p, n, dtype, A, n, 0, nullptr);
  if (rc) return rc;
  rc = jacobi_plan_solve(p, b, x0, max_iter, tol, x_out, iters_out, nullptr);
  std::string keep = g_err;
  jacobi_plan_destroy(p);
  g_err = keep;
  return rc;
}

extern "C" int jacobi_solve(int64_t n, const double* A, const double* b, const double* x0, int64_t max_iter,
                            double tol, double* x_out, int64_t* iters_out) {
  return solve_oneshot(n, JACOBI_F64, A, b, x0, max_iter, tol, x_out, iters_out);
}

extern "C" int jacobi_solve_f32a(int64_t n, const float* A, const double* b, const double* x0, int64_t max_iter,
                                 double tol, double* x_out, int64_t* iters_out) {
  return solve_oneshot(n, JACOBI_F32, A, b, x0, max_iter, tol, x_out, iters_out);
}

extern "C" int jacobi_bwprobe(int64_t nbytes, int reps, double* best_gbs) {
  if (nbytes < (1 << 20) || reps < 1 || !best_gbs) return jacobi_set_error(JACOBI_EINVAL, "jacobi_bwprobe: bad argument");
  double g = jacobi::bwprobe(nbytes, reps);
  if (g < 0) return jacobi_set_error(JACOBI_ECUDA, "jacobi_bwprobe: CUDA failure");
  *best_gbs = g;
  return 0;
}
