// cluster.cu — small-n solver: a whole solve in one thread-block-cluster
// launch, A resident in shared memory, x exchanged through distributed shared memory (DSMEM).
//
// For small n the graph-of-sweeps path is launch-latency bound (c1, n = 256: ~7 µs per sweep for
// ~1 µs of work).  Here a cluster of C CTAs (16 when the part allows non-portable clusters, else 8)
// splits the rows; CTA r loads its rows of A into shared memory once, and each sweep
//   1. computes its rows in the canonical summation order of sweep.cu (chunks of chunk(n, dtype)
//      columns; lane l owns columns c0 + (32 s + l)·E + e, one DFMA chain, shfl_xor butterfly, chunk
//      sums ascending; diagonal and j >= n skipped — PAPER.md:55), so every bit equals the sweep
//      kernels' result;
//   2. pushes x_i^(k) into every CTA's copy of x (st.async DSMEM stores, lanes 0..C-1 one peer each),
//      and its max |dx| bits (or, for the Euclidean rule, dx^2) into every CTA's slots; each store
//      completes transaction bytes on the receiver's mbarrier, so there is no fence and no cluster
//      barrier per sweep (ncu showed ERRBAR + barrier at ~30 % of the samples with plain stores);
//   3. once its mbarrier phase completes, every CTA evaluates the same stop test:
//      max of the C slots, or the fixed 256-row tree + strided warp sum of k_l2_partials/k_l2_final.
// A launch runs at most kMaxSweepsPerLaunch sweeps and writes x and the stop state back, so long
// runs stay interruptible; the next launch resumes from global x.
#include "internal.h"
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace jacobi {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kCT = 512;  // threads per CTA (16 warps: one row per warp for n = 256, C = 16)
constexpr int kMaxC = 16;
static_assert(kCT >= kL2Block, "the in-kernel L2 tree uses one thread per row of a block");

template <typename T> struct EOf;
template <> struct EOf<double> { static constexpr int E = 4; };
template <> struct EOf<float> { static constexpr int E = 8; };

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~(size_t)15; }

// Shared-memory order of a row of A and of x (bank-conflict-free 16-byte loads).  In the canonical
// summation order lane l of step s owns columns s S + l E + e (S = 32 E, e < E); storing column
// s S + l E + e at s S + (e / V) 32 V + l V + e % V, V = elements per 16-byte load (2 doubles,
// 4 floats), makes each 16-byte ld.shared of the warp read 512 contiguous bytes (4 wavefronts; the
// natural order, lanes 32 bytes apart, takes 8).  Only the placement changes, not the arithmetic.
template <int E, int V>
__host__ __device__ inline int perm(int j) {
  constexpr int S = 32 * E;
  const int s = j / S, w = j - s * S, l = w / E, e = w - l * E;
  return s * S + (e / V) * (32 * V) + l * V + e % V;
}

struct Layout {  // dynamic shared memory of one CTA
  size_t a_off, xs_off, sq_off, dsl_off, red_off, blk_off, total;
  int lds, xlen, n256;
};

__host__ __device__ inline Layout layout(int n, int C, int esz) {
  Layout L;
  const int rows_max = (n + C - 1) / C;
  const int S = 32 * (esz == 8 ? 4 : 8);  // columns per warp step (whole step blocks: see perm)
  L.lds = (n + S - 1) / S * S;
  L.xlen = L.lds;
  L.n256 = (n + kL2Block - 1) / kL2Block * kL2Block;
  L.a_off = 0;
  L.xs_off = align16((size_t)rows_max * L.lds * esz);
  L.sq_off = L.xs_off + align16((size_t)2 * L.xlen * 8);
  L.dsl_off = L.sq_off + align16((size_t)2 * L.n256 * 8);
  L.red_off = L.dsl_off + align16((size_t)2 * kMaxC * 8);
  L.blk_off = L.red_off + align16((size_t)kCT * 8);
  L.total = L.blk_off + align16((size_t)(L.n256 / kL2Block) * 8 + 8 * 8);
  return L;
}

// DSMEM push with completion on the receiver's mbarrier (no fence, no cluster barrier per sweep).
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned laddr, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(laddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_b64(unsigned raddr, unsigned long long v, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr), "l"(v),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_init_local(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
// Default (.acquire.cta) semantics, as for TMA-multicast data: the st.async bytes are visible once
// the phase completes; a .cluster-scope acquire would add an L1 invalidate (CCTL.IVALL) per sweep.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}

// A lane's E elements of one step block (see perm): 16-byte shared loads at lane stride 16 bytes.
__device__ __forceinline__ void lds2(const double* p, double& v0, double& v1) {
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v0), "=d"(v1) : "r"(smem_addr(p)) : "memory");
}
__device__ __forceinline__ void lds_a(const double* blk, int lane, double (&v)[4]) {
  lds2(blk + 2 * lane, v[0], v[1]);
  lds2(blk + 64 + 2 * lane, v[2], v[3]);
}
__device__ __forceinline__ void lds_a(const float* blk, int lane, float (&v)[8]) {
#pragma unroll
  for (int q = 0; q < 2; ++q)
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v[4 * q]), "=f"(v[4 * q + 1]), "=f"(v[4 * q + 2]), "=f"(v[4 * q + 3])
                 : "r"(smem_addr(blk + 128 * q + 4 * lane))
                 : "memory");
}
template <int E>
__device__ __forceinline__ void lds_x(const double* blk, int lane, double (&v)[E]) {
#pragma unroll
  for (int q = 0; q < E / 2; ++q) lds2(blk + 64 * q + 2 * lane, v[2 * q], v[2 * q + 1]);
}

struct ClusterArgs {
  const void* A;
  int64_t lda;
  int n, chunk, nchunks, norm;
  const double* diag;
  const double* b;
  double* x0buf;
  double* x1buf;
  State* st;
  // Fused start (device solves in one launch): x0_src non-null -> the kernel itself initialises the
  // stop state (max_iter, tol, hist below), scans b (= the caller's b) and x0 for NaN/Inf and loads
  // x^(0) from x0_src; x_out non-null -> it also writes X^(iters) there when the solve has finished.
  const double* x0_src;
  double* x_out;
  int64_t max_iter;
  double tol;
  double* hist;
  HostDone* done;  // non-null (fused start): completion record in mapped host memory, tagged seq
  unsigned long long seq;
};

// Rank 0's last act: the completion record, seq after a system fence (every CTA's x_out stores were
// fenced at system scope before the cluster barrier that precedes this).
__device__ __forceinline__ void publish_done(HostDone* d, unsigned long long seq, int status, int nonfinite,
                                             int64_t iters) {
  d->status = status;
  d->nonfinite = nonfinite;
  d->iters = iters;
  __threadfence_system();
  *(volatile unsigned long long*)&d->seq = seq;
}

template <typename T>
__global__ void __launch_bounds__(kCT, 1) k_solve_cluster(const ClusterArgs a, const int64_t k0, const int64_t k1) {
  constexpr int E = EOf<T>::E;
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = a.n;
  const Layout L = layout(n, C, (int)sizeof(T));
  extern __shared__ __align__(16) unsigned char sm[];
  T* As = reinterpret_cast<T*>(sm + L.a_off);
  double* xs = reinterpret_cast<double*>(sm + L.xs_off);
  double* sq = reinterpret_cast<double*>(sm + L.sq_off);
  unsigned long long* dsl = reinterpret_cast<unsigned long long*>(sm + L.dsl_off);
  double* red = reinterpret_cast<double*>(sm + L.red_off);
  double* blk = reinterpret_cast<double*>(sm + L.blk_off);
  __shared__ unsigned long long s_wmax[kCT / 32];
  __shared__ __align__(8) uint64_t s_full[2];  // per parity: x^(k), the C maxima (and dx^2) have landed

  State* st = a.st;
  const bool fused = a.x0_src != nullptr;
  if (fused) {
    if (rank == 0 && tid == 0) {  // the whole stop state of a fresh solve (no host memset / k_prepare)
      st->kbase = 0;
      st->max_iter = a.max_iter;
      st->tol = a.tol;
      st->hist = a.hist;
      st->done = 0;
      st->status = 0;
      st->iters = 0;
      st->nonfinite = 0;
      st->fault = 0;
    }
  } else if (*(volatile int32_t*)&st->done || st->nonfinite) {
    return;  // uniform for the whole cluster
  }
  const double tol = fused ? a.tol : st->tol;
  const int64_t max_iter = fused ? a.max_iter : st->max_iter;
  double* hist = fused ? a.hist : st->hist;
  __shared__ int s_bad;
  const int r_begin = (int)((int64_t)rank * n / C), r_end = (int)((int64_t)(rank + 1) * n / C);
  const int nr = r_end - r_begin;

  // Resident data: own rows of A (zero padded to lds), x^(k0-1), zeroed L2 buffers.
  const T* Ag = static_cast<const T*>(a.A);
  {  // 8 independent loads in flight per thread, then their shared-memory stores (one latency per
     // batch instead of one per element: the prologue of a 1-sweep c1 solve fell from ~11 µs)
    constexpr int UN = 8;
    const int total = nr * L.lds;
    for (int base = 0; base < total; base += kCT * UN) {
      T v[UN];
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        const int idx = base + u * kCT + tid;
        const int r = idx / L.lds, c = idx - r * L.lds;
        v[u] = idx < total && c < n ? __ldg(Ag + (int64_t)(r_begin + r) * a.lda + c) : T(0);
      }
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        const int idx = base + u * kCT + tid;
        const int r = idx / L.lds, c = idx - r * L.lds;
        if (idx < total) As[r * L.lds + perm<E, 16 / (int)sizeof(T)>(c)] = v[u];
      }
    }
  }
  const int p0 = (int)((k0 - 1) & 1);
  const double* xg = fused ? a.x0_src : (p0 ? a.x1buf : a.x0buf);
  if (tid == 0) s_bad = 0;
  __syncthreads();
  bool bad = false;
  for (int i = tid; i < L.xlen; i += kCT) {
    const double v = i < n ? xg[i] : 0.0;
    xs[p0 * L.xlen + perm<E, 2>(i)] = v;
    if (fused && i >= r_begin && i < r_end)  // this CTA's slice of x0 and b (PAPER.md:59 inputs)
      bad |= !isfinite(v) || !isfinite(a.b[i]);
  }
  if (bad) atomicOr(&s_bad, 1);
  for (int i = tid; i < 2 * L.n256; i += kCT) sq[i] = 0.0;
  if (tid == 0) {
    mbar_init_local(&s_full[0], 1);
    mbar_init_local(&s_full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();  // every CTA's barriers and buffers are ready before the first remote store
  if (fused) {  // any non-finite input anywhere in the cluster: ENONFINITE, no sweep
    int any = 0;
    for (int q = 0; q < C; ++q) any |= *cl.map_shared_rank(&s_bad, q);
    cl.sync();  // no CTA leaves while a peer may still read its flag
    if (any) {
      if (rank == 0 && tid == 0) {
        st->nonfinite = 1;
        if (a.done) publish_done(a.done, a.seq, 0, 1, 0);
      }
      return;
    }
  }
  // bytes that land in each CTA per sweep: all n values of x^(k), C maxima, and n dx^2 for L2
  const unsigned tx_bytes = (unsigned)(8 * n + 8 * C + (a.norm == JACOBI_NORM_L2 ? 8 * n : 0));
  unsigned phase = 0u;  // bit p: the parity of the next phase of s_full[p] (a register, not a local array)

  const int nsteps = a.chunk / (32 * E);
#ifdef JACOBI_CLUSTER_PROF  // probe build: per-phase clock64 sums of CTA 0 thread 0, printed at exit
  long long pt[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, tprev = clock64();
#define CPROF(i)                              \
  do {                                        \
    if (rank == 0 && tid == 0) {              \
      const long long t_ = clock64();         \
      pt[i] += t_ - tprev;                    \
      tprev = t_;                             \
    }                                         \
  } while (0)
#else
#define CPROF(i) \
  do {           \
  } while (0)
#endif
  int stop = 0;  // 1 converged, 2 iteration limit
  int64_t k = k0;
  // Each barrier phase takes one arrival (with the expected bytes) from thread 0.  The phases of
  // sweeps k0 and k0 + 1 are armed here, the phase of sweep k + 2 right after sweep k's wait on the
  // same barrier — off the loop top, where the arrive waited ~350 cycles behind the thread's DSMEM
  // stores.  No peer can start sweep k + 2 before this CTA has pushed x^(k+1), so the arming always
  // precedes that phase's bytes.
  if (tid == 0) {
    mbar_expect(&s_full[k0 & 1], tx_bytes);
    mbar_expect(&s_full[(k0 + 1) & 1], tx_bytes);
  }
  for (; k <= k1; ++k) {
    const int par = (int)(k & 1);
    const double* xo = xs + (1 - par) * L.xlen;
    CPROF(8);
    unsigned long long dmax = 0ull;
    for (int r = warp; r < nr; r += kCT / 32) {
      const int grow = r_begin + r;
      const T* arow = As + (size_t)r * L.lds;
      const double bi = a.b[grow], dii = a.diag[grow];  // issued before the row's FMA chain
      CPROF(9);
      double s = 0.0;
      for (int c = 0; c < a.nchunks; ++c) {
        const int c0 = c * a.chunk;
        double acc = 0.0;
        for (int step = 0; step < nsteps; ++step) {
          const int col = c0 + (step * 32 + lane) * E;
          if (col < n) {  // rows are zero padded to whole step blocks (lds): 16-byte loads, see perm
            T av[E];
            double xv[E];
            const int blk = col - lane * E;  // s S: this step's block
            lds_a(arow + blk, lane, av);
            lds_x(xo + blk, lane, xv);
            CPROF(10);
#pragma unroll
            for (int e = 0; e < E; ++e) {
              const int cc = col + e;
              if (cc < n && cc != grow) acc = __fma_rn((double)av[e], xv[e], acc);
            }
          }
        }
        CPROF(0);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(kFull, acc, off);
        s = c == 0 ? acc : s + acc;
        CPROF(1);
      }
      const double xnew = __ddiv_rn(__dsub_rn(bi, s), dii);
      const int gp = perm<E, 2>(grow);  // x_i's place in the shared-memory order
      const double dx = __dsub_rn(xnew, xo[gp]);
      CPROF(2);
      if (lane < C) {  // lane q pushes x_i^(k) (and dx^2) into CTA q
        const unsigned rbar = mapa(smem_addr(&s_full[par]), lane);
        st_async_b64(mapa(smem_addr(xs + par * L.xlen + gp), lane), (unsigned long long)__double_as_longlong(xnew),
                     rbar);
        if (a.norm == JACOBI_NORM_L2)
          st_async_b64(mapa(smem_addr(sq + par * L.n256 + grow), lane),
                       (unsigned long long)__double_as_longlong(__dmul_rn(dx, dx)), rbar);
      }
      const unsigned long long bits = (unsigned long long)__double_as_longlong(dx) & 0x7fffffffffffffffull;
      dmax = bits > dmax ? bits : dmax;
      CPROF(3);
    }
    if (lane == 0) s_wmax[warp] = dmax;
    __syncthreads();
    CPROF(4);
    if (warp == 0) {  // CTA max of the 16 warp maxima (a 16-lane butterfly), lane q pushes it to CTA q
      static_assert(kCT / 32 == 16 && kMaxC == 16, "16-lane butterflies");
      unsigned long long m = s_wmax[lane & 15];
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(kFull, m, off);
        m = o > m ? o : m;
      }
      if (lane < C) st_async_b64(mapa(smem_addr(dsl + par * kMaxC + rank), lane), m, mapa(smem_addr(&s_full[par]), lane));
    }
    CPROF(5);
    mbar_wait_cluster(&s_full[par], (phase >> par) & 1u);  // x^(k), the maxima and dx^2 of every row have landed
    phase ^= 1u << par;
    if (tid == 0) mbar_expect(&s_full[par], tx_bytes);  // arm this barrier's next phase (sweep k + 2)
    CPROF(6);

    double d;
    if (a.norm == JACOBI_NORM_L2) {  // identical arithmetic to k_l2_partials + k_l2_final
      const double* sqk = sq + par * L.n256;
      const int nblk = L.n256 / kL2Block;
      for (int q = 0; q < nblk; ++q) {
        if (tid < kL2Block) red[tid] = sqk[q * kL2Block + tid];  // rows >= n hold 0.0
        __syncthreads();
        for (int off = kL2Block / 2; off > 0; off >>= 1) {
          if (tid < off) red[tid] = __dadd_rn(red[tid], red[tid + off]);
          __syncthreads();
        }
        if (tid == 0) blk[q] = red[0];
        __syncthreads();
      }
      double t = 0.0;
      for (int q = lane; q < nblk; q += 32) t = __dadd_rn(t, blk[q]);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) t = __dadd_rn(t, __shfl_xor_sync(kFull, t, off));
      d = __dsqrt_rn(t);
    } else {  // max of the C slots: one load per lane (both half-warps), then a 16-lane butterfly
      unsigned long long m = (lane & 15) < C ? dsl[par * kMaxC + (lane & 15)] : 0ull;
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(kFull, m, off);
        m = o > m ? o : m;
      }
      d = __longlong_as_double((long long)m);
    }
    if (rank == 0 && tid == 0 && hist) hist[k - 1] = d;
    CPROF(7);
    if (d < tol) { stop = 1; break; }        // return X
    if (k == max_iter) { stop = 2; break; }  // iteration limit
  }
#ifdef JACOBI_CLUSTER_PROF
  if (rank == 0 && tid == 0) {
    const double ns = (double)(k - k0 + 1);
    printf("{\"cluster_prof\": true, \"n\": %d, \"C\": %d, \"sweeps\": %.0f, \"cycles\": [%.1f, %.1f, %.1f, %.1f, %.1f, "
           "%.1f, %.1f, %.1f], \"top\": [%.1f, %.1f, %.1f]}\n", n, C, ns, pt[0] / ns, pt[1] / ns, pt[2] / ns, pt[3] / ns,
           pt[4] / ns, pt[5] / ns, pt[6] / ns, pt[7] / ns, pt[8] / ns, pt[9] / ns, pt[10] / ns);
  }
#endif
  const int64_t klast = stop ? k : k1;
  double* xgo = (klast & 1) ? a.x1buf : a.x0buf;
  const double* xsl = xs + (int)(klast & 1) * L.xlen;
  for (int r = tid; r < nr; r += kCT) xgo[r_begin + r] = xsl[perm<E, 2>(r_begin + r)];
  if (stop && a.x_out)  // finished: X^(iters) straight to the caller's buffer (iters = klast)
    for (int r = tid; r < nr; r += kCT) a.x_out[r_begin + r] = xsl[perm<E, 2>(r_begin + r)];
  if (rank == 0 && tid == 0) {
    if (stop == 1) { st->status = JACOBI_CONVERGED; st->iters = klast; st->done = 1; }
    if (stop == 2) { st->status = JACOBI_MAX_ITER; st->iters = max_iter; st->done = 1; }
    st->kbase = klast;
  }
  if (a.done) __threadfence_system();  // this thread's x_out stores, before the barrier below
  cl.sync();  // no CTA leaves while a peer may still write into its shared memory
  if (a.done && stop && rank == 0 && tid == 0)
    publish_done(a.done, a.seq, stop == 1 ? JACOBI_CONVERGED : JACOBI_MAX_ITER, 0, stop == 1 ? klast : max_iter);
}

template <typename T>
cudaError_t try_cluster(int n, int C, size_t* smem_out, int* ok) {
  const Layout L = layout(n, C, (int)sizeof(T));
  *ok = 0;
  *smem_out = L.total;
  int maxsm = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (L.total > (size_t)maxsm) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_solve_cluster<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  if (C > 8) {
    e = cudaFuncSetAttribute(k_solve_cluster<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) { cudaGetLastError(); return cudaSuccess; }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kCT);
  cfg.dynamicSmemBytes = L.total;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  e = cudaOccupancyMaxActiveClusters(&nclusters, k_solve_cluster<T>, &cfg);
  if (e != cudaSuccess) { cudaGetLastError(); return cudaSuccess; }
  *ok = nclusters >= 1;
  return cudaSuccess;
}

}  // namespace

// Largest usable cluster (16, else 8) for an n x n system of this dtype; 0 when A does not fit.
int cluster_plan(int64_t n, int dtype, size_t* smem) {
  if (n < 1 || n > 4096) return 0;
  int only = 0;  // JACOBI_CLUSTER_C=16|8|4|2: tuning override (that size or nothing)
  if (const char* e = getenv("JACOBI_CLUSTER_C")) only = atoi(e);
  for (int C : {16, 8, 4, 2}) {
    if (only ? C != only : C < 8) continue;
    int ok = 0;
    cudaError_t e = dtype == JACOBI_F32 ? try_cluster<float>((int)n, C, smem, &ok)
                                        : try_cluster<double>((int)n, C, smem, &ok);
    if (e != cudaSuccess) { cudaGetLastError(); return 0; }
    if (ok) return C;
  }
  return 0;
}

cudaError_t launch_solve_cluster(int dtype, int C, size_t smem, const void* A, int64_t lda, int64_t n, int chunk,
                                 int norm, const double* diag, const double* b, double* x0buf, double* x1buf,
                                 State* st, int64_t k0, int64_t k1, cudaStream_t s, const double* x0_src,
                                 double* x_out, int64_t max_iter, double tol, double* hist, HostDone* done,
                                 unsigned long long seq) {
  ClusterArgs a;
  a.done = done;
  a.seq = seq;
  a.x0_src = x0_src;
  a.x_out = x_out;
  a.max_iter = max_iter;
  a.tol = tol;
  a.hist = hist;
  a.A = A;
  a.lda = lda;
  a.n = (int)n;
  a.chunk = chunk;
  a.nchunks = (int)((n + chunk - 1) / chunk);
  a.norm = norm;
  a.diag = diag;
  a.b = b;
  a.x0buf = x0buf;
  a.x1buf = x1buf;
  a.st = st;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kCT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (dtype == JACOBI_F32) return cudaLaunchKernelEx(&cfg, k_solve_cluster<float>, a, k0, k1);
  return cudaLaunchKernelEx(&cfg, k_solve_cluster<double>, a, k0, k1);
}

}  // namespace jacobi
