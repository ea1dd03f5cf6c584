// sweep.cu — sm_100a kernels of the dense Jacobi sweep.
//
// One Jacobi sweep over a launch's rows, fused with the max-norm change
// d_k = max_i |x_i^(k) - x_i^(k-1)| and the device-side stop test of PAPER.md:61-66.  Three work
// decompositions share one summation order, so every kernel (and every instance: R rows per tile,
// U steps in flight, CTA size) gives the same bits:
//   k_sweep       (item kernel, n with < 16 chunks): work item = (tile of R rows, column chunk),
//                 round-robin over a persistent grid; chunk partials in global memory, the last
//                 warp to arrive on a tile's counter finalizes it;
//   k_sweep_cta   (fp64 default): CTA b owns rows [b*m/G, (b+1)*m/G) — or, with DYN (large row
//                 blocks, c4), takes tiles from a launch-wide counter; warp w streams chunks
//                 w, w+16, ... of each tile; partials meet in a shared-memory ring (mbarriers) and a
//                 finalizer warp per tile applies the epilogue; also the L2-keep (POL) and the
//                 fused-exchange (PUSH, NEXT-1) instances; its body is each sweep of the persistent
//                 grid solver (k_solve_gridsync, mid-size n);
//   k_sweep_panel (fp32-A default): each warp owns whole rows and walks all chunks in order;
//                 optionally x^(k-1) staged in shared memory by a TMA chunk ring (XSN).
//
// Summation order (fixed; depends only on column indices, never on the rank count, the row
// placement, R or the grid): columns are cut into chunks of chunk_for(n, dtype) columns; within a
// chunk lane l accumulates columns c0 + (32 s + l)*E + e (E = 4 doubles / 8 floats per 256-bit
// load) in ascending s then e with one DFMA chain per row; the 32 lane sums are combined by a
// shfl_xor butterfly (16, 8, 4, 2, 1); the chunk sums are added in ascending chunk order.  The
// epilogue is x_i = (b_i - s_i) / a_ii (one IEEE division), and |x_i^(k) - x_i^(k-1)| is folded
// into the sweep's max with an unsigned 64-bit atomicMax on the bit pattern (sign cleared):
// NaN > +Inf > finite, so the max is NaN-sticky and order independent.
#include "internal.h"
#include <cstdio>

namespace jacobi {
namespace {

constexpr unsigned kFull = 0xffffffffu;

template <typename T> struct VecOf;
template <> struct VecOf<double> { static constexpr int E = 4; };
template <> struct VecOf<float> { static constexpr int E = 8; };

#ifdef JACOBI_BOUNDS_CHECK
__device__ unsigned long long g_oob = 0ull;
#define JB_CHECK(cond, bit)                                        \
  do {                                                             \
    if (!(cond)) atomicOr(&g_oob, 1ull << (bit));                  \
  } while (0)
#else
#define JB_CHECK(cond, bit) \
  do {                      \
  } while (0)
#endif

// Bounds of one tile x chunk: the R row pointers (indexed by global column), the columns the
// accumulate loop loads ([c0, top): the whole chunk when it is full, else up to n rounded to the
// 32-byte load), and the x range read.  Bits: 0 A below the block, 1 A past the block, 2 A past the
// row pitch, 3 x past its buffer.
template <typename T, int R>
__device__ __forceinline__ void check_tile(const SweepArgs& a, const T* const (&rowp)[R], int64_t c0, int64_t c1) {
#ifdef JACOBI_BOUNDS_CHECK
  constexpr int E = VecOf<T>::E;
  const int64_t last = min(c1, a.cend);
  const int64_t top = (c1 - c0 == a.chunk) ? c0 + a.chunk : c0 + ((last - c0 + E - 1) / E) * E;
  const T* base = static_cast<const T*>(a.a_base);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    JB_CHECK(rowp[r] + c0 >= base, 0);
    JB_CHECK(rowp[r] + top <= base + a.a_elems, 1);
    JB_CHECK(top - a.col0 <= a.lda, 2);
  }
  JB_CHECK(top <= a.x_len, 3);
#endif
}

// 256-bit streaming load of A (read exactly once per sweep): no L1 allocation.
__device__ __forceinline__ void ld_a(const double* p, double (&v)[4]) {
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void ld_a(const float* p, float (&v)[8]) {
  asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
      : "l"(p));
}
// Same loads with an L2 eviction-priority policy (createpolicy): used to keep part of A resident in
// L2 across sweeps when A is about the L2 size (c2: 134 MB vs 126 MB of L2).
__device__ __forceinline__ void ld_a(const double* p, double (&v)[4], uint64_t pol) {
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld_a(const float* p, float (&v)[8], uint64_t pol) {
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
      : "l"(p), "l"(pol));
}
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t pol;
  if (keep) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <bool POL, typename T, int E>
__device__ __forceinline__ void ld_a_p(const T* p, T (&v)[E], uint64_t pol) {
  if constexpr (POL) ld_a(p, v, pol);
  else ld_a(p, v);
}
// x^(k-1) is read-only during the sweep (it lives in the other ping-pong buffer): L1-cached loads.
// XL = 2: x^(k-1) was written by other SMs earlier in the same (persistent) launch — read it at L2
// (ld.global.cg), never through a possibly stale L1 line.
template <int XL>
__device__ __forceinline__ void ld_x4(const double* p, double* v) {
  if (XL == 1)  // keep x^(k-1) in L1 with priority over everything else
    asm("ld.global.nc.L1::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
  else if (XL == 2)
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
  else if (XL == 3)  // weak, L1-cacheable: coherent after the launch's acquire + barrier (memory model)
    asm("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p) : "memory");
  else
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
template <int XL>
__device__ __forceinline__ double ld_x1(const double* p) {
  if constexpr (XL == 2) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
  } else {
    return *p;
  }
}
template <int E, int XL = 0>
__device__ __forceinline__ void ld_x(const double* p, double (&v)[E]) {
#pragma unroll
  for (int q = 0; q < E; q += 4) ld_x4<XL>(p + q, v + q);
}

// x^(k-1) from a shared-memory chunk staged by the bulk-copy engine (k_sweep_panel with XSN > 0).
template <int E>
__device__ __forceinline__ void ld_xs(const double* p, double (&v)[E]) {
#pragma unroll
  for (int q = 0; q < E; q += 2)
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];"
                 : "=d"(v[q]), "=d"(v[q + 1]) : "r"((unsigned)__cvta_generic_to_shared(p + q)));
}

// Prologue of sweep k (PAPER.md:64-66 evaluated on the device): decides whether sweep k runs.
// Every CTA evaluates the same inputs and reaches the same decision; only the leader writes.
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Probe build only (-DJACOBI_SM_TIMING): per CTA of the last sweep-kernel launch, its SM id and the
// %globaltimer at its start and end (jacobi_debug_sm_times) — to see how the static row partition
// finishes across SMs and dies.
#ifdef JACOBI_SM_TIMING
__device__ unsigned long long g_smt[3 * 4096];
__device__ int g_rot = 0;  // row-panel kernel: CTA b takes the rows of block (b + g_rot) mod G
#define SMT_BEGIN()                              \
  unsigned long long smt0_ = 0;                  \
  if (threadIdx.x == 0) smt0_ = global_ns()
#define SMT_END()                                                            \
  do {                                                                       \
    __syncthreads();                                                         \
    if (threadIdx.x == 0 && blockIdx.x < 4096) {                             \
      unsigned sm_;                                                          \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                      \
      g_smt[3 * blockIdx.x] = sm_;                                           \
      g_smt[3 * blockIdx.x + 1] = smt0_;                                     \
      g_smt[3 * blockIdx.x + 2] = global_ns();                               \
    }                                                                        \
  } while (0)
#else
#define SMT_BEGIN() \
  do {              \
  } while (0)
#define SMT_END() \
  do {            \
  } while (0)
#endif

// All state loads are issued together (one L2 round trip instead of a chain of dependent ones: the
// short-circuit `done || nonfinite || fault` and the kbase -> slot dependency each cost a round trip,
// ~1-2 µs per sweep kernel).  The distance slot of sweep k-1 is (kbase + j) & 3 = j & 3 because kbase
// is a multiple of the graph batch, itself a multiple of 4 (jacobi_plan_set_batch); with the fused
// exchange it is re-read after the wait for the peers' atomics.
__device__ __forceinline__ bool sweep_prologue(const SweepArgs& a, int j, bool leader, long long* k_out) {
  State* st = a.st;
  const int32_t done = *(volatile int32_t*)&st->done, nonf = st->nonfinite, fault = *(volatile int32_t*)&st->fault;
  const int64_t kbase = st->kbase, max_iter = st->max_iter;
  const double tol = st->tol;
  double* const hist = st->hist;
  unsigned long long dbits = *(volatile unsigned long long*)&a.dslot[j & 3];
  if (done | nonf | fault) return false;
  JB_CHECK((kbase & 3) == 0, 7);  // bit 7: the slot shortcut's premise
  const int64_t k = kbase + j + 1;
  *k_out = k;  // broadcast through shared memory: the sweep body needs no second read of the state
  if (k >= 2 && a.peers) {
    // NEXT-1: wait until every CTA of every rank has pushed its x^(k-1) rows and max|dx| bits here.
    // Bounded: after pe->wait_ns (10 s by default) the plan is marked faulted (the host reports JACOBI_ECUDA) and every
    // later sweep is a no-op, so a failed peer cannot hang this GPU.
    const PeerArgs* pe = a.peers;
    const unsigned long long kp = (unsigned long long)(k - 1);
    const unsigned long long target = ((kp + (kp & 1)) / 2) * pe->total_ctas;  // sweeps of this parity
    const unsigned long long* f = pe->flags[pe->rank] + (kp & 1);
    unsigned long long t0 = 0;
    for (unsigned i = 0; ld_acquire_sys(f) < target; ++i) {
      __nanosleep(64);
      if ((i & 4095) == 4095) {
        const unsigned long long t = global_ns();
        if (t0 == 0) t0 = t;
        else if (t - t0 > pe->wait_ns || *(volatile int32_t*)&st->fault) {
          st->fault = 1;
          return false;
        }
      }
    }
    dbits = *(volatile unsigned long long*)&a.dslot[j & 3];  // after the acquire: every peer's atomicMax
  }
  if (k >= 2) {
    const double d = __longlong_as_double((long long)dbits);
    if (leader && hist) hist[k - 2] = d;
    if (d < tol) {  // (b): ||X - X^t|| < tol  -> return X^(k-1)
      if (leader) { st->status = JACOBI_CONVERGED; st->iters = k - 1; st->done = 1; }
      return false;
    }
  }
  if (k > max_iter) {  // step 3: iteration limit reached
    if (leader) { st->status = JACOBI_MAX_ITER; st->iters = max_iter; st->done = 1; }
    return false;
  }
  if (leader) a.dslot[(k + 1) & 3] = 0ull;  // next sweep's max accumulator
  return true;
}

// Sum of one column chunk [c0, c1) of R rows against x^(k-1), in the fixed order every kernel
// variant shares: lane l owns columns c0 + (32*s + l)*E + e, accumulated in ascending s then e with
// one DFMA chain per row; j == i (the diagonal) and j >= n are skipped.  Rows r >= nv
// are not loaded (their sums are unused).
// XSM: x^(k-1) of this chunk comes from shared memory, xs[col - c0] (else from global, xo[col]).
// PIN: see the step loop below.
// Row count nv in [1, R] as a compile-time constant: f(std::integral_constant<int, nv>).
template <int N>
struct NvConst { static constexpr int value = N; };
template <int R, typename F>
__device__ __forceinline__ void with_nv(const int nv, F&& f) {
  if constexpr (R <= 1) {
    f(NvConst<1>{});
  } else {
    if (nv >= R) f(NvConst<R>{});
    else with_nv<R - 1>(nv, f);
  }
}

template <typename T, int R, int U, int XL = 0, bool POL = false, bool XSM = false, bool PIN = false>
__device__ __forceinline__ void accumulate_chunk(const T* const (&rowp)[R], const int nv,
                                                 const double* __restrict__ xo, const int64_t c0,
                                                 const int64_t c1, const int chunk, const int64_t n,
                                                 const int64_t g0, const int lane, double (&acc)[R],
                                                 const uint64_t pol = 0, const double* xs = nullptr) {
  constexpr int E = VecOf<T>::E;
  constexpr int S = 32 * E;  // columns per warp step
  const int nsteps = chunk / S;
  const bool masked = (c1 - c0 != chunk) || (g0 < c1 && g0 + R > c0);
  if (!masked) {
    auto step = [&](const int s) {
      T av[U][R][E];
      double xv[U][E];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t col = c0 + (int64_t)((s + u) * 32 + lane) * E;
        if constexpr (XSM) ld_xs<E>(xs + (col - c0), xv[u]);
        else ld_x<E, XL>(xo + col, xv[u]);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (r < nv) ld_a_p<POL>(rowp[r] + col, av[u][r], pol);
          else {
#pragma unroll
            for (int e = 0; e < E; ++e) av[u][r][e] = T(0);
          }
        }
      }
#ifdef JACOBI_PROBE_NOFMA
      // Probe build only (wrong results): the same loads, each A element folded into the sum's bits
      // with one integer XOR instead of convert + DFMA, x^(k-1) once per step — separates the load
      // pattern's rate from the arithmetic's (profiles/nofma_probe_r02.txt).
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          long long bits = __double_as_longlong(acc[r]) ^ __double_as_longlong(xv[u][r % E]);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            if constexpr (sizeof(T) == 4) bits ^= (long long)__float_as_int((float)av[u][r][e]) << (e & 1) * 32;
            else bits ^= __double_as_longlong((double)av[u][r][e]);
          }
          acc[r] = __longlong_as_double(bits);
        }
#else
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int e = 0; e < E; ++e) acc[r] = __fma_rn((double)av[u][r][e], xv[u][e], acc[r]);
#endif
    };
    // PIN: one step per loop trip (no compiler unrolling).  In the persistent solver's register
    // budget an unrolled pair of steps is interleaved so that the first FMA waits on the first loads
    // with only ~4 of the 9 loads issued; one step per trip issues all 9 first (c2: -4 %).  The
    // HBM-streaming kernels are faster unrolled (c3/c5 +1-2.6 %).
    if constexpr (PIN) {
#pragma unroll 1
      for (int s = 0; s < nsteps; s += U) step(s);
    } else {
      for (int s = 0; s < nsteps; s += U) step(s);
    }
  } else {
    // Diagonal chunk or ragged tail: same order, j == i and j >= n terms skipped.
    for (int s = 0; s < nsteps; ++s) {
      const int64_t col = c0 + (int64_t)(s * 32 + lane) * E;
      if (col < n) {
        T av[R][E];
        double xv[E];
        if constexpr (XSM) ld_xs<E>(xs + (col - c0), xv);
        else ld_x<E, XL>(xo + col, xv);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (r < nv) ld_a_p<POL>(rowp[r] + col, av[r], pol);
          else {
#pragma unroll
            for (int e = 0; e < E; ++e) av[r][e] = T(0);
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int64_t cc = col + e;
            if (cc < n && cc != g0 + r) acc[r] = __fma_rn((double)av[r][e], xv[e], acc[r]);
          }
      }
    }
  }
}

// L2-resident share of A (POL instances).  The kept set is made of work units — (tile, column chunk[,
// row group]) — not whole tiles: a unit is 16-64 KB, a tile up to 1 MB (8 rows of 16384 fp64), and an
// L2 budget of ~60 MB is less than one tile per CTA once rows are that long (c3 shards).  Unit i of a
// CTA's sequence (offset by a per-CTA phase) is kept iff frac(i * phi) < keep_pm / 1000 (a Weyl
// sequence: the kept units are spread evenly along every CTA's sequence and every warp's share, and
// the kept count is the share to within a couple of units), so at any moment some CTAs stream kept
// units from L2 while others stream from HBM.  32-bit integer hash: two instructions per unit (an exact
// Bresenham split needed 64-bit divisions and pushed the persistent kernels into register spills).
// The same units are kept every sweep (static rows), so they hit in L2 from the second sweep on.
__device__ __forceinline__ unsigned keep_threshold(int keep_pm) {
  return keep_pm >= 1000 ? 0xffffffffu : (unsigned)(((unsigned long long)max(keep_pm, 0) << 32) / 1000ull);
}
__device__ __forceinline__ bool keep_unit(unsigned i, unsigned thr) { return i * 2654435769u < thr; }

// POL: A loaded with an L2 policy per work item — evict_last for the kept share (keep_unit over the
// item index, a.l2_keep_pm), evict_first for the rest (column slabs of a few chunks, NEXT-4).
template <typename T, int R, int U, int NT, bool POL = false>
__global__ void __launch_bounds__(NT, (NT < 512 ? 512 / NT : 1)) k_sweep(const SweepArgs a, const int j) {
  __shared__ int s_go;
  __shared__ long long s_k;
  if (threadIdx.x == 0) s_go = sweep_prologue(a, j, blockIdx.x == 0, &s_k);
  __syncthreads();
  if (!s_go) return;

  const int64_t k = s_k;
  const double* __restrict__ xo = (k & 1) ? a.x0buf : a.x1buf;  // x^(k-1)
  double* __restrict__ xn = (k & 1) ? a.x1buf : a.x0buf;        // x^(k)
  const T* __restrict__ A = static_cast<const T*>(a.A);
  const int lane = threadIdx.x & 31;
  const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t items = (int64_t)a.tiles * a.nchunks;

  for (int64_t it = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); it < items; it += W) {
    const int tile = (int)(it % a.tiles);
    const int c = (int)(it / a.tiles);
    const int64_t r0 = (int64_t)tile * R;
    const int64_t c0 = a.col0 + (int64_t)c * a.chunk;
    const int64_t c1 = min(c0 + (int64_t)a.chunk, a.cend);
    const int64_t g0 = a.row0 + r0;  // global index of the tile's first row
    const T* rowp[R];  // indexed by global column
#pragma unroll
    for (int r = 0; r < R; ++r) rowp[r] = A + min(r0 + r, a.m - 1) * a.lda - a.col0;
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;

    check_tile<T, R>(a, rowp, c0, c1);
    uint64_t pol = 0;
    if constexpr (POL) pol = l2_policy(keep_unit((unsigned)it, keep_threshold(a.l2_keep_pm)));
    accumulate_chunk<T, R, U, 0, POL>(rowp, R, xo, c0, c1, a.chunk, a.cend, g0, lane, acc, pol);
    // Butterfly: every lane ends with the same, order-fixed row sums.
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(kFull, acc[r], off);

    // Publish the chunk partials, then count arrivals for the tile.
    double mine = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (lane == r) mine = acc[r];
    if (lane < R && r0 + lane < a.m) a.part[(int64_t)c * a.m + r0 + lane] = mine;
    __threadfence();
    __syncwarp();
    unsigned last = 0;
    if (lane == 0) last = (atomicAdd(&a.cnt[tile], 1u) == (unsigned)(a.nchunks - 1));
    last = __shfl_sync(kFull, last, 0);
    if (!last) continue;

    // Finalize the tile (fused epilogue, PAPER.md:55 and the max-norm distance).
    __threadfence();
    unsigned long long dbits = 0ull;
    if (lane < R && r0 + lane < a.m) {
      const int64_t row = r0 + lane;
      JB_CHECK(a.row0 + row < a.x_len, 5);
      double s = __ldcg(a.part + row);
      for (int cc = 1; cc < a.nchunks; ++cc) s += __ldcg(a.part + (int64_t)cc * a.m + row);
      if (a.rsum) {  // column-wise partial product of this slab (epilogue after the reduction)
        a.rsum[row] = s;
      } else {
        const double xnew = __ddiv_rn(__dsub_rn(a.b[row], s), a.diag[row]);
        const int64_t gi = a.row0 + row;
        const double dx = __dsub_rn(xnew, xo[gi]);
        xn[gi] = xnew;
        dbits = (unsigned long long)__double_as_longlong(dx) & 0x7fffffffffffffffull;
        if (a.norm == JACOBI_NORM_L2) a.sq[row] = __dmul_rn(dx, dx);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(kFull, dbits, off);
      dbits = o > dbits ? o : dbits;
    }
    if (lane == 0) {
      atomicMax(&a.dslot[k & 3], dbits);
      a.cnt[tile] = 0u;
    }
  }
}


// ---------------------------------------------------------------------------------------------
// k_sweep_cta: the large-n sweep.  CTA b of G owns the contiguous rows [b*m/G, (b+1)*m/G) (balanced
// to one row), processed in tiles of R rows.  For each tile, warp w streams the chunks c = w, w+NW,
// ... of the tile's rows (same per-chunk order as accumulate_chunk) and lane 0 publishes the R
// butterfly sums to a shared-memory slot; an mbarrier per slot counts the NW contributions.  The
// tile's finalizer warp (tile % NW, one tile late so it never idles on its own tile) adds the chunk
// partials in ascending chunk order — exactly the order of k_sweep — and applies the fused epilogue.
// No global atomics or fences per tile: one atomicMax of the warp's max|dx| bits per sweep.
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}

constexpr int kSlots = 4;


// Fused exchange, end of sweep k in one CTA (thread 0, after a CTA barrier that follows every thread's
// x stores): fold the CTA's max|dx| bits into every rank's distance slot, then — behind one system-scope
// fence, cumulative over the stores the barrier ordered before it — add one arrival to every rank's
// counter for the parity of k.
// The reductions are system-scoped (red.global.sys): the counters and slots live in other GPUs' memory
// and are read there with ld.acquire.sys, so both sides of the synchronisation are morally strong at
// the same scope (global-space PTX, so no generic-address fallback is generated).
__device__ __forceinline__ void red_max_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("red.global.sys.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("red.global.sys.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void push_signal(const PeerArgs* pe, int64_t k, unsigned long long m) {
  const int P = pe->P;
  for (int p = 0; p < P; ++p) red_max_sys(pe->dslot[p] + (k & 3), m);
  asm volatile("fence.acq_rel.sys;" ::: "memory");  // release: the pushes and maxima before the arrivals
  for (int p = 0; p < P; ++p) red_add_sys(pe->flags[p] + (k & 1), 1ull);
}

// CTA-wide max of the warps' max|dx| bits (every thread must call it; returns the max in thread 0).
// Used by the fused exchange, where each atomic crosses NVLink to every peer: one remote atomic per
// CTA per peer instead of one per warp (16x fewer same-address atomics arriving at each rank: 1184
// instead of 18944 per sweep at P = 8).  Local slots keep one atomic per warp (measured faster for
// the persistent solver, whose sweep-end barrier is on the critical path).
template <int NW>
__device__ __forceinline__ unsigned long long cta_max_bits(unsigned long long wmax, unsigned long long* s_w) {
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = wmax;
  __syncthreads();
  unsigned long long m = 0ull;
  if (threadIdx.x == 0)
    for (int q = 0; q < NW; ++q) m = s_w[q] > m ? s_w[q] : m;
  return m;
}

// One sweep k over the CTA's rows (the body of k_sweep_cta, shared with the persistent grid solver).
// Tiles are numbered from tbase (a running count across the sweeps of a persistent launch) for the
// slots and mbarrier parities of the partial-sum ring.  Returns this warp's max|dx| bits.
// GR > 1: a work unit is (chunk, group of R/GR rows of the tile) instead of (chunk, tile): with
// nchunks not a multiple of the warp count, nchunks x GR units balance the warps (24 chunks: 1.5
// chunks per warp per tile — warps 0-7 do two — become 3 units each).  Same per-row order.
// DYN: tiles are taken from a launch-wide counter (a.dyn[0]) instead of a static row range, so SMs
// that stream faster take more tiles (the static partition leaves a fixed minority of slower SMs
// finishing last: profiles/sm_tail_r01.jsonl).  Sequence t's tile index sits in s_tile[t & 7]:
// thread 0 claims the tile of sequence t + kSlots when it starts sequence t (the atomic's latency
// hides behind its unit) and publishes it before its arrival on s_full of t; a warp reads it only
// after s_empty of that slot, which orders the publication before the read.  -1 = no tiles left.
template <typename T, int R, int NW, int U, int XL, bool PUSH, bool POL, int GR = 1, bool PIN = false,
          bool DYN = false>
__device__ __forceinline__ unsigned long long cta_sweep(const SweepArgs& a, const int64_t k, const int64_t tbase,
                                                        double* s_part, uint64_t* s_full, uint64_t* s_empty,
                                                        const int cta, const int ncta, volatile int* s_tile = nullptr) {
  const double* __restrict__ xo = (k & 1) ? a.x0buf : a.x1buf;  // x^(k-1)
  double* __restrict__ xn = (k & 1) ? a.x1buf : a.x0buf;        // x^(k)
  const T* __restrict__ A = static_cast<const T*>(a.A);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nch = a.nchunks;
  const int64_t rb = DYN ? 0 : (int64_t)cta * a.m / ncta;  // this CTA's rows of the launch (rank)
  const int64_t re = DYN ? a.m : (int64_t)(cta + 1) * a.m / ncta;
  const int ntile = (int)((re - rb + R - 1) / R);
  // POL keep pattern over the CTA's units (DYN: over the launch's units, tiles numbered globally)
  const unsigned kthr = POL ? keep_threshold(a.l2_keep_pm) : 0u;
  const unsigned koff = DYN ? 0u : (unsigned)cta * 40503u;
  unsigned long long dmax = 0ull;

  auto finalize = [&](int t) {
    const int64_t tt = tbase + t;
    const int q = (int)(tt % kSlots);
    const int64_t r0 = DYN ? (int64_t)s_tile[t & 7] * R : rb + (int64_t)t * R;
    const int nv = (int)min((int64_t)R, re - r0);
    // The epilogue's own operands (b_i, a_ii, x_i^(k-1)) do not depend on the partial sums: load
    // them before waiting for the tile, so their latency hides behind the other warps' work.
    double bi = 0.0, dii = 1.0, xoi = 0.0;
    if (lane < nv && !a.rsum) {
      bi = a.b[r0 + lane];
      dii = a.diag[r0 + lane];
      xoi = ld_x1<XL>(xo + a.row0 + r0 + lane);
    }
    mbar_wait(&s_full[q], (unsigned)((tt / kSlots) & 1));
    if (lane < nv) {
      const double* sp = s_part + (size_t)q * nch * R + lane;
      double s = sp[0];
      for (int c = 1; c < nch; ++c) s += sp[(size_t)c * R];
      const int64_t row = r0 + lane;
      JB_CHECK(row >= 0 && row < a.m && a.row0 + row < a.x_len, 5);  // bit 5: epilogue row
      if (a.rsum) {  // column-wise partial product of this slab (epilogue after the reduction)
        a.rsum[row] = s;
      } else {
        const double xnew = __ddiv_rn(__dsub_rn(bi, s), dii);
        const int64_t gi = a.row0 + row;
        const double dx = __dsub_rn(xnew, xoi);
        if constexpr (PUSH) {  // NEXT-1: push x_i^(k) into every rank's x^(k) buffer (NVLink stores)
          const PeerArgs* pe = a.peers;
          for (int p = 0; p < pe->P; ++p) ((k & 1) ? pe->x1[p] : pe->x0[p])[gi] = xnew;
        } else {
          xn[gi] = xnew;
        }
        const unsigned long long bits = (unsigned long long)__double_as_longlong(dx) & 0x7fffffffffffffffull;
        dmax = bits > dmax ? bits : dmax;
        if (a.norm == JACOBI_NORM_L2) a.sq[row] = __dmul_rn(dx, dx);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_empty[q]);
  };

  unsigned pend = 0u;  // DYN: thread 0's claim for sequence t + kSlots
  int t = 0;
  for (;; ++t) {
    if (!DYN && t >= ntile) break;
    const int64_t tt = tbase + t;
    const int q = (int)(tt % kSlots);
    if (tt >= kSlots) mbar_wait(&s_empty[q], (unsigned)(((tt / kSlots) - 1) & 1));
    int64_t r0;
    if constexpr (DYN) {
      const int tile = s_tile[t & 7];
      if (tile < 0) break;
      r0 = (int64_t)tile * R;
      if (threadIdx.x == 0) pend = atomicAdd(a.dyn, 1u);
    } else {
      r0 = rb + (int64_t)t * R;
    }
    const int nv = (int)min((int64_t)R, re - r0);
    const T* rowp[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rowp[r] = A + (r0 + min(r, nv - 1)) * a.lda - a.col0;  // global columns
    const int64_t g0 = a.row0 + r0;
    // Pattern index of unit u of this tile: u * (tiles) + tile, i.e. each unit position — each warp's
    // share, since warp w takes u = w, w + NW, ... — walks its own tiles consecutively in the Weyl
    // sequence, so every warp keeps the same number of units (to within one) and no warp is left with
    // only HBM-served units at the end of the sweep (the intra-CTA tail).
    const unsigned tix = (unsigned)(DYN ? (r0 / R) : (int64_t)t) + koff;
    const unsigned ustride = (unsigned)(DYN ? a.tiles : ntile);
    constexpr int RG = R / GR;  // rows per unit
    for (int u = w; u < nch * GR; u += NW) {
      const int c = u / GR, rg = u % GR;
      uint64_t pol = 0;  // POL: evict_last for the kept units, evict_first for the streamed ones
      if constexpr (POL) pol = l2_policy(keep_unit((unsigned)u * ustride + tix, kthr));
      const int nvg = min(RG, nv - rg * RG);  // rows of this group that exist (last tile)
      if (nvg <= 0) continue;
      const T* rp[RG];
#pragma unroll
      for (int r = 0; r < RG; ++r)
        rp[r] = GR == 1 ? rowp[r] : A + (r0 + min(rg * RG + r, nv - 1)) * a.lda - a.col0;
      double acc[RG];
#pragma unroll
      for (int r = 0; r < RG; ++r) acc[r] = 0.0;
      const int64_t c0 = a.col0 + (int64_t)c * a.chunk;
      const int64_t c1 = min(c0 + (int64_t)a.chunk, a.cend);
      // Full units take the constant-row-count instance: with a run-time row count nvcc wraps each
      // row's load (and, for fp32, its converts) in a branch and keeps one A load in flight per warp
      // (c5 fell to 3.97 TB/s); with nv = R the loads are unconditional and software-pipelined.
      // Partial units (a CTA's last tile: c2 has 27-28 rows per CTA, a c3 P = 8 shard 13-14) dispatch
      // their row count to a compile-time constant too, so they keep every load in flight.
      check_tile<T, RG>(a, rp, c0, c1);
      with_nv<RG>(nvg, [&](auto nvc) {
        accumulate_chunk<T, RG, U, XL, POL, false, PIN>(rp, decltype(nvc)::value, xo, c0, c1, a.chunk, a.cend,
                                                        g0 + rg * RG, lane, acc, pol);
      });
#pragma unroll
      for (int r = 0; r < RG; ++r)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(kFull, acc[r], off);
      if (lane == 0) {
        double* dst = s_part + ((size_t)q * nch + c) * R + rg * RG;
#pragma unroll
        for (int r = 0; r < RG; ++r) dst[r] = acc[r];
      }
    }
    __syncwarp();
    if constexpr (DYN)
      if (threadIdx.x == 0) s_tile[(t + kSlots) & 7] = pend < (unsigned)a.tiles ? (int)pend : -1;
    if (lane == 0) mbar_arrive(&s_full[q]);
    if (t >= 1 && (t - 1) % NW == w) finalize(t - 1);
  }
  if (t >= 1 && (t - 1) % NW == w) finalize(t - 1);  // t = tiles processed
  if constexpr (DYN) {  // the launch's last CTA resets the counters for the next launch (all claims are done)
#ifdef JACOBI_BOUNDS_CHECK
    if (threadIdx.x == 0) __threadfence();  // this CTA's claims before its finish count (checked build)
#endif
    if (threadIdx.x == 0 && atomicAdd(a.dyn + 1, 1u) == (unsigned)ncta - 1u) {
      // Every CTA claimed kSlots tiles up front and one more per tile it processed, so a launch that
      // started from a zero counter and dealt every tile once ends at ncta * kSlots + tiles (bit 6).
      JB_CHECK(atomicAdd(a.dyn, 0u) == (unsigned)ncta * kSlots + (unsigned)a.tiles, 6);
      a.dyn[0] = 0u;
      a.dyn[1] = 0u;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(kFull, dmax, off);
    dmax = o > dmax ? o : dmax;
  }
  return dmax;
}

template <typename T, int R, int NW, int U = 1, int XL = 0, bool PUSH = false, bool POL = false, int GR = 1,
          bool DYN = false>
__global__ void __launch_bounds__(NW * 32, 1) k_sweep_cta(const SweepArgs a, const int j) {
  SMT_BEGIN();
  extern __shared__ __align__(16) double s_part[];  // [kSlots][nchunks][R]
  __shared__ __align__(8) uint64_t s_full[kSlots], s_empty[kSlots];
  __shared__ int s_go;
  __shared__ int s_tile[8];  // DYN: tile of sequence t at [t & 7]
  __shared__ long long s_k;
  if (threadIdx.x == 0) {
    s_go = sweep_prologue(a, j, blockIdx.x == 0, &s_k);
    if (DYN && s_go) {  // the tiles of sequences 0 .. kSlots-1
      const unsigned base = atomicAdd(a.dyn, (unsigned)kSlots);
      for (int q = 0; q < kSlots; ++q) s_tile[q] = base + q < (unsigned)a.tiles ? (int)(base + q) : -1;
    }
    for (int q = 0; q < kSlots; ++q) {
      mbar_init(&s_full[q], NW);
      mbar_init(&s_empty[q], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (!s_go) return;

  const int64_t k = s_k;
  __shared__ unsigned long long s_wmax[NW];
  const unsigned long long dmax =
      cta_sweep<T, R, NW, U, XL, PUSH, POL, GR, false, DYN>(a, k, 0, s_part, s_full, s_empty, blockIdx.x, gridDim.x,
                                                           s_tile);
  if constexpr (!PUSH) {
    if ((threadIdx.x & 31) == 0 && dmax) atomicMax(&a.dslot[k & 3], dmax);  // local L2: one per warp is fine
  } else {
    // NEXT-1: the CTA's max|dx| bits go into every rank's slot and, after a system-scope fence, one
    // arrival per CTA on every rank's counter for this parity; the next sweep's prologue waits for all
    // of them.  The CTA barrier inside cta_max_bits orders every thread's NVLink x pushes before thread
    // 0's fence, whose release is cumulative — one fence per CTA instead of one per thread (512
    // fence.sc.sys per CTA per sweep cost ~12 µs per sweep in the persistent kernel).
    const unsigned long long m = cta_max_bits<NW>(dmax, s_wmax);
    if (threadIdx.x == 0) push_signal(a.peers, k, m);
  }
  SMT_END();
}

// ---------------------------------------------------------------------------------------------
// k_solve_gridsync: sweeps k0..k1 in one cooperative launch (NEXT-3 for mid-size n: the graph of
// sweep kernels pays ~8 µs per sweep in kernel boundaries and dependent global round trips when A
// fits in or near the L2).  Each sweep is cta_sweep (same bits as k_sweep_cta) with x read at L2;
// between sweeps a grid barrier (one release atomic per CTA on a global counter, an acquire spin by
// one thread per CTA); after it every CTA evaluates the same stop test of PAPER.md:64-66 from the
// same distance slot.  Waits are bounded (fault flag -> JACOBI_ECUDA instead of a hung GPU).
#ifndef JACOBI_GRID_XL
#define JACOBI_GRID_XL 3
#endif
constexpr int kGridXL = JACOBI_GRID_XL;  // x loads in the persistent solver (2: ld.cg, 3: weak ld)
constexpr int kGridMaxL2Blocks = 64;  // Euclidean rule in the persistent solver: m <= 64 * kL2Block rows

template <typename T, int R, int NW, bool POL, int GR = 1>
__global__ void __launch_bounds__(NW * 32, 1) k_solve_gridsync(const SweepArgs a, unsigned long long* gbar,
                                                               const int64_t k0, const int64_t k1) {
  extern __shared__ __align__(16) double s_part[];  // [kSlots][nchunks][R]
  __shared__ __align__(8) uint64_t s_full[kSlots], s_empty[kSlots];
  __shared__ int s_go;
  __shared__ double s_red[NW * 32];             // Euclidean rule: two 256-row block trees at a time
  __shared__ double s_blk[kGridMaxL2Blocks];    // ... and the block partials
  __shared__ double s_d2;                       // ... and sum of squares
  State* st = a.st;
  if (threadIdx.x == 0) {
    for (int q = 0; q < kSlots; ++q) {
      mbar_init(&s_full[q], NW);
      mbar_init(&s_empty[q], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (*(volatile int32_t*)&st->done || st->nonfinite || *(volatile int32_t*)&st->fault) return;  // uniform
  const int64_t rb = (int64_t)blockIdx.x * a.m / gridDim.x;
  const int64_t re = (int64_t)(blockIdx.x + 1) * a.m / gridDim.x;
  const int64_t ntile = (re - rb + R - 1) / R;
  const int lane = threadIdx.x & 31;
  const bool l2 = a.norm == JACOBI_NORM_L2;
  // The stop test's parameters do not change during a launch: read once, so thread 0's per-sweep chain
  // is barrier spin -> distance slot -> decision (each extra dependent L2 read cost ~0.3 µs per sweep).
  const double tol = st->tol;
  const int64_t max_iter = st->max_iter;
  double* const hist = st->hist;
  // A fixed-count run (tol = 0: d_k < tol never holds) needs d_{k-1} only for the
  // history, i.e. in CTA 0 when one is recorded: the other CTAs skip its L2 round trip (max norm) or
  // its all-rows reduction (Euclidean) on the way from the barrier to the next sweep.
  const bool need_d = tol > 0.0 || (blockIdx.x == 0 && hist);
  for (int64_t k = k0;; ++k) {
    if (threadIdx.x == 0) {
      int go = 1;
      if (k > k0) {  // grid barrier: every CTA has stored its x_i^(k-1), max|dx| bits (and dx^2)
        const unsigned long long target = (unsigned long long)gridDim.x * (unsigned long long)(k - 1);
        unsigned long long t0 = 0;
        for (unsigned i = 0; ld_acquire_gpu(gbar) < target; ++i) {
          if ((i & 1023) == 1023) {
            const unsigned long long t = global_ns();
            if (t0 == 0) t0 = t;
            else if (t - t0 > 2000000000ull || *(volatile int32_t*)&st->fault) {
              st->fault = 1;
              go = 0;
              break;
            }
          }
        }
      }
      s_go = go;
    }
    if (l2) __syncthreads();  // max norm: thread 0 goes straight on to the stop test below
    if (l2 && need_d && s_go && k >= 2) {
      // The Euclidean distance of PAPER.md:94 over all rows, computed redundantly by every CTA in the
      // order of k_l2_partials / k_l2_final (256-row shared-memory trees, then a strided ascending
      // warp sum and a butterfly), so the bits equal the graph path's.  dx^2 of sweep k-1 lives in
      // the half (k-1) & 1 of the double-buffered sq array; sweep k writes the other half.
      const double* sq = a.sq + ((k - 1) & 1) * a.m;
      const int64_t nblk = (a.m + kL2Block - 1) / kL2Block;
      const int half = threadIdx.x / kL2Block, t = threadIdx.x % kL2Block;
      for (int64_t b0 = 0; b0 < nblk; b0 += NW * 32 / kL2Block) {
        const int64_t blk = b0 + half, i = blk * kL2Block + t;
        s_red[threadIdx.x] = (blk < nblk && i < a.m) ? ld_x1<2>(sq + i) : 0.0;
        __syncthreads();
        for (int off = kL2Block / 2; off > 0; off >>= 1) {
          if (t < off) s_red[threadIdx.x] = __dadd_rn(s_red[threadIdx.x], s_red[threadIdx.x + off]);
          __syncthreads();
        }
        if (t == 0 && blk < nblk) s_blk[blk] = s_red[threadIdx.x];
        __syncthreads();
      }
      if (threadIdx.x < 32) {
        double v = 0.0;
        for (int64_t q = threadIdx.x; q < nblk; q += 32) v = __dadd_rn(v, s_blk[q]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(kFull, v, off));
        if (threadIdx.x == 0) s_d2 = __dsqrt_rn(v);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      int go = s_go;
      if (go && need_d && k >= 2) {  // stop test for sweep k-1, identical in every CTA
        const double d = l2 ? s_d2 : ld_x1<2>(reinterpret_cast<const double*>(a.dslot + ((k - 1) & 3)));
        if (blockIdx.x == 0 && hist) hist[k - 2] = d;
        if (d < tol) {
          if (blockIdx.x == 0) { st->status = JACOBI_CONVERGED; st->iters = k - 1; st->done = 1; }
          go = 0;
        }
      }
      if (go && k > max_iter) {
        if (blockIdx.x == 0) { st->status = JACOBI_MAX_ITER; st->iters = max_iter; st->done = 1; }
        go = 0;
      }
      if (go && k > k1) go = 0;  // end of this launch's segment; the next launch resumes at k
      if (go && blockIdx.x == 0) a.dslot[(k + 1) & 3] = 0ull;
      s_go = go;
    }
    __syncthreads();
    if (!s_go) break;
#ifdef JACOBI_SM_TIMING
    // probe build: sweeps k0+20 .. k0+23 of the launch, per CTA: SM id, start of the sweep's work (after
    // the barrier and stop test), end of it (before the barrier arrival)
    const int64_t smt_i = k - k0 - 20;
    unsigned long long smt_go = 0;
    if (threadIdx.x == 0 && smt_i >= 0 && smt_i < 4) smt_go = global_ns();
#endif
    SweepArgs ak = a;
    ak.sq = a.sq + (k & 1) * a.m;  // double-buffered dx^2 (Euclidean rule)
    const unsigned long long dmax =
        cta_sweep<T, R, NW, 1, kGridXL, false, POL, GR, GR == 1>(ak, k, (k - k0) * ntile, s_part, s_full, s_empty,
                                                                 blockIdx.x, gridDim.x);
    if (lane == 0 && dmax) atomicMax(&a.dslot[k & 3], dmax);
    __syncthreads();  // every x_i^(k) store and max|dx| atomic of this CTA has been issued
    if (threadIdx.x == 0) {
#ifdef JACOBI_SM_TIMING
      if (smt_i >= 0 && smt_i < 4 && blockIdx.x < 1024) {
        unsigned sm_;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));
        const size_t o = 3 * ((size_t)smt_i * 1024 + blockIdx.x);
        g_smt[o] = sm_;
        g_smt[o + 1] = smt_go;
        g_smt[o + 2] = global_ns();
      }
#endif
      asm volatile("fence.acq_rel.gpu;" ::: "memory");  // release, cumulative over the CTA's stores
      atomicAdd(gbar, 1ull);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// k_solve_gridsync_push: the persistent solver over P ranks with the fused exchange (NEXT-1 x
// NEXT-3).  Each rank runs one cooperative launch of G CTAs for the sweeps k0..k1; each sweep is
// cta_sweep with the NVLink push of x_i^(k) into every rank's buffer, then per CTA one remote
// atomicMax of the max|dx| bits into every rank's slot and, after a system fence, one arrival on
// every rank's counter for the sweep's parity.  Before sweep k >= 2 a CTA waits on its own rank's
// counter (all CTAs of all ranks have pushed x^(k-1)) — also at k = k0, since other GPUs may still
// be finishing the previous launch — and then every CTA of every rank takes the same stop decision
// from its own copy of the distance slot.  x^(k-1) is read with weak loads (kGridXL = 3), as in
// k_solve_gridsync: thread 0's ld.acquire.sys of the arrival counter and the CTA barrier that follows
// order every peer's and every local CTA's stores of x^(k-1) before them (ld.global.cg here — L2 on
// every tile, asm volatile — measured 1.6x slower per sweep: c3 shard 491 vs 299 µs).
// Single-GPU emulation: one launch holds nvr virtual ranks (CTA groups) with their own x copies,
// slots and counters (jacobi_plan_set_p2p_emulation) — the whole protocol in one co-resident grid.
template <typename T, int R, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_solve_gridsync_push(const SweepArgs* __restrict__ ranks, const int nvr,
                                                                    const int64_t k0, const int64_t k1) {
  extern __shared__ __align__(16) double s_part[];  // [kSlots][nchunks][R]
  __shared__ __align__(8) uint64_t s_full[kSlots], s_empty[kSlots];
  __shared__ unsigned long long s_wmax[NW];
  __shared__ int s_go;
  // this CTA's virtual rank and its CTA range within it (balanced split of the grid)
  int vr = 0;
  while (vr + 1 < nvr && (int64_t)(vr + 1) * gridDim.x / nvr <= (int64_t)blockIdx.x) ++vr;
  const int c0 = (int)((int64_t)vr * gridDim.x / nvr), c1 = (int)((int64_t)(vr + 1) * gridDim.x / nvr);
  const SweepArgs a = ranks[vr];
  const PeerArgs* pe = a.peers;
  State* st = a.st;
  if (threadIdx.x == 0) {
    for (int q = 0; q < kSlots; ++q) {
      mbar_init(&s_full[q], NW);
      mbar_init(&s_empty[q], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (*(volatile int32_t*)&st->done || st->nonfinite || *(volatile int32_t*)&st->fault) return;  // uniform
  const int64_t rb = (int64_t)(blockIdx.x - c0) * a.m / (c1 - c0);
  const int64_t re = (int64_t)(blockIdx.x - c0 + 1) * a.m / (c1 - c0);
  const int64_t ntile = (re - rb + R - 1) / R;
  const bool leader = blockIdx.x == c0;  // writes this rank's state, history and slot clears
  const double tol = st->tol;            // fixed during the launch (see k_solve_gridsync)
  const int64_t max_iter = st->max_iter;
  double* const hist = st->hist;
  const bool need_d = tol > 0.0 || (leader && hist);  // as in k_solve_gridsync
  for (int64_t k = k0;; ++k) {
    if (threadIdx.x == 0) {
      int go = 1;
      if (k >= 2) {  // every CTA of every rank has pushed x^(k-1) and its max|dx| bits here
        const unsigned long long kp = (unsigned long long)(k - 1);
        const unsigned long long target = ((kp + (kp & 1)) / 2) * pe->total_ctas;  // sweeps of this parity
        const unsigned long long* f = pe->flags[pe->rank] + (kp & 1);
        unsigned long long t0 = 0;
        for (unsigned i = 0; ld_acquire_sys(f) < target; ++i) {
          if ((i & 1023) == 1023) {
            const unsigned long long t = global_ns();
            if (t0 == 0) t0 = t;
            else if (t - t0 > pe->wait_ns || *(volatile int32_t*)&st->fault) {
              st->fault = 1;
              go = 0;
              break;
            }
          }
        }
      }
      if (go && need_d && k >= 2) {  // stop test for sweep k-1, identical on every rank
        const double d = ld_x1<2>(reinterpret_cast<const double*>(a.dslot + ((k - 1) & 3)));
        if (leader && hist) hist[k - 2] = d;
        if (d < tol) {
          if (leader) { st->status = JACOBI_CONVERGED; st->iters = k - 1; st->done = 1; }
          go = 0;
        }
      }
      if (go && k > max_iter) {
        if (leader) { st->status = JACOBI_MAX_ITER; st->iters = max_iter; st->done = 1; }
        go = 0;
      }
      if (go && k > k1) go = 0;  // end of this launch's segment; the next launch resumes at k
      if (go && leader) a.dslot[(k + 1) & 3] = 0ull;
      s_go = go;
    }
    __syncthreads();
    if (!s_go) break;
    const unsigned long long dmax =
        cta_sweep<T, R, NW, 1, kGridXL, true, true, 1, true>(a, k, (k - k0) * ntile, s_part, s_full, s_empty, blockIdx.x - c0,
                                                   c1 - c0);
    const unsigned long long m = cta_max_bits<NW>(dmax, s_wmax);  // CTA barrier: every x push issued
    if (threadIdx.x == 0) push_signal(pe, k, m);
  }
}

// ---------------------------------------------------------------------------------------------
// k_sweep_panel: every warp owns whole rows.  CTA b of G owns rows [b*m/G, (b+1)*m/G); warp w of NW
// owns an equal share of them (balanced to one row) and walks its tiles of R rows across all column
// chunks in ascending order, adding each chunk's butterfly sum to the row's running sum — exactly the
// canonical order (s = chunk_0; s += chunk_c for c = 1, 2, ...) — and applies the fused epilogue
// itself.  No shared memory, no barriers, no cross-warp handoff.  Because the CTA's warps march
// across the same column chunks at the same rate, each x^(k-1) chunk is fetched from L2 once per CTA
// and served to the other warps from L1 (in k_sweep_cta every warp reads a different chunk, so x
// streams from L2 once per tile: +25 % of the A bytes for fp64, +50 % for fp32 A).
// Shared-memory ring of x^(k-1) chunks (k_sweep_panel with XSN slots).  Item i = t * nchunks + c is
// chunk c for the warps' t-th tiles; it lives in slot i mod XSN and lands on full[slot] (mbarrier
// parity (i / XSN) & 1).  Every warp still at its t-th tile consumes every item of round t in order;
// the last of them (smem arrival counter) refills the slot with item i + XSN.  A warp waits for item
// i only after consuming item i - XSN, so the parity never aliases a phase two rounds back.
struct XRing {
  double* xs;          // [XSN][chunk]
  uint64_t* full;      // [XSN]
  unsigned* cnt;       // [XSN]
  int64_t items;       // rounds * nchunks
  int xsn;
};
__device__ __forceinline__ void xring_issue(const XRing& q, const SweepArgs& a, const double* xo, int64_t i) {
  if (i >= q.items) return;
  const int slot = (int)(i % q.xsn);
  const int64_t c0 = a.col0 + (i % a.nchunks) * (int64_t)a.chunk;
  const int64_t cols = min((int64_t)a.chunk, a.cend - c0);
  const unsigned bytes = (unsigned)((cols * 8 + 15) & ~(int64_t)15);  // x is padded past n
  JB_CHECK(c0 + (int64_t)(bytes / 8) <= a.x_len && (int64_t)(bytes / 8) <= a.chunk, 4);  // bit 4: x ring copy
  double* dst = q.xs + (size_t)slot * a.chunk;
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&q.full[slot]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot before the async write
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(xo + c0), "r"(bytes), "r"(bar)
               : "memory");
}

template <typename T, int R, int U, int XL, bool POL, int NV, int XSN = 0>
__device__ __forceinline__ void panel_tile(const SweepArgs& a, const T* A, const double* __restrict__ xo,
                                           const int64_t r0, const int lane, double (&s)[R], const uint64_t pol,
                                           const XRing* ring = nullptr, int64_t item0 = 0, unsigned arrivals = 0) {
  const T* rowp[R];
#pragma unroll
  for (int r = 0; r < R; ++r) rowp[r] = A + (r0 + (r < NV ? r : NV - 1)) * a.lda - a.col0;
  const int64_t g0 = a.row0 + r0;
  for (int c = 0; c < a.nchunks; ++c) {
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    const int64_t c0 = a.col0 + (int64_t)c * a.chunk;
    const int64_t c1 = min(c0 + (int64_t)a.chunk, a.cend);
    check_tile<T, R>(a, rowp, c0, c1);
    if constexpr (XSN > 0) {
      const int64_t i = item0 + c;
      const int slot = (int)(i % XSN);
      mbar_wait(&ring->full[slot], (unsigned)((i / XSN) & 1));
      accumulate_chunk<T, R, U, XL, POL, true>(rowp, NV, xo, c0, c1, a.chunk, a.cend, g0, lane, acc, pol,
                                               ring->xs + (size_t)slot * a.chunk);
      __syncwarp();
      if (lane == 0 && atomicAdd(&ring->cnt[slot], 1u) + 1u == arrivals) {  // last reader of item i
        ring->cnt[slot] = 0u;
        xring_issue(*ring, a, xo, i + XSN);
      }
    } else {
      accumulate_chunk<T, R, U, XL, POL>(rowp, NV, xo, c0, c1, a.chunk, a.cend, g0, lane, acc, pol);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(kFull, acc[r], off);
      s[r] = c == 0 ? acc[r] : s[r] + acc[r];
    }
  }
}

// Row count nv in [1, R] as a compile-time constant (a run-time count serialises the loads, see
// k_sweep_cta).
template <typename T, int R, int U, int XL, bool POL, int XSN, int NV = R>
__device__ __forceinline__ void panel_tile_nv(const int nv, const SweepArgs& a, const T* A,
                                              const double* __restrict__ xo, const int64_t r0, const int lane,
                                              double (&s)[R], const uint64_t pol, const XRing* ring,
                                              int64_t item0, unsigned arrivals) {
  if constexpr (NV == 1) {
    panel_tile<T, R, U, XL, POL, 1, XSN>(a, A, xo, r0, lane, s, pol, ring, item0, arrivals);
  } else {
    if (nv == NV) panel_tile<T, R, U, XL, POL, NV, XSN>(a, A, xo, r0, lane, s, pol, ring, item0, arrivals);
    else panel_tile_nv<T, R, U, XL, POL, XSN, NV - 1>(nv, a, A, xo, r0, lane, s, pol, ring, item0, arrivals);
  }
}

// POL: rows in the first l2_keep_pm/1000 of each warp's share are loaded with L2 evict_last (kept
// resident across sweeps), the rest with evict_first.
// XSN > 0: x^(k-1) is staged in shared memory, chunk by chunk, through an XSN-slot ring filled by the
// bulk-copy engine (XRing); else each warp reads it with L1-cached global loads.
constexpr int kMaxXSN = 16;
template <typename T, int R, int NW, int U = 1, int XL = 0, bool POL = false, int XSN = 0>
__global__ void __launch_bounds__(NW * 32, 1) k_sweep_panel(const SweepArgs a, const int j) {
  SMT_BEGIN();
  static_assert(XSN <= kMaxXSN, "x ring slots");
  extern __shared__ __align__(128) double s_xring[];  // [XSN][chunk] when XSN > 0
  __shared__ __align__(8) uint64_t s_xfull[XSN > 0 ? XSN : 1];
  __shared__ unsigned s_xcnt[XSN > 0 ? XSN : 1];
  __shared__ int s_go;
  __shared__ long long s_k;
  if (threadIdx.x == 0) {
    s_go = sweep_prologue(a, j, blockIdx.x == 0, &s_k);
    if constexpr (XSN > 0) {
      for (int q = 0; q < XSN; ++q) {
        mbar_init(&s_xfull[q], 1);
        s_xcnt[q] = 0u;
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  if (!s_go) return;

  const int64_t k = s_k;
  const double* __restrict__ xo = (k & 1) ? a.x0buf : a.x1buf;  // x^(k-1)
  double* __restrict__ xn = (k & 1) ? a.x1buf : a.x0buf;        // x^(k)
  const T* __restrict__ A = static_cast<const T*>(a.A);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#ifdef JACOBI_SM_TIMING
  const int64_t cb = (blockIdx.x + g_rot) % gridDim.x;  // probe build: rotate the CTA -> row-block map
#else
  const int64_t cb = blockIdx.x;
#endif
  const int64_t rb = cb * a.m / gridDim.x;
  const int64_t re = (cb + 1) * a.m / gridDim.x;
  const int64_t wb = rb + (re - rb) * w / NW, we = rb + (re - rb) * (w + 1) / NW;
  // x ring schedule: round t = every warp's t-th tile; arrivals of round t = warps with > t tiles.
  XRing ring{};
  auto tiles_of = [&](int ww) {
    const int64_t b0 = rb + (re - rb) * ww / NW, b1 = rb + (re - rb) * (ww + 1) / NW;
    return (int)((b1 - b0 + R - 1) / R);
  };
  if constexpr (XSN > 0) {
    int rounds = 0;
    for (int ww = 0; ww < NW; ++ww) rounds = max(rounds, tiles_of(ww));
    ring = XRing{s_xring, s_xfull, s_xcnt, (int64_t)rounds * a.nchunks, XSN};
    if (threadIdx.x == 0)
      for (int64_t i = 0; i < XSN; ++i) xring_issue(ring, a, xo, i);
  }
  unsigned long long dmax = 0ull;
  int t = 0;
  for (int64_t r0 = wb; r0 < we; r0 += R, ++t) {
    const int nv = (int)min((int64_t)R, we - r0);
    double s[R];
    uint64_t pol = 0;
    if constexpr (POL) pol = l2_policy((r0 - wb) * 1000 < (we - wb) * (int64_t)a.l2_keep_pm);
    unsigned arrivals = 0;
    if constexpr (XSN > 0)
      for (int ww = 0; ww < NW; ++ww) arrivals += tiles_of(ww) > t ? 1u : 0u;
    panel_tile_nv<T, R, U, XL, POL, XSN>(nv, a, A, xo, r0, lane, s, pol, &ring, (int64_t)t * a.nchunks, arrivals);
    double mine = s[0];
#pragma unroll
    for (int r = 1; r < R; ++r)
      if (lane == r) mine = s[r];
    if (lane < nv) {
      const int64_t row = r0 + lane;
      JB_CHECK(row >= 0 && row < a.m && a.row0 + row < a.x_len, 5);
      if (a.rsum) {  // column-wise partial product of this slab (epilogue after the reduction)
        a.rsum[row] = mine;
      } else {
        const double xnew = __ddiv_rn(__dsub_rn(a.b[row], mine), a.diag[row]);
        const int64_t gi = a.row0 + row;
        const double dx = __dsub_rn(xnew, xo[gi]);
        xn[gi] = xnew;
        const unsigned long long bits = (unsigned long long)__double_as_longlong(dx) & 0x7fffffffffffffffull;
        dmax = bits > dmax ? bits : dmax;
        if (a.norm == JACOBI_NORM_L2) a.sq[row] = __dmul_rn(dx, dx);
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(kFull, dmax, off);
    dmax = o > dmax ? o : dmax;
  }
  if (lane == 0 && dmax) atomicMax(&a.dslot[k & 3], dmax);
  SMT_END();
}

// k_sweep_group: the row-panel kernel with G warps per tile.  The CTA's NW warps form NW/G groups;
// group p owns an equal share of the CTA's rows and walks them in tiles of R rows; warp q of the group
// takes the tile's chunks q, q + G, ... (each chunk's lane chains and butterfly exactly as in the panel
// kernel), writes the chunk sums to the group's shared-memory partials (double-buffered by tile
// parity), and after a group barrier warp 0 folds them in ascending chunk order — the canonical order
// again — and applies the fused epilogue.  Why: a group streams G chunks of each of its rows at once,
// so the chip keeps 1/G as many DRAM rows open as the panel kernel (probes/tma_warp_probe.cu, c5's
// pattern: 7.10 TB/s for one warp per 4-row tile, 7.21-7.28 for 2-16), while x^(k-1) still comes from
// the CTA's shared-memory ring (each chunk read by one warp of every group).
template <typename T, int R, int NW, int G, int XSN>
__global__ void __launch_bounds__(NW * 32, 1) k_sweep_group(const SweepArgs a, const int j) {
  SMT_BEGIN();
  static_assert(XSN > 0 && XSN <= kMaxXSN && NW % G == 0 && NW / G <= 15, "group kernel shape");
  constexpr int NG = NW / G;
  extern __shared__ __align__(128) double s_xring[];  // [XSN][chunk] x ring, then [NG][2][R][nchunks] partials
  __shared__ __align__(8) uint64_t s_xfull[XSN];
  __shared__ unsigned s_xcnt[XSN];
  __shared__ int s_go;
  __shared__ long long s_k;
  if (threadIdx.x == 0) {
    s_go = sweep_prologue(a, j, blockIdx.x == 0, &s_k);
    for (int q = 0; q < XSN; ++q) {
      mbar_init(&s_xfull[q], 1);
      s_xcnt[q] = 0u;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (!s_go) return;

  const int64_t k = s_k;
  const double* __restrict__ xo = (k & 1) ? a.x0buf : a.x1buf;  // x^(k-1)
  double* __restrict__ xn = (k & 1) ? a.x1buf : a.x0buf;        // x^(k)
  const T* __restrict__ A = static_cast<const T*>(a.A);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, grp = w / G, q = w % G;
  const int64_t rb = blockIdx.x * a.m / gridDim.x, re = (blockIdx.x + 1) * a.m / gridDim.x;
  auto tiles_of = [&](int gg) {
    const int64_t b0 = rb + (re - rb) * gg / NG, b1 = rb + (re - rb) * (gg + 1) / NG;
    return (int)((b1 - b0 + R - 1) / R);
  };
  const int64_t gb = rb + (re - rb) * grp / NG, ge = rb + (re - rb) * (grp + 1) / NG;
  int rounds = 0;
  for (int gg = 0; gg < NG; ++gg) rounds = max(rounds, tiles_of(gg));
  const int nch = a.nchunks;
  const XRing ring{s_xring, s_xfull, s_xcnt, (int64_t)rounds * nch, XSN};
  if (threadIdx.x == 0)
    for (int64_t i = 0; i < XSN; ++i) xring_issue(ring, a, xo, i);
  double* const part0 = s_xring + (size_t)XSN * a.chunk + (size_t)grp * 2 * R * nch;
  unsigned long long dmax = 0ull;
  int t = 0;
  for (int64_t r0 = gb; r0 < ge; r0 += R, ++t) {
    const int nv = (int)min((int64_t)R, ge - r0);
    unsigned arrivals = 0;  // groups with a t-th tile: one warp of each reads every item of round t
    for (int gg = 0; gg < NG; ++gg) arrivals += tiles_of(gg) > t ? 1u : 0u;
    double* const part = part0 + (size_t)(t & 1) * R * nch;
    const int64_t g0 = a.row0 + r0;
    with_nv<R>(nv, [&](auto NVc) {
      constexpr int NV = decltype(NVc)::value;
      const T* rowp[R];
#pragma unroll
      for (int r = 0; r < R; ++r) rowp[r] = A + (r0 + (r < NV ? r : NV - 1)) * a.lda - a.col0;
      for (int c = q; c < nch; c += G) {
        double acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.0;
        const int64_t c0 = a.col0 + (int64_t)c * a.chunk;
        const int64_t c1 = min(c0 + (int64_t)a.chunk, a.cend);
        check_tile<T, R>(a, rowp, c0, c1);
        const int64_t i = (int64_t)t * nch + c;
        const int slot = (int)(i % XSN);
        mbar_wait(&ring.full[slot], (unsigned)((i / XSN) & 1));
        accumulate_chunk<T, R, 1, 0, false, true>(rowp, NV, xo, c0, c1, a.chunk, a.cend, g0, lane, acc, 0,
                                                  ring.xs + (size_t)slot * a.chunk);
        __syncwarp();
        if (lane == 0 && atomicAdd(&ring.cnt[slot], 1u) + 1u == arrivals) {  // last reader of item i
          ring.cnt[slot] = 0u;
          xring_issue(ring, a, xo, i + XSN);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(kFull, acc[r], off);
          if (lane == r) part[r * nch + c] = acc[r];
        }
      }
    });
    // the group's chunk sums of this tile are in `part`; the barrier of tile t + 1 orders warp 0's
    // fold of tile t before any write of tile t + 2 into the same buffer
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(G * 32) : "memory");
    if (q == 0 && lane < nv) {
      double mine = part[lane * nch];
      for (int c = 1; c < nch; ++c) mine += part[lane * nch + c];  // ascending chunk order
      const int64_t row = r0 + lane;
      JB_CHECK(row >= 0 && row < a.m && a.row0 + row < a.x_len, 5);
      if (a.rsum) {  // column-wise partial product of this slab (epilogue after the reduction)
        a.rsum[row] = mine;
      } else {
        const double xnew = __ddiv_rn(__dsub_rn(a.b[row], mine), a.diag[row]);
        const int64_t gi = a.row0 + row;
        const double dx = __dsub_rn(xnew, xo[gi]);
        xn[gi] = xnew;
        const unsigned long long bits = (unsigned long long)__double_as_longlong(dx) & 0x7fffffffffffffffull;
        dmax = bits > dmax ? bits : dmax;
        if (a.norm == JACOBI_NORM_L2) a.sq[row] = __dmul_rn(dx, dx);
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(kFull, dmax, off);
    dmax = o > dmax ? o : dmax;
  }
  if (lane == 0 && dmax) atomicMax(&a.dslot[k & 3], dmax);
  SMT_END();
}

// Euclidean distance (NEXT-2 row), deterministic: k_l2_partials sums each block of
// kL2Block rows' squared changes with a fixed smem tree; k_l2_final (one warp) sums the block partials
// of all ranks (lane l: blocks l, l+32, ... ascending; then a shfl_xor butterfly) and stores the
// bits of sqrt(sum) in the sweep's distance slot, overwriting the max-norm bits.
__global__ void __launch_bounds__(kL2Block) k_l2_partials(const double* __restrict__ sq, int64_t m,
                                                          double* __restrict__ blk, const State* st) {
  if (*(volatile const int32_t*)&st->done) return;
  __shared__ double s[kL2Block];
  const int64_t i = (int64_t)blockIdx.x * kL2Block + threadIdx.x;
  s[threadIdx.x] = i < m ? sq[i] : 0.0;
  __syncthreads();
  for (int off = kL2Block / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) s[threadIdx.x] = __dadd_rn(s[threadIdx.x], s[threadIdx.x + off]);
    __syncthreads();
  }
  if (threadIdx.x == 0) blk[blockIdx.x] = s[0];
}

__global__ void k_l2_final(const double* __restrict__ blk, int64_t nblk, unsigned long long* dslot, State* st,
                           int j) {
  if (*(volatile int32_t*)&st->done) return;
  const int64_t k = st->kbase + j + 1;
  double s = 0.0;
  for (int64_t q = threadIdx.x; q < nblk; q += 32) s = __dadd_rn(s, blk[q]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_xor_sync(kFull, s, off));
  if (threadIdx.x == 0) dslot[k & 3] = (unsigned long long)__double_as_longlong(__dsqrt_rn(s));
}

// Column-wise epilogue (NEXT-4, "partial values ... added together and subtracted by the
// value of the corresponding cell of the B vector"): s_i = sum of the nb slab partials in ascending
// slab order, then x_i^(k) = (b_i - s_i)/a_ii and |dx| for the rows [row0, row0 + rows).
__global__ void k_colsum_epilogue(const double* __restrict__ rsum, int nb, int64_t stride, int64_t rows,
                                  int64_t row0, const double* __restrict__ b, const double* __restrict__ diag,
                                  double* x0buf, double* x1buf, unsigned long long* dslot, double* sq, int norm,
                                  State* st, int j) {
  if (*(volatile int32_t*)&st->done || st->nonfinite || st->fault) return;
  const int64_t k = st->kbase + j + 1;
  const double* xo = (k & 1) ? x0buf : x1buf;
  double* xn = (k & 1) ? x1buf : x0buf;
  unsigned long long dmax = 0ull;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    double s = rsum[r];
    for (int q = 1; q < nb; ++q) s += rsum[(int64_t)q * stride + r];
    const double xnew = __ddiv_rn(__dsub_rn(b[r], s), diag[r]);
    const int64_t gi = row0 + r;
    const double dx = __dsub_rn(xnew, xo[gi]);
    xn[gi] = xnew;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(dx) & 0x7fffffffffffffffull;
    dmax = bits > dmax ? bits : dmax;
    if (norm == JACOBI_NORM_L2) sq[r] = __dmul_rn(dx, dx);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(kFull, dmax, off);
    dmax = o > dmax ? o : dmax;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(&dslot[k & 3], dmax);
}

// After a graph batch of K sweeps: settle the stop decision for the batch's last sweep (same rule
// as the prologue) and advance the sweep counter.
__device__ __forceinline__ bool advance(State* st, const unsigned long long* dslot, int K) {
  if (st->done || st->nonfinite || st->fault) return false;
  const int64_t k = st->kbase + K + 1;  // the sweep that would come next
  const double d = __longlong_as_double((long long)dslot[(k - 1) & 3]);
  if (st->hist) st->hist[k - 2] = d;
  if (d < st->tol) { st->status = JACOBI_CONVERGED; st->iters = k - 1; st->done = 1; return false; }
  if (k > st->max_iter) { st->status = JACOBI_MAX_ITER; st->iters = st->max_iter; st->done = 1; return false; }
  st->kbase += K;
  return true;
}
__global__ void k_advance(State* st, const unsigned long long* dslot, int K) { advance(st, dslot, K); }
// ... and, as the last node of the body of a device-side while loop (conditional graph node), decide
// whether the loop runs another batch: the solve needs one graph launch and no host polling.
__global__ void k_advance_while(State* st, const unsigned long long* dslot, int K, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, advance(st, dslot, K) ? 1u : 0u);
}

template <typename T>
__global__ void k_setup_diag(const T* __restrict__ A, int64_t lda, int64_t m, int64_t row0,
                             double* __restrict__ diag, unsigned long long* zero_min) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)A[r * lda + row0 + r];
    diag[r] = v;
    if (v == 0.0) atomicMin(zero_min, (unsigned long long)(row0 + r));
  }
}

__device__ __forceinline__ bool nonfinite(double v) {
  return ((unsigned long long)__double_as_longlong(v) & 0x7ff0000000000000ull) == 0x7ff0000000000000ull;
}
__device__ __forceinline__ bool nonfinite(float v) {
  return ((unsigned)__float_as_uint(v) & 0x7f800000u) == 0x7f800000u;
}

template <typename T>
__global__ void k_scan_A(const T* __restrict__ A, int64_t lda, int64_t m, int64_t n, int* flag) {
  const int lane = threadIdx.x & 31;
  bool bad = false;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < m;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const T* row = A + r * lda;
    for (int64_t jj = lane; jj < n; jj += 32) bad |= nonfinite(row[jj]);
  }
  if (__any_sync(kFull, bad) && lane == 0) *flag = 1;
}

// Solve start (one launch, no host round trip): stop-state parameters, distance slots and tile
// counters cleared, and the non-finite scan of b and x0 (PAPER.md:59 inputs; ENONFINITE is reported
// when the host reads the final state).  The state was zeroed by a memset just before.
__global__ void k_prepare(State* st, int64_t max_iter, double tol, double* hist, unsigned long long* dslot,
                          unsigned* cnt, int64_t ncnt, double* __restrict__ b, const double* __restrict__ b_src,
                          int64_t m, double* __restrict__ x0, const double* __restrict__ x0_src, int64_t n,
                          unsigned long long* flags, unsigned long long* gbar) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0) {
    st->max_iter = max_iter;
    st->tol = tol;
    st->hist = hist;
    if (gbar) *gbar = 0ull;
  }
  if (tid < 4) dslot[tid] = 0ull;
  if (flags && tid < 2) flags[tid] = 0ull;
  for (int64_t i = tid; i < ncnt; i += stride) cnt[i] = 0u;
  bool bad = false;
  // Device inputs are copied in here (one launch instead of two memcpys); host inputs were copied
  // by the caller, and are only scanned.
  for (int64_t i = tid; i < m; i += stride) {
    const double v = b_src ? b_src[i] : b[i];
    if (b_src) b[i] = v;
    bad |= nonfinite(v);
  }
  for (int64_t i = tid; i < n; i += stride) {
    const double v = x0_src ? x0_src[i] : x0[i];
    if (x0_src) x0[i] = v;
    bad |= nonfinite(v);
  }
  if (bad) st->nonfinite = 1;
}

// Solve end, device x_out: copy x^(iters) (ping-pong buffer iters & 1) to the caller's buffer, decided
// on the device from the final state — enqueued after every solver launch, before the state is read
// back, so a device solve needs one host synchronisation.  Nothing is written unless the solve has
// finished (done) without failing (non-finite input, a wait fault): x_out is only written for a
// status >= 0.
__global__ void k_finalize(const State* st, const double* __restrict__ x0buf, const double* __restrict__ x1buf,
                           double* __restrict__ dst, int64_t n) {
  if (!st->done || st->nonfinite || st->fault) return;  // only a finished, successful solve
  const double* src = (st->iters & 1) ? x1buf : x0buf;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

template <typename T>
__global__ void k_copy_pitched(const T* __restrict__ src, int64_t sld, T* __restrict__ dst, int64_t dld,
                               int64_t rows, int64_t n) {
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < dld; c += (int64_t)gridDim.x * blockDim.x)
      dst[r * dld + c] = c < n ? src[r * sld + c] : T(0);
}

__global__ void k_probe(const double* __restrict__ buf, int64_t nvec, double* out) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + stride < nvec; i += 2 * stride) {
    double v0[4], v1[4];
    ld_a(buf + 4 * i, v0);
    ld_a(buf + 4 * (i + stride), v1);
    acc += (v0[0] + v0[1]) + (v0[2] + v0[3]) + (v1[0] + v1[1]) + (v1[2] + v1[3]);
  }
  for (; i < nvec; i += stride) {
    double v0[4];
    ld_a(buf + 4 * i, v0);
    acc += (v0[0] + v0[1]) + (v0[2] + v0[3]);
  }
  if (acc == 1234.5678) *out = acc;  // keeps the loads alive
}

__global__ void k_fill(double* buf, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = (double)(i & 1023);
}

// Sweep variants: (R rows per warp, U steps in flight per lane, threads per CTA).  All variants
// produce identical bits (the summation order does not depend on R, U or the grid); the default is
// chosen from measurements (profiles/), others stay selectable with JACOBI_SWEEP_VARIANT for tuning.
struct Variant {
  const char* name;
  int R, threads, cta;  // cta = 1: k_sweep_cta (needs nchunks >= threads/32 and its partial slots)
  int R32;              // rows per tile of the fp32 instance (R: fp64)
  int u64, u32;         // steps in flight (fp64 / fp32 instance): the chunk must be a multiple of 32*E*U
  void (*f64)(const SweepArgs, const int);
  void (*f32)(const SweepArgs, const int);
};
const Variant kVariants[] = {
    // item kernel (defaults below 16 column chunks: 0 for fp32 A, 1 for fp64 A)
    {"k_sweep R4 U2", 4, 512, 0, 4, 2, 1, k_sweep<double, 4, 2, 512>, k_sweep<float, 4, 1, 512>},
    {"k_sweep R8 U1", 8, 512, 0, 8, 1, 1, k_sweep<double, 8, 1, 512>, k_sweep<float, 8, 1, 512>},
    // CTA kernel with plain loads: the baselines the L2-policy (7) and dynamic (10) instances are measured against
    {"k_sweep_cta R8 U1", 8, 512, 1, 8, 1, 1, k_sweep_cta<double, 8, 16>, k_sweep_cta<float, 8, 16>},
    {"k_sweep_cta R4 U1", 4, 512, 1, 4, 1, 1, k_sweep_cta<double, 4, 16>, k_sweep_cta<float, 4, 16>},
    // fused-exchange (NEXT-1) instance of the fp64 default; selected only by jacobi_plan_ipc_attach /
    // jacobi_plan_set_p2p_emulation (it needs SweepArgs.peers).  x^(k-1) is read with weak
    // (L1-cacheable) loads, XL = 3, never ld.global.nc: peers store into it over NVLink while this
    // kernel may already be resident (spinning in sweep_prologue); the prologue's ld.acquire.sys of
    // the arrival counter plus the CTA barrier order those stores before every load of the sweep.
    // (CTA kernel R = 8 for fp64; the fp32 instances keep R = 4, R = 8 spills.)
    {"k_sweep_cta R8 U1 fused-exchange", 8, 512, 2, 4, 1, 1, k_sweep_cta<double, 8, 16, 1, 3, true, true>, k_sweep_cta<float, 4, 16, 1, 3, true>},
    // row-panel kernel (cta = 3): warps own whole rows, x chunks shared through L1 (fp32 fallback)
    {"k_sweep_panel R4 U1", 4, 512, 3, 4, 1, 1, k_sweep_panel<double, 4, 16>, k_sweep_panel<float, 4, 16>},
    // row-panel kernel with x^(k-1) staged in shared memory (8-slot chunk ring, cta = 4): fp32 default
    {"k_sweep_panel R4 U1 x-smem", 4, 512, 4, 4, 1, 1, k_sweep_panel<double, 4, 16, 1, 0, false, 8>, k_sweep_panel<float, 4, 16, 1, 0, false, 8>},
    // CTA kernel R8 with an L2 cache policy on A (evict_first, or evict_last for the kept share): fp64 default
    {"k_sweep_cta R8 U1 L2-policy", 8, 512, 1, 4, 1, 1, k_sweep_cta<double, 8, 16, 1, 0, false, true>, k_sweep_cta<float, 4, 16, 1, 0, false, true>},
    // ... with (chunk, half-tile) units: balanced when nchunks (17-31) is not a multiple of 16
    {"k_sweep_cta R8 U1 L2-policy rows/2", 8, 512, 1, 4, 1, 1, k_sweep_cta<double, 8, 16, 1, 0, false, true, 2>, k_sweep_cta<float, 4, 16, 1, 0, false, true, 2>},
    // ... with dynamic tile assignment (a launch-wide counter) instead of static row ranges
    {"k_sweep_cta R8 U1 L2-policy dynamic", 8, 512, 1, 4, 1, 1, k_sweep_cta<double, 8, 16, 1, 0, false, true, 1, true>, k_sweep_cta<float, 4, 16, 1, 0, false, true, 1, true>},
    {"k_sweep_cta R4 U2 L2-policy dynamic", 4, 512, 1, 4, 2, 2, k_sweep_cta<double, 4, 16, 2, 0, false, true, 1, true>, k_sweep_cta<float, 4, 16, 2, 0, false, true, 1, true>},
    // fused-exchange instance of 10 (large row blocks per rank, e.g. c4 at P <= 2)
    {"k_sweep_cta R4 U2 dynamic fused-exchange", 4, 512, 2, 4, 2, 2, k_sweep_cta<double, 4, 16, 2, 3, true, true, 1, true>, k_sweep_cta<float, 4, 16, 2, 3, true, true, 1, true>},
    // row-panel kernel with 4 warps per 8-row tile (cta = 6: G = 4 warps per group), x ring as 6: fp32
    // default with few rows per SM (c5 shards at P >= 2)
    {"k_sweep_group R8 G4 x-smem", 8, 512, 6, 8, 1, 1, k_sweep_group<double, 8, 16, 4, 8>, k_sweep_group<float, 8, 16, 4, 8>},
    // item kernel R4 U2 with the L2 policy on A: column slabs of fewer than 4 chunks (NEXT-4), whose
    // L2-resident share the plain item kernel cannot keep
    {"k_sweep R4 U2 L2-policy", 4, 512, 0, 4, 2, 1, k_sweep<double, 4, 2, 512, true>, k_sweep<float, 4, 1, 512, true>},
};
// Round 1 also compiled item kernels R2 U4 / R4 U1 / 256 and 1024 threads, CTA kernels R8 256t / R4 U2 /
// R2 U4 / R4 fused-exchange / R4 L2-keep / rows/4 / R4 U1 dynamic, and panel kernels x-evict_last / R8 /
// R4 U2 / L2-keep / x-smem L2-keep: all slower than the instances above on every config they were
// measured on (profiles/variants*_r01_*.jsonl, shard_variants_r02.jsonl), so they were removed.
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);

}  // namespace

unsigned long long bounds_violations(bool reset) {
#ifdef JACOBI_BOUNDS_CHECK
  unsigned long long v = 0;
  cudaMemcpyFromSymbol(&v, g_oob, sizeof(v));
  if (reset) {
    const unsigned long long z = 0;
    cudaMemcpyToSymbol(g_oob, &z, sizeof(z));
  }
  return v;
#else
  (void)reset;
  return 0;
#endif
}

int num_variants() { return kNumVariants; }
const char* variant_name(int v) { return v >= 0 && v < kNumVariants ? kVariants[v].name : nullptr; }
bool variant_is_cta(int v) { return kVariants[v].cta != 0; }
// Fused-exchange kernel for a rank's row block: the dynamic-tile instance under the same rule as
// default_variant (>= 32 four-row tiles per CTA), else the static R8 instance.
int push_variant(int dtype, int64_t rows, int num_sms) {
  return (dtype == JACOBI_F64 && num_sms > 0 && rows >= (int64_t)32 * 4 * num_sms) ? 11 : 4;
}
// Shared memory of a variant: the CTA kernel's partial slots.
size_t variant_smem(int v, int nchunks, int dtype, int chunk) {
  const Variant& V = kVariants[v];
  if (V.cta == 4) return (size_t)8 * chunk * 8;  // x ring: 8 slots of one chunk of fp64 x
  if (V.cta >= 5) {  // x ring + per group two tiles' chunk sums (cta 5 / 6 / 7: 2 / 4 / 8 warps per group)
    const int R = dtype == JACOBI_F32 ? V.R32 : V.R, groups = V.threads / (32 << (V.cta - 4));
    return (size_t)8 * chunk * 8 + (size_t)groups * 2 * R * nchunks * 8;
  }
  const int R = dtype == JACOBI_F32 ? V.R32 : V.R;
  return (V.cta == 1 || V.cta == 2) ? (size_t)kSlots * nchunks * R * 8 : 0;  // 2: fused exchange
}
bool variant_fits(int v, int nchunks, int dtype, int chunk) {
  const Variant& V = kVariants[v];
  const int step_cols = 32 * (dtype == JACOBI_F32 ? 8 : 4) * (dtype == JACOBI_F32 ? V.u32 : V.u64);
  if (chunk % step_cols != 0) return false;
  if (V.cta >= 4) return variant_smem(v, nchunks, dtype, chunk) <= 200 * 1024;
  return !V.cta || V.cta == 3 || (nchunks >= V.threads / 32 && variant_smem(v, nchunks, dtype, chunk) <= 48 * 1024);
}
bool variant_is_push(int v) { return kVariants[v].cta == 2; }
int variant_rows_dt(int v, int dtype) { return dtype == JACOBI_F32 ? kVariants[v].R32 : kVariants[v].R; }
// Defaults from B200 measurements (profiles/variants*_r01_*.jsonl; sustained = 100-sweep graph solves):
// - fp64, n with >= 16 chunks: CTA-cooperative R=8 (c4: 7316 burst / 7278 sustained GB/s vs 7274 /
//   7170 for R=4; c3: 7006 / 7115 vs 6732 / 6839; every P-way shard of c3/c4 faster too,
//   profiles/shard_rates_r01.jsonl; the panel kernel ties R=4 at c4, U=2 instances sit at the
//   128-register cap and measured lower); with an L2-resident share of A (l2_keep_pm > 0, A within
//   4x the L2) its POL instance (c2: 4976 -> 6051 effective GB/s with R=4 at 55 % kept, R=8 +2.5 %);
//   the POL instance is the default for every fp64 size: with nothing kept it loads A with
//   L2::evict_first, +0.3 % over plain loads (c4 7416 vs 7396, c3 7199 vs 7179 sustained, 3 runs);
// - fp32 A, >= 16 chunks: the row-panel kernel R=4 with x^(k-1) staged in shared memory (c5: 7103 /
//   6878; with L1-served x 6973 / 6783; the CTA kernel 6983 / 6415, which re-reads x from L2 once per
//   tile: +50 % of the A bytes with fp32 A).  For fp64 A the shared-memory ring measured 1-2.5 %
//   slower than the CTA kernel (c4 7092 / 7076, c3 6564 / 6676), so fp64 keeps the CTA kernel;
// - fewer chunks: the item kernel R=8,U=1 (fp64) or R=4,U=1 (fp32).
int default_variant(int dtype, int nchunks, int chunk, bool l2_keep, int64_t rows, int num_sms) {
  (void)l2_keep;  // every default instance with an L2 policy handles any kept share (0 included)
  // fp32 A with fewer than 512 rows per SM (c5 shards at P >= 2): the group kernel, whose 4 warps per
  // 8-row tile stream 4 chunks of each row at once (sustained 100-sweep shard times, panel / group:
  // P = 2 4909-4927 / 4866-4873 µs, P = 4 2582-2586 / 2459-2464, P = 8 1300-1302 / 1242-1244; at
  // P = 1, 885 rows per SM, 7055-7066 / 7041 GB/s, so the panel kernel stays).
  if (dtype == JACOBI_F32 && nchunks >= 16 && num_sms > 0 && rows < (int64_t)512 * num_sms &&
      variant_fits(12, nchunks, dtype, chunk))
    return 12;
  if (dtype == JACOBI_F32 && nchunks >= 16) return variant_fits(6, nchunks, dtype, chunk) ? 6 : 5;
  // Dynamic tiles of 4 rows, two column steps in flight (10) once a CTA has >= 32 such tiles: the
  // expected idle of dynamic assignment, about half a tile, then undercuts the static partition's
  // tail (a fixed minority of slower SMs).  µs per sweep, static default / 10 (R8 dynamic, 9, in
  // between): n = 20000 491 / 485, 24576 688 / 681, 32768 1186 / 1188, 49152 2667 / 2631, 65536
  // 4704 / 4668; below the threshold it loses (16384: 302 / 305; 12288: 178 / 180).
  // (its L2 keep pattern numbers the units by global tile, so it holds with dynamic tiles too)
  if (dtype == JACOBI_F64 && nchunks >= 16 && num_sms > 0 && rows >= (int64_t)32 * 4 * num_sms &&
      variant_fits(10, nchunks, dtype, chunk))
    return 10;
  // 16 < nchunks < 32, not a multiple of 16: (chunk, half-tile) units balance the 16 warps (n = 12288 /
  // 20000 / 24576: +3 / +4 / +2 %; from 40 chunks on, and for multiples of 16, whole-tile units win).
  const int big = (dtype == JACOBI_F64 && nchunks > 16 && nchunks < 32 && nchunks % 16 != 0) ? 8 : 7;
  if (variant_fits(big, nchunks, dtype, chunk)) return big;
  return dtype == JACOBI_F32 ? 0 : 1;  // item kernel: fits every chunk
}
// Column slabs (NEXT-4: all n rows, m < n columns) with fewer than 16 column chunks, where
// default_variant falls back to the item kernel: per-rank slab rates (jacobi_plan_time_shard mode 3,
// profiles/colslab_rates_r02.txt), item R8 U1 / R4 U2 / panel / group GB/s: c3 P = 2 (8 chunks) 6374 /
// 6357 / 6220 / 6683, P = 4 (4) 5989 / 6148 / 6228 / 6345, P = 8 (2) 5152 / 5594 / 5536 / 4631; c4 P = 8 (8)
// 6833 / 6674 / 6998 / 7072; c5 P = 8 (8, fp32) 6233 / 6605 / 6942 / 7052.  The group kernel from 4
// chunks up; below, the item kernel R4 U2 with the L2 policy (variant 13), which keeps the slab's
// L2-resident share (c3 P = 8: 47.5 -> 40.0 us).  (A group instance with the L2 policy measured c3 P = 2
// +2.3 %, P = 4 -0.2 %, c4 P = 8 -2.1 %: not kept.)
int slab_variant(int dtype, int nchunks, int chunk, int fallback) {
  if (nchunks >= 16) return fallback;
  if (nchunks >= 4 && variant_fits(12, nchunks, dtype, chunk)) return 12;
  if (variant_fits(13, nchunks, dtype, chunk)) return 13;
  return fallback;
}
int variant_rows(int v) { return kVariants[v].R; }
int variant_threads(int v) { return kVariants[v].threads; }

#ifdef JACOBI_SM_TIMING
extern "C" int jacobi_debug_sm_times(unsigned long long* out, int nctas) {
  return cudaMemcpyFromSymbol(out, g_smt, sizeof(unsigned long long) * 3 * (size_t)nctas) == cudaSuccess ? 0 : -5;
}
extern "C" int jacobi_debug_set_rotation(int rot) {
  return cudaMemcpyToSymbol(g_rot, &rot, sizeof(rot)) == cudaSuccess ? 0 : -5;
}
#endif

int chunk_for(int64_t n, int dtype) {
  // 8 KB of row data per chunk (1024 fp64 / 2048 fp32 columns) when n has >= 16 such chunks, halved
  // down to 256 columns otherwise (c2, n = 4096: 16 chunks of 256).  A function of (n, dtype) only,
  // so every rank count and every kernel variant sums each row in the same order.
  int c = dtype == JACOBI_F32 ? 2048 : 1024;
  while (c > 256 && (int64_t)c * 16 > n) c /= 2;
  return c;
}

int sweep_grid(int dtype, int v, int num_sms, int nchunks, int chunk) {
  int per_sm = 0;
  const Variant& V = kVariants[v];
  const size_t smem = variant_smem(v, nchunks, dtype, chunk);
  auto fn = dtype == JACOBI_F32 ? V.f32 : V.f64;
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, V.threads, smem);
  if (e != cudaSuccess || per_sm < 1) per_sm = 1;
  return num_sms * per_sm;
}

cudaError_t launch_sweep(int dtype, int v, const SweepArgs& a, int j, int grid, cudaStream_t s) {
  const Variant& V = kVariants[v];
  const size_t smem = variant_smem(v, a.nchunks, dtype, a.chunk);
  if (dtype == JACOBI_F32) V.f32<<<grid, V.threads, smem, s>>>(a, j);
  else V.f64<<<grid, V.threads, smem, s>>>(a, j);
  return cudaGetLastError();
}

// Persistent grid solver (k_solve_gridsync): one CTA per SM, co-resident (cooperative launch).
// Instance with (chunk, row-group) units for A with few chunks: measured per sweep (fp64, 400-sweep
// solves, GR = 1 / 2 / 4): n = 1024 (4 chunks) 4.83 / 4.27 / 4.25 µs; 1536 (6) 7.10 / 6.11 / 7.09;
// 2048 (8) 7.38 / 6.64 / 7.38; 2560 (10) 10.23 / 10.93 / 11.72; 3072 (12) 10.91 / 11.75 / 11.87;
// 3584 (14) 16.6 / 18.0 / 23.2 — half-tile units pay off up to 8 chunks only.
static int gridsync_gr(int dtype, int nchunks) {
  if (const char* e = getenv("JACOBI_GRID_GR")) {  // tuning override: 1, 2, 4 (, 8 fp64)
    const int g = atoi(e);
    if (g == 1 || g == 2 || g == 4 || (g == 8 && dtype != JACOBI_F32)) return g;
  }
  return nchunks <= 8 ? 2 : 1;
}
// Rows per tile: 8 for fp64; for fp32 8 with few chunks (the half-tile units of 4 rows: 400-sweep
// solves, R = 4 / 8: n = 1024 5.20 / 4.73 µs, 2048 7.96 / 6.61) and 4 beyond (the R = 8 one-chunk
// units spill: 4096 14.4 / 17.1, 8192 47.5 / 59.9).  JACOBI_GRID_R = 4 | 8 overrides.
static int gridsync_r(int dtype, int nchunks) {
  if (dtype != JACOBI_F32) return 8;
  if (gridsync_gr(dtype, nchunks) == 1) return 4;  // no fp32 R = 8 one-chunk-unit instance (it spills)
  if (const char* e = getenv("JACOBI_GRID_R")) return atoi(e) == 8 ? 8 : 4;
  return 8;
}
static const void* gridsync_fn(int dtype, int nchunks) {
  const int gr = gridsync_gr(dtype, nchunks);
  if (dtype == JACOBI_F32 && gridsync_r(dtype, nchunks) == 8) {
    switch (gr) {
      case 2: return (const void*)k_solve_gridsync<float, 8, 16, true, 2>;
      default: return (const void*)k_solve_gridsync<float, 8, 16, true, 4>;
    }
  }
  if (dtype == JACOBI_F32) {
    switch (gr) {
      case 1: return (const void*)k_solve_gridsync<float, 4, 16, true, 1>;
      case 2: return (const void*)k_solve_gridsync<float, 4, 16, true, 2>;
      default: return (const void*)k_solve_gridsync<float, 4, 16, true, 4>;
    }
  }
  switch (gr) {
    case 1: return (const void*)k_solve_gridsync<double, 8, 16, true, 1>;
    case 2: return (const void*)k_solve_gridsync<double, 8, 16, true, 2>;
    case 4: return (const void*)k_solve_gridsync<double, 8, 16, true, 4>;
    default: return (const void*)k_solve_gridsync<double, 8, 16, true, 8>;
  }
}

int gridsync_plan(int dtype, int nchunks, int num_sms, size_t* smem) {
  const int R = gridsync_r(dtype, nchunks);
  *smem = (size_t)kSlots * nchunks * R * 8;
  if (*smem > 200 * 1024) return 0;
  const void* fn = gridsync_fn(dtype, nchunks);
  if (*smem > 48 * 1024 && cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem) != cudaSuccess)
    return 0;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 512, *smem) != cudaSuccess || per_sm < 1) return 0;
  return num_sms;
}

cudaError_t launch_solve_gridsync(int dtype, const SweepArgs& a, unsigned long long* gbar, int64_t k0, int64_t k1,
                                  int grid, size_t smem, cudaStream_t s) {
  SweepArgs aa = a;
  void* args[] = {&aa, &gbar, &k0, &k1};
  return cudaLaunchCooperativeKernel(gridsync_fn(dtype, a.nchunks), dim3(grid), dim3(512), args, smem, s);
}

int gridsync_push_plan(int dtype, int nchunks, int num_sms, size_t* smem) {
  const int R = dtype == JACOBI_F32 ? 4 : 8;
  *smem = (size_t)kSlots * nchunks * R * 8;
  if (*smem > 200 * 1024) return 0;
  auto fn = dtype == JACOBI_F32 ? k_solve_gridsync_push<float, 4, 16> : k_solve_gridsync_push<double, 8, 16>;
  if (*smem > 48 * 1024 && cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem) != cudaSuccess)
    return 0;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 512, *smem) != cudaSuccess || per_sm < 1) return 0;
  return num_sms;
}

cudaError_t launch_solve_gridsync_push(int dtype, const SweepArgs* ranks_dev, int nvr, int64_t k0, int64_t k1,
                                       int grid, size_t smem, cudaStream_t s) {
  void* args[] = {&ranks_dev, &nvr, &k0, &k1};
  const void* fn = dtype == JACOBI_F32 ? (const void*)k_solve_gridsync_push<float, 4, 16>
                                       : (const void*)k_solve_gridsync_push<double, 8, 16>;
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(512), args, smem, s);
}

cudaError_t launch_l2_partials(const double* sq, int64_t m, double* blk, const State* st, cudaStream_t s) {
  k_l2_partials<<<(unsigned)((m + kL2Block - 1) / kL2Block), kL2Block, 0, s>>>(sq, m, blk, st);
  return cudaGetLastError();
}

cudaError_t launch_l2_final(const double* blk, int64_t nblk, unsigned long long* dslot, State* st, int j,
                            cudaStream_t s) {
  k_l2_final<<<1, 32, 0, s>>>(blk, nblk, dslot, st, j);
  return cudaGetLastError();
}

cudaError_t launch_colsum_epilogue(const double* rsum, int nb, int64_t stride, int64_t rows, int64_t row0,
                                   const double* b, const double* diag, double* x0buf, double* x1buf,
                                   unsigned long long* dslot, double* sq, int norm, State* st, int j,
                                   cudaStream_t s) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((rows + 255) / 256, 592));
  k_colsum_epilogue<<<grid, 256, 0, s>>>(rsum, nb, stride, rows, row0, b, diag, x0buf, x1buf, dslot, sq, norm, st, j);
  return cudaGetLastError();
}

cudaError_t launch_advance(State* st, unsigned long long* dslot, int K, cudaStream_t s) {
  k_advance<<<1, 1, 0, s>>>(st, dslot, K);
  return cudaGetLastError();
}

cudaError_t launch_advance_while(State* st, unsigned long long* dslot, int K, cudaGraphConditionalHandle h,
                                 cudaStream_t s) {
  k_advance_while<<<1, 1, 0, s>>>(st, dslot, K, h);
  return cudaGetLastError();
}

cudaError_t launch_setup_diag(int dtype, const void* A, int64_t lda, int64_t m, int64_t row0, double* diag,
                              unsigned long long* zero_min, cudaStream_t s) {
  const int grid = (int)std::min<int64_t>((m + 255) / 256, 4096);
  if (dtype == JACOBI_F32) k_setup_diag<float><<<grid, 256, 0, s>>>((const float*)A, lda, m, row0, diag, zero_min);
  else k_setup_diag<double><<<grid, 256, 0, s>>>((const double*)A, lda, m, row0, diag, zero_min);
  return cudaGetLastError();
}

cudaError_t launch_scan_nonfinite_A(int dtype, const void* A, int64_t lda, int64_t m, int64_t n, int* flag,
                                    cudaStream_t s) {
  const int grid = (int)std::min<int64_t>((m + 7) / 8, 148 * 16);
  if (dtype == JACOBI_F32) k_scan_A<float><<<grid, 256, 0, s>>>((const float*)A, lda, m, n, flag);
  else k_scan_A<double><<<grid, 256, 0, s>>>((const double*)A, lda, m, n, flag);
  return cudaGetLastError();
}

cudaError_t launch_prepare(State* st, int64_t max_iter, double tol, double* hist, unsigned long long* dslot,
                           unsigned* cnt, int64_t ncnt, double* b, const double* b_src, int64_t m, double* x0,
                           const double* x0_src, int64_t n, unsigned long long* flags, unsigned long long* gbar,
                           cudaStream_t s) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((std::max(n, ncnt) + 255) / 256, 592));
  k_prepare<<<grid, 256, 0, s>>>(st, max_iter, tol, hist, dslot, cnt, ncnt, b, b_src, m, x0, x0_src, n, flags, gbar);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const State* st, const double* x0buf, const double* x1buf, double* dst, int64_t n,
                            cudaStream_t s) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 592));
  k_finalize<<<grid, 256, 0, s>>>(st, x0buf, x1buf, dst, n);
  return cudaGetLastError();
}

cudaError_t launch_copy_pitched(int dtype, const void* src, int64_t sld, void* dst, int64_t dld, int64_t rows,
                                int64_t n, cudaStream_t s) {
  dim3 grid((unsigned)std::min<int64_t>((dld + 255) / 256, 64), (unsigned)std::min<int64_t>(rows, 65535));
  if (dtype == JACOBI_F32) k_copy_pitched<float><<<grid, 256, 0, s>>>((const float*)src, sld, (float*)dst, dld, rows, n);
  else k_copy_pitched<double><<<grid, 256, 0, s>>>((const double*)src, sld, (double*)dst, dld, rows, n);
  return cudaGetLastError();
}

double bwprobe(int64_t nbytes, int reps) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* buf = nullptr;
  double* out = nullptr;
  if (cudaMalloc(&buf, nbytes) != cudaSuccess) return -1.0;
  if (cudaMalloc(&out, 8) != cudaSuccess) { cudaFree(buf); return -1.0; }
  const int64_t n = nbytes / 8, nvec = n / 4;
  k_fill<<<sms * 8, 256>>>(buf, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < reps + 1; ++r) {
    cudaEventRecord(e0);
    k_probe<<<sms * 2, 1024>>>(buf, nvec, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;  // first pass is a warm-up
  }
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  cudaFree(out);
  if (err != cudaSuccess) return -1.0;
  return (double)(nvec * 32) / (best * 1e-3) / 1e9;
}

}  // namespace jacobi
