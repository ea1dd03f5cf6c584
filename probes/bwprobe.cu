// Read-only HBM ceiling probe (SURVEY.md §2.2 "k_bwprobe", finding F6).
// Standalone executable: streams a >= 32 GiB buffer with several load flavours
// and reports GB/s (CUDA events, best of R). Used to pick the sweep kernel's
// load strategy and to give the roofline a read-only denominator.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void ld128(const void* p, double& a, double& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
}
__device__ __forceinline__ void ld128ef(const void* p, double& a, double& b, uint64_t pol) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(a), "=d"(b) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld256(const void* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

// mode 0: 128-bit nc no_allocate; 1: + L2 evict_first policy; 2: 256-bit
template <int U, int MODE>
__global__ void k_read(const double* __restrict__ buf, size_t nelem, double* out, int reps = 1) {
  uint64_t pol = 0;
  if (MODE == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int V = (MODE == 2) ? 4 : 2;
  size_t nvec = nelem / V;
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (int rep = 0; rep < reps; ++rep) {  // several passes in one launch (L2-resident buffers)
  size_t i = tid;
  for (; i + (U - 1) * stride < nvec; i += U * stride) {
    double v[U][V];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double* p = buf + (i + u * stride) * V;
      if (MODE == 0) ld128(p, v[u][0], v[u][1]);
      else if (MODE == 1) ld128ef(p, v[u][0], v[u][1], pol);
      else ld256(p, v[u][0], v[u][1], v[u][2], v[u][3]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < V; ++q) acc += v[u][q];
  }
  for (; i < nvec; i += stride) {
    double a, b;
    ld128(buf + i * V, a, b);
    acc += a + b;
  }
  }
  if (acc == 12345.678) out[0] = acc;  // keep loads alive
}

// Mixed L2 policy (the persistent solver's traffic without its arithmetic, barriers or stop test):
// 8 KB unit u is loaded with L2 evict_last iff frac(u * phi) < keep / 1000 (the solver's Weyl keep
// rule), else evict_first; 256-bit no-L1 loads, U in flight per thread, `reps` passes per launch.
__device__ __forceinline__ void ld256p(const void* p, double& a, double& b, double& c, double& d, uint64_t pol) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p), "l"(pol));
}
template <int U>
__global__ void k_read_keep(const double* __restrict__ buf, size_t nelem, double* out, int reps, unsigned thr) {
  uint64_t pk, ps;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pk));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(ps));
  const size_t nvec = nelem / 4;
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (int rep = 0; rep < reps; ++rep) {
    for (size_t i = tid; i + (U - 1) * stride < nvec; i += U * stride) {
      double v[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t j = i + u * stride;
        const unsigned unit = (unsigned)(j >> 8);  // 256 vectors of 32 B = 8 KB
        ld256p(buf + j * 4, v[u][0], v[u][1], v[u][2], v[u][3], unit * 2654435769u < thr ? pk : ps);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc += (v[u][0] + v[u][1]) + (v[u][2] + v[u][3]);
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void k_fill(double* buf, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) buf[i] = (double)(i & 1023) * 1e-3;
}

__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[i];
}

// cp.async.bulk ring: one CTA per SM, S stages of CH bytes, one producer thread.
template <int S, int CH>
__global__ void __launch_bounds__(256) k_bulk(const char* __restrict__ buf, size_t nbytes, double* out, int reps = 1) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[S], empty_[S];
  const int nwarps = blockDim.x / 32;
  const size_t nreal = nbytes / CH;
  size_t nchunks = nreal * reps;  // virtual chunk c reads chunk c % nreal
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&full[s]);
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(a));
      a = (uint32_t)__cvta_generic_to_shared(&empty_[s]);
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(a), "r"(nwarps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  double acc = 0.0;
  int it = 0;
  // producer: thread 0 issues; all warps consume
  size_t first = blockIdx.x;
  size_t step = gridDim.x;
  // prologue
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      size_t c = first + s * step;
      if (c >= nchunks) break;
      uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[s]);
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem + s * CH);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(fb), "r"(CH));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(dst), "l"(buf + (c % nreal) * CH), "r"(CH), "r"(fb) : "memory");
    }
  }
  for (size_t c = first; c < nchunks; c += step, ++it) {
    int s = it % S;
    uint32_t ph = (it / S) & 1;
    uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[s]);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" :: "r"(fb), "r"(ph));
    const double2* t = (const double2*)(smem + s * CH);
    for (int q = threadIdx.x; q < CH / 16; q += blockDim.x) { double2 v = t[q]; acc += v.x + v.y; }
    __syncwarp();
    uint32_t eb = (uint32_t)__cvta_generic_to_shared(&empty_[s]);
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" :: "r"(eb));
    if (threadIdx.x == 0) {
      size_t cn = c + S * step;
      if (cn < nchunks) {
        asm volatile("{ .reg .pred p; W2: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W2; }" :: "r"(eb), "r"(ph));
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem + s * CH);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(fb), "r"(CH));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(dst), "l"(buf + (cn % nreal) * CH), "r"(CH), "r"(fb) : "memory");
      }
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

template <typename F>
static double time_best(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

int main(int argc, char** argv) {
  size_t gib = argc > 1 ? atoll(argv[1]) : 32;
  // "probes/bwprobe N mib": an N MiB buffer — L2-resident after the first pass when N is below ~100,
  // i.e. the L2-hit streaming rate of the same load flavours
  const bool mib = argc > 2 && argv[2][0] == 'm';
  size_t nbytes = mib ? gib << 20 : gib << 30, n = nbytes / 8;
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  int bus, memclk, l2;
  CK(cudaDeviceGetAttribute(&bus, cudaDevAttrGlobalMemoryBusWidth, 0));
  CK(cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, 0));
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  printf("{\"probe\":\"attrs\",\"sms\":%d,\"bus_bits\":%d,\"memclk_khz\":%d,\"l2_bytes\":%d,\"theoretical_gbs\":%.1f}\n",
         nsm, bus, memclk, l2, 2.0 * memclk * 1e3 * bus / 8 / 1e9);
  double* buf; CK(cudaMalloc(&buf, nbytes));
  double* out; CK(cudaMalloc(&out, 8));
  k_fill<<<nsm * 8, 512>>>(buf, n); CK(cudaDeviceSynchronize());
  auto rep = [&](const char* name, int tpb, int bps, double ms, double bytes) {
    printf("{\"probe\":\"%s\",\"tpb\":%d,\"blocks_per_sm\":%d,\"ms\":%.3f,\"gbs\":%.1f}\n", name, tpb, bps, ms, bytes / ms / 1e6);
    fflush(stdout);
  };
  const int passes = mib ? 20 : 1;  // small buffers: 20 passes per launch so the launch does not dominate
  if (argc > 4 && argv[3][0] == 'k') {  // "probes/bwprobe N mib keep P": mixed-policy streaming only
    const int keep = atoi(argv[4]);
    const unsigned thr = keep >= 1000 ? 0xffffffffu : (unsigned)(((unsigned long long)keep << 32) / 1000ull);
#define RUNK(U, TPB, BPS) { double ms = time_best([&]{ k_read_keep<U><<<nsm * BPS, TPB>>>(buf, n, out, passes, thr); }, 5); \
    char nm[64]; snprintf(nm, 64, "keep%d_u%d", keep, U); rep(nm, TPB, BPS, ms, (double)nbytes * passes); }
    RUNK(8, 512, 1); RUNK(4, 1024, 1); RUNK(16, 512, 1); RUNK(8, 256, 4); RUNK(4, 512, 4);  // 128/128/256/256/256 KB in flight per SM
    return 0;
  }
#define RUN(U, MODE, TPB, BPS) { double ms = time_best([&]{ k_read<U, MODE><<<nsm * BPS, TPB>>>(buf, n, out, passes); }, 5); \
    char nm[64]; snprintf(nm, 64, "read_m%d_u%d", MODE, U); rep(nm, TPB, BPS, ms, (double)nbytes * passes); }
  RUN(4, 0, 256, 8); RUN(8, 0, 256, 8); RUN(16, 0, 256, 4); RUN(8, 0, 512, 4); RUN(8, 0, 1024, 2);
  RUN(4, 0, 512, 4); RUN(2, 0, 1024, 2);
  RUN(8, 1, 256, 8); RUN(16, 1, 256, 4);
  RUN(4, 2, 256, 8); RUN(8, 2, 256, 4); RUN(4, 2, 512, 4);
  {
    size_t half = nbytes / 2 / 16;
    double ms = time_best([&]{ k_copy<<<nsm * 8, 256>>>((const double2*)buf, (double2*)((char*)buf + nbytes / 2), half); }, 5);
    rep("copy_rw", 256, 8, ms, (double)nbytes);
  }
#define RUNB(S, CH) { auto kf = k_bulk<S, CH>; CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, S * CH)); \
    double ms = time_best([&]{ kf<<<nsm, 256, S * CH>>>((const char*)buf, nbytes, out, passes); }, 5); \
    char nm[64]; snprintf(nm, 64, "bulk_s%d_ch%d", S, CH); rep(nm, 256, 1, ms, (double)nbytes * passes); }
  RUNB(4, 32768); RUNB(6, 32768); RUNB(8, 16384); RUNB(12, 16384); RUNB(3, 65536);
  return 0;
}
