// tma_probe.cu — throughput of cp.async.bulk (1D TMA) streaming into a shared-memory ring.
// One producer lane per CTA issues `copies_per_stage` bulk copies of `bytes` each per stage into a
// ring of `stages` slots; 16 consumer warps wait for a stage (mbarrier), optionally touch it, and
// release it.  Prints GB/s for each configuration.  Build: make tma_probe; run: probes/tma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool test(uint64_t* b, unsigned par) {
  unsigned ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
               : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
  return ok;
}

template <int HINT>
__global__ void __launch_bounds__(544, 1) k(const char* src, size_t total, int bytes, int cps, int stages, double* out) {
  extern __shared__ __align__(128) char ring[];
  __shared__ __align__(8) uint64_t full[32], empty[32];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t stage_bytes = (size_t)bytes * cps;
  const size_t per_cta = total / gridDim.x / stage_bytes * stage_bytes;
  const char* base = src + per_cta * blockIdx.x;
  const long long nst = per_cta / stage_bytes;
  if (w == 16) {
    if (lane) return;
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (long long g = 0; g < nst; ++g) {
      const int s = (int)(g % stages);
      if (g >= stages) {
        long long it = 0;
        while (!test(&empty[s], (unsigned)(((g / stages) - 1) & 1)))
          if (++it > (1ll << 24)) { *out = -1.0; return; }
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"((unsigned)stage_bytes));
      for (int c = 0; c < cps; ++c) {
        const char* p = base + g * stage_bytes + (size_t)c * bytes;
        char* d = ring + (size_t)s * stage_bytes + (size_t)c * bytes;
        if (HINT)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                       ::"r"(sa(d)), "l"(p), "r"(bytes), "r"(sa(&full[s])), "l"(pol) : "memory");
        else
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(sa(d)), "l"(p), "r"(bytes), "r"(sa(&full[s])) : "memory");
      }
    }
    return;
  }
  double acc = 0;
  for (long long g = w; g < nst; g += 16) {
    const int s = (int)(g % stages);
    long long it = 0;
    while (!test(&full[s], (unsigned)((g / stages) & 1)))
      if (++it > (1ll << 24)) { *out = -2.0; return; }
    acc += ((const double*)(ring + (size_t)s * stage_bytes))[lane];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
  }
  if (acc == 12345.0) *out = acc;
}

int main() {
  const size_t total = 4ull << 30;
  char* src;
  double* out;
  cudaMalloc(&src, total);
  cudaMalloc(&out, 8);
  cudaMemset(src, 1, total);
  cudaMemset(out, 0, 8);
  setvbuf(stdout, nullptr, _IONBF, 0);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct C { int bytes, cps, stages, hint; } cs[] = {
      {2048, 4, 24, 1}, {2048, 4, 24, 0}, {2048, 1, 24, 0}, {8192, 1, 24, 0}, {8192, 1, 12, 0},
      {16384, 1, 12, 0}, {32768, 1, 6, 0}, {4096, 2, 24, 0}, {1024, 8, 24, 0}, {2048, 4, 12, 0}};
  for (auto c : cs) {
    const size_t smem = (size_t)c.bytes * c.cps * c.stages;
    auto fn = c.hint ? k<1> : k<0>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0);
      fn<<<sms, 544, smem>>>(src, total, c.bytes, c.cps, c.stages, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"bytes\": %d, \"copies_per_stage\": %d, \"stages\": %d, \"hint\": %d, \"in_flight_kb\": %zu, \"gbs\": %.1f, \"err\": \"%s\"}\n",
           c.bytes, c.cps, c.stages, c.hint, smem / 1024, total / (best * 1e-3) / 1e9, cudaGetErrorString(e));
    double o = 0;
    cudaMemcpy(&o, out, 8, cudaMemcpyDeviceToHost);
    if (o < 0) printf("  (a wait gave up: %g)\n", o);
    fflush(stdout);
  }
  return 0;
}
