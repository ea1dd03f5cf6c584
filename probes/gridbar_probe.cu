// gridbar_probe.cu — cost of one grid-wide barrier on B200 (148 co-resident CTAs x 512 threads),
// the floor of the persistent grid solver's sweep.  Variants:
//   0: atomicAdd on one counter + ld.acquire.gpu spin by thread 0 (the solver's barrier)
//   1: red.release.gpu.global.add + ld.acquire.gpu spin
//   2: cooperative_groups::this_grid().sync()
//   3: variant 0 plus a dependent L2 read after the barrier (the solver's stop-test read)
//   4: two-level: 8 group counters, each group's last arriver adds to a top counter that all poll
//   5: per-CTA epoch flags (st.release), warp 0 of every CTA polls all flags (ld.acquire) with a vote
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o probes/gridbar_probe probes/gridbar_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int V>
__global__ void __launch_bounds__(512, 1) k(unsigned long long* ctr, double* slot, int iters, double* out) {
  double acc = 0.0;
  for (int it = 1; it <= iters; ++it) {
    if constexpr (V == 2) {
      cg::this_grid().sync();
    } else if constexpr (V == 4) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned G = gridDim.x, grp = blockIdx.x & 7u;
        const unsigned gsize = G / 8u + (grp < (G & 7u) ? 1u : 0u);
        __threadfence();
        const unsigned long long old = atomicAdd(ctr + 16 + 16 * grp, 1ull);
        if (old == (unsigned long long)gsize * it - 1ull) atomicAdd(ctr, 1ull);
        const unsigned long long target = 8ull * it;
        while (ld_acq(ctr) < target) {
        }
      }
      __syncthreads();
    } else if constexpr (V == 5) {
      __syncthreads();
      if (threadIdx.x < 32) {
        if (threadIdx.x == 0) {
          __threadfence();
          st_rel(ctr + 256 + blockIdx.x, (unsigned long long)it);
        }
        bool done = false;
        while (!done) {
          bool mine = true;
          for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) mine &= ld_acq(ctr + 256 + b) >= (unsigned long long)it;
          done = __all_sync(0xffffffffu, mine);
        }
      }
      __syncthreads();
    } else {
      __syncthreads();
      if (threadIdx.x == 0) {
        if constexpr (V == 1) {
          asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        } else {
          __threadfence();
          atomicAdd(ctr, 1ull);
        }
        const unsigned long long target = (unsigned long long)gridDim.x * it;
        while (ld_acq(ctr) < target) {
        }
        if constexpr (V == 3) acc += *(volatile double*)slot;
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0 && acc == 1234.5) *out = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* ctr;
  double *slot, *out;
  cudaMalloc(&ctr, 8 * 1024);
  cudaMalloc(&slot, 8);
  cudaMalloc(&out, 8);
  const int iters = 20000;
  void (*fns[])(unsigned long long*, double*, int, double*) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>};
  for (int v = 0; v < 6; ++v) {
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaMemset(ctr, 0, 8 * 1024);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      int it = iters;
      void* args[] = {&ctr, &slot, &it, &out};
      cudaEventRecord(e0);
      cudaError_t e = cudaLaunchCooperativeKernel((const void*)fns[v], dim3(sms), dim3(512), args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (e != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(e));
      if (ms < best) best = ms;
    }
    printf("{\"variant\": %d, \"ctas\": %d, \"us_per_barrier\": %.3f}\n", v, sms, 1e3 * best / iters);
  }
  return 0;
}
