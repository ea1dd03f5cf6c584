// tma_warp_probe.cu — can 1D bulk copies (cp.async.bulk, TMA) feed a row-panel sweep at the HBM
// read ceiling?  Pattern of k_sweep_panel at c5: rows of 512 KB (131072 fp32), each warp streams
// tiles of 4 rows along the columns.  Mode "tma": every warp is its own producer and consumer — lane
// 0 issues one bulk copy per row segment (B bytes) into the warp's S-slot shared-memory ring, the warp
// waits on the slot's mbarrier, reads the slot with 16-byte shared loads and re-issues it.  Mode
// "ldg": the same tiles with 256-bit LDG (8 floats per lane per row per step, as the panel kernel).
// Prints GB/s (CUDA events, best of 4).  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int64_t kRowBytes = 512 * 1024;
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512, 1) k_tma(const char* A, int64_t nrows, int B, int S, float* out) {
  extern __shared__ __align__(128) char ring[];  // [NW][S][4][B]
  __shared__ __align__(8) uint64_t full[16 * 16];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
  uint64_t* fb = full + w * 16;
  char* my = ring + (size_t)w * S * 4 * B;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&fb[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t ntiles = nrows / 4, gw = blockIdx.x * (int64_t)NW + w, nw = (int64_t)gridDim.x * NW;
  const int64_t segs = kRowBytes / B;
  float acc = 0.f;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  // flattened item stream of this warp: (tile, seg)
  const int64_t mytiles = gw < ntiles ? (ntiles - gw + nw - 1) / nw : 0;
  const int64_t items = mytiles * segs;
  auto issue = [&](int64_t it) {
    if (it >= items) return;
    const int s = (int)(it % S);
    const int64_t tile = gw + (it / segs) * nw, seg = it % segs;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&fb[s])), "r"(4 * B) : "memory");
    for (int r = 0; r < 4; ++r) {
      const char* src = A + (tile * 4 + r) * kRowBytes + seg * B;
      char* dst = my + ((size_t)s * 4 + r) * B;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                   ::"r"(sa(dst)), "l"(src), "r"(B), "r"(sa(&fb[s])), "l"(pol) : "memory");
    }
  };
  if (lane == 0)
    for (int64_t i = 0; i < S; ++i) issue(i);
  for (int64_t it = 0; it < items; ++it) {
    const int s = (int)(it % S);
    const unsigned par = (unsigned)((it / S) & 1);
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 ::"r"(sa(&fb[s])), "r"(par) : "memory");
    const float4* p = (const float4*)(my + (size_t)s * 4 * B);
    for (int q = lane; q < B / 4; q += 32) {  // 4 rows x B bytes as float4
      const float4 v = p[q];
      acc += v.x + v.y + v.z + v.w;
    }
    __syncwarp();
    if (lane == 0) issue(it + S);
  }
  if (acc == 1234.5f) out[0] = acc;
}

// G warps share each 4-row tile: warp q of the group streams chunks q, q + G, ... (chunk = 2048 fp32 =
// 8 KB per row, 8 steps of 256 columns), so a group reads G x 8 KB of every row at once.
template <int G>
__global__ void __launch_bounds__(512, 1) k_ldg(const float* A, int64_t nrows, float* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const int q = w % G, grp = w / G, ngrp = NW / G;
  const int64_t ntiles = nrows / 4, gg = blockIdx.x * (int64_t)ngrp + grp, ng = (int64_t)gridDim.x * ngrp;
  const int64_t cols = kRowBytes / 4, nch = cols / 2048;
  float acc = 0.f;
  for (int64_t t = gg; t < ntiles; t += ng) {
    for (int64_t ch = q; ch < nch; ch += G) {
      for (int64_t c = ch * 2048 + lane * 8; c < (ch + 1) * 2048; c += 256) {
        float v[4][8];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float* p = A + (t * 4 + r) * cols + c;
          asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=f"(v[r][0]), "=f"(v[r][1]), "=f"(v[r][2]), "=f"(v[r][3]), "=f"(v[r][4]), "=f"(v[r][5]),
                         "=f"(v[r][6]), "=f"(v[r][7])
                       : "l"(p));
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int e = 0; e < 8; ++e) acc += v[r][e];
      }
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t nrows = argc > 1 ? atoll(argv[1]) : 32768;  // 16 GiB
  const size_t total = (size_t)nrows * kRowBytes;
  char* A;
  float* out;
  CK(cudaMalloc(&A, total));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(A, 0, total));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](auto launch) {
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r && ms < best) best = ms;
    }
    CK(cudaGetLastError());
    return total / (best * 1e-3) / 1e9;
  };
  printf("{\"mode\": \"ldg\", \"warps_per_tile\": 1, \"gbs\": %.1f}\n", timeit([&] { k_ldg<1><<<sms, 512>>>((const float*)A, nrows, out); }));
  printf("{\"mode\": \"ldg\", \"warps_per_tile\": 2, \"gbs\": %.1f}\n", timeit([&] { k_ldg<2><<<sms, 512>>>((const float*)A, nrows, out); }));
  printf("{\"mode\": \"ldg\", \"warps_per_tile\": 4, \"gbs\": %.1f}\n", timeit([&] { k_ldg<4><<<sms, 512>>>((const float*)A, nrows, out); }));
  printf("{\"mode\": \"ldg\", \"warps_per_tile\": 8, \"gbs\": %.1f}\n", timeit([&] { k_ldg<8><<<sms, 512>>>((const float*)A, nrows, out); }));
  printf("{\"mode\": \"ldg\", \"warps_per_tile\": 16, \"gbs\": %.1f}\n", timeit([&] { k_ldg<16><<<sms, 512>>>((const float*)A, nrows, out); }));
  struct C { int nw, B, S; } cs[] = {{16, 512, 6}, {16, 1024, 3}, {16, 512, 4}, {16, 1024, 2}, {16, 256, 12},
                                     {8, 1024, 6}, {8, 2048, 3}, {4, 2048, 6}, {4, 4096, 3}, {16, 2048, 1}};
  for (auto c : cs) {
    const size_t smem = (size_t)c.nw * c.S * 4 * c.B;
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const double g = timeit([&] { k_tma<<<sms, c.nw * 32, smem>>>(A, nrows, c.B, c.S, out); });
    printf("{\"mode\": \"tma\", \"warps\": %d, \"seg_bytes\": %d, \"slots\": %d, \"in_flight_kb_per_sm\": %zu, \"gbs\": %.1f}\n",
           c.nw, c.B, c.S, smem / 1024, g);
  }
  return 0;
}
