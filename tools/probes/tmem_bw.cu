// Probe: tcgen05.ld / tcgen05.st throughput per SM (bytes per cycle) vs warps.
#include <cstdio>
#include "../../paper_2505_14708_b200/csrc/common.cuh"

using namespace da;

template <bool STORE>
__global__ void tmem_bw(int reps, long long* out, float* sink) {
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t col = (uint32_t)((warp >> 2) * 64) & 511;
  float acc = 0.f;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = (float)i;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (STORE) {
      tmem_st32(tmem_base + lane_off + col, v);
      tmem_st32(tmem_base + lane_off + col + 32, v);
      tmem_st_wait();
    } else {
      float a[32], b[32];
      tmem_ld32(tmem_base + lane_off + col, a);
      tmem_ld32(tmem_base + lane_off + col + 32, b);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += a[i] + b[i];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 12345.f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem_base);
  }
}

int main() {
  long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 8);
  cudaMalloc(&sink, 4);
  const int reps = 4000;
  for (int store = 0; store < 2; ++store) {
    for (int warps : {4, 8, 16}) {
      if (store) tmem_bw<true><<<148, warps * 32>>>(reps, d_out, sink);
      else tmem_bw<false><<<148, warps * 32>>>(reps, d_out, sink);
      cudaDeviceSynchronize();
      long long cyc = 0;
      cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)warps * reps * 2 * 32 * 32 * 4;
      printf("%s warps=%2d: %7.1f B/clk/SM (%lld cycles) %s\n", store ? "tcgen05.st" : "tcgen05.ld", warps,
             bytes / cyc, cyc, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
