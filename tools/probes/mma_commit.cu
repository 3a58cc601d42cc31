// Probe: cost of tcgen05.commit between groups of tcgen05.mma (TS, kind::f16).
// One thread issues R groups of 8 MMAs; after each group it commits to C
// distinct mbarriers (nobody waits on them). Cycles per group vs C and N.
#include <cstdio>
#include "../../paper_2505_14708_b200/csrc/common.cuh"

using namespace da;

template <int N, int C, int MODE>
__global__ void __launch_bounds__(128, 1) commit_rate(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t bar[8];
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t IDESC = umma_idesc_bf16(128, N, 0, 0);
    const uint32_t b = smem_u32(smem);
    const uint64_t db = umma_desc_sw128(b, 16, 1024);
    long long issue = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      long long a0 = clock64();
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t bo = (uint64_t)((k >> 2) * (16384 >> 4) + (k & 3) * 2);
        umma_bf16_ts(tmem_base + 256, tmem_base + k * 8, db + bo, IDESC, (r | k) ? 1u : 0u);
      }
      issue += clock64() - a0;
      if (MODE == 0) {
#pragma unroll
        for (int c = 0; c < C; ++c) umma_commit(&bar[c]);
      } else if (MODE == 1) {  // same barrier every time
#pragma unroll
        for (int c = 0; c < C; ++c) umma_commit(&bar[0]);
      } else if (MODE == 2) {  // commit every other group
        if (r & 1) {
#pragma unroll
          for (int c = 0; c < C; ++c) umma_commit(&bar[c]);
        }
      } else if (MODE == 3) {  // multicast form (cluster of 1)
#pragma unroll
        for (int c = 0; c < C; ++c)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                       ::"r"(smem_u32(&bar[c])), "h"((uint16_t)1) : "memory");
      }
    }
    umma_commit(&bar[7]);
    mbar_wait(&bar[7], 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = issue; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem_base);
  }
}

template <int N, int C, int MODE = 0>
void run() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(commit_rate<N, C, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int reps = 2000;
  commit_rate<N, C, MODE><<<148, 128, 64 * 1024>>>(reps, d);
  cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("mode %d N=%3d commits/group=%d: %7.1f cycles/group (8 MMAs), issue %7.1f cycles/group  (%s)\n", MODE, N, C,
         (double)h[0] / reps, (double)h[1] / reps, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64, 0>(); run<64, 1>(); run<128, 0>(); run<128, 1>(); run<128, 2>();
  run<128, 1, 1>(); run<128, 2, 1>(); run<128, 1, 2>(); run<128, 1, 3>();
  return 0;
}
