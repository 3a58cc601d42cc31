// Probe: L2->SM bandwidth for random 16 KB block fetches (the K4 access pattern:
// every kept (query block, key block) pair pulls a 16 KB K block and a 16 KB V
// block). Bulk async copies (cp.async.bulk) into a multi-stage smem ring.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t addr = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" :: "r"(addr), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem), "r"(bytes),
                  "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

template <int STAGES, int BLK>
__global__ void __launch_bounds__(32, 1) l2bw_kernel(const uint8_t* __restrict__ buf, size_t nblocks, int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  uint32_t x = blockIdx.x * 2654435761u + 12345u;
  unsigned long long acc = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES && s < iters; ++s) {
      x = x * 1664525u + 1013904223u;
      size_t b = (x >> 8) % nblocks;
      mbar_expect_tx(&bars[s], BLK);
      bulk_g2s(smem + s * BLK, buf + b * BLK, BLK, &bars[s]);
    }
    for (int it = 0; it < iters; ++it) {
      int s = it % STAGES;
      uint32_t ph = (it / STAGES) & 1;
      mbar_wait(&bars[s], ph);
      acc += smem[s * BLK + (it & 1023)];
      int nxt = it + STAGES;
      if (nxt < iters) {
        x = x * 1664525u + 1013904223u;
        size_t b = (x >> 8) % nblocks;
        mbar_expect_tx(&bars[s], BLK);
        bulk_g2s(smem + s * BLK, buf + b * BLK, BLK, &bars[s]);
      }
    }
    atomicAdd(sink, acc);
  }
}

// plain LDG.128 streaming reads of random 16 KB blocks, 256 threads
__global__ void __launch_bounds__(256) ldg_kernel(const int4* __restrict__ buf, size_t nblocks, int iters, unsigned long long* sink) {
  uint32_t x = blockIdx.x * 2654435761u + 777u;
  int4 acc = make_int4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    size_t b = (x >> 8) % nblocks;
    const int4* p = buf + b * 1024;  // 16 KB block = 1024 int4
    int4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldg(p + threadIdx.x + j * 256);
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc.x ^= v[j].x; acc.y ^= v[j].y; acc.z ^= v[j].z; acc.w ^= v[j].w; }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678) atomicAdd(sink, 1ull);
}

int main() {
  int dev = 0;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  printf("device %s SMs %d L2 %d MB\n", prop.name, prop.multiProcessorCount, prop.l2CacheSize >> 20);
  size_t max_bytes = size_t(2048) << 20;
  uint8_t* buf;
  cudaMalloc(&buf, max_bytes);
  cudaMemset(buf, 1, max_bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  constexpr int BLK = 16384;
  auto run_bulk = [&](auto kern, int stages, size_t nblocks) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, stages * BLK);
    int grid = prop.multiProcessorCount;
    int iters = 4000;
    kern<<<grid, 32, stages * BLK>>>(buf, nblocks, 200, sink);
    cudaEventRecord(e0);
    kern<<<grid, 32, stages * BLK>>>(buf, nblocks, iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = double(grid) * iters * BLK;
    printf("bulk stages %2d (%3d KB in flight/SM) 64 MB buf: %.1f GB/s err=%s\n", stages, stages * 16,
           bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  {
    size_t nb = (size_t(64) << 20) / BLK;
    run_bulk(l2bw_kernel<4, BLK>, 4, nb);
    run_bulk(l2bw_kernel<8, BLK>, 8, nb);
    run_bulk(l2bw_kernel<10, BLK>, 10, nb);
    run_bulk(l2bw_kernel<13, BLK>, 13, nb);
  }
  constexpr int STAGES = 8;
  cudaFuncSetAttribute(l2bw_kernel<STAGES, BLK>, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * BLK);
  size_t sizes_mb[] = {32, 64, 96, 2048};
  for (size_t mb : sizes_mb) {
    size_t nblocks = (mb << 20) / BLK;
    for (int ctas_per_sm : {1, 2}) {
      int grid = prop.multiProcessorCount * ctas_per_sm;
      int iters = 4000;
      l2bw_kernel<STAGES, BLK><<<grid, 32, STAGES * BLK>>>(buf, nblocks, 200, sink);
      cudaEventRecord(e0);
      l2bw_kernel<STAGES, BLK><<<grid, 32, STAGES * BLK>>>(buf, nblocks, iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = double(grid) * iters * BLK;
      printf("bulk  buf %5zu MB ctas/SM %d stages %d: %.1f GB/s  (%.3f ms) err=%s\n", mb, ctas_per_sm, STAGES,
             bytes / ms / 1e6, ms, cudaGetErrorString(cudaGetLastError()));
    }
    for (int ctas_per_sm : {4, 8}) {
      int grid = prop.multiProcessorCount * ctas_per_sm;
      int iters = 1000;
      ldg_kernel<<<grid, 256>>>((const int4*)buf, nblocks, 50, sink);
      cudaEventRecord(e0);
      ldg_kernel<<<grid, 256>>>((const int4*)buf, nblocks, iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = double(grid) * iters * BLK;
      printf("ldg   buf %5zu MB ctas/SM %d: %.1f GB/s  (%.3f ms) err=%s\n", mb, ctas_per_sm,
             bytes / ms / 1e6, ms, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
