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


// cp.async (LDGSTS, 16 B per thread) of random 16 KB blocks into a smem ring,
// NT threads per CTA, STAGES blocks in flight
template <int STAGES, int NT>
__global__ void __launch_bounds__(NT, 1) ldgsts_kernel(const uint8_t* __restrict__ buf, size_t nblocks, int iters,
                                                      unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t x = blockIdx.x * 2654435761u + 999u;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  unsigned long long acc = 0;
  auto issue = [&](int it) {
    x = x * 1664525u + 1013904223u;
    const size_t b = (x >> 8) % nblocks;
    const uint8_t* src = buf + b * 16384;
    const uint32_t dst = sb + (it % STAGES) * 16384;
#pragma unroll
    for (int j = 0; j < 16384 / 16 / NT; ++j) {
      const int off = (threadIdx.x + j * NT) * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + off), "l"(src + off) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < STAGES - 1; ++s) issue(s);
  for (int it = 0; it < iters; ++it) {
    issue(it + STAGES - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");
    acc += smem[(it % STAGES) * 16384 + threadIdx.x * 16];
  }
  if (acc == 0x123456789ull) atomicAdd(sink, acc);
}

// mixed: warp 0 streams random 16 KB blocks with bulk copies (TMA engine),
// warps 1..NW-1 with cp.async (LSU path), each into its own ring
template <int NW>
__global__ void __launch_bounds__(32 * NW, 1) mixed_kernel(const uint8_t* __restrict__ buf, size_t nblocks, int iters,
                                                          unsigned long long* sink, int use_bulk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[4];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t x = blockIdx.x * 2654435761u + 31u * warp;
  unsigned long long acc = 0;
  if (warp == 0) {
    if (!use_bulk) return;
    if (lane == 0) {
      for (int s = 0; s < 4; ++s) {
        x = x * 1664525u + 1013904223u;
        mbar_expect_tx(&bars[s], 16384);
        bulk_g2s(smem + s * 16384, buf + ((x >> 8) % nblocks) * 16384, 16384, &bars[s]);
      }
      for (int it = 0; it < iters; ++it) {
        const int s = it % 4;
        mbar_wait(&bars[s], (it / 4) & 1);
        acc += smem[s * 16384 + (it & 1023)];
        if (it + 4 < iters) {
          x = x * 1664525u + 1013904223u;
          mbar_expect_tx(&bars[s], 16384);
          bulk_g2s(smem + s * 16384, buf + ((x >> 8) % nblocks) * 16384, 16384, &bars[s]);
        }
      }
    }
  } else {
    // each cp.async warp: its own 4-stage ring of 16 KB after the bulk ring
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem) + 4 * 16384 + (warp - 1) * 4 * 16384;
    auto issue = [&](int it) {
      x = x * 1664525u + 1013904223u;
      const uint8_t* src = buf + ((x >> 8) % nblocks) * 16384;
      const uint32_t dst = sb + (it % 4) * 16384;
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const int off = (lane + j * 32) * 16;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + off), "l"(src + off) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int s = 0; s < 3; ++s) issue(s);
    for (int it = 0; it < iters; ++it) {
      issue(it + 3);
      asm volatile("cp.async.wait_group 3;" ::: "memory");
      acc += smem[4 * 16384 + (warp - 1) * 4 * 16384 + (it % 4) * 16384 + lane * 16];
    }
  }
  if (acc == 0x123456789ull) atomicAdd(sink, acc);
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

  {
    size_t nb = (size_t(64) << 20) / BLK;
    auto run_ldgsts = [&](auto kern, int stages, int nt, const char* name) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, stages * BLK);
      int grid = prop.multiProcessorCount;
      int iters = 4000;
      kern<<<grid, nt, stages * BLK>>>(buf, nb, 200, sink);
      cudaEventRecord(e0);
      kern<<<grid, nt, stages * BLK>>>(buf, nb, iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = double(grid) * iters * BLK;
      printf("ldgsts %s stages %2d threads %d 64 MB buf: %.1f GB/s err=%s\n", name, stages, nt, bytes / ms / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    };
    run_ldgsts(ldgsts_kernel<4, 128>, 4, 128, "");
    run_ldgsts(ldgsts_kernel<8, 128>, 8, 128, "");
    run_ldgsts(ldgsts_kernel<8, 256>, 8, 256, "");
    run_ldgsts(ldgsts_kernel<12, 256>, 12, 256, "");
    run_ldgsts(ldgsts_kernel<8, 64>, 8, 64, "");
    run_ldgsts(ldgsts_kernel<8, 32>, 8, 32, "");
  }

  {
    size_t nb = (size_t(64) << 20) / BLK;
    auto run_mixed = [&](auto kern, int nw, int use_bulk) {
      const int smem_bytes = (4 + 4 * (nw - 1)) * BLK;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
      int grid = prop.multiProcessorCount;
      int iters = 2000;
      kern<<<grid, 32 * nw, smem_bytes>>>(buf, nb, 100, sink, use_bulk);
      cudaEventRecord(e0);
      kern<<<grid, 32 * nw, smem_bytes>>>(buf, nb, iters, sink, use_bulk);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = double(grid) * iters * BLK * ((nw - 1) + use_bulk);
      printf("mixed bulk=%d + %d cp.async warps: %.1f GB/s err=%s\n", use_bulk, nw - 1, bytes / ms / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    };
    run_mixed(mixed_kernel<2>, 2, 0);
    run_mixed(mixed_kernel<2>, 2, 1);
    run_mixed(mixed_kernel<3>, 3, 0);
    run_mixed(mixed_kernel<3>, 3, 1);
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
