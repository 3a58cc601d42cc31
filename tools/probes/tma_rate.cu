// Probe: L2->SMEM throughput of TMA tensor boxes shaped like K4's K/V tiles
// (2-D map over (rows, 128) bf16, box 64 x 64 with SWIZZLE_128B: 64 rows of
// 128 B at a 256 B stride) vs contiguous cp.async.bulk of the same 16 KB.
#include <cstdio>
#include <cuda.h>
#include "../../paper_2505_14708_b200/csrc/common.cuh"

using namespace da;

template <int STAGES, bool TENSOR>
__global__ void __launch_bounds__(32, 1) rate(const __grid_constant__ CUtensorMap map, const uint8_t* buf,
                                              int nblk, int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  uint32_t x = blockIdx.x * 2654435761u + 12345u;
  unsigned long long acc = 0;
  auto issue = [&](int s) {
    x = x * 1664525u + 1013904223u;
    const int b = (x >> 8) % nblk;  // a 64-row block (16 KB)
    mbar_expect_tx(&bars[s], 16384);
    if (TENSOR) {
      tma_load_2d(smem + s * 16384, &map, &bars[s], 0, b * 64);
      tma_load_2d(smem + s * 16384 + 8192, &map, &bars[s], 64, b * 64);
    } else {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(smem + s * 16384)), "l"(buf + (size_t)b * 16384), "r"(16384), "r"(smem_u32(&bars[s]))
                   : "memory");
    }
  };
  for (int s = 0; s < STAGES; ++s) issue(s);
  for (int it = 0; it < iters; ++it) {
    const int s = it % STAGES;
    mbar_wait(&bars[s], (it / STAGES) & 1);
    acc += smem[s * 16384 + (it & 1023)];
    if (it + STAGES < iters) issue(s);
  }
  atomicAdd(sink, acc);
}

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int STAGES, bool TENSOR>
void run(const CUtensorMap& m, const uint8_t* buf, int nblk, unsigned long long* sink, int sms) {
  auto k = rate<STAGES, TENSOR>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * 16384);
  const int iters = 3000;
  k<<<sms, 32, STAGES * 16384>>>(m, buf, nblk, 100, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms, 32, STAGES * 16384>>>(m, buf, nblk, iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%s stages %2d: %8.1f GB/s (%s)\n", TENSOR ? "tensor 2x(64x128B)" : "bulk 16KB        ", STAGES,
         (double)sms * iters * 16384 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = size_t(64) << 20;  // 64 MB: L2 resident
  uint8_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  PFN enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m;
  const cuuint64_t rows = bytes / 256;
  cuuint64_t dims[2] = {128, rows};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t estr[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int nblk = (int)(rows / 64);
  run<4, false>(m, buf, nblk, sink, sms);
  run<8, false>(m, buf, nblk, sink, sms);
  run<12, false>(m, buf, nblk, sink, sms);
  run<4, true>(m, buf, nblk, sink, sms);
  run<8, true>(m, buf, nblk, sink, sms);
  run<12, true>(m, buf, nblk, sink, sms);
  return 0;
}
