// Probe: does L2->smem bulk-copy traffic slow tcgen05.mma operand reads from
// shared memory? Warp 0 issues R TS MMAs (M = 64, N = 64 or 128; B from smem),
// warp 1 (optional) streams random 16 KB blocks into a separate 4-stage ring
// with cp.async.bulk for the whole duration. Cycles per MMA with / without.
#include <cstdio>
#include "../../paper_2505_14708_b200/csrc/common.cuh"

using namespace da;

template <int N, int M>
__global__ void __launch_bounds__(64, 1) contend(int reps, const uint8_t* buf, size_t nblocks, int stream,
                                                long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t bar, lbar[8];
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int s = 0; s < 8; ++s) mbar_init(&lbar[s], 1);
    done = 0;
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (threadIdx.x == 0) {
      constexpr uint32_t IDESC = umma_idesc_bf16(M, N, 0, 0);
      const uint64_t db = umma_desc_sw128(smem_u32(smem), 16, 1024);
      long long t0 = clock64();
      if (stream == 2) {  // no MMAs: just let the copy stream run for ~1.4M cycles
        while (clock64() - t0 < 1430000) {
        }
        reps = 0;
      }
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t bo = (uint64_t)((k >> 2) * (16384 >> 4) + (k & 3) * 2);
          umma_bf16_ts(tmem_base + 256, tmem_base + k * 8, db + bo, IDESC, (r | k) ? 1u : 0u);
        }
      }
      if (reps) {
        umma_commit(&bar);
        mbar_wait(&bar, 0);
      }
      long long t1 = clock64();
      done = 1;
      if (blockIdx.x == 0) out[0] = t1 - t0;
    }
  } else if (stream && threadIdx.x == 32) {
    uint8_t* ring = smem + 32 * 1024;
    uint32_t x = blockIdx.x * 2654435761u + 1u;
    long long n = 0;
    for (int s = 0; s < 8; ++s) {
      x = x * 1664525u + 1013904223u;
      mbar_expect_tx(&lbar[s], 16384);
      bulk_g2s(ring + s * 16384, buf + ((x >> 8) % nblocks) * 16384, 16384, &lbar[s]);
    }
    for (int it = 0;; ++it) {
      const int s = it % 8;
      mbar_wait(&lbar[s], (it / 8) & 1);
      ++n;
      if (done) break;
      x = x * 1664525u + 1013904223u;
      mbar_expect_tx(&lbar[s], 16384);
      bulk_g2s(ring + s * 16384, buf + ((x >> 8) % nblocks) * 16384, 16384, &lbar[s]);
    }
    // drain the copies still in flight
    for (int it2 = 1; it2 < 8; ++it2) {
      const int it = (int)n - 1 + it2;
      mbar_wait(&lbar[it % 8], (it / 8) & 1);
    }
    if (blockIdx.x == 0) out[1] = n;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem_base);
  }
}

template <int N, int M>
void run(int sms, const uint8_t* buf, size_t nb, int stream, long long* d_out) {
  const int reps = 4000;
  cudaFuncSetAttribute(contend<N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaMemset(d_out, 0, 16);
  contend<N, M><<<sms, 64, 160 * 1024>>>(reps, buf, nb, stream, d_out);
  cudaDeviceSynchronize();
  long long o[2];
  cudaMemcpy(o, d_out, 16, cudaMemcpyDeviceToHost);
  const double per = (double)o[0] / (reps * 8);
  printf("M=%3d N=%3d stream=%d: %6.1f cycles/MMA; copies %lld (%.1f B/clk/SM of L2->smem)  (%s)\n", M, N, stream, per,
         o[1], o[1] * 16384.0 / o[0], cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* buf;
  const size_t bytes = size_t(64) << 20;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  long long* d_out;
  cudaMalloc(&d_out, 16);
  const size_t nb = bytes / 16384;
  run<64, 64>(sms, buf, nb, 2, d_out);
  for (int s = 0; s < 2; ++s) {
    run<64, 64>(sms, buf, nb, s, d_out);
    run<128, 64>(sms, buf, nb, s, d_out);
    run<64, 128>(sms, buf, nb, s, d_out);
    run<128, 128>(sms, buf, nb, s, d_out);
    run<256, 128>(sms, buf, nb, s, d_out);
  }
  return 0;
}
