// Probe: cycles per K4 "pair step" (two kept 64 x 64 x 128 blocks of one query
// region) for the tcgen05 formulations, with the shared-memory traffic that
// goes with them, on all SMs.
//
//   lh  (current K4): GEMM1 S[64 q x 128 k] = Q K^T   TS, M = 64, N = 128 (A = Q in TMEM, B = K pair in smem)
//                     GEMM2 O[64 q x 128 d] += P V    TS, M = 64, N = 128 (A = P in TMEM, B = V pair, MN-major)
//   tr  (transposed): GEMM1 S^T[128 k x 64 q] = K Q^T SS, M = 128, N = 64 (A = K pair, B = Q tile)
//                     GEMM2 O^T[128 d x 64 q] += V^T P^T SS, M = 128, N = 64 (A = V pair MN-major, B = P^T MN-major)
//
// Per step the producer bulk-copies COPY bytes of random 16 KB tiles from an
// L2-resident buffer into a 2-slot ring (the K and V tiles), and (tr, STS=1)
// four warps write a 16 KB P^T tile with st.shared (the softmax output), each
// gated like the real pipeline. Reports cycles per step.
#include <cstdio>
#include "../../paper_2505_14708_b200/csrc/common.cuh"

using namespace da;

constexpr int SLOT = 65536;  // K pair (32 KB) + V pair (32 KB)
constexpr int NSLOT = 2;
constexpr int OFF_Q = NSLOT * SLOT;      // 16 KB Q tile
constexpr int OFF_P = OFF_Q + 16384;     // 2 x 16 KB P^T tiles
constexpr int SMEM = OFF_P + 2 * 16384;  // 176 KB

__global__ void __launch_bounds__(256, 1) step_pipe(int mode, int copy_bytes, int sts, int steps, const uint8_t* buf,
                                                     size_t ntiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t full[NSLOT], empty[NSLOT], pfull[2], pfree[2], done_bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < SMEM / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSLOT; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&pfull[s], 128); mbar_init(&pfree[s], 1); }
    mbar_init(&done_bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  long long t0 = clock64();
  if (warp == 0) {
    if (lane == 0) {
      uint32_t x = blockIdx.x * 2654435761u + 1u;
      for (int s = 0; s < steps; ++s) {
        const int sl = s % NSLOT;
        if (s >= NSLOT) mbar_wait(&empty[sl], ((s / NSLOT) - 1) & 1);
        if (copy_bytes == 0) {
          mbar_arrive(&full[sl]);
          continue;
        }
        mbar_expect_tx(&full[sl], copy_bytes);
        for (int c = 0; c < copy_bytes; c += 16384) {
          x = x * 1664525u + 1013904223u;
          bulk_g2s(smem + sl * SLOT + c, buf + (size_t)((x >> 8) % ntiles) * 16384, 16384, &full[sl]);
        }
      }
    }
  } else if (warp == 1) {
    const uint64_t dK = umma_desc_sw128(0, 16, 2048) + (smem_u32(smem) >> 4);       // K pair, K-major
    const uint64_t dV = umma_desc_sw128(0, 1024, 2048) + (smem_u32(smem + 32768) >> 4);  // V pair, MN-major
    const uint64_t dQ = umma_desc_sw128(0, 16, 1024) + (smem_u32(smem + OFF_Q) >> 4);   // Q [half][64 x 128 B]
    const uint64_t dP = umma_desc_sw128(0, 16, 1024) + (smem_u32(smem + OFF_P) >> 4);   // P^T [8-key group][8 x 128 B]
    for (int s = 0; s < steps; ++s) {
      const int sl = s % NSLOT, pb = s & 1;
      mbar_wait_spin(&full[sl], (s / NSLOT) & 1);
      if (mode == 1 && sts) mbar_wait_spin(&pfull[pb], (s >> 1) & 1);
      tc_fence_after();
      if (elect_one_sync()) {
        const uint64_t so = (uint64_t)(sl * (SLOT >> 4));
        if (mode == 0) {
          constexpr uint32_t I1 = umma_idesc_bf16(64, 128, 0, 0);
          constexpr uint32_t I2 = umma_idesc_bf16(64, 128, 0, 1);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts(tmem + 64, tmem + kk * 8, dK + so + (uint64_t)((kk >> 2) * 64 + (kk & 3) * 2), I1, kk > 0);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts(tmem + 256, tmem + 192 + kk * 8, dV + so + (uint64_t)(kk * 256), I2, 1u);
        } else {
          constexpr uint32_t I1 = umma_idesc_bf16(128, 64, 0, 0);
          constexpr uint32_t I2 = umma_idesc_bf16(128, 64, 1, 1);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(tmem + 64 * pb, dK + so + (uint64_t)((kk >> 2) * 64 + (kk & 3) * 2),
                      dQ + (uint64_t)((kk >> 2) * 512 + (kk & 3) * 2), I1, kk > 0);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(tmem + 256, dV + so + (uint64_t)(kk * 256), dP + (uint64_t)(pb * 1024 + kk * 128), I2, 1u);
        }
        umma_commit(&empty[sl]);
        umma_commit(&pfree[pb]);
        if (s == steps - 1) umma_commit(&done_bar);
      }
      __syncwarp();
    }
    mbar_wait(&done_bar, 0);
    if (lane == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
  } else if (warp >= 4 && mode == 1 && sts) {
    // P^T writers: thread t = key row t of the 128-key step; 8 x 16 B swizzled stores
    const int t = threadIdx.x - 128;
    for (int s = 0; s < steps; ++s) {
      const int pb = s & 1;
      if (s >= 2) mbar_wait(&pfree[pb], ((s >> 1) - 1) & 1);
      const uint32_t base = smem_u32(smem + OFF_P + pb * 16384) + (uint32_t)((t >> 3) * 1024 + (t & 7) * 128);
#pragma unroll
      for (int c = 0; c < 8; ++c) sts128(base + (((c ^ t) & 7) << 4), s, c, t, 0x3c003c00u);
      fence_proxy_async_smem();
      mbar_arrive(&pfull[pb]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* buf;
  const size_t bytes = size_t(64) << 20;  // L2-resident tile pool
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  long long* d_out;
  cudaMalloc(&d_out, 16);
  cudaFuncSetAttribute(step_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const int steps = 4000;
  struct Cfg { int mode, copy, sts; const char* name; };
  const Cfg cfgs[] = {
      {0, 0, 0, "lh  TS M64 N128, no copies"},
      {0, 65536, 0, "lh  TS M64 N128, 64 KB copies/step"},
      {1, 0, 0, "tr  SS M128 N64, no copies, no P^T stores"},
      {1, 0, 1, "tr  SS M128 N64, P^T stores"},
      {1, 65536, 0, "tr  SS M128 N64, 64 KB copies/step"},
      {1, 65536, 1, "tr  SS M128 N64, 64 KB copies + P^T stores"},
      {1, 32768, 1, "tr  SS M128 N64, 32 KB copies + P^T stores"},
  };
  for (int rep = 0; rep < 2; ++rep)
    for (const Cfg& c : cfgs) {
      cudaMemset(d_out, 0, 16);
      step_pipe<<<sms, 256, SMEM>>>(c.mode, c.copy, c.sts, steps, buf, bytes / 16384, d_out);
      cudaError_t e = cudaDeviceSynchronize();
      long long cyc = 0;
      cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
      printf("%-48s %7.1f cycles/step (%6.1f per block)  %s\n", c.name, (double)cyc / steps,
             (double)cyc / steps / 2, cudaGetErrorString(e));
    }
  return 0;
}
