// Probe: tcgen05.mma (kind::f16, SS operands, cta_group::1) issue rate by shape
// and operand majorness. One CTA per SM; one elected thread issues R MMAs into
// the same TMEM accumulator; cycles per MMA = total / R.
#include <cstdio>
#include "../../paper_2505_14708_b200/csrc/common.cuh"

using namespace da;

template <int N, int AMN, int BMN>
__global__ void __launch_bounds__(128, 1) mma_rate(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t IDESC = umma_idesc_bf16(128, N, AMN, BMN);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32 * 1024);
    const uint64_t da_ = umma_desc_sw128(a, AMN ? 8192 : 16, 1024);
    const uint64_t db = umma_desc_sw128(b, BMN ? 8192 : 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t ao = AMN ? (uint64_t)((k * 2048) >> 4) : (uint64_t)((k >> 2) * (16384 >> 4) + (k & 3) * 2);
        const uint64_t bo = BMN ? (uint64_t)((k * 2048) >> 4) : (uint64_t)((k >> 2) * (8192 >> 4) + (k & 3) * 2);
        umma_bf16(tmem_base, da_ + ao, db + bo, IDESC, (r | k) ? 1u : 0u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<256>(tmem_base);
  }
}

// A from TMEM (K-major, packed bf16 pairs), B from shared memory.
template <int N, int BMN>
__global__ void __launch_bounds__(128, 1) mma_rate_ts(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t IDESC = umma_idesc_bf16(128, N, 0, BMN);
    const uint32_t b = smem_u32(smem);
    const uint64_t db = umma_desc_sw128(b, BMN ? 8192 : 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t bo = BMN ? (uint64_t)((k * 2048) >> 4) : (uint64_t)((k >> 2) * (16384 >> 4) + (k & 3) * 2);
        umma_bf16_ts(tmem_base + 256, tmem_base + k * 8, db + bo, IDESC, (r | k) ? 1u : 0u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem_base);
  }
}

template <int N, int BMN>
void run_ts(const char* name, int sms, long long* d_out) {
  const int reps = 2000;
  cudaFuncSetAttribute(mma_rate_ts<N, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  mma_rate_ts<N, BMN><<<sms, 128, 64 * 1024>>>(reps, d_out);
  cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  double per = (double)cyc / (reps * 8);
  printf("%-28s N=%3d: %7.1f cycles/MMA  %7.0f MAC/clk/SM  (%s)\n", name, N, per, 128.0 * N * 16 / per,
         cudaGetErrorString(cudaGetLastError()));
}


// TS with M = 64: ALT = 1 alternates 8-MMA groups between the two lane halves
// (TMEM lane offset 0 / 16, separate accumulators) as the K4 pair kernel does.
template <int M, int N, int ALT>
__global__ void __launch_bounds__(128, 1) mma_rate_m(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t IDESC = umma_idesc_bf16(M, N, 0, 0);
    const uint32_t b = smem_u32(smem);
    const uint64_t db = umma_desc_sw128(b, 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t loff = ALT ? ((uint32_t)(16 * (r & 1)) << 16) : 0u;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t bo = (uint64_t)((k >> 2) * (16384 >> 4) + (k & 3) * 2);
        umma_bf16_ts(tmem_base + loff + 256, tmem_base + loff + k * 8, db + bo, IDESC, (r > 1 || k) ? 1u : 0u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem_base);
  }
}

template <int M, int N, int ALT>
void run_m(const char* name, int sms, long long* d_out) {
  const int reps = 2000;
  cudaFuncSetAttribute(mma_rate_m<M, N, ALT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  mma_rate_m<M, N, ALT><<<sms, 128, 64 * 1024>>>(reps, d_out);
  cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  double per = (double)cyc / (reps * 8);
  printf("%-28s M=%3d N=%3d: %7.1f cycles/MMA  %7.0f MAC/clk/SM  (%s)\n", name, M, N, per, (double)M * N * 16 / per,
         cudaGetErrorString(cudaGetLastError()));
}

template <int N, int AMN, int BMN>
void run(const char* name, int sms, long long* d_out) {
  const int reps = 2000;
  cudaFuncSetAttribute(mma_rate<N, AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  mma_rate<N, AMN, BMN><<<sms, 128, 96 * 1024>>>(reps, d_out);
  cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  double per = (double)cyc / (reps * 8);
  double macs = 128.0 * N * 16;
  printf("%-28s N=%3d: %7.1f cycles/MMA  %7.0f MAC/clk/SM  (%s)\n", name, N, per, macs / per,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d_out;
  cudaMalloc(&d_out, 8);
  run<64, 0, 0>("K-major A, K-major B", sms, d_out);
  run<64, 1, 1>("MN-major A, MN-major B", sms, d_out);
  run<128, 0, 0>("K-major A, K-major B", sms, d_out);
  run<128, 1, 1>("MN-major A, MN-major B", sms, d_out);
  run<256, 0, 0>("K-major A, K-major B", sms, d_out);
  run_ts<128, 0>("TS: A tmem, B K-major", sms, d_out);
  run_ts<128, 1>("TS: A tmem, B MN-major", sms, d_out);
  run_ts<64, 0>("TS: A tmem, B K-major", sms, d_out);
  run_ts<256, 0>("TS: A tmem, B K-major", sms, d_out);
  run_m<128, 64, 0>("TS", sms, d_out);
  run_m<128, 128, 0>("TS", sms, d_out);
  run_m<128, 256, 0>("TS", sms, d_out);
  run_m<64, 64, 0>("TS M64", sms, d_out);
  run_m<64, 128, 0>("TS M64", sms, d_out);
  run_m<64, 256, 0>("TS M64", sms, d_out);
  run_m<64, 64, 1>("TS M64 alternating halves", sms, d_out);
  run_m<64, 128, 1>("TS M64 alternating halves", sms, d_out);
  run_m<64, 256, 1>("TS M64 alternating halves", sms, d_out);
  run<64, 0, 0>("K/K single CTA", 1, d_out);
  run<64, 1, 1>("MN/MN single CTA", 1, d_out);
  return 0;
}
