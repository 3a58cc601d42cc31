// Probe: tcgen05.mma kind::f16 with M = 64 (cta_group::1), A from TMEM (TS).
// Checks the TMEM lane layout the K4 two-tile design relies on: an M=64 tile
// occupies lanes {0-15, 32-47, 64-79, 96-111} (lane offset 0) or the other
// half-subpartitions {16-31, ...} (lane offset 16), for both D and A.
#include <cstdio>
#include <cmath>
#include <vector>
#include "../../paper_2505_14708_b200/csrc/common.cuh"
using namespace da;

__global__ void __launch_bounds__(128, 1) m64(const float* q, const float* k, float* s_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, t = threadIdx.x;
  // K tile (64 keys x 128 d) into smem, SWIZZLE_128B K-major [half][64 rows x 128 B]
  for (int i = t; i < 64 * 128; i += 128) {
    const int r = i / 128, c = i % 128, hf = c / 64, cc = c % 64;
    const int chunk = cc / 8, e = cc % 8;
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(smem + hf * 8192 + r * 128 + ((chunk ^ (r & 7)) * 16)) + e;
    *dst = __float2bfloat16(k[r * 128 + c]);
  }
  if (t == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  // Q: thread = TMEM lane L; tile = (L % 32) >= 16; row = 16 * (L / 32) + L % 16
  {
    const int L = t, tile = (L % 32) >= 16, row = 16 * (L / 32) + (L % 16);
    uint32_t qv[64];
    for (int c = 0; c < 64; ++c) qv[c] = pack_bf16(q[(tile * 64 + row) * 128 + 2 * c], q[(tile * 64 + row) * 128 + 2 * c + 1]);
    const uint32_t la = tm + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 4; ++c) tmem_st16u(la + c * 16, *reinterpret_cast<uint32_t(*)[16]>(&qv[c * 16]));
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    constexpr uint32_t IDESC = umma_idesc_bf16(64, 64, 0, 0);
    const uint64_t dK = umma_desc_sw128(smem_u32(smem), 16, 1024);
    for (int tile = 0; tile < 2; ++tile) {
      const uint32_t loff = (uint32_t)(16 * tile) << 16;
      for (int kk = 0; kk < 8; ++kk)
        umma_bf16_ts(tm + loff + 128, tm + loff + kk * 8, dK + (uint64_t)((kk >> 2) * (8192 >> 4) + (kk & 3) * 2), IDESC,
                     kk > 0 ? 1u : 0u);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float s[64];
  tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + 128, *reinterpret_cast<float(*)[32]>(&s[0]));
  tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + 160, *reinterpret_cast<float(*)[32]>(&s[32]));
  tmem_ld_wait();
  for (int c = 0; c < 64; ++c) s_out[t * 64 + c] = s[c];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_free<256>(tm); }
}

int main() {
  std::vector<float> q(128 * 128), k(64 * 128), s(128 * 64);
  for (size_t i = 0; i < q.size(); ++i) q[i] = (float)((i * 7919 % 17) - 8) / 8.f;
  for (size_t i = 0; i < k.size(); ++i) k[i] = (float)((i * 104729 % 13) - 6) / 8.f;
  float *dq, *dk, *ds;
  cudaMalloc(&dq, q.size() * 4); cudaMalloc(&dk, k.size() * 4); cudaMalloc(&ds, s.size() * 4);
  cudaMemcpy(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, k.data(), k.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(m64, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  m64<<<1, 128, 16384>>>(dq, dk, ds);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(s.data(), ds, s.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  int bad = 0;
  for (int L = 0; L < 128; ++L) {
    const int tile = (L % 32) >= 16, row = 16 * (L / 32) + (L % 16);
    for (int c = 0; c < 64; ++c) {
      double ref = 0;
      for (int d = 0; d < 128; ++d) ref += (double)q[(tile * 64 + row) * 128 + d] * k[c * 128 + d];
      const double err = fabs(ref - s[L * 64 + c]);
      if (err > 1e-2) ++bad;
      maxerr = fmax(maxerr, err);
    }
  }
  printf("M=64 two-tile TS MMA: %s, max err %.3g, bad %d of %d\n", cudaGetErrorString(e), maxerr, bad, 128 * 64);
  return 0;
}
