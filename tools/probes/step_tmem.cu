// Probe: cycles per K4 pair step (two kept 64 x 64 x 128 blocks of one query
// region) for the TRANSPOSED formulation with BOTH A operands in TMEM:
//
//   GEMM1  S^T[128 keys x 64 q]  = K_pair . Q^T      TS, M = 128, N = 64 (A = K pair in TMEM, B = Q tile in smem)
//   GEMM2  O^T[128 d x 64 q]    += V_pair^T . P^T    TS, M = 128, N = 64 (A = V^T pair in TMEM, B = P^T in smem)
//
// K and V^T reach TMEM from L2 through registers (LDG.128, tcgen05.st), so
// the only shared-memory traffic per step is the 16 KB P^T tile (written with
// st.shared, read by GEMM2) and GEMM1's Q^T reads. Loader groups of 4 warps
// (lane = key row for K, lane = feature row for V^T) alternate steps; four
// more warps write P^T. Compare with step_pipe.cu (lh: 1546 cycles per step
// with its 64 KB of bulk copies).
#include <cstdio>
#include "../../paper_2505_14708_b200/csrc/common.cuh"

using namespace da;

constexpr int OFF_Q = 0;                 // 16 KB Q tile [half][64 x 128 B]
constexpr int OFF_P = 16384;             // 2 x 16 KB P^T tiles [8-key group][8 x 128 B]
constexpr int SMEM = OFF_P + 2 * 16384;  // 48 KB
// TMEM columns: K pair buffers [0,128), V^T pair buffers [128,256), S^T [256,384), O^T [384,448)
constexpr uint32_t COL_K = 0, COL_V = 128, COL_S = 256, COL_O = 384;
constexpr int LG = 2;  // loader groups per tensor (alternating steps)

DA_DEV void ldg_row(const uint8_t* base, int row, uint32_t (&r)[64]) {
  // 16 chunks of 16 B; chunk c of all 128 rows is contiguous ([c][row][16 B])
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(base + c * 2048 + row * 16));
    r[4 * c] = v.x; r[4 * c + 1] = v.y; r[4 * c + 2] = v.z; r[4 * c + 3] = v.w;
  }
}

__global__ void __launch_bounds__(32 * (4 + 8 * LG) + 128, 1) step_tmem(int steps, int mode, const uint8_t* buf,
                                                                    size_t ntiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t kfull[2], kempty[2], vfull[2], vempty[2], pfull[2], pfree[2], sfull[2], done_bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < SMEM / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kfull[s], 128); mbar_init(&kempty[s], 1);
      mbar_init(&vfull[s], 128); mbar_init(&vempty[s], 1);
      mbar_init(&pfull[s], 128); mbar_init(&pfree[s], 1);
      mbar_init(&sfull[s], 1);
    }
    mbar_init(&done_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const long long t0 = clock64();
  if (warp == 1 || warp == 2) {
    // ---------------- MMA issuers: warp 1 GEMM1, warp 2 GEMM2 ----------------
    const uint64_t dQ = umma_desc_sw128(0, 16, 1024) + (smem_u32(smem + OFF_Q) >> 4);
    const uint64_t dP = umma_desc_sw128(0, 16, 1024) + (smem_u32(smem + OFF_P) >> 4);
    constexpr uint32_t I1 = umma_idesc_bf16(128, 64, 0, 0);  // A K-major (TMEM), B K-major
    constexpr uint32_t I2 = umma_idesc_bf16(128, 64, 0, 1);  // A (TMEM), B MN-major
    for (int s = 0; s < steps; ++s) {
      const int b = s & 1;
      const uint32_t par = (s >> 1) & 1;
      if (warp == 1) {
        mbar_wait_spin(&kfull[b], par);
        // S^T buffer b: the softmax stand-in of step s - 2 has produced its P^T
        // (without it: GEMM2 of step s - 2 is done), as in the real pipeline
        if (s >= 2) mbar_wait_spin((mode & 1) ? &pfull[b] : &pfree[b], par ^ 1u);
        tc_fence_after();
        if (elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts(tmem + COL_S + 64 * b, tmem + COL_K + 64 * b + 8 * kk,
                         dQ + (uint64_t)((kk >> 2) * 512 + (kk & 3) * 2), I1, kk > 0);
          umma_commit(&kempty[b]);
          umma_commit(&sfull[b]);
        }
        __syncwarp();
      } else {
        mbar_wait_spin(&vfull[b], par);
        if (mode & 1) mbar_wait_spin(&pfull[b], par);
        else mbar_wait_spin(&sfull[b], par);
        tc_fence_after();
        if (elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts(tmem + COL_O, tmem + COL_V + 64 * b + 8 * kk, dP + (uint64_t)(b * 1024 + kk * 128), I2, 1u);
          umma_commit(&vempty[b]);
          umma_commit(&pfree[b]);
          if (s == steps - 1) umma_commit(&done_bar);
        }
        __syncwarp();
      }
    }
    if (warp == 2) {
      mbar_wait(&done_bar, 0);
      if (lane == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
    }
  } else if (warp >= 4 && warp < 4 + 8 * LG) {
    // ---------------- loaders: group gi of tensor z takes steps s = gi (mod LG) ----------------
    const int lw = warp - 4;
    const int z = lw / (4 * LG);            // 0: K, 1: V^T
    const int gi = (lw / 4) % LG;
    const int row = 32 * (lw % 4) + lane;   // TMEM lane = key (K) or feature (V^T)
    const uint32_t tl = tmem + ((uint32_t)(32 * (lw % 4)) << 16);
    uint64_t* full = z ? vfull : kfull;
    uint64_t* empty = z ? vempty : kempty;
    const uint32_t col = z ? COL_V : COL_K;
    uint32_t x = blockIdx.x * 2654435761u + 17u * (uint32_t)(z * LG + gi) + 1u;
    uint32_t r[64];
    for (int s = gi; s < steps; s += LG) {
      x = x * 1664525u + 1013904223u;
      if (mode & 2) {
        ldg_row(buf + (size_t)((x >> 8) % ntiles) * 32768, row, r);
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i) r[i] = x + i;
      }
      const int b = s & 1;
      if (s >= 2) mbar_wait_spin(&empty[b], ((s >> 1) - 1) & 1);
      tc_fence_after();
      tmem_st32(tl + col + 64 * b, *reinterpret_cast<float(*)[32]>(&r[0]));
      tmem_st32(tl + col + 64 * b + 32, *reinterpret_cast<float(*)[32]>(&r[32]));
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&full[b]);
    }
  } else if (warp >= 4 + 8 * LG && (mode & 1)) {
    // ---------------- P^T writers (stand-in for the softmax): 128 key rows x 128 B ----------------
    const int t = threadIdx.x - 32 * (4 + 8 * LG);
    if (t < 128) {
      for (int s = 0; s < steps; ++s) {
        const int b = s & 1;
        mbar_wait_spin(&sfull[b], (s >> 1) & 1);  // S^T of the step is in TMEM (not read here)
        if (s >= 2) mbar_wait_spin(&pfree[b], ((s >> 1) - 1) & 1);
        const uint32_t base = smem_u32(smem + OFF_P + b * 16384) + (uint32_t)((t >> 3) * 1024 + (t & 7) * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c) sts128(base + (((c ^ t) & 7) << 4), s, c, t, 0x3c003c00u);
        fence_proxy_async_smem();
        mbar_arrive(&pfull[b]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* buf;
  const size_t bytes = size_t(64) << 20;  // L2-resident tile-pair pool
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  long long* d_out;
  cudaMalloc(&d_out, 16);
  const int threads = 32 * (4 + 8 * LG) + 128;
  cudaFuncSetAttribute(step_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const int steps = 4000;
  const char* names[] = {"MMAs only (register data, no P^T)", "MMAs + P^T st.shared",
                         "MMAs + LDG K/V (L2 tiles)", "MMAs + LDG K/V + P^T st.shared"};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 4; ++mode) {
      cudaMemset(d_out, 0, 16);
      step_tmem<<<sms, threads, SMEM>>>(steps, mode, buf, bytes / 32768, d_out);
      cudaError_t e = cudaDeviceSynchronize();
      long long cyc = 0;
      cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
      printf("tr-TMEM %-36s %7.1f cycles/step (%6.1f per block)  %s\n", names[mode], (double)cyc / steps,
             (double)cyc / steps / 2, cudaGetErrorString(e));
    }
  return 0;
}
