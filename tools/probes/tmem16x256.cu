// Probe: tcgen05.ld .16x256b mapping. Fill TMEM with 32x32b stores (value =
// lane * 1000 + column), read .16x256b.x4 at lane base 0 (column 0) and print
// which (lane, column) each of the 16 registers of each thread received.
#include <cstdio>
#include "../../paper_2505_14708_b200/csrc/common.cuh"
using namespace da;

DA_DEV void ld16x256_x4(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
}

__global__ void probe(int* out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc<64>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase + ((uint32_t)(warp * 32) << 16);
  for (int c0 = 0; c0 < 64; c0 += 32) {
    float v[32];
    for (int c = 0; c < 32; ++c) v[c] = (float)((warp * 32 + lane) * 1000 + c0 + c);
    tmem_st32(tm + c0, v);
  }
  tmem_st_wait();
  uint32_t r[16];
  ld16x256_x4(tm + (16u << 16), r);  // lane base 16, column 0
  tmem_ld_wait();
  if (warp == 0)
    for (int i = 0; i < 16; ++i) out[lane * 16 + i] = (int)__uint_as_float(r[i]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<64>(tbase);
}

int main() {
  int* d;
  cudaMalloc(&d, 32 * 16 * sizeof(int));
  probe<<<1, 128>>>(d);
  int h[32 * 16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int t = 0; t < 32; ++t) {
    printf("t%2d:", t);
    for (int i = 0; i < 16; ++i) printf(" %d/%d", h[t * 16 + i] / 1000, h[t * 16 + i] % 1000);
    printf("\n");
  }
}
