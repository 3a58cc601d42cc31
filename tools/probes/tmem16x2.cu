// Probe: tcgen05.ld / st .16x32bx2 mapping. Fill TMEM with 32x32b stores
// (value = lane * 1000 + column), read with 16x32bx2 at lane base 0 and 16,
// half-split offset 64; print which (lane, column) each thread received.
#include <cstdio>
#include "../../paper_2505_14708_b200/csrc/common.cuh"
using namespace da;

DA_DEV void ld16x2_x4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], 64;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
}
DA_DEV void st16x2_x2(uint32_t taddr, uint32_t a, uint32_t b) {
  asm volatile("tcgen05.st.sync.aligned.16x32bx2.x2.b32 [%0], 64, {%1,%2};" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}

__global__ void probe(int* out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc<256>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase + ((uint32_t)(warp * 32) << 16);
  for (int c0 = 0; c0 < 256; c0 += 32) {
    float v[32];
    for (int c = 0; c < 32; ++c) v[c] = (float)((warp * 32 + lane) * 1000 + c0 + c);
    tmem_st32(tm + c0, v);
  }
  tmem_st_wait();
  uint32_t r[4];
  ld16x2_x4(tm + 8, r);  // lane base 0, column 8
  tmem_ld_wait();
  if (warp == 0) for (int i = 0; i < 4; ++i) out[lane * 4 + i] = (int)__uint_as_float(r[i]);
  ld16x2_x4(tm + (16u << 16) + 8, r);  // lane base 16
  tmem_ld_wait();
  if (warp == 0) for (int i = 0; i < 4; ++i) out[128 + lane * 4 + i] = (int)__uint_as_float(r[i]);
  // store round trip: 16x32bx2 .x2 at lane base 16, column 200, split 64 -> read back with 32x32b
  st16x2_x2(tm + (16u << 16) + 200, __float_as_uint(-1.f - lane), __float_as_uint(-100.f - lane));
  tmem_st_wait();
  float w[32];
  tmem_ld32(tm + 200, w);
  tmem_ld_wait();
  if (warp == 0) { out[256 + lane * 2] = (int)w[0]; out[256 + lane * 2 + 1] = (int)w[1]; }
  tmem_ld32(tm + 224, w);  // not written by the store (column 264 is beyond): sanity
  float w2[32];
  tmem_ld32(tm + 256 - 32, w2);
  tmem_ld_wait();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_free<256>(tbase); }
}

int main() {
  int* d; cudaMalloc(&d, 4096 * 4); cudaMemset(d, 0, 4096 * 4);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  int h[512]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(e));
  for (int t = 0; t < 32; t += 5) printf("base0 t%2d: %d %d %d %d\n", t, h[t*4], h[t*4+1], h[t*4+2], h[t*4+3]);
  for (int t = 0; t < 32; t += 5) printf("base16 t%2d: %d %d %d %d\n", t, h[128+t*4], h[128+t*4+1], h[128+t*4+2], h[128+t*4+3]);
  for (int l = 0; l < 32; l += 3) printf("st lane %2d: col200 %d col201 %d\n", l, h[256+l*2], h[256+l*2+1]);
  return 0;
}
