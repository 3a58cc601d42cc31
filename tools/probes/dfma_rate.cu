// Probe: DFMA throughput per SM (fp64 CUDA-core ceiling for the draft GEMM).
#include <cstdio>
__global__ void dfma(int reps, double* out, long long* cyc) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 8); cudaMalloc(&c, 8 * 148);
  for (int threads : {256, 512, 1024}) {
    const int reps = 2000;
    dfma<<<148, threads>>>(reps, o, c);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d: %.1f DFMA/clk/SM\n", threads, (double)threads * reps * 16 / h);
  }
  return 0;
}
