// K1 permute-in, K5 permute-out, K2 region pooling, K3a draft scores.
//
// K1/K5 and K2 are HBM-bound: one CTA per (head, region) moves the region's p
// rows with 16-byte vector accesses; the region's coordinates are decoded once
// per CTA so the per-chunk index math is a shift and an add. K3a is a small
// float64 GEMM (g x d x g per head) tiled through shared memory.
#include "common.cuh"
#include "kernels.h"

namespace da {

// ---------------------------------------------------------------------------
// K1 / K5
// ---------------------------------------------------------------------------
struct RegionCoord {
  int f, y0, x0;
};

DA_DEV RegionCoord region_coord(const Geo& g, int i) {
  int f = i / (g.Ph * g.Pw);
  int rest = i - f * g.Ph * g.Pw;
  int a = rest / g.Pw, b = rest - a * g.Pw;
  return {f, a * g.ph, b * g.pw};
}

// Real row of offset r inside the region, or -1.
DA_DEV long long region_real_row(const Geo& g, const RegionCoord& rc, int r) {
  int u = r / g.pw, v = r - u * g.pw;
  int y = rc.y0 + u, x = rc.x0 + v;
  if (y >= g.H || x >= g.W) return -1;
  return ((long long)rc.f * g.H + y) * g.W + x;
}

// grid: (g regions, heads); block 256. d8 = d / 8 sixteen-byte chunks per row.
__global__ void __launch_bounds__(256) permute_in_kernel(const uint4* __restrict__ x, long long head_stride8,
                                                         long long row_stride8, uint4* __restrict__ x_r, int d8,
                                                         Geo g) {
  const int i = blockIdx.x, h = blockIdx.y;
  const RegionCoord rc = region_coord(g, i);
  const uint4* src = x + h * head_stride8;
  uint4* dst = x_r + ((long long)h * g.n_pad + (long long)i * g.p) * d8;
  const int total = g.p * d8;
  for (int c = threadIdx.x; c < total; c += blockDim.x) {
    int r = c / d8, k = c - r * d8;
    long long row = region_real_row(g, rc, r);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row >= 0) v = __ldg(src + row * row_stride8 + k);
    dst[c] = v;
  }
}

__global__ void __launch_bounds__(256) permute_out_kernel(const uint4* __restrict__ o_r, uint4* __restrict__ out,
                                                          long long head_stride8, long long row_stride8, int d8,
                                                          Geo g) {
  const int i = blockIdx.x, h = blockIdx.y;
  const RegionCoord rc = region_coord(g, i);
  const uint4* src = o_r + ((long long)h * g.n_pad + (long long)i * g.p) * d8;
  uint4* dst = out + h * head_stride8;
  const int total = g.p * d8;
  for (int c = threadIdx.x; c < total; c += blockDim.x) {
    int r = c / d8, k = c - r * d8;
    long long row = region_real_row(g, rc, r);
    if (row >= 0) dst[row * row_stride8 + k] = __ldg(src + c);
  }
}

// ---------------------------------------------------------------------------
// K2 pooling: float64 sums of bf16 values (exact), one division by the valid
// count (padding.py:91-92), or a coordinatewise max (pooling.py:31-32).
// grid: (g, heads); block 256 = RG row groups x d8 column chunks.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) pool_kernel(const __nv_bfloat16* __restrict__ x, long long head_stride,
                                                   long long row_stride, double* __restrict__ pooled, int d,
                                                   int mode, Geo g) {
  extern __shared__ double red[];  // [RG][d]
  const int i = blockIdx.x, h = blockIdx.y;
  const int d8 = d / 8;
  const int RG = blockDim.x / d8;  // row groups
  const int tid = threadIdx.x;
  const int k = tid % d8, rg = tid / d8;
  const RegionCoord rc = region_coord(g, i);
  const __nv_bfloat16* src = x + h * head_stride;
  double acc[8];
  const double init = mode == 0 ? 0.0 : -INFINITY;
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = init;
  int count = 0;
  if (rg < RG) {
    for (int r = rg; r < g.p; r += RG) {
      long long row = region_real_row(g, rc, r);
      if (row < 0) continue;
      ++count;
      uint4 v = __ldg(reinterpret_cast<const uint4*>(src + row * row_stride) + k);
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        double xv = (double)__bfloat162float(b[e]);
        acc[e] = mode == 0 ? acc[e] + xv : fmax(acc[e], xv);
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) red[rg * d + k * 8 + e] = acc[e];
  }
  __syncthreads();
  // valid count of the region (closed form, same for every column)
  if (tid < d) {
    const int vy = min(g.ph, g.H - rc.y0), vx = min(g.pw, g.W - rc.x0);
    const int cnt = vy * vx;
    double s = red[tid];
    for (int q = 1; q < RG; ++q) s = mode == 0 ? s + red[q * d + tid] : fmax(s, red[q * d + tid]);
    double outv;
    if (mode == 0) {
      outv = s / (double)(cnt > 1 ? cnt : 1);
    } else {
      outv = cnt > 0 ? s : 0.0;
    }
    pooled[((long long)h * g.g + i) * d + tid] = outv;
  }
  (void)count;
}

// ---------------------------------------------------------------------------
// K3a: scores[h] = (qp[h] kp[h]^T) * scale in float64.
// 64x64 output tile per CTA, 256 threads, 4x4 outputs per thread, k-chunks of
// 16 staged in shared memory (transposed so the inner loop reads broadcast-
// free float64 pairs).
// ---------------------------------------------------------------------------
constexpr int DT = 64, DK = 16;
__global__ void __launch_bounds__(256) draft_gemm_kernel(const double* __restrict__ qp, const double* __restrict__ kp,
                                                         double* __restrict__ scores, int g, int d, double scale) {
  __shared__ double sq[DK][DT + 1];
  __shared__ double sk[DK][DT + 1];
  const int h = blockIdx.z;
  const int i0 = blockIdx.y * DT, j0 = blockIdx.x * DT;
  const double* Q = qp + (long long)h * g * d;
  const double* K = kp + (long long)h * g * d;
  const int tid = threadIdx.x;
  const int ty = tid / 16, tx = tid % 16;  // 16 x 16 threads, 4 x 4 outputs each
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int k0 = 0; k0 < d; k0 += DK) {
    for (int e = tid; e < DT * DK; e += 256) {
      int r = e / DK, c = e % DK;
      int gi = i0 + r, gj = j0 + r, kk = k0 + c;
      sq[c][r] = (gi < g && kk < d) ? Q[(long long)gi * d + kk] : 0.0;
      sk[c][r] = (gj < g && kk < d) ? K[(long long)gj * d + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < DK; ++c) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = sq[c][ty + 16 * u];
        b[u] = sk[c][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
  double* S = scores + (long long)h * g * g;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    int gi = i0 + ty + 16 * u;
    if (gi >= g) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      int gj = j0 + tx + 16 * v;
      if (gj < g) S[(long long)gi * g + gj] = acc[u][v] * scale;
    }
  }
}

// Row softmax in float64 (core.py:38-54), one warp per row.
__global__ void __launch_bounds__(256) row_softmax_kernel(double* __restrict__ scores, int g, long long rows) {
  long long row = (long long)blockIdx.x * 8 + threadIdx.x / 32;
  int lane = threadIdx.x % 32;
  if (row >= rows) return;
  double* s = scores + row * g;
  double mx = -INFINITY;
  for (int j = lane; j < g; j += 32) mx = fmax(mx, s[j]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double shift = isfinite(mx) ? mx : 0.0;
  double sum = 0.0;
  for (int j = lane; j < g; j += 32) sum += exp(s[j] - shift);
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  double den = isfinite(mx) ? sum : 1.0;
  for (int j = lane; j < g; j += 32) s[j] = exp(s[j] - shift) / den;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_permute_in(const void* x, long long hs, long long rs, void* x_r, int heads, int d, const Geo& g,
                              cudaStream_t st) {
  dim3 grid(g.g, heads);
  permute_in_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(x), hs / 8, rs / 8,
                                          reinterpret_cast<uint4*>(x_r), d / 8, g);
  return cudaGetLastError();
}

cudaError_t launch_permute_out(const void* o_r, void* out, long long hs, long long rs, int heads, int d,
                               const Geo& g, cudaStream_t st) {
  dim3 grid(g.g, heads);
  permute_out_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(o_r), reinterpret_cast<uint4*>(out),
                                           hs / 8, rs / 8, d / 8, g);
  return cudaGetLastError();
}

cudaError_t launch_pool(const void* x, long long hs, long long rs, double* pooled, int heads, int d, int mode,
                        const Geo& g, cudaStream_t st) {
  int d8 = d / 8;
  int rg = 256 / d8;
  if (rg < 1) rg = 1;
  int threads = rg * d8;
  size_t smem = sizeof(double) * rg * d;
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(pool_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  dim3 grid(g.g, heads);
  pool_kernel<<<grid, threads, smem, st>>>(reinterpret_cast<const __nv_bfloat16*>(x), hs, rs, pooled, d, mode, g);
  return cudaGetLastError();
}

cudaError_t launch_draft_scores(const double* qp, const double* kp, double* scores, int heads, int g, int d,
                                double scale, int softmax, cudaStream_t st) {
  dim3 grid((g + DT - 1) / DT, (g + DT - 1) / DT, heads);
  draft_gemm_kernel<<<grid, 256, 0, st>>>(qp, kp, scores, g, d, scale);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !softmax) return e;
  long long rows = (long long)heads * g;
  row_softmax_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(scores, g, rows);
  return cudaGetLastError();
}

}  // namespace da
