// K1 permute-in, K5 permute-out, K2 region pooling, K3a draft scores.
//
// K1/K5 and K2 are HBM-bound: one CTA per (head, region) moves the region's p
// rows with 16-byte vector accesses; the region's coordinates are decoded once
// per CTA. K3a is a float64 GEMM (g x d x g per head): 128 x 128 output tiles,
// 8 x 8 register blocking, k-chunks staged through shared memory; its epilogue
// can also histogram the top 11 bits of the selection keys (digit 0 of K3b).
#include "common.cuh"
#include "kernels.h"

namespace da {

// ---------------------------------------------------------------------------
// K1 / K5
// ---------------------------------------------------------------------------
struct RegionCoord {
  int f, y0, x0, vy, vx;  // frame, first row / column, valid rows / columns
};

DA_DEV RegionCoord region_coord(const Geo& g, int i) {
  int f = i / (g.Ph * g.Pw);
  int rest = i - f * g.Ph * g.Pw;
  int a = rest / g.Pw, b = rest - a * g.Pw;
  RegionCoord rc{f, a * g.ph, b * g.pw, 0, 0};
  rc.vy = min(g.ph, g.H - rc.y0);
  rc.vx = min(g.pw, g.W - rc.x0);
  return rc;
}

// Real row of offset r inside the region, or -1.
DA_DEV long long region_real_row(const Geo& g, const RegionCoord& rc, int r) {
  int u = r / g.pw, v = r - u * g.pw;
  if (u >= rc.vy || v >= rc.vx) return -1;
  return ((long long)rc.f * g.H + rc.y0 + u) * g.W + rc.x0 + v;
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
// grid: (g, heads, tensors); block = RG row groups x d8 column chunks. Up to
// two tensors (Q and K) per launch.
// ---------------------------------------------------------------------------
struct PoolSrc {
  const __nv_bfloat16* x[3];  // Q, K (pooled) and V (tiled only)
  long long hs[3], rs[3];
  double* out[2];
  uint8_t* tile[2];           // optional K / V region tiles for the attention kernel (z = 1, 2)
  unsigned long long* pnorm;  // optional [heads][2]: largest pooled row norm^2 of Q (0) and K (1), as double bits
  Shards sh;                  // sequence shards of Q, K, V (z = 0, 1, 2), or unsplit
};
// element z of a 2- or 3-entry parameter array, selected without dynamic
// indexing (which would copy the kernel parameters to local memory)
template <class T>
DA_DEV T pick3(const T (&a)[3], int z) { return z == 0 ? a[0] : (z == 1 ? a[1] : a[2]); }
template <class T>
DA_DEV T pick2(const T (&a)[2], int z) { return z == 0 ? a[0] : a[1]; }

__global__ void __launch_bounds__(256) pool_kernel(const __grid_constant__ PoolSrc src, int d, int mode, Geo g) {
  extern __shared__ double red[];  // [RG][d]
  const int i = blockIdx.x, h = blockIdx.y, z = blockIdx.z;
  const int d8 = d / 8;
  const int RG = blockDim.x / d8;
  const int tid = threadIdx.x;
  const int k = tid % d8, rg = tid / d8;
  const RegionCoord rc = region_coord(g, i);
  const __nv_bfloat16* xz = pick3(src.x, z);
  const long long ho = h * pick3(src.hs, z);
  const long long rs = pick3(src.rs, z);
  double acc[8];
  const double init = mode == 0 ? 0.0 : -INFINITY;
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = init;
  // rows of the region: (u, v) with u < vy, v < vx, visited as r = u*pw + v
  if (mode == 0 && g.p == 4 * RG) {
    // common case (8x8 pool, d = 128: four rows per thread): all four 16-byte
    // loads in flight before any accumulation
    uint4 q[4];
    bool ok[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = rg + i * RG;
      const int u = r / g.pw, v = r - u * g.pw;
      ok[i] = u < rc.vy && v < rc.vx;
      const long long row = ((long long)rc.f * g.H + rc.y0 + u) * g.W + rc.x0 + v;
      q[i] = ok[i] ? __ldg(reinterpret_cast<const uint4*>(shard_addr(src.sh, z, xz, ho, row, rs)) + k)
                   : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!ok[i]) continue;  // padding rows are not summed (keeps -0.0 sums bit-exact)
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&q[i]);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += (double)__bfloat162float(b[e]);
    }
  } else
  for (int r = rg; r < g.p; r += RG) {
    const int u = r / g.pw, v = r - u * g.pw;
    if (u >= rc.vy || v >= rc.vx) continue;
    const long long row = ((long long)rc.f * g.H + rc.y0 + u) * g.W + rc.x0 + v;
    uint4 q = __ldg(reinterpret_cast<const uint4*>(shard_addr(src.sh, z, xz, ho, row, rs)) + k);
    const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&q);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const double xv = (double)__bfloat162float(b[e]);
      acc[e] = mode == 0 ? acc[e] + xv : fmax(acc[e], xv);
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[rg * d + k * 8 + e] = acc[e];
  __syncthreads();
  for (int c = tid; c < d; c += blockDim.x) {
    const int cnt = rc.vy * rc.vx;
    double s = red[c];
    for (int q = 1; q < RG; ++q) s = mode == 0 ? s + red[q * d + c] : fmax(s, red[q * d + c]);
    double outv;
    if (mode == 0) outv = s / (double)(cnt > 1 ? cnt : 1);
    else outv = cnt > 0 ? s : 0.0;
    pick2(src.out, z)[((long long)h * g.g + i) * d + c] = outv;
  }
}

// ---------------------------------------------------------------------------
// K3a: scores[h] = (qp[h] kp[h]^T) * scale in float64.
// 128x128 output tile per CTA, 256 threads (16 x 16), 8 x 8 outputs per thread
// at stride 16 (broadcast / conflict-free shared reads), k-chunks of 8 with a
// register prefetch of the next chunk.
// ---------------------------------------------------------------------------
constexpr int DT = 128, DK = 8;

__global__ void __launch_bounds__(256) draft_gemm_kernel(const double* __restrict__ qp, const double* __restrict__ kp,
                                                         double* __restrict__ scores, int g, int d, double scale,
                                                         unsigned int* __restrict__ hist0, const int* __restrict__ gate = nullptr) {
  if (gate != nullptr && *gate == 0) return;  // fp64 path gated off (fp32 selection succeeded)
  __shared__ double sq[DK][DT + 1];  // +1: the transposing stores hit distinct banks
  __shared__ double sk[DK][DT + 1];
  __shared__ unsigned int sh[2048];
  const int h = blockIdx.z;
  const int i0 = blockIdx.y * DT, j0 = blockIdx.x * DT;
  const double* Q = qp + (long long)h * g * d;
  const double* K = kp + (long long)h * g * d;
  const int tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;
  if (hist0)
    for (int b = tid; b < 2048; b += 256) sh[b] = 0;
  // loader mapping: 1024 doubles per operand chunk -> 4 per thread
  // element e = tid + 256*t: row = e / DK, col = e % DK
  double pq[4], pk[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int e = tid + 256 * t;
      const int r = e / DK, c = e % DK;
      const int kk = k0 + c;
      pq[t] = (i0 + r < g && kk < d) ? __ldg(Q + (long long)(i0 + r) * d + kk) : 0.0;
      pk[t] = (j0 + r < g && kk < d) ? __ldg(K + (long long)(j0 + r) * d + kk) : 0.0;
    }
  };
  double acc[8][8];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[u][v] = 0.0;
  load(0);
  for (int k0 = 0; k0 < d; k0 += DK) {
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int e = tid + 256 * t;
      sq[e % DK][e / DK] = pq[t];
      sk[e % DK][e / DK] = pk[t];
    }
    __syncthreads();
    if (k0 + DK < d) load(k0 + DK);
#pragma unroll
    for (int c = 0; c < DK; ++c) {
      double a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = sq[c][ty + 16 * u];
#pragma unroll
      for (int v = 0; v < 8; ++v) b[v] = sk[c][tx + 16 * v];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
  }
  double* S = scores + (long long)h * g * g;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int gi = i0 + ty + 16 * u;
    if (gi >= g) continue;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int gj = j0 + tx + 16 * v;
      if (gj < g) {
        const double s = acc[u][v] * scale;
        S[(long long)gi * g + gj] = s;
        if (hist0) atomicAdd(&sh[(unsigned)(score_key(s) >> 53)], 1u);
      }
    }
  }
  if (hist0) {
    __syncthreads();
    for (int b = tid; b < 2048; b += 256)
      if (sh[b]) atomicAdd(&hist0[(long long)h * 2048 + b], sh[b]);
  }
}

// Row softmax in float64 (core.py:38-54), one warp per row.
__global__ void __launch_bounds__(256) row_softmax_kernel(double* __restrict__ scores, int g, long long rows, const int* __restrict__ gate = nullptr) {
  if (gate != nullptr && *gate == 0) return;
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

// Average pooling with one thread per (region, 8-feature chunk): the TPR = d/8
// threads of a region read its rows whole (256 B per row at d = 128, coalesced),
// eight rows in flight, and keep exact float64 sums in registers (no shared-
// memory reduction); one division by the valid count (padding.py:91-92). For
// the second tensor (K) the kernel also records the largest key row norm per
// block (kpart[h][blockIdx.x]), the bound the attention kernel's fixed softmax
// offset needs, so K is read once.
template <int TPR, bool SPLIT>  // SPLIT: rows in sequence shards (PoolSrc::sh)
#ifndef DA_POOL_MINB
#define DA_POOL_MINB 4  // 64 registers: 8 CTAs of 256 threads per SM (memory-latency bound at 2)
#endif
__global__ void __launch_bounds__(256, DA_POOL_MINB) pool_avg_kernel(const __grid_constant__ PoolSrc src, int d, Geo g,
                                                                   float* __restrict__ kpart) {
  constexpr int RPB = 256 / TPR;  // regions per block
  __shared__ float wmax[8];
  const int h = blockIdx.y, z = blockIdx.z;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * RPB + threadIdx.x / TPR;
  const int k = threadIdx.x % TPR;
  const bool live = i < g.g;
  const RegionCoord rc = region_coord(g, live ? i : 0);
  const __nv_bfloat16* xz = pick3(src.x, z);
  const long long ho = h * pick3(src.hs, z), rs = pick3(src.rs, z);
  const bool norms = z == 1 && kpart != nullptr;
  // K / V tiles ([half][64 rows x 128 B], 128-byte swizzle, zero padding rows):
  // byte-for-byte the shared-memory image the attention MMAs read (d = 128, p = 64)
  uint8_t* const tz = z >= 1 ? pick2(src.tile, z - 1) : nullptr;
  // 64 x 2^s-token regions: the tiles of their 2^s column parts, 2^s i + part
  // (the attention kernel's split mode; region_parts_shift)
  const int split = max(0, region_parts_shift(g));
  uint8_t* tdst = (tz != nullptr && live) ? tz + ((long long)h * g.g + i) * (16384 << split) : nullptr;
#ifdef DA_K4_TK
  uint4 vprev[4];  // V^T tiles (the experimental transposed K4's layout): the previous 4-row batch
#endif
  // fp64 sums of bf16 values are exact, in any order
  double acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0;
  float nmax = 0.f;
#ifndef DA_POOL_RB
#define DA_POOL_RB 4
#endif
  constexpr int RB = DA_POOL_RB;  // rows per batch (loads in flight per thread); occupancy supplies the rest
  for (int r0 = 0; r0 < g.p; r0 += RB) {
    uint4 q[RB];
    bool ok[RB];
#pragma unroll
    for (int t = 0; t < RB; ++t) {
      const int r = r0 + t;
      const int u = r / g.pw, v = r - u * g.pw;
      ok[t] = live && r < g.p && u < rc.vy && v < rc.vx;
      const long long row = ((long long)rc.f * g.H + rc.y0 + u) * g.W + rc.x0 + v;
      q[t] = ok[t] ? __ldg(reinterpret_cast<const uint4*>(shard_at<SPLIT>(src.sh, z, xz, ho, row, rs)) + k)
                   : make_uint4(0, 0, 0, 0);
    }
    if (tdst != nullptr) {
#ifndef DA_K4_TK
#pragma unroll
      for (int t = 0; t < RB; ++t) {
        const int r = r0 + t;
        if (r >= g.p) continue;
        int rt = r, half = 0;
        if (split) {
          const int pw = g.pw >> split, u = r / g.pw, v = r - u * g.pw;
          half = v / pw;  // the column part
          rt = u * pw + v - half * pw;
        }
        *reinterpret_cast<uint4*>(tdst + half * 16384 + kv_tile_offset_grouped(rt, k >> 3, k & 7)) = q[t];
      }
#else
      // the experimental transposed K4 (attn_tk.cu; probe builds only): K as
      // the GROUPED smem image, V as V^T
      if (z == 1) {
#pragma unroll
        for (int t = 0; t < RB; ++t) {
          const int r = r0 + t;
          if (r < g.p) *reinterpret_cast<uint4*>(tdst + kv_tile_offset_grouped(r, k >> 3, k & 7)) = q[t];
        }
      } else {
        // V^T: this thread holds features 8k..8k+7 of rows r0 .. r0 + RB - 1;
        // two batches make an 8 x 8 block, transposed in registers into key
        // chunk r0 / 8 (keys r0 - 4 .. r0 + 3) of feature rows 8k .. 8k + 7
        static_assert(RB == 4, "V^T tiles pair two 4-row batches");
        if ((r0 & 4) == 0) {
#pragma unroll
          for (int t = 0; t < 4; ++t) vprev[t] = q[t];
        } else {
          const uint4 rows[8] = {vprev[0], vprev[1], vprev[2], vprev[3], q[0], q[1], q[2], q[3]};
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t a = (&rows[2 * i].x)[e >> 1], b = (&rows[2 * i + 1].x)[e >> 1];
              w[i] = __byte_perm(a, b, (e & 1) ? 0x7632 : 0x5410);
            }
            *reinterpret_cast<uint4*>(tdst + ((r0 - 4) >> 3) * 2048 + (8 * k + e) * 16) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
#endif
    }
    if (z == 2) continue;  // V: tiles only
#pragma unroll
    for (int t = 0; t < RB; ++t) {
      const uint32_t wv[4] = {q[t].x, q[t].y, q[t].z, q[t].w};
      if (ok[t]) {  // padding rows are not summed (keeps -0.0 sums bit-exact)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          acc[2 * e] += (double)__uint_as_float(wv[e] << 16);
          acc[2 * e + 1] += (double)__uint_as_float(wv[e] & 0xffff0000u);
        }
      }
      if (norms) {
        float s2 = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float lo = __uint_as_float(wv[e] << 16), hi = __uint_as_float(wv[e] & 0xffff0000u);
          s2 = fmaf(lo, lo, fmaf(hi, hi, s2));
        }
#pragma unroll
        for (int o = TPR / 2; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        nmax = fmaxf(nmax, s2);
      }
    }
  }
  double pn2 = 0.0;  // this thread's share of the pooled row's squared norm
  if (live && z < 2) {
    const int cnt = rc.vy * rc.vx;
    const double div = (double)(cnt > 1 ? cnt : 1);
    double* o = pick2(src.out, z) + ((long long)h * g.g + i) * d + k * 8;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      o[e] = acc[e] / div;
      pn2 = fma(o[e], o[e], pn2);
    }
  }
  if (z < 2 && src.pnorm != nullptr) {
    // the pooled row's squared norm (its TPR threads), then the warp's largest;
    // NaN stays visible (its bits sort above every finite value)
#pragma unroll
    for (int o = TPR / 2; o; o >>= 1) pn2 += __shfl_xor_sync(0xffffffffu, pn2, o);
#pragma unroll
    for (int o = 16; o >= TPR; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, pn2, o);
      pn2 = (y != y || pn2 != pn2) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(pn2, y);
    }
    if (lane == 0) atomicMax(&src.pnorm[(long long)h * 2 + z], (unsigned long long)__double_as_longlong(pn2));
  }
  if (norms) {
#pragma unroll
    for (int o = 16; o; o >>= 1) nmax = fmaxf(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
    if (lane == 0) wmax[w] = nmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      float b = wmax[0];
      for (int j = 1; j < 8; ++j) b = fmaxf(b, wmax[j]);
      kpart[(long long)h * gridDim.x + blockIdx.x] = sqrtf(b);
    }
  }
}

template <bool SPLIT>
static void launch_pool_avg(int d, dim3 grid, const PoolSrc& src, const Geo& g, float* kp, cudaStream_t st) {
  switch (d / 8) {
    case 1: pool_avg_kernel<1, SPLIT><<<grid, 256, 0, st>>>(src, d, g, kp); break;
    case 2: pool_avg_kernel<2, SPLIT><<<grid, 256, 0, st>>>(src, d, g, kp); break;
    case 4: pool_avg_kernel<4, SPLIT><<<grid, 256, 0, st>>>(src, d, g, kp); break;
    case 8: pool_avg_kernel<8, SPLIT><<<grid, 256, 0, st>>>(src, d, g, kp); break;
    case 16: pool_avg_kernel<16, SPLIT><<<grid, 256, 0, st>>>(src, d, g, kp); break;
    default: pool_avg_kernel<32, SPLIT><<<grid, 256, 0, st>>>(src, d, g, kp); break;
  }
}

int pool_norm_blocks(int d, const Geo& g) {
  const int tpr = d / 8;
  return (tpr >= 1 && tpr <= 32 && (tpr & (tpr - 1)) == 0 && d % 8 == 0) ? (g.g + 256 / tpr - 1) / (256 / tpr) : 0;
}

cudaError_t launch_pool2(const void* x0, long long hs0, long long rs0, double* out0, const void* x1, long long hs1,
                         long long rs1, double* out1, int heads, int d, int mode, const Geo& g, cudaStream_t st,
                         float* kpart, const void* x2, long long hs2, long long rs2, uint8_t* ktile,
                         uint8_t* vtile, unsigned long long* pnorm, const Shards* sh) {
  const Shards shards = sh ? *sh : no_shards();
  if (mode == 0 && pool_norm_blocks(d, g) > 0 && rs0 % 8 == 0 && (!x1 || rs1 % 8 == 0)) {
    PoolSrc src;
    src.x[0] = static_cast<const __nv_bfloat16*>(x0);
    src.hs[0] = hs0; src.rs[0] = rs0; src.out[0] = out0;
    src.x[1] = static_cast<const __nv_bfloat16*>(x1 ? x1 : x0);
    src.hs[1] = x1 ? hs1 : hs0; src.rs[1] = x1 ? rs1 : rs0; src.out[1] = x1 ? out1 : out0;
    const bool tiles = x1 && x2 && ktile && vtile && d == 128 && region_parts_shift(g) >= 0 && rs2 % 8 == 0;
    src.x[2] = static_cast<const __nv_bfloat16*>(tiles ? x2 : x0);
    src.hs[2] = tiles ? hs2 : hs0; src.rs[2] = tiles ? rs2 : rs0;
    src.tile[0] = tiles ? ktile : nullptr;
    src.tile[1] = tiles ? vtile : nullptr;
    src.pnorm = pnorm;
    src.sh = shards;
    dim3 grid(pool_norm_blocks(d, g), heads, x1 ? (tiles ? 3 : 2) : 1);
    float* kp = x1 ? kpart : nullptr;
    if (shards.n > 1) launch_pool_avg<true>(d, grid, src, g, kp, st);
    else launch_pool_avg<false>(d, grid, src, g, kp, st);
    return cudaGetLastError();
  }
  if (kpart) return cudaErrorInvalidValue;  // norms only on the fast path

  PoolSrc src;
  src.x[0] = static_cast<const __nv_bfloat16*>(x0);
  src.hs[0] = hs0; src.rs[0] = rs0; src.out[0] = out0;
  src.x[1] = static_cast<const __nv_bfloat16*>(x1 ? x1 : x0);
  src.hs[1] = x1 ? hs1 : hs0; src.rs[1] = x1 ? rs1 : rs0; src.out[1] = x1 ? out1 : out0;
  src.sh = shards;
  const int d8 = d / 8;
  int rg = 256 / d8;
  if (rg < 1) rg = 1;
  const int threads = rg * d8;
  const size_t smem = sizeof(double) * rg * d;
  if (smem > 48 * 1024) {
    cudaError_t e = ensure_smem_optin((const void*)pool_kernel, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(g.g, heads, x1 ? 2 : 1);
  pool_kernel<<<grid, threads, smem, st>>>(src, d, mode, g);
  return cudaGetLastError();
}

cudaError_t launch_pool(const void* x, long long hs, long long rs, double* pooled, int heads, int d, int mode,
                        const Geo& g, cudaStream_t st) {
  return launch_pool2(x, hs, rs, pooled, nullptr, 0, 0, nullptr, heads, d, mode, g, st, nullptr, nullptr, 0, 0,
                      nullptr, nullptr, nullptr, nullptr);
}

cudaError_t launch_draft_scores(const double* qp, const double* kp, double* scores, int heads, int g, int d,
                                double scale, int softmax, cudaStream_t st, unsigned int* hist0, const int* gate) {
  dim3 grid((g + DT - 1) / DT, (g + DT - 1) / DT, heads);
  draft_gemm_kernel<<<grid, 256, 0, st>>>(qp, kp, scores, g, d, scale, softmax ? nullptr : hist0, gate);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !softmax) return e;
  long long rows = (long long)heads * g;
  row_softmax_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(scores, g, rows, gate);
  return cudaGetLastError();
}

}  // namespace da
