// Portable block-sparse attention forward (CUDA cores, fp32 math) for region
// sizes / head dims the tcgen05 kernel does not cover (e.g. the tiny config:
// 4x4 pool, d=64). Same semantics as the reference executor
// (sparse.py:88-166): per query region, kept key regions in ascending order,
// streaming softmax over valid keys, fully dropped rows -> 0.
//
// grid: (g, heads); block 256. Shared memory: a chunk of qc query rows (Q and
// the output accumulator, fp32), per-row m / l, and one key chunk: K and V
// rows (fp32) and the qc x kc score tile. Large regions run as several query
// chunks (each streams the region's keys again).
#include "common.cuh"
#include "kernels.h"

namespace da {

struct PortableArgs {
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  __nv_bfloat16* out;
  long long qh, qr, kh, kr, vh, vr, oh, orow;
  int d, dv, layout;
  float scale;
  const int* row_ptr;
  const int* col_idx;
  long long cap;
  const uint8_t* key_valid;
  int mask_h;  // 1 = per-head masks, 0 = head 0's mask for all heads
  int kc;      // key rows per chunk (portable_chunks)
  int qc;      // query rows per chunk
  Geo geo;
  Shards sh;   // sequence shards (original layout), or unsplit
};

// row of token (region, offset) in the caller's tensor; -1 = not stored
DA_DEV long long token_row(const PortableArgs& a, int region, int r) {
  if (a.layout == DA_LAYOUT_REORDERED) return (long long)region * a.geo.p + r;
  return real_row(a.geo, region, r);
}

DA_DEV bool key_ok(const PortableArgs& a, int region, int r) {
  if (a.key_valid != nullptr) return a.key_valid[(long long)region * a.geo.p + r] != 0;
  return key_is_valid(a.geo, region, r);
}

// One query region i of head h (the whole block; block-uniform control flow).
// Each kept key region is consumed in chunks of kc key rows so that large
// regions (8x16 pools: p = 128) fit in shared memory with d = 128.
__device__ void portable_region(const PortableArgs& a, int i, int h, float* sm) {
  const int p = a.geo.p, d = a.d, dv = a.dv, kc = a.kc, qc = a.qc;
  float* Qs = sm;                 // qc*d
  float* O = Qs + qc * d;         // qc*dv
  float* M = O + qc * dv;         // qc
  float* L = M + qc;              // qc
  float* alpha = L + qc;          // qc
  float* Ks = alpha + qc;         // kc*d
  float* Vs = Ks + kc * d;        // kc*dv
  float* S = Vs + kc * dv;        // qc*kc
  int* kval = reinterpret_cast<int*>(S + qc * kc);  // kc

  const int tid = threadIdx.x, nt = blockDim.x;
  const int g = a.geo.g;
  const int* rp = a.row_ptr + (long long)(h * a.mask_h) * (g + 1);
  const int beg = rp[i], end = rp[i + 1];
  const int* cols = a.col_idx + (long long)(h * a.mask_h) * a.cap;

  for (int q0 = 0; q0 < p; q0 += qc) {
    const int nq = min(qc, p - q0);
    for (int e = tid; e < nq * d; e += nt) {
      int r = e / d, c = e - r * d;
      long long row = token_row(a, i, q0 + r);
      Qs[e] = row >= 0 ? __bfloat162float(*shard_addr(a.sh, SH_Q, a.q, h * a.qh + c, row, a.qr)) : 0.f;
    }
    for (int e = tid; e < nq * dv; e += nt) O[e] = 0.f;
    for (int r = tid; r < nq; r += nt) { M[r] = -INFINITY; L[r] = 0.f; }
    __syncthreads();

    for (int t = beg; t < end; ++t) {
      const int j = cols[t];
      for (int c0 = 0; c0 < p; c0 += kc) {
        const int nc = min(kc, p - c0);
        for (int e = tid; e < nc * d; e += nt) {
          int r = e / d, c = e - r * d;
          long long row = token_row(a, j, c0 + r);
          Ks[e] = row >= 0 ? __bfloat162float(*shard_addr(a.sh, SH_K, a.k, h * a.kh + c, row, a.kr)) : 0.f;
        }
        for (int e = tid; e < nc * dv; e += nt) {
          int r = e / dv, c = e - r * dv;
          long long row = token_row(a, j, c0 + r);
          Vs[e] = row >= 0 ? __bfloat162float(*shard_addr(a.sh, SH_V, a.v, h * a.vh + c, row, a.vr)) : 0.f;
        }
        for (int r = tid; r < nc; r += nt) kval[r] = key_ok(a, j, c0 + r);
        __syncthreads();
        for (int e = tid; e < nq * nc; e += nt) {
          int r = e / nc, c = e - r * nc;
          float s = -INFINITY;
          if (kval[c]) {
            float acc = 0.f;
            for (int kk = 0; kk < d; ++kk) acc = fmaf(Qs[r * d + kk], Ks[c * d + kk], acc);
            s = acc * a.scale;
          }
          S[r * kc + c] = s;
        }
        __syncthreads();
        // per-row online softmax update, one warp per row
        const int lane = tid % 32, w = tid / 32, nw = nt / 32;
        for (int r = w; r < nq; r += nw) {
          float mx = -INFINITY;
          for (int c = lane; c < nc; c += 32) mx = fmaxf(mx, S[r * kc + c]);
#pragma unroll
          for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
          float mold = M[r];
          float mnew = fmaxf(mold, mx);
          float sum = 0.f;
          if (mnew == -INFINITY) {  // chunk entirely invalid for this row: skip
            for (int c = lane; c < nc; c += 32) S[r * kc + c] = 0.f;
          } else {
            for (int c = lane; c < nc; c += 32) {
              float s = S[r * kc + c];
              float pr = s == -INFINITY ? 0.f : expf(s - mnew);
              S[r * kc + c] = pr;
              sum += pr;
            }
          }
#pragma unroll
          for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
          __syncwarp();  // every lane has read M[r] before lane 0 rewrites it
          if (lane == 0) {
            float al = (mold == -INFINITY) ? 0.f : expf(mold - mnew);
            if (mnew == -INFINITY) al = 1.f;
            alpha[r] = al;
            L[r] = L[r] * al + sum;
            M[r] = mnew;
          }
        }
        __syncthreads();
        for (int e = tid; e < nq * dv; e += nt) {
          int r = e / dv, c = e - r * dv;
          float acc = O[e] * alpha[r];
          for (int kk = 0; kk < nc; ++kk) acc = fmaf(S[r * kc + kk], Vs[kk * dv + c], acc);
          O[e] = acc;
        }
        __syncthreads();
      }
    }
    for (int e = tid; e < nq * dv; e += nt) {
      int r = e / dv, c = e - r * dv;
      long long row = token_row(a, i, q0 + r);
      if (row < 0) continue;
      float l = L[r];
      float o = l > 0.f ? O[e] / l : 0.f;
      *shard_addr(a.sh, SH_O, a.out, h * a.oh + c, row, a.orow) = __float2bfloat16_rn(o);
    }
    __syncthreads();  // shared tiles are reused by the next query chunk / region
  }
  if (a.sh.n > 1) __threadfence_system();  // rows stored into peer GPUs' shards
}

__global__ void __launch_bounds__(256) portable_attn_kernel(const __grid_constant__ PortableArgs a) {
  extern __shared__ float sm[];
  portable_region(a, blockIdx.x, blockIdx.y, sm);
}

// Regions listed in items[0 .. *count): the tcgen05 kernel's fallback rows.
__global__ void __launch_bounds__(256) portable_list_kernel(const __grid_constant__ PortableArgs a, const int* __restrict__ items,
                                                            const int* __restrict__ count) {
  extern __shared__ float sm[];
  const int n = *count;
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const int it = items[b];
    portable_region(a, it % a.geo.g, it / a.geo.g, sm);
  }
}

static size_t portable_smem_for(int qc, int d, int dv, int kc) {
  return sizeof(float) * ((size_t)qc * d + (size_t)qc * dv + 3 * (size_t)qc + (size_t)kc * (d + dv + qc)) +
         sizeof(int) * kc;
}

// Query and key chunks whose tiles fit in the 227 KB of shared memory a CTA
// may opt into: the whole region if possible, else the most query rows (each
// query chunk re-streams the keys) with the largest key chunk; {0, 0} if none.
struct Chunks {
  int qc, kc;
};
static Chunks portable_chunks(int p, int d, int dv) {
  constexpr size_t kMax = 227 * 1024;
  auto fit = [&](int qc, Chunks& out) {
    if (portable_smem_for(qc, d, dv, p) <= kMax) {
      out = {qc, p};
      return true;
    }
    for (int kc = 256; kc >= 1; kc >>= 1)
      if (kc < p && portable_smem_for(qc, d, dv, kc) <= kMax) {
        out = {qc, kc};
        return true;
      }
    return false;
  };
  Chunks c = {0, 0};
  if (fit(p, c)) return c;
  int q = 1;
  while (2 * q < p) q *= 2;  // the largest power of two below p
  for (; q >= 1; q >>= 1)
    if (fit(q, c)) return c;
  return c;
}

size_t portable_smem_bytes(int p, int d, int dv) {
  const Chunks c = portable_chunks(p, d, dv);
  return c.qc ? portable_smem_for(c.qc, d, dv, c.kc) : ~size_t(0);
}

static PortableArgs portable_args(const da_attn_args& args, const Geo& geo) {
  PortableArgs a;
  a.q = static_cast<const __nv_bfloat16*>(args.q);
  a.k = static_cast<const __nv_bfloat16*>(args.k);
  a.v = static_cast<const __nv_bfloat16*>(args.v);
  a.out = static_cast<__nv_bfloat16*>(args.out);
  a.qh = args.q_head_stride; a.qr = args.q_row_stride;
  a.kh = args.k_head_stride; a.kr = args.k_row_stride;
  a.vh = args.v_head_stride; a.vr = args.v_row_stride;
  a.oh = args.o_head_stride; a.orow = args.o_row_stride;
  a.d = args.d; a.dv = args.dv; a.layout = args.layout;
  a.scale = (float)args.scale;
  a.row_ptr = args.row_ptr; a.col_idx = args.col_idx; a.cap = args.mask_cap;
  a.key_valid = args.key_valid;
  a.mask_h = args.shared_mask ? 0 : 1;
  const Chunks ch = portable_chunks(geo.p, args.d, args.dv);
  a.kc = ch.kc;
  a.qc = ch.qc;
  a.geo = geo;
  a.sh = make_shards(args);
  return a;
}

cudaError_t launch_portable_attn(const da_attn_args& args, const Geo& geo, cudaStream_t st) {
  const PortableArgs a = portable_args(args, geo);
  size_t smem = portable_smem_bytes(geo.p, args.d, args.dv);
  cudaError_t e = ensure_smem_optin((const void*)portable_attn_kernel, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(geo.g, args.heads);
  portable_attn_kernel<<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_portable_list(const da_attn_args& args, const Geo& geo, cudaStream_t st, const int* items,
                                 const int* count, int blocks) {
  const PortableArgs a = portable_args(args, geo);
  size_t smem = portable_smem_bytes(geo.p, args.d, args.dv);
  cudaError_t e = ensure_smem_optin((const void*)portable_list_kernel, (int)smem);
  if (e != cudaSuccess) return e;
  portable_list_kernel<<<blocks, 256, smem, st>>>(a, items, count);
  return cudaGetLastError();
}

}  // namespace da
