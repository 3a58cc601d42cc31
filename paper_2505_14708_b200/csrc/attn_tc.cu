// K4: block-sparse FlashAttention forward on tcgen05 / TMEM / TMA (sm_100a).
//
// Shape: region size p = 64 (8x8 pool), d = dv = 128, bf16 in, fp32 accumulate.
//
// Transposed formulation. A query region has only 64 rows, but the tcgen05
// tile that runs at full rate has M = 128. Instead of pairing two query
// regions (whose kept key lists differ), each step takes TWO kept key regions
// of ONE query region and puts the 128 keys on M:
//     GEMM1  S^T[128 keys x 64 q]  = K_pair[128 x 128d] . Q^T          (K-major A and B)
//     GEMM2  O^T[128 d  x 64 q]   += V_pair^T[128d x 128 keys] . P^T    (MN-major A and B)
// S^T and O^T live in TMEM (lane = key / feature, column = query). The
// softmax warpgroup owns one TMEM lane per thread, i.e. one KEY per thread:
// masking invalid (padded) keys is a per-thread predicate and P^T rows are
// written to shared memory as 128-byte swizzled rows. Softmax statistics are
// per query column: the running max m[q] is kept in shared memory and only
// recomputed (a cross-lane column reduction, plus an O^T/l rescale) when some
// score exceeds it by more than TAU (log2 units) — a barrier.red.or vote per
// step; row sums l[q] are per-thread partials reduced once per region.
//
// Roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer (+ TMEM
// owner), warps 4..7 = softmax / epilogue warpgroup. Persistent CTAs walk the
// (head, query region) items round-robin. Key/value blocks are fetched with
// TMA either from the reordered (heads, n_pad, 128) tensors (2-D maps) or
// straight from the ORIGINAL (f, y, x)-ordered tensors with 5-D maps whose box
// is one 8x8 region (out-of-bounds rows of ragged edge regions are zero-filled
// by TMA), so the patch permutation of padding.py:139-143 costs no extra pass.
// The epilogue writes rows back in original order (padding.py:157 fused).
#include "common.cuh"
#include "kernels.h"

namespace da {
namespace tc {

constexpr int P = 64;           // region size
constexpr int D = 128;          // head dim
constexpr int KST = 3;          // K ring stages (one pair of key regions each)
constexpr int VST = 2;          // V ring stages
constexpr int BOX = 64 * 128;   // one TMA box: 64 rows x 64 bf16 = 8 KB
constexpr int Q_BYTES = 2 * BOX;
constexpr int KV_BYTES = 4 * BOX;  // two regions x two feature halves
constexpr int P_BYTES = 128 * 128; // 128 keys x 64 queries bf16
constexpr float TAU = 8.0f;

constexpr int SMEM_Q = 0;
constexpr int SMEM_K = SMEM_Q + Q_BYTES;
constexpr int SMEM_V = SMEM_K + KST * KV_BYTES;
constexpr int SMEM_P = SMEM_V + VST * KV_BYTES;
constexpr int SMEM_END = SMEM_P + 2 * P_BYTES;
constexpr int SMEM_ALLOC = SMEM_END + 1024;  // + alignment slack

constexpr uint32_t TMEM_COLS = 256;
constexpr uint32_t COL_S0 = 0, COL_S1 = 64, COL_O = 128;

struct Params {
  __nv_bfloat16* out;
  long long oh, orow;
  int heads;
  int layout;
  float scale_log2;
  const int* row_ptr;
  const int* col_idx;
  long long cap;
  const uint8_t* key_valid;
  int mask_h;  // 1 = per-head masks, 0 = shared
  Geo geo;
  long long n_pad;
};

struct __align__(8) Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[KST], k_empty[KST];
  uint64_t v_full[VST], v_empty[VST];
  uint64_t s_full[2], s_free[2];
  uint64_t p_full[2], p_free[2];
  uint64_t o_full, o_empty;
};

struct SmemAux {
  Bars bars;
  uint32_t tmem_base;
  float m[P];          // running column max (log2 units)
  float alpha[P];
  float red[4][P];     // per-warp column partials
};

DA_DEV void load_region(const CUtensorMap* map, void* dst, uint64_t* bar, const Params& p, int h, int region,
                        int half) {
  if (p.layout == DA_LAYOUT_REORDERED) {
    tma_load_2d(dst, map, bar, half * 64, (int)(h * p.n_pad + (long long)region * P));
  } else {
    const Geo& g = p.geo;
    int f = region / (g.Ph * g.Pw);
    int rest = region - f * g.Ph * g.Pw;
    int a = rest / g.Pw, b = rest - a * g.Pw;
    tma_load_5d(dst, map, bar, half * 64, b * g.pw, a * g.ph, f, h);
  }
}

DA_DEV bool key_valid_at(const Params& p, int region, int r) {
  if (p.key_valid != nullptr) return p.key_valid[(long long)region * P + r] != 0;
  return key_is_valid(p.geo, region, r);
}

DA_DEV long long out_row(const Params& p, int region, int r) {
  if (p.layout == DA_LAYOUT_REORDERED) return (long long)region * P + r;
  return real_row(p.geo, region, r);
}

// Column reduction of 32 values held one row per thread across the 32 lanes
// of a warp ("transpose-reduce": each step trades half of the remaining
// columns with lane ^ off). Lane L ends up holding column L.
template <bool IS_MAX>
DA_DEV float warp_col_reduce32(float (&v)[32], int lane) {
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int half = 16 >> k;
    const int off = 16 >> k;
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int c = 0; c < half; ++c) {
      float mine = upper ? v[c + half] : v[c];
      float send = upper ? v[c] : v[c + half];
      float recv = __shfl_xor_sync(0xffffffffu, send, off);
      v[c] = IS_MAX ? fmaxf(mine, recv) : mine + recv;
    }
  }
  return v[0];
}

__global__ void __launch_bounds__(256, 1)
    sparse_attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ SmemAux aux;
  Bars& B = aux.bars;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const Geo& geo = p.geo;
  const int g = geo.g;
  const long long items = (long long)p.heads * g;

  if (threadIdx.x == 0) {
    mbar_init(&B.q_full, 1);
    mbar_init(&B.q_empty, 1);
    for (int s = 0; s < KST; ++s) { mbar_init(&B.k_full[s], 1); mbar_init(&B.k_empty[s], 1); }
    for (int s = 0; s < VST; ++s) { mbar_init(&B.v_full[s], 1); mbar_init(&B.v_empty[s], 1); }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&B.s_full[s], 1);
      mbar_init(&B.s_free[s], 128);
      mbar_init(&B.p_full[s], 128);
      mbar_init(&B.p_free[s], 1);
    }
    mbar_init(&B.o_full, 1);
    mbar_init(&B.o_empty, 128);
    fence_barrier_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(&aux.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = aux.tmem_base;

  uint8_t* sQ = smem + SMEM_Q;
  uint8_t* sK = smem + SMEM_K;
  uint8_t* sV = smem + SMEM_V;
  uint8_t* sP = smem + SMEM_P;

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      int kq = 0, vq = 0, qi = 0;
      for (long long it = blockIdx.x; it < items; it += gridDim.x) {
        const int h = (int)(it / g), i = (int)(it % g);
        const int* rp = p.row_ptr + (long long)(h * p.mask_h) * (g + 1);
        const int beg = rp[i], n = rp[i + 1] - beg;
        if (n == 0) continue;
        const int* cols = p.col_idx + (long long)(h * p.mask_h) * p.cap + beg;
        const int steps = (n + 1) / 2;
        if (qi > 0) mbar_wait(&B.q_empty, (qi - 1) & 1);
        mbar_expect_tx(&B.q_full, Q_BYTES);
        load_region(&tm_q, sQ, &B.q_full, p, h, i, 0);
        load_region(&tm_q, sQ + BOX, &B.q_full, p, h, i, 1);
        for (int t = 0; t < steps; ++t) {
          const int j0 = cols[2 * t];
          const int j1 = (2 * t + 1 < n) ? cols[2 * t + 1] : j0;
          const int ks = kq % KST;
          if (kq >= KST) mbar_wait(&B.k_empty[ks], ((kq / KST) - 1) & 1);
          uint8_t* kb = sK + ks * KV_BYTES;  // [half][slot][64 x 128B]
          mbar_expect_tx(&B.k_full[ks], KV_BYTES);
          load_region(&tm_k, kb, &B.k_full[ks], p, h, j0, 0);
          load_region(&tm_k, kb + BOX, &B.k_full[ks], p, h, j1, 0);
          load_region(&tm_k, kb + 2 * BOX, &B.k_full[ks], p, h, j0, 1);
          load_region(&tm_k, kb + 3 * BOX, &B.k_full[ks], p, h, j1, 1);
          ++kq;
          const int vs = vq % VST;
          if (vq >= VST) mbar_wait(&B.v_empty[vs], ((vq / VST) - 1) & 1);
          uint8_t* vb = sV + vs * KV_BYTES;  // [slot][half][64 x 128B]
          mbar_expect_tx(&B.v_full[vs], KV_BYTES);
          load_region(&tm_v, vb, &B.v_full[vs], p, h, j0, 0);
          load_region(&tm_v, vb + BOX, &B.v_full[vs], p, h, j0, 1);
          load_region(&tm_v, vb + 2 * BOX, &B.v_full[vs], p, h, j1, 0);
          load_region(&tm_v, vb + 3 * BOX, &B.v_full[vs], p, h, j1, 1);
          ++vq;
        }
        ++qi;
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    if (lane == 0) {
      constexpr uint32_t IDESC1 = umma_idesc_bf16(128, 64, 0, 0);  // K-major A, K-major B
      constexpr uint32_t IDESC2 = umma_idesc_bf16(128, 64, 1, 1);  // MN-major A, MN-major B
      const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV), aP = smem_u32(sP);
      int kq = 0, vq = 0, qi = 0;
      long long G = 0;
      auto gemm2 = [&](long long Gp, bool first) {
        const int vs = vq % VST;
        mbar_wait(&B.v_full[vs], (vq / VST) & 1);
        const int pb = (int)(Gp & 1);
        mbar_wait(&B.p_full[pb], (uint32_t)((Gp >> 1) & 1));
        if (first && qi > 0) mbar_wait(&B.o_empty, (qi - 1) & 1);
        tc_fence_after();
        const uint32_t vbase = aV + vs * KV_BYTES;
        const uint32_t pbase = aP + pb * P_BYTES;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t slot = kk >> 2;
          uint64_t a = umma_desc_sw128(vbase + slot * 2 * BOX + (kk & 3) * 2048, 2 * BOX / 2, 1024);
          uint64_t b = umma_desc_sw128(pbase + kk * 2048, BOX, 1024);
          umma_bf16(tmem + COL_O, a, b, IDESC2, (first && kk == 0) ? 0u : 1u);
        }
        umma_commit(&B.v_empty[vs]);
        umma_commit(&B.p_free[pb]);
        ++vq;
      };
      for (long long it = blockIdx.x; it < items; it += gridDim.x) {
        const int h = (int)(it / g), i = (int)(it % g);
        const int* rp = p.row_ptr + (long long)(h * p.mask_h) * (g + 1);
        const int n = rp[i + 1] - rp[i];
        if (n == 0) continue;
        const int steps = (n + 1) / 2;
        mbar_wait(&B.q_full, qi & 1);
        for (int t = 0; t < steps; ++t) {
          const int ks = kq % KST;
          mbar_wait(&B.k_full[ks], (kq / KST) & 1);
          const int b = (int)(G & 1);
          if (G >= 2) mbar_wait(&B.s_free[b], (uint32_t)(((G >> 1) - 1) & 1));
          tc_fence_after();
          const uint32_t kbase = aK + ks * KV_BYTES;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            uint64_t a = umma_desc_sw128(kbase + (kk >> 2) * 2 * BOX + (kk & 3) * 32, 16, 1024);
            uint64_t bq = umma_desc_sw128(aQ + (kk >> 2) * BOX + (kk & 3) * 32, 16, 1024);
            umma_bf16(tmem + (b ? COL_S1 : COL_S0), a, bq, IDESC1, kk > 0 ? 1u : 0u);
          }
          umma_commit(&B.k_empty[ks]);
          umma_commit(&B.s_full[b]);
          if (t == steps - 1) umma_commit(&B.q_empty);
          ++kq;
          if (t >= 1) gemm2(G - 1, t == 1);
          ++G;
        }
        gemm2(G - 1, steps == 1);
        umma_commit(&B.o_full);
        ++qi;
      }
    }
  } else if (warp >= 4) {
    // ======================= softmax / epilogue warpgroup ====================
    const int tid = threadIdx.x - 128;  // key / feature lane 0..127
    const int q4 = tid >> 5;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const int slot = tid >> 6, r = tid & 63;
    long long G = 0;
    int qi = 0;
    for (long long it = blockIdx.x; it < items; it += gridDim.x) {
      const int h = (int)(it / g), i = (int)(it % g);
      const int* rp = p.row_ptr + (long long)(h * p.mask_h) * (g + 1);
      const int beg = rp[i], n = rp[i + 1] - beg;
      __nv_bfloat16* outh = p.out + h * p.oh;
      if (n == 0) {
        // no kept key region: zero rows (sparse.py:137-138)
        for (int c = tid; c < P * (D / 8); c += 128) {
          int q = c >> 4, part = c & 15;
          long long row = out_row(p, i, q);
          if (row >= 0) reinterpret_cast<uint4*>(outh + row * p.orow)[part] = make_uint4(0, 0, 0, 0);
        }
        continue;
      }
      const int* cols = p.col_idx + (long long)(h * p.mask_h) * p.cap + beg;
      const int steps = (n + 1) / 2;
      float l[P];
#pragma unroll
      for (int c = 0; c < P; ++c) l[c] = 0.f;
      bool mvalid = false;
      for (int t = 0; t < steps; ++t) {
        const int b = (int)(G & 1);
        const int js = 2 * t + slot;
        const bool valid = js < n && key_valid_at(p, cols[js], r);
        mbar_wait(&B.s_full[b], (uint32_t)((G >> 1) & 1));
        tc_fence_after();
        const uint32_t sa = tmem + lane_off + (b ? COL_S1 : COL_S0);
        float x[P];
        tmem_ld32_at<0>(sa, x);
        tmem_ld32_at<32>(sa + 32, x);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < P; ++c) x[c] = valid ? x[c] * p.scale_log2 : -INFINITY;
        bool exceed = !mvalid;
        if (mvalid) {
#pragma unroll
          for (int c = 0; c < P; ++c) exceed |= (x[c] - aux.m[c]) > TAU;
        }
        const bool need = bar_red_or(1, 128, exceed);
        if (need) {
          // column max over the 128 keys of this step (two 32-column halves)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            float tmp[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) tmp[c] = x[hf * 32 + c];
            aux.red[q4][hf * 32 + lane] = warp_col_reduce32<true>(tmp, lane);
          }
          bar_sync(1, 128);
          if (tid < P) {
            float ms = fmaxf(fmaxf(aux.red[0][tid], aux.red[1][tid]), fmaxf(aux.red[2][tid], aux.red[3][tid]));
            float mold = mvalid ? aux.m[tid] : -INFINITY;
            float mnew = fmaxf(mold, ms);
            aux.alpha[tid] = (mold == -INFINITY || mnew == -INFINITY) ? 0.f : exp2f(mold - mnew);
            aux.m[tid] = mnew;
          }
          bar_sync(1, 128);
          const bool now_valid = aux.m[0] != -INFINITY;
          if (mvalid) {
#pragma unroll
            for (int c = 0; c < P; ++c) l[c] *= aux.alpha[c];
            if (t > 0) {
              // O^T holds GEMM2 results up to step t-1: wait for it, rescale columns
              const long long Gp = G - 1;
              mbar_wait(&B.p_free[Gp & 1], (uint32_t)((Gp >> 1) & 1));
              tc_fence_after();
#pragma unroll
              for (int hf = 0; hf < 2; ++hf) {
                float o[32];
                const uint32_t oa = tmem + lane_off + COL_O + hf * 32;
                tmem_ld32(oa, o);
                tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 32; ++c) o[c] *= aux.alpha[hf * 32 + c];
                tmem_st32(oa, o);
              }
              tmem_st_wait();
            }
          }
          mvalid = now_valid;
        }
        // P^T row for this key -> shared memory (128B-swizzled, MN-major)
        if (G >= 2) mbar_wait(&B.p_free[b], (uint32_t)(((G >> 1) - 1) & 1));
        uint8_t* prow = sP + b * P_BYTES + tid * 128;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = cc * 8 + 2 * e;
            float p0 = 0.f, p1 = 0.f;
            if (mvalid) {  // invalid keys carry x = -inf -> exp2 = +0
              p0 = fast_exp2(x[c] - aux.m[c]);
              p1 = fast_exp2(x[c + 1] - aux.m[c + 1]);
            }
            l[c] += p0;
            l[c + 1] += p1;
            w[e] = pack_bf16(p0, p1);
          }
          *reinterpret_cast<uint4*>(prow + ((cc ^ (tid & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&B.p_full[b]);
        mbar_arrive(&B.s_free[b]);  // S[b] no longer needed (re-read above on the rare rescale path)
        ++G;
      }
      // ------------------------------ epilogue ------------------------------
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float tmp[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) tmp[c] = l[hf * 32 + c];
        aux.red[q4][hf * 32 + lane] = warp_col_reduce32<false>(tmp, lane);
      }
      mbar_wait(&B.o_full, qi & 1);
      tc_fence_after();
      bar_sync(1, 128);
      if (tid < P) aux.alpha[tid] = aux.red[0][tid] + aux.red[1][tid] + aux.red[2][tid] + aux.red[3][tid];
      bar_sync(1, 128);
      // O^T row d = tid -> normalised bf16 into the staging tile [64 q][128 d]
      __nv_bfloat16* stage = reinterpret_cast<__nv_bfloat16*>(sP);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float o[32];
        tmem_ld32(tmem + lane_off + COL_O + half * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float lq = aux.alpha[half * 32 + c];
          const float v = lq > 0.f ? o[c] / lq : 0.f;
          stage[(half * 32 + c) * D + tid] = __float2bfloat16_rn(v);
        }
      }
      tc_fence_before();
      mbar_arrive(&B.o_empty);
      bar_sync(1, 128);
      for (int c = tid; c < P * (D / 8); c += 128) {
        const int q = c >> 4, part = c & 15;
        const long long row = out_row(p, i, q);
        if (row >= 0)
          reinterpret_cast<uint4*>(outh + row * p.orow)[part] = reinterpret_cast<const uint4*>(stage + q * D)[part];
      }
      bar_sync(1, 128);
      ++qi;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<TMEM_COLS>(tmem);
  }
}

}  // namespace tc

// ---------------------------------------------------------------------------
// host side: tensor maps + launch
// ---------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(ptr);
  }
  return fn;
}

// 2-D map over (rows, 128) dense bf16; box 64 rows x 64 features, 128B swizzle.
static bool make_map_2d(CUtensorMap* m, const void* base, long long rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  cuuint64_t strides[1] = {128 * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 5-D map over the original token grid (d, x, y, f, head); box = one region.
static bool make_map_5d(CUtensorMap* m, const void* base, long long head_stride, long long row_stride,
                        const Geo& g, int heads) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[5] = {128, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.F, (cuuint64_t)heads};
  cuuint64_t strides[4] = {(cuuint64_t)row_stride * 2, (cuuint64_t)row_stride * 2 * g.W,
                           (cuuint64_t)row_stride * 2 * g.W * g.H, (cuuint64_t)head_stride * 2};
  cuuint32_t box[5] = {64, (cuuint32_t)g.pw, (cuuint32_t)g.ph, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tc_supported(const da_attn_args& a, const Geo& g) {
  if (a.d != 128 || a.dv != 128 || g.p != 64) return false;
  if (a.layout == DA_LAYOUT_ORIGINAL && (g.ph != 8 || g.pw != 8)) return false;
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  if (!al16(a.q) || !al16(a.k) || !al16(a.v) || !al16(a.out)) return false;
  if (a.layout == DA_LAYOUT_REORDERED) {
    // dense (heads, n_pad, 128) tensors
    if (a.q_row_stride != 128 || a.k_row_stride != 128 || a.v_row_stride != 128) return false;
    if (a.q_head_stride != g.n_pad * 128 || a.k_head_stride != g.n_pad * 128 || a.v_head_stride != g.n_pad * 128)
      return false;
  } else {
    if (a.q_row_stride % 8 || a.k_row_stride % 8 || a.v_row_stride % 8) return false;
    if (a.q_head_stride % 8 || a.k_head_stride % 8 || a.v_head_stride % 8) return false;
  }
  if (a.o_row_stride % 8 || a.o_head_stride % 8) return false;
  return true;
}

cudaError_t launch_tc_attn(const da_attn_args& a, const Geo& g, cudaStream_t st, const char** why) {
  CUtensorMap mq, mk, mv;
  bool ok;
  if (a.layout == DA_LAYOUT_REORDERED) {
    long long rows = (long long)a.heads * g.n_pad;
    ok = make_map_2d(&mq, a.q, rows) && make_map_2d(&mk, a.k, rows) && make_map_2d(&mv, a.v, rows);
  } else {
    ok = make_map_5d(&mq, a.q, a.q_head_stride, a.q_row_stride, g, a.heads) &&
         make_map_5d(&mk, a.k, a.k_head_stride, a.k_row_stride, g, a.heads) &&
         make_map_5d(&mv, a.v, a.v_head_stride, a.v_row_stride, g, a.heads);
  }
  if (!ok) {
    *why = "cuTensorMapEncodeTiled failed";
    return cudaErrorInvalidValue;
  }
  tc::Params p;
  p.out = static_cast<__nv_bfloat16*>(a.out);
  p.oh = a.o_head_stride;
  p.orow = a.o_row_stride;
  p.heads = a.heads;
  p.layout = a.layout;
  p.scale_log2 = (float)(a.scale * 1.4426950408889634);
  p.row_ptr = a.row_ptr;
  p.col_idx = a.col_idx;
  p.cap = a.mask_cap;
  p.key_valid = a.key_valid;
  p.mask_h = a.shared_mask ? 0 : 1;
  p.geo = g;
  p.n_pad = g.n_pad;
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  cudaError_t e = cudaFuncSetAttribute(tc::sparse_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       tc::SMEM_ALLOC);
  if (e != cudaSuccess) return e;
  long long items = (long long)a.heads * g.g;
  int grid = (int)(items < num_sms ? items : num_sms);
  tc::sparse_attn_tc_kernel<<<grid, 256, tc::SMEM_ALLOC, st>>>(mq, mk, mv, p);
  return cudaGetLastError();
}

}  // namespace da
