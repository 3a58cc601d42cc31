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
// S^T and O^T live in TMEM (lane = key / feature, column = query). A softmax
// thread owns one TMEM lane, i.e. one KEY: masking padded keys is a per-thread
// predicate and P^T rows go to shared memory as 128-byte swizzled rows.
// Softmax statistics are per query column: the running max m[q] lives in
// shared memory and is only recomputed (a cross-lane column reduction plus an
// O^T / l rescale of the affected columns) when a score exceeds it by more
// than TAU (log2 units) — one barrier.red.or vote per half step; row sums l[q]
// are per-thread partials reduced once per region.
//
// Roles (384 threads): warp 0 = TMA producer, warp 1 = MMA issuer (+ TMEM
// owner), warps 4-7 and 8-11 = two softmax/epilogue warpgroups. Each CTA walks
// its (head, query region) items; even items go to warpgroup 0, odd ones to
// warpgroup 1, and the producer / MMA interleave the two warpgroups step by
// step so one warpgroup's exponentials overlap the other's matrix products.
// K/V blocks are fetched by TMA either from reordered (heads, n_pad, 128)
// tensors (2-D maps) or straight from the ORIGINAL (f, y, x)-ordered tensors
// with 5-D maps whose box is one 8x8 region (out-of-bounds rows of ragged edge
// regions are zero-filled), so the patch permutation of padding.py:139-143
// costs no extra pass; the epilogue writes rows back in original order
// (padding.py:157 fused).
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace da {
namespace tc {

constexpr int P = 64;            // region size
constexpr int D = 128;           // head dim
constexpr int NWG = 2;           // softmax warpgroups
constexpr int KST = 2;           // K ring stages (one pair of key regions each)
constexpr int VST = 3;           // V ring stages (V is recycled only after the softmax + GEMM2)
constexpr int BOX = 64 * 128;    // one TMA box: 64 rows x 64 bf16 = 8 KB
constexpr int Q_BYTES = 2 * BOX;
constexpr int KV_BYTES = 4 * BOX;   // two regions x two feature halves
constexpr int P_BYTES = 128 * 128;  // 128 keys x 64 queries bf16
constexpr float TAU = 8.0f;

constexpr int SMEM_Q = 0;
constexpr int SMEM_K = SMEM_Q + NWG * Q_BYTES;
constexpr int SMEM_V = SMEM_K + KST * KV_BYTES;
constexpr int SMEM_P = SMEM_V + VST * KV_BYTES;
constexpr int SMEM_END = SMEM_P + NWG * P_BYTES;
// barriers and softmax state follow the tiles in dynamic shared memory (no
// static shared memory, so the dynamic window starts 1024-byte aligned)

constexpr uint32_t TMEM_COLS = 512;
// per warpgroup: S0 [0,64), S1 [64,128), O0 [128,192), O1 [192,256); the O
// accumulator alternates between items so the next item's GEMM2 does not wait
// for this item's epilogue
constexpr uint32_t WG_COLS = 256;
constexpr uint32_t COL_O = 128;

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
  RegionDecoder dec;
  FastDiv per_head;  // g
  long long n_pad;
  long long* trace;  // diagnostics: per-step clock64 stamps of CTA 0 (nullptr = off)
};

constexpr int TRACE_N = 1024;
#define DA_TRACE(ev, idx)                                                     \
  do {                                                                        \
    if (p.trace != nullptr && blockIdx.x == 0 && (idx) < TRACE_N)             \
      p.trace[(ev) * TRACE_N + (idx)] = (long long)clock64();                 \
  } while (0)

struct WgBars {
  uint64_t q_full, q_empty;
  uint64_t s_full[2], s_free[2];
  uint64_t p_full, p_free;
  uint64_t o_full[2], o_empty[2];
};
struct __align__(8) Bars {
  uint64_t k_full[KST], k_empty[KST];
  uint64_t v_full[VST], v_empty[VST];
  WgBars wg[NWG];
};
struct __align__(16) WgAux {
  float neg_m[P];  // -(running column max), log2 units (read as float2)
  float alpha[P];
  float red[4][P / 2];  // per-warp column partials of one 32-column half
};
struct SmemAux {
  Bars bars;
  uint32_t tmem_base;
  WgAux wg[NWG];
};
constexpr int SMEM_ALLOC = SMEM_END + (int)sizeof(SmemAux);
static_assert(SMEM_ALLOC <= 227 * 1024, "shared memory budget");

struct Item {
  int h, i, n;
  const int* cols;
};

DA_DEV bool fetch_item(const Params& p, long long it, long long items, Item& out) {
  if (it >= items) return false;
  const int g = p.geo.g;
  const int h = (int)fdiv((uint32_t)it, p.per_head);
  const int i = (int)(it - (long long)h * g);
  const int* rp = p.row_ptr + (long long)(h * p.mask_h) * (g + 1);
  const int beg = rp[i];
  out.h = h;
  out.i = i;
  out.n = rp[i + 1] - beg;
  out.cols = p.col_idx + (long long)(h * p.mask_h) * p.cap + beg;
  return true;
}

// Cursor over one warpgroup's NONEMPTY items (producer and MMA views).
struct Cursor {
  long long k;  // CTA-local item index (item = blockIdx.x + k * gridDim.x)
  Item item;
  int steps, t;
  bool active;
};

DA_DEV void cursor_seek(Cursor& c, const Params& p, long long items) {
  while (true) {
    const long long it = blockIdx.x + c.k * (long long)gridDim.x;
    if (!fetch_item(p, it, items, c.item)) {
      c.active = false;
      return;
    }
    if (c.item.n > 0) {
      c.steps = (c.item.n + 1) / 2;
      c.t = 0;
      c.active = true;
      return;
    }
    c.k += NWG;
  }
}

// Q blocks are read once (evict first); K/V blocks are re-read by ~10% of the
// head's query regions while the head is in flight (normal priority).
DA_DEV void load_region(const CUtensorMap* map, void* dst, uint64_t* bar, const Params& p, int h, int region,
                        int half, uint64_t policy = L2_EVICT_NORMAL) {
  if (p.layout == DA_LAYOUT_REORDERED) {
    tma_load_2d(dst, map, bar, half * 64, (int)(h * p.n_pad + (long long)region * P), policy);
  } else {
    const RegionXY rc = p.dec(region);
    tma_load_5d(dst, map, bar, half * 64, rc.x0, rc.y0, rc.f, h, policy);
  }
}

DA_DEV long long out_row(const Params& p, const RegionXY& rc, int region, int r) {
  if (p.layout == DA_LAYOUT_REORDERED) return (long long)region * P + r;
  const int u = r / p.geo.pw, v = r - u * p.geo.pw;
  const int y = rc.y0 + u, x = rc.x0 + v;
  if (y >= p.geo.H || x >= p.geo.W) return -1;
  return ((long long)rc.f * p.geo.H + y) * p.geo.W + x;
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

__global__ void __launch_bounds__(384, 1)
    sparse_attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();  // SWIZZLE_128B tiles need 1024-byte alignment
  SmemAux& aux = *reinterpret_cast<SmemAux*>(smem + SMEM_END);
  Bars& B = aux.bars;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long items = (long long)p.heads * p.geo.g;

  if (threadIdx.x == 0) {
    for (int s = 0; s < KST; ++s) { mbar_init(&B.k_full[s], 1); mbar_init(&B.k_empty[s], 1); }
    for (int s = 0; s < VST; ++s) { mbar_init(&B.v_full[s], 1); mbar_init(&B.v_empty[s], 1); }
    for (int w = 0; w < NWG; ++w) {
      WgBars& wb = B.wg[w];
      mbar_init(&wb.q_full, 1);
      mbar_init(&wb.q_empty, 1);
      for (int s = 0; s < 2; ++s) { mbar_init(&wb.s_full[s], 1); mbar_init(&wb.s_free[s], 128); }
      mbar_init(&wb.p_full, 128);
      mbar_init(&wb.p_free, 1);
      for (int s = 0; s < 2; ++s) { mbar_init(&wb.o_full[s], 1); mbar_init(&wb.o_empty[s], 128); }
    }
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

  // registers: the producer / MMA warpgroup hands its budget to the softmax warpgroups
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 104;");
  if (warp == 0 || warp == 2) {
    // ================= TMA producers: warp 0 = Q and K, warp 2 = V =================
    // Separate threads so the K ring (freed right after GEMM1) is never held
    // back by the V ring (freed only after the softmax and GEMM2).
    if (lane == 0) {
      const bool is_k = warp == 0;
      Cursor c[NWG];
      int qi[NWG];
      for (int w = 0; w < NWG; ++w) {
        c[w].k = w;
        qi[w] = 0;
        cursor_seek(c[w], p, items);
      }
      int kq = 0;
      while (c[0].active || c[1].active) {
#pragma unroll
        for (int w = 0; w < NWG; ++w) {
          if (!c[w].active) continue;
          Cursor& cu = c[w];
          WgBars& wb = B.wg[w];
          const int j0 = cu.item.cols[2 * cu.t];
          const int j1 = (2 * cu.t + 1 < cu.item.n) ? cu.item.cols[2 * cu.t + 1] : j0;
          if (is_k) {
            if (cu.t == 0) {
              if (qi[w] > 0) mbar_wait(&wb.q_empty, (qi[w] - 1) & 1);
              mbar_expect_tx(&wb.q_full, Q_BYTES);
              uint8_t* q = sQ + w * Q_BYTES;
              load_region(&tm_q, q, &wb.q_full, p, cu.item.h, cu.item.i, 0, L2_EVICT_FIRST);
              load_region(&tm_q, q + BOX, &wb.q_full, p, cu.item.h, cu.item.i, 1, L2_EVICT_FIRST);
            }
            const int ks = kq % KST;
            if (kq >= KST) mbar_wait(&B.k_empty[ks], ((kq / KST) - 1) & 1);
            DA_TRACE(0, kq);
            uint8_t* kb = sK + ks * KV_BYTES;  // [half][slot][64 x 128B]
            mbar_expect_tx(&B.k_full[ks], KV_BYTES);
            load_region(&tm_k, kb, &B.k_full[ks], p, cu.item.h, j0, 0);
            load_region(&tm_k, kb + BOX, &B.k_full[ks], p, cu.item.h, j1, 0);
            load_region(&tm_k, kb + 2 * BOX, &B.k_full[ks], p, cu.item.h, j0, 1);
            load_region(&tm_k, kb + 3 * BOX, &B.k_full[ks], p, cu.item.h, j1, 1);
          } else {
            const int vs = kq % VST;
            if (kq >= VST) mbar_wait(&B.v_empty[vs], ((kq / VST) - 1) & 1);
            DA_TRACE(1, kq);
            uint8_t* vb = sV + vs * KV_BYTES;  // [slot][half][64 x 128B]
            mbar_expect_tx(&B.v_full[vs], KV_BYTES);
            load_region(&tm_v, vb, &B.v_full[vs], p, cu.item.h, j0, 0);
            load_region(&tm_v, vb + BOX, &B.v_full[vs], p, cu.item.h, j0, 1);
            load_region(&tm_v, vb + 2 * BOX, &B.v_full[vs], p, cu.item.h, j1, 0);
            load_region(&tm_v, vb + 3 * BOX, &B.v_full[vs], p, cu.item.h, j1, 1);
          }
          ++kq;
          if (++cu.t == cu.steps) {
            ++qi[w];
            cu.k += NWG;
            cursor_seek(cu, p, items);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    if (lane == 0) {
      constexpr uint32_t IDESC1 = umma_idesc_bf16(128, 64, 0, 0);  // K-major A, K-major B
      constexpr uint32_t IDESC2 = umma_idesc_bf16(128, 64, 1, 1);  // MN-major A, MN-major B
      // descriptor templates; start addresses (>> 4) are added to the low word
      const uint64_t dK = umma_desc_sw128(0, 16, 1024);
      const uint64_t dV = umma_desc_sw128(0, BOX, 1024);
      const uint32_t aQ = smem_u32(sQ) >> 4, aK = smem_u32(sK) >> 4, aV = smem_u32(sV) >> 4;
      const uint32_t aP = smem_u32(sP) >> 4;
      Cursor c[NWG];
      int qi[NWG];
      long long G[NWG];
      for (int w = 0; w < NWG; ++w) {
        c[w].k = w;
        qi[w] = 0;
        G[w] = 0;
        cursor_seek(c[w], p, items);
      }
      int kq = 0, vq = 0;
      // GEMM2 of a warpgroup's step is issued after the GEMM1 of its NEXT step,
      // so S(t+1) is computed while the softmax of step t runs (per-warpgroup
      // lookahead); issue order stays the global step order, as the V ring needs
      struct Pend {
        int w, qi;
        long long G;
        bool first, last, valid;
      } pend[NWG];
      for (int w = 0; w < NWG; ++w) pend[w].valid = false;
      auto gemm2 = [&](const Pend& s) {
        WgBars& wb = B.wg[s.w];
        const int vs = vq % VST;
        DA_TRACE(13, vq);
        mbar_wait(&B.v_full[vs], (vq / VST) & 1);
        DA_TRACE(3, vq);
        mbar_wait(&wb.p_full, (uint32_t)(s.G & 1));
        DA_TRACE(4, vq);
        const int ob = s.qi & 1;  // O buffer of this item
        if (s.first && s.qi >= 2) mbar_wait(&wb.o_empty[ob], ((s.qi >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t vbase = aV + vs * (KV_BYTES >> 4);
        const uint32_t pbase = aP + s.w * (P_BYTES >> 4);
        const uint32_t dO = tmem + s.w * WG_COLS + COL_O + ob * 64;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a = dV + (uint64_t)(vbase + (kk >> 2) * (2 * BOX >> 4) + (kk & 3) * (2048 >> 4));
          const uint64_t b = dV + (uint64_t)(pbase + kk * (2048 >> 4));
          umma_bf16(dO, a, b, IDESC2, (s.first && kk == 0) ? 0u : 1u);
        }
        umma_commit(&B.v_empty[vs]);
        umma_commit(&wb.p_free);
        if (s.last) umma_commit(&wb.o_full[ob]);
        ++vq;
      };
      while (c[0].active || c[1].active) {
#pragma unroll
        for (int w = 0; w < NWG; ++w) {
          if (!c[w].active) {
            if (pend[w].valid) {  // this warpgroup has no more steps: retire its last GEMM2 in order
              gemm2(pend[w]);
              pend[w].valid = false;
            }
            continue;
          }
          Cursor& cu = c[w];
          WgBars& wb = B.wg[w];
          if (cu.t == 0) mbar_wait(&wb.q_full, qi[w] & 1);
          const int ks = kq % KST;
          DA_TRACE(15, kq);
          mbar_wait(&B.k_full[ks], (kq / KST) & 1);
          DA_TRACE(2, kq);
          const int b = (int)(G[w] & 1);
          if (G[w] >= 2) mbar_wait(&wb.s_free[b], (uint32_t)(((G[w] >> 1) - 1) & 1));
          DA_TRACE(12, kq);
          tc_fence_after();
          const uint32_t kbase = aK + ks * (KV_BYTES >> 4);
          const uint32_t qbase = aQ + w * (Q_BYTES >> 4);
          const uint32_t dS = tmem + w * WG_COLS + b * 64;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t a = dK + (uint64_t)(kbase + (kk >> 2) * (2 * BOX >> 4) + (kk & 3) * 2);
            const uint64_t bq = dK + (uint64_t)(qbase + (kk >> 2) * (BOX >> 4) + (kk & 3) * 2);
            umma_bf16(dS, a, bq, IDESC1, kk > 0 ? 1u : 0u);
          }
          umma_commit(&B.k_empty[ks]);
          umma_commit(&wb.s_full[b]);
          if (cu.t == cu.steps - 1) umma_commit(&wb.q_empty);
          ++kq;
          if (pend[w].valid) gemm2(pend[w]);
          pend[w].w = w;
          pend[w].qi = qi[w];
          pend[w].G = G[w];
          pend[w].first = cu.t == 0;
          pend[w].last = cu.t == cu.steps - 1;
          pend[w].valid = true;
          ++G[w];
          if (++cu.t == cu.steps) {
            ++qi[w];
            cu.k += NWG;
            cursor_seek(cu, p, items);
          }
        }
      }
      for (int w = 0; w < NWG; ++w)
        if (pend[w].valid) gemm2(pend[w]);
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
    // ===================== softmax / epilogue warpgroups ====================
    const int wg = (warp - 4) >> 2;
    const int tid = threadIdx.x - 128 - wg * 128;  // key / feature lane 0..127
    const int q4 = tid >> 5;
    const int bar_id = 1 + wg;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t tbase = tmem + wg * WG_COLS + lane_off;
    WgBars& wb = B.wg[wg];
    WgAux& X = aux.wg[wg];
    uint8_t* myP = sP + wg * P_BYTES;
    const int slot = tid >> 6, r = tid & 63;
    const int ru = r / p.geo.pw, rv = r - ru * p.geo.pw;  // in-patch row / column of my key
    const float sl2 = p.scale_log2;
    long long G = 0;
    int qi = 0;
    for (long long k = wg;; k += NWG) {
      Item itm;
      if (!fetch_item(p, blockIdx.x + k * (long long)gridDim.x, items, itm)) break;
      const int i = itm.i, n = itm.n;
      __nv_bfloat16* outh = p.out + itm.h * p.oh;
      const RegionXY qrc = p.layout == DA_LAYOUT_REORDERED ? RegionXY{0, 0, 0} : p.dec(i);
      if (n == 0) {
        // no kept key region: zero rows (sparse.py:137-138)
        for (int c = tid; c < P * (D / 8); c += 128) {
          const long long row = out_row(p, qrc, i, c >> 4);
          if (row >= 0) reinterpret_cast<uint4*>(outh + row * p.orow)[c & 15] = make_uint4(0, 0, 0, 0);
        }
        continue;
      }
      const int steps = (n + 1) / 2;
      const int ob = qi & 1;
      const uint32_t tO = tbase + COL_O + ob * 64;  // this item's O^T accumulator
      float2 l2[P / 2];
#pragma unroll
      for (int c = 0; c < P / 2; ++c) l2[c] = make_float2(0.f, 0.f);
      bool mvalid = false;
      for (int t = 0; t < steps; ++t) {
        const int b = (int)(G & 1);
        const int js = 2 * t + slot;
        bool valid = false;
        if (js < n) {
          const int j = itm.cols[js];
          if (p.key_valid != nullptr) {
            valid = p.key_valid[(long long)j * P + r] != 0;
          } else {
            const RegionXY kc = p.dec(j);
            valid = (kc.y0 + ru < p.geo.H) && (kc.x0 + rv < p.geo.W);
          }
        }
        const float vf = valid ? 1.f : 0.f;
        const uint32_t vmask = valid ? 0xffffffffu : 0u;
        if (tid == 0) DA_TRACE(11 + 3 * wg, G);
        mbar_wait(&wb.s_full[b], (uint32_t)((G >> 1) & 1));
        if (tid == 0) DA_TRACE(5 + 3 * wg, G);
        tc_fence_after();
        const uint32_t sa = tbase + b * 64;
        const uint32_t prow = smem_u32(myP) + tid * 128;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          float x[32];
          tmem_ld32(sa + hf * 32, x);
          tmem_ld_wait();
          bool exceed = !mvalid;
          if (mvalid) {
            float emax = -INFINITY;
#pragma unroll
            for (int c = 0; c < 32; c += 2) {
              const float2 nm = *reinterpret_cast<const float2*>(&X.neg_m[hf * 32 + c]);
              const float2 e = ffma2(make_float2(x[c], x[c + 1]), make_float2(sl2, sl2), nm);
              x[c] = e.x;
              x[c + 1] = e.y;
              emax = fmaxf(emax, fmaxf(e.x, e.y));
            }
            exceed = valid && emax > TAU;
          }
          if (bar_red_or(bar_id, 128, exceed)) {
            // (re)establish the running max of these 32 columns over this step's keys
            tmem_ld32(sa + hf * 32, x);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 32; ++c) x[c] = valid ? x[c] * sl2 : -INFINITY;
            {
              float tmp[32];
#pragma unroll
              for (int c = 0; c < 32; ++c) tmp[c] = x[c];
              X.red[q4][lane] = warp_col_reduce32<true>(tmp, lane);
            }
            bar_sync(bar_id, 128);
            if (tid < 32) {
              const int c = hf * 32 + tid;
              const float ms =
                  fmaxf(fmaxf(X.red[0][tid], X.red[1][tid]), fmaxf(X.red[2][tid], X.red[3][tid]));
              const float mold = mvalid ? -X.neg_m[c] : -INFINITY;
              const float mnew = fmaxf(mold, ms);
              X.alpha[c] = (mold == -INFINITY || mnew == -INFINITY) ? 0.f : exp2f(mold - mnew);
              X.neg_m[c] = -mnew;
            }
            bar_sync(bar_id, 128);
            if (mvalid) {
#pragma unroll
              for (int c = 0; c < 16; ++c) {
                l2[hf * 16 + c].x *= X.alpha[hf * 32 + 2 * c];
                l2[hf * 16 + c].y *= X.alpha[hf * 32 + 2 * c + 1];
              }
              if (t > 0) {
                // O^T holds GEMM2 results up to the previous step: wait, rescale these columns
                mbar_wait(&wb.p_free, (uint32_t)((G - 1) & 1));
                tc_fence_after();
                float o[32];
                const uint32_t oa = tO + hf * 32;
                tmem_ld32(oa, o);
                tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 32; ++c) o[c] *= X.alpha[hf * 32 + c];
                tmem_st32(oa, o);
                tmem_st_wait();
              }
            }
            const bool any = X.neg_m[hf * 32] != INFINITY;  // m finite <=> some valid key seen
#pragma unroll
            for (int c = 0; c < 32; ++c) x[c] = any ? x[c] + X.neg_m[hf * 32 + c] : -INFINITY;
          }
          // probabilities of my key for these 32 queries -> P^T row (128B-swizzled, MN-major)
          uint32_t w16[16];
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const float p0 = fast_exp2(x[c]);
            const float p1 = fast_exp2(x[c + 1]);
            l2[hf * 16 + c / 2] = ffma2(make_float2(p0, p1), make_float2(vf, vf), l2[hf * 16 + c / 2]);
            w16[c / 2] = pack_bf16(p0, p1) & vmask;
          }
          // the P^T buffer is free once the previous step's GEMM2 has consumed it
          if (hf == 0 && tid == 0) DA_TRACE(6 + 3 * wg, G);
          if (hf == 0 && G >= 1) mbar_wait(&wb.p_free, (uint32_t)((G - 1) & 1));
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            sts128(prow + (((hf * 4 + cc) ^ (tid & 7)) << 4), w16[4 * cc], w16[4 * cc + 1], w16[4 * cc + 2],
                   w16[4 * cc + 3]);
        }
        if (!mvalid) mvalid = X.neg_m[0] != INFINITY;
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&wb.p_full);
        if (tid == 0) DA_TRACE(7 + 3 * wg, G);
        mbar_arrive(&wb.s_free[b]);
        ++G;
      }
      // ------------------------------ epilogue ------------------------------
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float tmp[32];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          tmp[2 * c] = l2[hf * 16 + c].x;
          tmp[2 * c + 1] = l2[hf * 16 + c].y;
        }
        const float part = warp_col_reduce32<false>(tmp, lane);
        bar_sync(bar_id, 128);  // previous readers of red are done
        X.red[q4][lane] = part;
        bar_sync(bar_id, 128);
        if (tid < 32) X.alpha[hf * 32 + tid] = X.red[0][tid] + X.red[1][tid] + X.red[2][tid] + X.red[3][tid];
      }
      mbar_wait(&wb.o_full[ob], (uint32_t)((qi >> 1) & 1));
      tc_fence_after();
      bar_sync(bar_id, 128);
      // O^T row d = tid -> normalised bf16 into the staging tile [64 q][128 d]
      __nv_bfloat16* stage = reinterpret_cast<__nv_bfloat16*>(myP);
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float o[32];
        tmem_ld32(tO + hf * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float lq = X.alpha[hf * 32 + c];
          stage[(hf * 32 + c) * D + tid] = __float2bfloat16_rn(lq > 0.f ? o[c] / lq : 0.f);
        }
      }
      tc_fence_before();
      mbar_arrive(&wb.o_empty[ob]);
      bar_sync(bar_id, 128);
      for (int c = tid; c < P * (D / 8); c += 128) {
        const int q = c >> 4;
        const long long row = out_row(p, qrc, i, q);
        if (row >= 0)
          reinterpret_cast<uint4*>(outh + row * p.orow)[c & 15] = reinterpret_cast<const uint4*>(stage + q * D)[c & 15];
      }
      bar_sync(bar_id, 128);
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
static long long* g_trace = nullptr;  // diagnostics (da_debug_trace)
void set_tc_trace(void* buf) { g_trace = static_cast<long long*>(buf); }

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
  if (!(a.scale > 0.0)) return false;  // the fixed softmax offset bounds scale * |q| |k| from above
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
  return (long long)a.heads * g.g < (1ll << 31);
}

bool make_kv_maps(const da_attn_args& a, const Geo& g, CUtensorMap* mk, CUtensorMap* mv) {
  if (a.layout == DA_LAYOUT_REORDERED) {
    const long long rows = (long long)a.heads * g.n_pad;
    return make_map_2d(mk, a.k, rows) && make_map_2d(mv, a.v, rows);
  }
  return make_map_5d(mk, a.k, a.k_head_stride, a.k_row_stride, g, a.heads) &&
         make_map_5d(mv, a.v, a.v_head_stride, a.v_row_stride, g, a.heads);
}

cudaError_t launch_pair_attn(const da_attn_args& a, const Geo& g, cudaStream_t st, const char** why,
                             long long* trace, const float* kpart, int kblk, bool tiles_ready);

// Default: region-pair kernel (attn_pair.cu). DA_K4=transposed selects the
// single-region transposed kernel below (kept for A/B measurements).
// K4 variant: 2 lane-half kernel (attn_lh.cu, default), 0 pair kernel
// (DA_K4=pair; also the block-sparse seam), 1 transposed (DA_K4=transposed)
static int k4_variant() {
  static int variant = -1;
  if (variant < 0) {
    const char* env = getenv("DA_K4");
    variant = (env && strcmp(env, "transposed") == 0) ? 1 : (env && strcmp(env, "pair") == 0) ? 0 : 2;
  }
  return variant;
}
bool attn_tiles_grouped() { return k4_variant() == 2; }

cudaError_t launch_tc_attn(const da_attn_args& a, const Geo& g, cudaStream_t st, const char** why,
                           const float* kpart, int kblk, bool tiles_ready) {
  const int variant = k4_variant();
  if (variant == 0) return launch_pair_attn(a, g, st, why, g_trace, kpart, kblk, tiles_ready);
  if (variant == 2) return launch_lh_attn(a, g, st, why, g_trace, kpart, kblk, tiles_ready);
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
  p.dec = make_decoder(g);
  p.per_head = make_fastdiv((uint32_t)g.g);
  p.n_pad = g.n_pad;
  p.trace = g_trace;
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
  tc::sparse_attn_tc_kernel<<<grid, 384, tc::SMEM_ALLOC, st>>>(mq, mk, mv, p);
  return cudaGetLastError();
}

}  // namespace da
