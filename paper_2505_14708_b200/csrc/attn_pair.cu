// K4: block-sparse FlashAttention forward on tcgen05 / TMEM / TMA (sm_100a),
// region-pair tiles.
//
// Shape: region size p = 64 (8x8 pool), d = dv = 128, bf16 in, fp32 accumulate.
//
// A work item is a PAIR of query regions (2i, 2i+1) of one head: 128 query
// rows, one per TMEM lane and one per softmax thread. The item walks the
// ascending UNION of the two kept key-region lists, two key regions (128 keys)
// per step; a key region kept by only one of the two query regions is masked
// for the other region's rows (whole-warp predicate). Per step:
//     GEMM1  S[128 q x 128 k]  = Q[128 x 128d] . K_pair^T      A = Q in TMEM, B = K (smem, K-major)
//     GEMM2  O[128 q x 128 d] += P[128 x 128k] . V_pair        A = P in TMEM, B = V (smem, MN-major)
// Q and P live in TMEM, so shared memory only carries the K/V tiles: an SS
// MMA at N = 64 streams 6 KB of operands per 32-cycle instruction and is
// shared-memory bound (measured 48 cycles, tools/probes/mma_rate.cu), whereas
// these TS MMAs read 4 KB per 64-cycle instruction. The union costs ~1.9x the
// MMA work of the kept pairs for i.i.d. data, but each K/V tile is fetched once
// for 128 queries.
//
// Softmax is the classic per-row form: each thread owns its row's running max
// m (log2 units, lazily raised when a score exceeds it by > TAU, with an O-row
// rescale) and running sum l. P is written back over S in TMEM as packed bf16.
//
// Roles (384 threads): warp 0 = TMA producer for K, warp 2 = TMA producer
// for V, warp 1 = MMA issuer + TMEM owner, warps 4-7 and 8-11 = two
// softmax / Q-loader / epilogue warpgroups that split each step's two key
// regions (and the feature halves of Q and O) between them. TMEM: Q [0,64), S0 [64,192),
// S1 [192,320) (double-buffered so GEMM1 of step t+1 overlaps the softmax of
// step t), O [320,448).
//
// K/V tiles come from TMA: 2-D maps over reordered (heads, n_pad, 128) tensors
// or 5-D maps (d, x, y, f, head) over the ORIGINAL token order whose box is one
// 8x8 region (ragged rows zero-filled), so the permutation of
// padding.py:139-143 is free; Q rows are read straight from the original order
// and output rows are written back to it (padding.py:157).
#include "common.cuh"
#include "kernels.h"

namespace da {
namespace pairk {

constexpr int P = 64;
constexpr int D = 128;
constexpr int KST = 3;
constexpr int VST = 3;
constexpr int BOX = 64 * 128;       // 64 rows x 64 bf16 = 8 KB
constexpr int KV_BYTES = 4 * BOX;   // two key regions x two feature halves
constexpr float TAU = 8.0f;

constexpr int SMEM_K = 0;
constexpr int SMEM_V = SMEM_K + KST * KV_BYTES;
constexpr int SMEM_END = SMEM_V + VST * KV_BYTES;

constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t COL_Q = 0, COL_S0 = 64, COL_S1 = 192, COL_O = 320;

struct Params {
  const __nv_bfloat16* q;
  long long qh, qr;
  __nv_bfloat16* out;
  long long oh, orow;
  int heads;
  int layout;
  float scale_log2;
  const int* row_ptr;
  const int* col_idx;
  long long cap;
  const uint8_t* key_valid;
  int mask_h;
  Geo geo;
  RegionDecoder dec;
  FastDiv per_head;  // pairs per head
  int npairs;
  long long n_pad;
  long long* trace;
};

struct __align__(8) Bars {
  uint64_t k_full[KST], k_empty[KST];
  uint64_t v_full[VST], v_empty[VST];
  uint64_t s_full[2], p_full[2];
  uint64_t o_step, o_full, o_empty;
  uint64_t q_full, q_empty;
};
struct SmemAux {
  Bars bars;
  uint32_t tmem_base;
  float xch[2][2 * 128];  // [step parity][warpgroup x row] block maxima
  float lsum[2][128];     // [warpgroup][row] partial row sums
};
constexpr int SMEM_ALLOC = SMEM_END + (int)sizeof(SmemAux);
static_assert(SMEM_ALLOC <= 227 * 1024, "shared memory budget");

constexpr int TRACE_N = 1024;
#define PAIR_TRACE(ev, idx)                                                   \
  do {                                                                        \
    if (p.trace != nullptr && blockIdx.x == 0 && (idx) < TRACE_N)             \
      p.trace[(ev) * TRACE_N + (idx)] = (long long)clock64();                 \
  } while (0)

// An item: query regions a = 2*ip and b = 2*ip + 1 (b may not exist) of head h.
struct PairItem {
  int h, a, b;
  const int* la;
  const int* lb;
  int na, nb;
};

DA_DEV bool fetch_pair(const Params& p, long long it, long long items, PairItem& o) {
  if (it >= items) return false;
  const int g = p.geo.g;
  const int h = (int)fdiv((uint32_t)it, p.per_head);
  const int ip = (int)(it - (long long)h * p.npairs);
  o.h = h;
  o.a = 2 * ip;
  o.b = 2 * ip + 1;
  const int* rp = p.row_ptr + (long long)(h * p.mask_h) * (g + 1);
  const int* base = p.col_idx + (long long)(h * p.mask_h) * p.cap;
  const int a0 = rp[o.a];
  o.la = base + a0;
  o.na = rp[o.a + 1] - a0;
  if (o.b < g) {
    const int b0 = rp[o.b];
    o.lb = base + b0;
    o.nb = rp[o.b + 1] - b0;
  } else {
    o.lb = base;
    o.nb = 0;
  }
  return true;
}

// Ascending merge of the two kept lists, with membership flags.
struct UnionWalk {
  const int* a;
  const int* b;
  int na, nb, ia, ib;
  DA_DEV void init(const PairItem& it) {
    a = it.la; b = it.lb; na = it.na; nb = it.nb; ia = 0; ib = 0;
  }
  DA_DEV bool done() const { return ia >= na && ib >= nb; }
  // next key region and its membership (bit 0: kept by a, bit 1: kept by b)
  DA_DEV bool next(int& j, int& flags) {
    const int va = ia < na ? __ldg(a + ia) : 0x7fffffff;
    const int vb = ib < nb ? __ldg(b + ib) : 0x7fffffff;
    if (va == 0x7fffffff && vb == 0x7fffffff) return false;
    if (va <= vb) {
      j = va;
      flags = 1;
      ++ia;
      if (vb == va) { flags |= 2; ++ib; }
    } else {
      j = vb;
      flags = 2;
      ++ib;
    }
    return true;
  }
};

DA_DEV void load_region(const CUtensorMap* map, void* dst, uint64_t* bar, const Params& p, int h, int region,
                        int half) {
  if (p.layout == DA_LAYOUT_REORDERED) {
    tma_load_2d(dst, map, bar, half * 64, (int)(h * p.n_pad + (long long)region * P));
  } else {
    const RegionXY rc = p.dec(region);
    tma_load_5d(dst, map, bar, half * 64, rc.x0, rc.y0, rc.f, h);
  }
}

// Token row of (region, r) in the caller's q/out tensors, -1 if padding.
DA_DEV long long token_row(const Params& p, int region, int r) {
  if (p.layout == DA_LAYOUT_REORDERED) return (long long)region * P + r;
  const RegionXY rc = p.dec(region);
  const int u = r / p.geo.pw, v = r - u * p.geo.pw;
  const int y = rc.y0 + u, x = rc.x0 + v;
  if (y >= p.geo.H || x >= p.geo.W) return -1;
  return ((long long)rc.f * p.geo.H + y) * p.geo.W + x;
}

// 64-bit validity mask of the keys of region j (bit r = key r valid).
DA_DEV unsigned long long key_mask(const Params& p, int j) {
  if (p.key_valid != nullptr) {
    const uint8_t* kv = p.key_valid + (long long)j * P;
    unsigned long long m = 0;
#pragma unroll 8
    for (int r = 0; r < P; ++r) m |= (unsigned long long)(kv[r] != 0) << r;
    return m;
  }
  const RegionXY rc = p.dec(j);
  const int vy = min(p.geo.ph, p.geo.H - rc.y0), vx = min(p.geo.pw, p.geo.W - rc.x0);
  if (vy == p.geo.ph && vx == p.geo.pw) return ~0ull;
  // key r = u*pw + v is valid iff u < vy and v < vx: vy copies of the row mask
  const unsigned long long rowm = (1ull << vx) - 1ull;
  unsigned long long m = 0;
  for (int u = 0; u < vy; ++u) m |= rowm << (u * p.geo.pw);
  return m;
}

__global__ void __launch_bounds__(384, 1)
    sparse_attn_pair_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                            const Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  SmemAux& aux = *reinterpret_cast<SmemAux*>(smem + SMEM_END);
  Bars& B = aux.bars;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long items = (long long)p.heads * p.npairs;

  if (threadIdx.x == 0) {
    for (int s = 0; s < KST; ++s) { mbar_init(&B.k_full[s], 1); mbar_init(&B.k_empty[s], 1); }
    for (int s = 0; s < VST; ++s) { mbar_init(&B.v_full[s], 1); mbar_init(&B.v_empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&B.s_full[s], 1); mbar_init(&B.p_full[s], 256); }
    mbar_init(&B.o_step, 1);
    mbar_init(&B.o_full, 1);
    mbar_init(&B.o_empty, 256);
    mbar_init(&B.q_full, 256);
    mbar_init(&B.q_empty, 1);
    fence_barrier_init();
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(&aux.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = aux.tmem_base;
  uint8_t* sK = smem + SMEM_K;
  uint8_t* sV = smem + SMEM_V;

  if (warp == 0 || warp == 2) {
    // ===================== TMA producers (warp 0: K, warp 2: V) =====================
    if (lane == 0) {
      const bool is_k = warp == 0;
      const int ST = is_k ? KST : VST;
      uint8_t* ring = is_k ? sK : sV;
      uint64_t* full = is_k ? B.k_full : B.v_full;
      uint64_t* empty = is_k ? B.k_empty : B.v_empty;
      const CUtensorMap* map = is_k ? &tm_k : &tm_v;
      int kq = 0;
      for (long long it = blockIdx.x;; it += gridDim.x) {
        PairItem itm;
        if (!fetch_pair(p, it, items, itm)) break;
        UnionWalk u;
        u.init(itm);
        int j0, j1, f;
        while (u.next(j0, f)) {
          if (!u.next(j1, f)) j1 = j0;
          const int s = kq % ST;
          if (kq >= ST) mbar_wait(&empty[s], ((kq / ST) - 1) & 1);
          PAIR_TRACE(is_k ? 0 : 1, kq);
          uint8_t* st = ring + s * KV_BYTES;
          mbar_expect_tx(&full[s], KV_BYTES);
          if (is_k) {  // [half][slot][64 x 128B]: B operand rows 0..127 = keys of j0 then j1
            load_region(map, st, &full[s], p, itm.h, j0, 0);
            load_region(map, st + BOX, &full[s], p, itm.h, j1, 0);
            load_region(map, st + 2 * BOX, &full[s], p, itm.h, j0, 1);
            load_region(map, st + 3 * BOX, &full[s], p, itm.h, j1, 1);
          } else {     // [slot][half][64 x 128B]: MN-major B, keys = K dimension
            load_region(map, st, &full[s], p, itm.h, j0, 0);
            load_region(map, st + BOX, &full[s], p, itm.h, j0, 1);
            load_region(map, st + 2 * BOX, &full[s], p, itm.h, j1, 0);
            load_region(map, st + 3 * BOX, &full[s], p, itm.h, j1, 1);
          }
          ++kq;
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    if (lane == 0) {
      constexpr uint32_t IDESC1 = umma_idesc_bf16(128, 128, 0, 0);  // A (TMEM) K-major, B K-major
      constexpr uint32_t IDESC2 = umma_idesc_bf16(128, 128, 0, 1);  // A (TMEM) K-major, B MN-major
      const uint64_t dK = umma_desc_sw128(0, 16, 1024);
      const uint64_t dV = umma_desc_sw128(0, BOX, 1024);
      const uint32_t aK = smem_u32(sK) >> 4, aV = smem_u32(sV) >> 4;
      int kq = 0, vq = 0, qi = 0;
      long long G = 0;
      struct Pend {
        long long step;
        int qi;
        bool first, last, valid;
      } pend;
      pend.valid = false;
      auto gemm2 = [&](const Pend& s) {
        const int vs = vq % VST;
        mbar_wait(&B.v_full[vs], (vq / VST) & 1);
        const int b = (int)(s.step & 1);
        mbar_wait(&B.p_full[b], (uint32_t)((s.step >> 1) & 1));
        if (s.first && s.qi > 0) mbar_wait(&B.o_empty, (s.qi - 1) & 1);
        PAIR_TRACE(4, vq);
        tc_fence_after();
        const uint32_t vbase = aV + vs * (KV_BYTES >> 4);
        const uint32_t aP = tmem + (b ? COL_S1 : COL_S0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bv = dV + (uint64_t)(vbase + (kk >> 2) * (2 * BOX >> 4) + (kk & 3) * (2048 >> 4));
          umma_bf16_ts(tmem + COL_O, aP + kk * 8, bv, IDESC2, (s.first && kk == 0) ? 0u : 1u);
        }
        umma_commit(&B.v_empty[vs]);
        umma_commit(&B.o_step);
        if (s.last) umma_commit(&B.o_full);
        ++vq;
      };
      for (long long it = blockIdx.x;; it += gridDim.x) {
        PairItem itm;
        if (!fetch_pair(p, it, items, itm)) break;
        if (itm.na + itm.nb == 0) continue;
        UnionWalk u;
        u.init(itm);
        mbar_wait(&B.q_full, qi & 1);
        bool first = true;
        int j0, j1, f;
        while (u.next(j0, f)) {
          u.next(j1, f);
          const bool last = u.done();
          const int ks = kq % KST;
          mbar_wait(&B.k_full[ks], (kq / KST) & 1);
          PAIR_TRACE(2, kq);
          tc_fence_after();
          const uint32_t kbase = aK + ks * (KV_BYTES >> 4);
          const int b = (int)(G & 1);
          const uint32_t dS = tmem + (b ? COL_S1 : COL_S0);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t bk = dK + (uint64_t)(kbase + (kk >> 2) * (2 * BOX >> 4) + (kk & 3) * 2);
            umma_bf16_ts(dS, tmem + COL_Q + kk * 8, bk, IDESC1, kk > 0 ? 1u : 0u);
          }
          umma_commit(&B.k_empty[ks]);
          umma_commit(&B.s_full[b]);
          if (last) umma_commit(&B.q_empty);
          ++kq;
          if (pend.valid) gemm2(pend);
          pend.step = G;
          pend.qi = qi;
          pend.first = first;
          pend.last = last;
          pend.valid = true;
          first = false;
          ++G;
        }
        ++qi;
      }
      if (pend.valid) gemm2(pend);
    }
  } else if (warp >= 4) {
    // ============ softmax / Q loader / epilogue: two warpgroups split the step ============
    // Warpgroup wg handles key region wg of each step (S columns [64*wg, 64*wg+64))
    // and feature half wg of Q and O; thread t of a warpgroup owns query row t.
    // The two threads of a row agree on the running max through shared memory.
    const int wg = (warp - 4) >> 2;
    const int t = (threadIdx.x - 128) & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tq = tmem + lane_off;
    const int half = t >> 6;  // 0: rows of region a, 1: rows of region b
    const int r = t & 63;
    const float sl2 = p.scale_log2;
    long long G = 0;
    int qi = 0;
    // my half of the Q row of (item, row) -> TMEM columns [32*wg, 32*wg+32) as
    // packed bf16 pairs. The next nonempty item's Q is written as soon as the
    // current item's last GEMM1 is done, before this item's epilogue.
    auto load_q = [&](const PairItem& itm, int wait_parity) {
      const int region = half ? itm.b : itm.a;
      const long long qrow = region < p.geo.g ? token_row(p, region, r) : -1;
      uint32_t qv[32];
      if (qrow >= 0) {
        const uint4* src = reinterpret_cast<const uint4*>(p.q + itm.h * p.qh + qrow * p.qr) + wg * 8;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 w = __ldg(src + c);
          qv[4 * c] = w.x; qv[4 * c + 1] = w.y; qv[4 * c + 2] = w.z; qv[4 * c + 3] = w.w;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) qv[c] = 0u;
      }
      if (wait_parity >= 0) mbar_wait(&B.q_empty, (uint32_t)wait_parity);
      tc_fence_after();
      tmem_st16u(tq + COL_Q + wg * 32, *reinterpret_cast<uint32_t(*)[16]>(&qv[0]));
      tmem_st16u(tq + COL_Q + wg * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(&qv[16]));
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&B.q_full);
    };
    bool have_q = false;
    for (long long it = blockIdx.x;; it += gridDim.x) {
      PairItem itm;
      if (!fetch_pair(p, it, items, itm)) break;
      const int region = half ? itm.b : itm.a;
      const bool region_ok = region < p.geo.g;
      const long long row = region_ok ? token_row(p, region, r) : -1;
      __nv_bfloat16* orow = row >= 0 ? p.out + itm.h * p.oh + row * p.orow + wg * 64 : nullptr;
      if (itm.na + itm.nb == 0) {
        if (orow) {
#pragma unroll
          for (int c = 0; c < 8; ++c) reinterpret_cast<uint4*>(orow)[c] = make_uint4(0, 0, 0, 0);
        }
        continue;
      }
      if (!have_q) load_q(itm, -1);  // first nonempty item of this CTA
      float m = -INFINITY, l = 0.f;  // running max (both threads of a row agree), my partial sum
      bool mvalid = false;
      UnionWalk u;
      u.init(itm);
      int j[2], fl[2];
      bool first_step = true;
      while (u.next(j[0], fl[0])) {
        if (!u.next(j[1], fl[1])) { j[1] = j[0]; fl[1] = 0; }
        const int b = (int)(G & 1);
        const uint32_t cs = tq + (b ? COL_S1 : COL_S0);
        if (t == 0 && wg == 0) PAIR_TRACE(5, G);
        mbar_wait(&B.s_full[b], (uint32_t)((G >> 1) & 1));
        if (t == 0 && wg == 0) PAIR_TRACE(6, G);
        tc_fence_after();
        // my key region's scores (warp-uniform: a warp's rows share one query region)
        const bool keep = (fl[wg] >> half) & 1;
        float x[64];
        float bm_own = -INFINITY;
        if (keep) {
          tmem_ld32_at<0>(cs + wg * 64, x);
          tmem_ld32_at<32>(cs + wg * 64 + 32, x);
          const unsigned long long vm = key_mask(p, j[wg]);
          tmem_ld_wait();
          if (vm != ~0ull) {
#pragma unroll
            for (int c = 0; c < 64; ++c) x[c] = ((vm >> c) & 1ull) ? x[c] : -INFINITY;
          }
          float mx = x[0];
#pragma unroll
          for (int c = 1; c < 64; ++c) mx = fmaxf(mx, x[c]);
          bm_own = mx * sl2;
        }
        // step max of the row over both key regions (log2 units); the running
        // max is raised only when the step exceeds it by more than TAU
        float* xb = aux.xch[G & 1];
        xb[wg * 128 + t] = bm_own;
        bar_sync(1, 256);
        const float bm = fmaxf(bm_own, xb[(wg ^ 1) * 128 + t]);
        float alpha = 1.f;
        bool raise = false;
        if (!mvalid) {
          if (bm != -INFINITY) { m = bm; mvalid = true; }
        } else if (bm > m + TAU) {
          alpha = exp2f(m - bm);
          l *= alpha;
          m = bm;
          raise = true;
        }
        // warpgroup 0 rescales the O rows (warp-wide: tcgen05.ld/st are
        // .sync.aligned; rows that did not raise scale by 1) once the previous
        // step's GEMM2 has landed
        if (wg == 0 && __any_sync(0xffffffffu, raise) && !first_step) {
          mbar_wait(&B.o_step, (uint32_t)((G - 1) & 1));
          tc_fence_after();
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            float o[32];
            tmem_ld32(tq + COL_O + c4 * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] *= alpha;
            tmem_st32(tq + COL_O + c4 * 32, o);
          }
          tmem_st_wait();
        }
        uint32_t pk[32];
        if (keep && mvalid) {
          const float2 sc = make_float2(sl2, sl2), nm = make_float2(-m, -m);
          float2 acc = make_float2(0.f, 0.f);
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            const float2 e = ffma2(make_float2(x[c], x[c + 1]), sc, nm);
            const float p0 = fast_exp2(e.x), p1 = fast_exp2(e.y);
            acc.x += p0;
            acc.y += p1;
            pk[c / 2] = pack_bf16(p0, p1);
          }
          l += acc.x + acc.y;
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) pk[c] = 0u;
        }
        // P (bf16 pairs) over the first half of this S buffer: keys 64*wg.. -> columns 32*wg..
        tmem_st16u(cs + wg * 32, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
        tmem_st16u(cs + wg * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(&pk[16]));
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&B.p_full[b]);
        if (t == 0 && wg == 0) PAIR_TRACE(7, G);
        first_step = false;
        ++G;
      }
      // ---- next nonempty item's Q (its GEMM1s overlap this epilogue)
      have_q = false;
      for (long long it2 = it + gridDim.x;; it2 += gridDim.x) {
        PairItem nx;
        if (!fetch_pair(p, it2, items, nx)) break;
        if (nx.na + nx.nb == 0) continue;
        load_q(nx, qi & 1);  // q_empty completion #qi = this item's last GEMM1
        have_q = true;
        break;
      }
      // ------------------------------ epilogue ------------------------------
      aux.lsum[wg][t] = l;
      bar_sync(1, 256);
      const float lt = l + aux.lsum[wg ^ 1][t];
      mbar_wait(&B.o_full, qi & 1);
      tc_fence_after();
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        float o[32];
        tmem_ld32(tq + COL_O + wg * 64 + c2 * 32, o);
        tmem_ld_wait();
        if (orow) {
          uint32_t w[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) w[c] = pack_bf16(o[2 * c] * inv, o[2 * c + 1] * inv);
          uint4* dst = reinterpret_cast<uint4*>(orow) + c2 * 4;
#pragma unroll
          for (int c = 0; c < 4; ++c) dst[c] = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(&B.o_empty);
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

}  // namespace pairk

bool make_kv_maps(const da_attn_args& a, const Geo& g, CUtensorMap* mk, CUtensorMap* mv);

cudaError_t launch_pair_attn(const da_attn_args& a, const Geo& g, cudaStream_t st, const char** why,
                             long long* trace) {
  CUtensorMap mk, mv;
  if (!make_kv_maps(a, g, &mk, &mv)) {
    *why = "cuTensorMapEncodeTiled failed";
    return cudaErrorInvalidValue;
  }
  pairk::Params p;
  p.q = static_cast<const __nv_bfloat16*>(a.q);
  p.qh = a.q_head_stride;
  p.qr = a.q_row_stride;
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
  p.npairs = (g.g + 1) / 2;
  p.per_head = make_fastdiv((uint32_t)p.npairs);
  p.n_pad = g.n_pad;
  p.trace = trace;
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  cudaError_t e = cudaFuncSetAttribute(pairk::sparse_attn_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       pairk::SMEM_ALLOC);
  if (e != cudaSuccess) return e;
  const long long items = (long long)a.heads * p.npairs;
  const int grid = (int)(items < num_sms ? items : num_sms);
  pairk::sparse_attn_pair_kernel<<<grid, 384, pairk::SMEM_ALLOC, st>>>(mk, mv, p);
  return cudaGetLastError();
}

}  // namespace da
