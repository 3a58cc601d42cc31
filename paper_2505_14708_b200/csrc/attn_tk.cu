// K4 "tk" (experiment; probe builds with -DDA_K4_TK only): block-sparse
// FlashAttention forward, TRANSPOSED, with M = 128 tiles.
//
// Same semantics as the reference executor (sparse.py:88-166): per query
// region, its kept key regions in ascending order, padding keys masked out,
// softmax over the valid kept keys, rows with no valid kept key -> 0.
//
// A step takes TWO kept key regions of one query region and puts the 128 keys
// on M:
//
//     GEMM1  S^T[128 keys x 64 q]  = K_pair . Q^T      A = K pair (smem, bulk copies), B = Q tile (smem)
//     GEMM2  O^T[128 d   x 64 q]  += V_pair^T . P^T    A = V^T pair (TMEM), B = P^T (smem, MN-major)
//
// GEMM1 is an SS MMA fed like the lane-half kernel's (one contiguous bulk copy
// per pooled region tile, GROUPED layout); V^T reaches TMEM through registers
// (LDG.128 -> tcgen05.st), so the two L2 -> SM paths run side by side and
// shared memory carries K (write + read), Q^T and P^T only. Tensor time per
// step: 8 x 48 (SS, N = 64) + 8 x 32 (TS) = 640 cycles, against 1024 for the
// lane-half kernel's two M = 64 GEMMs.
//
// Softmax per query COLUMN with a fixed offset per (query, item): m[q] =
// |q| max|k| scale log2(e) - 64 (Cauchy-Schwarz bounds every score). Three
// softmax warpgroups take the steps in turn (step s -> warpgroup s % 3, S^T
// buffer and P^T buffer s % 3), so each has three step times for its serial
// chain (profiles/r02/tk/README.md: that chain, not the MMAs, bounded the
// two-warpgroup version). A thread owns 4 keys x 16 queries of a step
// (.16x256b fragments); row sums accumulate in registers across the item.
// Rows whose sum ends below 2^-80 are redone by the portable kernel.
//
// Roles (24 warps):
//   warp 0      scheduler + K producer: claims items, stages kept lists,
//               publishes item records and step entries, issues the K bulk
//               copies (ring of KSL slots of two tiles)
//   warp 1      GEMM1 issuer (and TMEM owner)      warp 2   GEMM2 issuer
//   warp 3      Q loader: the item's Q tile into smem + the offsets m[q]
//   warps 4-11  V^T loaders, two groups of 4 (group = step parity); lane = feature
//   warps 12-23 softmax, three warpgroups; warpgroups 0 and 1 also write the
//               item's output rows [0, 32) / [32, 64)
// TMEM: S^T [0,192) (three buffers), V^T [192,320) (two), O^T [320,448) (two:
// item parity).
#include "attn_k4.cuh"
#include "common.cuh"
#include "kernels.h"

#ifndef TK_REG_CTL
#define TK_REG_CTL 56
#endif
#ifndef TK_REG_LD
#define TK_REG_LD 80
#endif
#ifndef TK_REG_SM
#define TK_REG_SM 88
#endif
#ifndef TK_KSL
#define TK_KSL 3  // K ring slots (32 KB each)
#endif

// waits of the softmax warps (SMW) and of the MMA issuers (ISW): 0 sleep in
// try_wait, 1 every lane spins on test_wait, 2 lane 0 spins
#ifndef TK_SMW
#define TK_SMW 0
#endif
#ifndef TK_ISW
#define TK_ISW 1
#endif
#define TK_WAITF(kind, bar, par)         \
  do {                                   \
    if ((kind) == 0) mbar_wait(bar, par); \
    else if ((kind) == 1) mbar_wait_spin(bar, par); \
    else mbar_wait_warp(bar, par);        \
  } while (0)

#ifndef TK_POLY
#define TK_POLY 1  // every fourth exponential pair on the FMA pipe (exp2_poly2) instead of MUFU
#endif

// TK_PROF (probe builds, tools/probes/tk_prof.py): per-role cycle accounting of
// the waits, lane 0 of one warp per role, summed per CTA into the
// da_debug_trace buffer as [CTA][64] int64 (role r: slots 8 r .. 8 r + 7;
// slot 63: CTA cycles)
#ifdef TK_PROF
#define TK_T0() const long long _t0 = clock64()
#define TK_ACC(k) prof[k] += clock64() - _t0
#define TK_TIME(k, stmt) \
  {                      \
    TK_T0();             \
    stmt;                \
    TK_ACC(k);           \
  }
#else
#define TK_T0() \
  do {          \
  } while (0)
#define TK_ACC(k) \
  do {            \
  } while (0)
#define TK_TIME(k, stmt) \
  { stmt; }
#endif

// TK_TRACE (probe builds, tools/probes/tk_trace.py): CTA 0 records clock64()
// of per-step events into the da_debug_trace buffer as [event][TK_NT] int64:
// 0 GEMM1 issue, 1 GEMM2 issue, 2 S ready, 3 S read, 4 P written, 5 K copy
// issued, 6 V stored, 7 softmax step start
#ifdef TK_TRACE
constexpr int TK_NT = 4096;
#define TK_EV(ev, step)                                                                                   \
  do {                                                                                                    \
    if (blockIdx.x == 0 && p.trace != nullptr && (step) < TK_NT) p.trace[(ev) * TK_NT + (step)] = clock64(); \
  } while (0)
#else
#define TK_EV(ev, step) \
  do {                  \
  } while (0)
#endif

namespace da {
namespace tkk {

using k4::D;
using k4::Item;
using k4::item_from_record;
using k4::item_record;
using k4::key_mask;
using k4::LISTCAP;
using k4::P;
using k4::Params;
using k4::RAGW;
using k4::TILE;
using k4::token_row;

constexpr int KSL = TK_KSL;
constexpr int SLOT = 2 * TILE;
constexpr int NWG = 3;     // softmax warpgroups
constexpr int INFO = 24;   // step ring: a multiple of NWG (a slot always holds steps of one warpgroup) and of 2
constexpr int W_SCHED = 0, W_G1 = 1, W_G2 = 2, W_Q = 3, W_LD = 4, W_SM = 12;
constexpr int NWARPS = W_SM + 4 * NWG;
constexpr int THREADS = 32 * NWARPS;
constexpr int LAUNCH_REGS = (65536 / THREADS) & ~7;
#ifndef TK_NOASSERT
static_assert(4 * TK_REG_CTL + 8 * TK_REG_LD + 4 * NWG * TK_REG_SM <= NWARPS * LAUNCH_REGS, "register budget");
#endif
// step entries: GEMM1, GEMM2, the 8 loader warps and the 4 warps of the step's warpgroup
constexpr int INFO_CONSUMERS = 2 + 8 + 4;
constexpr int IR = 8;  // item ring: the Q warp and every softmax warp
constexpr int ITEM_CONSUMERS = 1 + 4 * NWG;
static_assert(INFO % NWG == 0 && INFO % 2 == 0, "step ring");

constexpr uint32_t COL_S = 0, COL_V = 64 * NWG, COL_O = COL_V + 128;

constexpr int SMEM_K = 0;                          // KSL x 32 KB K slots (GROUPED tiles)
constexpr int SMEM_Q = SMEM_K + KSL * SLOT;        // 2 x 16 KB Q tiles: [feature half][64 rows x 128 B], SW128
constexpr int SMEM_P = SMEM_Q + 2 * TILE;          // NWG x 16 KB P^T tiles: [8-key group][8 keys x 128 B], SW128
constexpr int SMEM_O = SMEM_P + NWG * TILE;        // 16 KB output staging [64 q][128 d] bf16
constexpr int SMEM_END = SMEM_O + TILE;

// step entry flags (int4.z low byte; head in the bits above)
constexpr int F_J1 = 1, F_RAG0 = 2, F_RAG1 = 4;
// int4.w: bit 0 last step of the item, bit 1 first step, bit 2 end of stream; region << 3
constexpr int W_LAST = 1, W_FIRST = 2, W_END = 4;

struct __align__(8) Bars {
  uint64_t k_full[KSL], k_empty[KSL], v_full[2], v_empty[2];
  uint64_t s_full[NWG], s_free[NWG], p_full[NWG], p_free[NWG];
  uint64_t q_full[2], q_empty[2], o_full[2], o_empty[2];
  uint64_t info_full[INFO], info_empty[INFO];
  uint64_t item_full[IR], item_empty[IR];
};
struct SmemAux {
  Bars bars;
  int4 info[INFO];
  int4 items[IR];  // (first global step, steps, head, region); steps < 0: end of work
  uint32_t tmem_base;
  alignas(16) float m[2][64];     // [item parity][query] fixed offsets (log2 units)
  float lsum[2][NWG][4][64];      // [item parity][warpgroup][warp slice][query] partial row sums
  float linv[2][32];              // [output warpgroup][column] 1 / l, or 0
  uint32_t ragged[RAGW];
  int list[LISTCAP];
};
constexpr int SMEM_ALLOC = SMEM_END + (int)sizeof(SmemAux);
static_assert(SMEM_ALLOC <= 227 * 1024, "shared memory budget");

// V^T tile layout (pooling pass): key chunk c (keys 8c..8c+7) of feature row d
DA_DEV uint32_t vt_off(int d, int c) { return (uint32_t)(c * 2048 + d * 16); }

template <int N>
DA_DEV void set_maxnreg() {
  if constexpr (N > LAUNCH_REGS) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N) : "memory");
  else if constexpr (N < LAUNCH_REGS) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N) : "memory");
}

// .16x256b.x4 load into v[0 .. 15] (mapping: tools/probes/tmem16x256.cu): register
// i holds lane base + t/4 + 8 ((i >> 1) & 1), column base + 8 (i >> 2) + 2 (t % 4) + (i & 1)
DA_DEV void tmem_ld16x256_x4(uint32_t taddr, float (&v)[16]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
DA_DEV void sts32(uint32_t saddr, uint32_t v) { asm volatile("st.shared.b32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory"); }

DA_DEV void ldg16x4(const uint8_t* src, uint32_t* r) {
  const uint4 v = __ldg(reinterpret_cast<const uint4*>(src));
  r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
}

__global__ void __launch_bounds__(THREADS, 1) sparse_attn_tk_kernel(const Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  SmemAux& aux = *reinterpret_cast<SmemAux*>(smem + SMEM_END);
  Bars& B = aux.bars;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long items = (long long)p.heads * p.geo.g;
#ifdef TK_PROF
  long long prof[8];
  for (int k = 0; k < 8; ++k) prof[k] = 0;
  const long long t_start = clock64();
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < KSL; ++s) {
      mbar_init(&B.k_full[s], 1);
      mbar_init(&B.k_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&B.v_full[b], 128);
      mbar_init(&B.v_empty[b], 1);
      mbar_init(&B.q_full[b], 32);
      mbar_init(&B.q_empty[b], 1 + 128 * NWG);  // GEMM1's last MMA of the item + every softmax thread
      mbar_init(&B.o_full[b], 1);
      mbar_init(&B.o_empty[b], 256);            // the two output warpgroups
    }
    for (int w = 0; w < NWG; ++w) {
      mbar_init(&B.s_full[w], 1);
      mbar_init(&B.s_free[w], 128);
      mbar_init(&B.p_full[w], 128);
      mbar_init(&B.p_free[w], 1);
    }
    for (int s = 0; s < INFO; ++s) {
      mbar_init(&B.info_full[s], 1);
      mbar_init(&B.info_empty[s], INFO_CONSUMERS);
    }
    for (int s = 0; s < IR; ++s) {
      mbar_init(&B.item_full[s], 1);
      mbar_init(&B.item_empty[s], ITEM_CONSUMERS);
    }
    fence_barrier_init();
  }
  if (p.key_valid == nullptr && p.geo.g <= 32 * RAGW) {
    for (int wd = threadIdx.x; wd < (p.geo.g + 31) / 32; wd += blockDim.x) {
      uint32_t bits = 0;
      for (int b = 0; b < 32; ++b) {
        const int j = wd * 32 + b;
        if (j < p.geo.g && key_mask(p, j) != ~0ull) bits |= 1u << b;
      }
      aux.ragged[wd] = bits;
    }
  }
  if (warp == W_G1) tmem_alloc<512>(&aux.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = aux.tmem_base;

  // a warp takes a ring entry (lane 0 reads it, releases the slot, broadcasts)
  auto take = [&](const int4* ring, uint64_t* full, uint64_t* empty, uint32_t parity) {
    int4 v = make_int4(0, 0, 0, 0);
    if (lane == 0) {
      mbar_wait(full, parity);
      v = *ring;
      mbar_arrive(empty);
    }
    v.x = __shfl_sync(0xffffffffu, v.x, 0);
    v.y = __shfl_sync(0xffffffffu, v.y, 0);
    v.z = __shfl_sync(0xffffffffu, v.z, 0);
    v.w = __shfl_sync(0xffffffffu, v.w, 0);
    return v;
  };
  int ii_item = 0;
  uint32_t iph_item = 0;
  auto next_item = [&]() {
    const int4 v = take(&aux.items[ii_item], &B.item_full[ii_item], &B.item_empty[ii_item], iph_item);
    if (++ii_item == IR) { ii_item = 0; iph_item ^= 1u; }
    return v;
  };
  int ri = 0;
  uint32_t rph = 0;
  auto next_step = [&]() {  // every step consumer but the softmax walks the ring in order
    TK_T0();
    const int4 e = take(&aux.info[ri], &B.info_full[ri], &B.info_empty[ri], rph);
    TK_ACC(0);
    if (++ri == INFO) { ri = 0; rph ^= 1u; }
    return e;
  };

  if (warp == W_SCHED) {
    // ======================== scheduler + K producer ========================
    set_maxnreg<TK_REG_CTL>();
    const bool bitmap = p.key_valid == nullptr && p.geo.g <= 32 * RAGW;
    const uint8_t* kt = p.kt;
    int kq = 0, kit = 0;
    long long claim = 0;
    int4 rec_next = make_int4(0, 0, -1, 0);
    {
      long long c0 = 0;
      if (lane == 0) {
        c0 = atomicAdd(p.work, 1);
        claim = atomicAdd(p.work, 1);
      }
      rec_next = item_record(p, __shfl_sync(0xffffffffu, c0, 0), items);
    }
    auto publish_item = [&](int4 v) {  // lane 0
      const int si = kit % IR;
      if (kit >= IR) mbar_wait(&B.item_empty[si], (uint32_t)(((kit / IR) - 1) & 1));
      aux.items[si] = v;
      mbar_arrive(&B.item_full[si]);
      ++kit;
    };
    auto ragged = [&](int j) {
      return bitmap ? ((aux.ragged[j >> 5] >> (j & 31)) & 1u) != 0 : key_mask(p, j) != ~0ull;
    };
    for (;;) {
      int4 rec;
      for (;;) {
        rec = rec_next;
        long long c = 0;
        if (lane == 0) {
          c = claim;
          claim = atomicAdd(p.work, 1);
        }
        rec_next = item_record(p, __shfl_sync(0xffffffffu, c, 0), items);
        if (rec.z != 0) break;
        // no kept key region: the region's output rows are zero (sparse.py:137-138)
        for (int e = lane; e < P * (D / 8); e += 32) {
          const long long row = token_row(p, rec.x, e / (D / 8));
          if (row >= 0) reinterpret_cast<uint4*>(p.out + rec.w * p.oh + row * p.orow)[e % (D / 8)] = make_uint4(0, 0, 0, 0);
        }
      }
      Item itm;
      if (!item_from_record(p, rec, itm)) break;
      const bool staged = itm.n <= LISTCAP;
      __syncwarp();
      if (staged)
        for (int e = lane; e < itm.n; e += 32) aux.list[e] = __ldg(itm.list + e);
      __syncwarp();
      if (lane == 0) {
        const int n = (itm.n + 1) / 2;
        publish_item(make_int4(kq, n, itm.h, itm.i));
        const uint8_t* hb = kt + (long long)itm.h * p.geo.g * TILE;
        for (int t = 0; t < n; ++t) {
          const int j0 = staged ? aux.list[2 * t] : __ldg(itm.list + 2 * t);
          const int j1 = 2 * t + 1 < itm.n ? (staged ? aux.list[2 * t + 1] : __ldg(itm.list + 2 * t + 1)) : -1;
          int fl = ragged(j0) ? F_RAG0 : 0;
          if (j1 >= 0) fl |= F_J1 | (ragged(j1) ? F_RAG1 : 0);
          const int ii = kq % INFO;
          if (kq >= INFO) TK_TIME(1, mbar_wait(&B.info_empty[ii], (uint32_t)(((kq / INFO) - 1) & 1)));
          aux.info[ii] = make_int4(j0, j1, fl | (itm.h << 8),
                                   (itm.i << 3) | (t == n - 1 ? W_LAST : 0) | (t == 0 ? W_FIRST : 0));
          mbar_arrive(&B.info_full[ii]);
          // K pair of this step into ring slot kq % KSL (the GROUPED tiles:
          // two adjacent tiles are one 128-row K-major operand)
          const int s = kq % KSL;
          if (kq >= KSL) TK_TIME(2, mbar_wait(&B.k_empty[s], (uint32_t)(((kq / KSL) - 1) & 1)));
          uint8_t* st = smem + SMEM_K + s * SLOT;
          mbar_expect_tx(&B.k_full[s], TILE * (j1 >= 0 ? 2 : 1));
          TK_EV(5, kq);
          bulk_g2s(st, hb + (long long)j0 * TILE, TILE, &B.k_full[s], p.pol_kv);
          if (j1 >= 0) bulk_g2s(st + TILE, hb + (long long)j1 * TILE, TILE, &B.k_full[s], p.pol_kv);
          ++kq;
        }
      }
      __syncwarp();
      kq = __shfl_sync(0xffffffffu, kq, 0);
    }
    if (lane == 0) {
      const int ii = kq % INFO;
      if (kq >= INFO) mbar_wait(&B.info_empty[ii], (uint32_t)(((kq / INFO) - 1) & 1));
      aux.info[ii] = make_int4(-1, -1, 0, W_END);
      mbar_arrive(&B.info_full[ii]);
      publish_item(make_int4(0, -1, 0, 0));
    }
  } else if (warp == W_G1 || warp == W_G2) {
    // ============================== MMA issuers ===============================
    set_maxnreg<TK_REG_CTL>();
    const bool g1 = warp == W_G1;
    constexpr uint32_t I1 = umma_idesc_bf16(128, 64, 0, 0);  // A = K pair (smem, K-major), B = Q tile (K-major)
    constexpr uint32_t I2 = umma_idesc_bf16(128, 64, 0, 1);  // A = V^T (TMEM), B = P^T (smem, MN-major)
    const uint64_t dK = umma_desc_sw128(0, 16, 2048) + (smem_u32(smem + SMEM_K) >> 4);
    const uint64_t dQ = umma_desc_sw128(0, 16, 1024) + (smem_u32(smem + SMEM_Q) >> 4);
    const uint64_t dP = umma_desc_sw128(0, 16, 1024) + (smem_u32(smem + SMEM_P) >> 4);
    int gs = 0, seq = 0;
    for (;;) {
      const int4 e = next_step();
      if (e.w & W_END) break;
      const int w = gs % NWG;                                 // S^T / P^T buffer
      const uint32_t wpar = (uint32_t)((gs / NWG) & 1);       // its phase
      const int xb = seq & 1;  // Q tile (GEMM1) / O^T buffer (GEMM2) of the item
      const bool first = e.w & W_FIRST, last = e.w & W_LAST;
      if (g1) {
        const int s = gs % KSL;
        if (first) TK_TIME(1, TK_WAITF(TK_ISW, &B.q_full[xb], (uint32_t)((seq >> 1) & 1)));
        TK_TIME(2, TK_WAITF(TK_ISW, &B.k_full[s], (uint32_t)((gs / KSL) & 1)));
        if (gs >= NWG) TK_TIME(3, TK_WAITF(TK_ISW, &B.s_free[w], wpar ^ 1u));
        tc_fence_after();
        if (lane == 0) TK_EV(0, gs);
        TK_T0();
        if (elect_one_sync()) {
          const uint64_t ak = dK + (uint64_t)(s * (SLOT >> 4));
          const uint64_t bq = dQ + (uint64_t)(xb * (TILE >> 4));
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(tmem + COL_S + 64 * w, ak + (uint64_t)((kk >> 2) * (1024 >> 4) + (kk & 3) * 2),
                      bq + (uint64_t)((kk >> 2) * (8192 >> 4) + (kk & 3) * 2), I1, kk > 0 ? 1u : 0u);
          umma_commit(&B.k_empty[s]);
          umma_commit(&B.s_full[w]);
          if (last) umma_commit(&B.q_empty[xb]);
        }
        __syncwarp();
        TK_ACC(4);
      } else {
        const int b = gs & 1;
        if (first && seq >= 2) TK_TIME(1, mbar_wait(&B.o_empty[xb], (uint32_t)(((seq >> 1) - 1) & 1)));
        TK_TIME(2, TK_WAITF(TK_ISW, &B.v_full[b], (uint32_t)((gs >> 1) & 1)));
        TK_TIME(3, TK_WAITF(TK_ISW, &B.p_full[w], wpar));
        tc_fence_after();
        if (lane == 0) TK_EV(1, gs);
        TK_T0();
        if (elect_one_sync()) {
          const int nk = (e.z & F_J1) ? 8 : 4;  // an odd last region: keys 64..127 absent
          for (int kk = 0; kk < nk; ++kk)
            umma_bf16_ts(tmem + COL_O + 64 * xb, tmem + COL_V + 64 * b + 8 * kk,
                         dP + (uint64_t)(w * (TILE >> 4) + kk * (2048 >> 4)), I2, (first && kk == 0) ? 0u : 1u);
          umma_commit(&B.v_empty[b]);
          umma_commit(&B.p_free[w]);
          if (last) umma_commit(&B.o_full[xb]);
        }
        __syncwarp();
        TK_ACC(4);
      }
      if (last) ++seq;
      ++gs;
    }
  } else if (warp == W_Q) {
    // ====================== Q tiles and fixed offsets ======================
    set_maxnreg<TK_REG_CTL>();
    // lane handles query rows lane and lane + 32 of the item
    int seq = 0, cur_head = -1;
    float kmax = 0.f;
    const float sl2 = p.scale_log2;
    for (;;) {
      const int4 it = next_item();
      if (it.y < 0) break;
      const int h = it.z, region = it.w;
      const int qb = seq & 1;
      if (h != cur_head) {
        cur_head = h;
        const float* kp = p.kpart + (long long)h * p.kblk;
        float mx = 0.f;
        for (int k = 0; k < p.kblk; ++k) mx = fmaxf(mx, __ldg(kp + k));
        kmax = mx;
      }
      if (seq >= 2) mbar_wait(&B.q_empty[qb], (uint32_t)(((seq >> 1) - 1) & 1));
      uint8_t* qt = smem + SMEM_Q + qb * TILE;
#pragma unroll 1
      for (int rr = 0; rr < 2; ++rr) {
        const int r = lane + 32 * rr;
        const long long row = token_row(p, region, r);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(p.q + h * p.qh + (row >= 0 ? row : 0) * p.qr);
        float s2 = 0.f;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          uint32_t w[4] = {0u, 0u, 0u, 0u};
          if (row >= 0) ldg16x4(src + 16 * c, w);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
            s2 = fmaf(f.x, f.x, fmaf(f.y, f.y, s2));
          }
          // [half c >> 3][row r][chunk c & 7 swizzled]
          sts128(smem_u32(qt + (c >> 3) * 8192 + r * 128 + ((((c & 7) ^ r) & 7) << 4)), w[0], w[1], w[2], w[3]);
        }
        aux.m[qb][r] = sqrtf(s2) * kmax * sl2 * 1.0001f - 64.f;
      }
      fence_proxy_async_smem();  // Q tile: generic-proxy stores -> the MMA's async-proxy reads
      mbar_arrive(&B.q_full[qb]);
      ++seq;
    }
  } else if (warp >= W_LD && warp < W_SM) {
    // ============================== V^T loaders ==============================
    set_maxnreg<TK_REG_LD>();
    const int grp = (warp - W_LD) >> 2, slice = (warp - W_LD) & 3;
    const int L = 32 * slice + lane;  // TMEM lane: feature d
    const long long hstride = (long long)p.geo.g * TILE;
    int gs = 0;
    for (;;) {
      const int4 e = next_step();
      if (e.w & W_END) break;
      if ((gs & 1) == grp) {
        const uint8_t* hb = p.vt + (long long)(e.z >> 8) * hstride;
        uint32_t r[64];
        const uint8_t* s0 = hb + (long long)e.x * TILE + vt_off(L, 0);
#pragma unroll
        for (int c = 0; c < 8; ++c) ldg16x4(s0 + c * 2048, r + 4 * c);
        if (e.y >= 0) {
          const uint8_t* s1 = hb + (long long)e.y * TILE + vt_off(L, 0);
#pragma unroll
          for (int c = 0; c < 8; ++c) ldg16x4(s1 + c * 2048, r + 32 + 4 * c);
        } else {
#pragma unroll
          for (int c = 32; c < 64; ++c) r[c] = 0u;
        }
        const int b = gs & 1;
        if (gs >= 2) TK_TIME(2, mbar_wait(&B.v_empty[b], (uint32_t)(((gs >> 1) - 1) & 1)));
        tc_fence_after();
        const uint32_t tl = tmem + ((uint32_t)(32 * slice) << 16) + COL_V + 64 * b;
        TK_TIME(3, tmem_st32(tl, *reinterpret_cast<float(*)[32]>(&r[0]));
                tmem_st32(tl + 32, *reinterpret_cast<float(*)[32]>(&r[32])); tmem_st_wait());
        tc_fence_before();
        mbar_arrive(&B.v_full[b]);
        if (slice == 0 && lane == 0) TK_EV(6, gs);
      }
      ++gs;
    }
  } else {
    // ========================= softmax + epilogue =========================
    // Warpgroup wg takes the steps gs with gs % 3 == wg (S^T / P^T buffer wg),
    // all 64 query columns; warp sp of it owns S^T lanes 32 sp .. 32 sp + 31
    // (keys), read in quarters (lane bases 0 / 16, column bases 0 / 32) with
    // .16x256b.x4: a thread holds 4 keys x 16 queries of the step.
    set_maxnreg<TK_REG_SM>();
    const int wg = (warp - W_SM) >> 2, sp = (warp - W_SM) & 3;
    const int c4 = lane & 3, r8 = lane >> 2;
    const uint32_t tl = tmem + ((uint32_t)(32 * sp) << 16);
    const float sl2 = p.scale_log2;
    // P^T tile: [8-key group][8 keys x 128 B], 128-byte swizzle; this thread's
    // words: key 32 sp + 8 kk + r8, 16-byte chunk jj ^ r8, word c4
    const uint32_t pbase = smem_u32(smem + SMEM_P + wg * TILE) + (uint32_t)(4 * sp * 1024 + r8 * 128 + 4 * c4);
    int seq = 0;
    float2 lsum[8], mq[8];
    bool anyv = false;
    for (;;) {
      const int4 it = next_item();
      if (it.y < 0) break;
      const int G = it.x, nst = it.y;
      const int qb = seq & 1;
      TK_TIME(1, mbar_wait(&B.q_full[qb], (uint32_t)((seq >> 1) & 1)));  // the item's offsets m[q]
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        mq[jj] = *reinterpret_cast<const float2*>(&aux.m[qb][8 * jj + 2 * c4]);
        lsum[jj] = make_float2(0.f, 0.f);
      }
      anyv = false;
      // this warpgroup's steps of the item: global steps G + t with (G + t) % 3 == wg
      for (int t = ((wg - G) % NWG + NWG) % NWG; t < nst; t += NWG) {
        const int gs = G + t;
        const int ii = gs % INFO;
        int4 e;
        TK_TIME(0, e = take(&aux.info[ii], &B.info_full[ii], &B.info_empty[ii], (uint32_t)((gs / INFO) & 1)));
        const uint32_t wpar = (uint32_t)((gs / NWG) & 1);
        if (sp == 0 && lane == 0) TK_EV(7, gs);
        // this warp's keys are rows 32 (sp & 1) + [0, 32) of region j0 (sp < 2) or j1
        const int sel = sp >> 1;
        const int j = sel ? e.y : e.x;
        if (j < 0) {
          // odd last step: keys 64..127 absent; GEMM2 reads only P^T rows 0..63
          TK_TIME(2, TK_WAITF(TK_SMW, &B.s_full[wg], wpar));
          tc_fence_before();
          mbar_arrive(&B.s_free[wg]);
          if (gs >= NWG) TK_TIME(4, TK_WAITF(TK_SMW, &B.p_free[wg], wpar ^ 1u));
          mbar_arrive(&B.p_full[wg]);
          continue;
        }
        uint32_t kvm = 0xfu;  // validity of keys kk = 0..3 (row 32 (sp & 1) + 8 kk + r8)
        if (e.z & (sel ? F_RAG1 : F_RAG0)) {
          const unsigned long long km = key_mask(p, j) >> (32 * (sp & 1) + r8);
          kvm = (uint32_t)((km & 1ull) | ((km >> 7) & 2ull) | ((km >> 14) & 4ull) | ((km >> 21) & 8ull));
        }
        anyv |= kvm != 0u;
        TK_TIME(2, TK_WAITF(TK_SMW, &B.s_full[wg], wpar));
        if (sp == 0 && lane == 0) TK_EV(2, gs);
        tc_fence_after();
        if (gs >= NWG) TK_TIME(4, TK_WAITF(TK_SMW, &B.p_free[wg], wpar ^ 1u));
        TK_T0();
        // four quarters: lane half hh (keys 16 hh + ..), column half cc (queries 32 cc + ..)
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const int hh = qq >> 1, cc = qq & 1;
          float x[16];
          tmem_ld16x256_x4(tl + ((uint32_t)(16 * hh) << 16) + COL_S + 64 * wg + 32 * cc, x);
          tmem_ld_wait();
          if (qq == 3) {
            tc_fence_before();
            mbar_arrive(&B.s_free[wg]);  // all of S^T in registers: GEMM1 may refill this buffer
            if (sp == 0 && lane == 0) TK_EV(3, gs);
          }
          // x[4 j + 2 kb + e]: key 8 (2 hh + kb) + r8, query 32 cc + 8 j + 2 c4 + e
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const int jj = 4 * cc + (i >> 2);
            const int kk = 2 * hh + ((i >> 1) & 1);
            float2 v = ffma2(make_float2(x[i], x[i + 1]), make_float2(sl2, sl2), make_float2(-mq[jj].x, -mq[jj].y));
            if (TK_POLY && (i & 6) == 6) v = exp2_poly2(v);
            else v = make_float2(fast_exp2(v.x), fast_exp2(v.y));
            if (kvm != 0xfu && !((kvm >> kk) & 1u)) v = make_float2(0.f, 0.f);  // ragged region / padding keys
            x[i] = v.x;
            x[i + 1] = v.y;
            sts32(pbase + (uint32_t)(kk * 1024) + (uint32_t)(((jj ^ r8) & 7) << 4), pack_bf16(v.x, v.y));
          }
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const int jj = 4 * cc + (i >> 2);
            lsum[jj] = fadd2(lsum[jj], make_float2(x[i], x[i + 1]));
          }
        }
        TK_ACC(3);
        fence_proxy_async_smem();
        mbar_arrive(&B.p_full[wg]);
        if (sp == 0 && lane == 0) TK_EV(4, gs);
      }
      // ---------------- item epilogue ----------------
      mbar_arrive(&B.q_empty[qb]);  // done with m[qb]
      const int h = it.z, region = it.w;
      // row sums: reduce the 8 key groups (lane bits 2..4) of each warp; the
      // 12 warps' partials meet in shared memory
#pragma unroll
      for (int o = 4; o < 32; o <<= 1)
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          lsum[jj].x += __shfl_xor_sync(0xffffffffu, lsum[jj].x, o);
          lsum[jj].y += __shfl_xor_sync(0xffffffffu, lsum[jj].y, o);
        }
      if (r8 == 0)
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          *reinterpret_cast<float2*>(&aux.lsum[qb][wg][sp][8 * jj + 2 * c4]) = lsum[jj];
      const bool had = bar_red_or(1, 128 * NWG, anyv);  // all warpgroups: partial sums written
      if (wg < 2) {
        // warpgroups 0 / 1 write query rows [0, 32) / [32, 64)
        if (sp == 0) {
          const int q = 32 * wg + lane;
          float l = 0.f;
#pragma unroll
          for (int w2 = 0; w2 < NWG; ++w2)
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) l += aux.lsum[qb][w2][s2][q];
          aux.linv[wg][lane] = l > 0.f ? 1.f / l : 0.f;
          const long long row = token_row(p, region, q);
          const bool bad = had && !(l >= 0x1p-80f) && row >= 0;
          const unsigned bal = __ballot_sync(0xffffffffu, bad);
          if (bal != 0u && lane == 0) {  // duplicates are harmless
            const int slot = atomicAdd(p.fb_count, 1);
            p.fb_items[slot] = h * p.geo.g + region;
          }
        }
        TK_TIME(5, mbar_wait(&B.o_full[qb], (uint32_t)((seq >> 1) & 1)));
        tc_fence_after();
        const int L = 32 * sp + lane;  // TMEM lane of O^T: feature d
        float o[32];
        tmem_ld32(tl + COL_O + 64 * qb + 32 * wg, o);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&B.o_empty[qb]);
        bar_sync(2 + wg, 128);  // linv written
        {
          // lane L = feature d: column i of O^T is query 32 wg + i
          uint16_t* st = reinterpret_cast<uint16_t*>(smem + SMEM_O);
          const float* li = aux.linv[wg];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const __nv_bfloat16 v = __float2bfloat16_rn(o[i] * li[i]);
            st[(32 * wg + i) * D + L] = *reinterpret_cast<const uint16_t*>(&v);
          }
        }
        bar_sync(2 + wg, 128);  // staging complete
        {
          const int t = threadIdx.x - 32 * (W_SM + 4 * wg);  // 0..127
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int id = t + 128 * k;  // 512 chunks: 32 rows x 16 chunks of 16 B
            const int q = 32 * wg + (id >> 4), c = id & 15;
            const long long row = token_row(p, region, q);
            if (row >= 0) {
              const uint4 v = *reinterpret_cast<const uint4*>(smem + SMEM_O + q * 256 + c * 16);
              reinterpret_cast<uint4*>(p.out + h * p.oh + row * p.orow)[c] = v;
            }
          }
        }
      }
      ++seq;
    }
  }
#ifdef TK_PROF
  {
    const int role = warp == W_G1 ? 0 : warp == W_G2 ? 1 : warp == W_LD ? 2 : warp == W_LD + 4 ? 3 : warp == W_SM ? 4
                     : warp == W_Q ? 5 : warp == W_SCHED ? 6 : -1;
    if (p.trace != nullptr && lane == 0 && role >= 0) {
      long long* o = p.trace + (long long)blockIdx.x * 64 + 8 * role;
      for (int k = 0; k < 8; ++k) o[k] = prof[k];
      if (role == 0) p.trace[(long long)blockIdx.x * 64 + 63] = clock64() - t_start;
    }
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == W_G1) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

}  // namespace tkk

cudaError_t launch_tk_kernel(const k4::Params& p, int grid, cudaStream_t st) {
  cudaError_t e = ensure_smem_optin((const void*)tkk::sparse_attn_tk_kernel, tkk::SMEM_ALLOC);
  if (e != cudaSuccess) return e;
  tkk::sparse_attn_tk_kernel<<<grid, tkk::THREADS, tkk::SMEM_ALLOC, st>>>(p);
  return cudaGetLastError();
}

}  // namespace da
