// K4, the lane-half kernel (the shipped tcgen05 path): block-sparse
// FlashAttention forward with ONE query region per item, two key regions per
// step (GEMM1 at N = 128), and the two TMEM lane halves of the M = 64 tile used
// as an even / odd step pipeline.
//
// Semantics of the reference executor (sparse.py:88-166): per query
// region, kept key regions in ascending order, padding keys masked, fixed
// per-row softmax offset with the portable-kernel fallback for rows whose sum
// underflows.
//
// Why: an M = 64 tcgen05.mma costs the cycles of an M = 128 one and an N = 64
// one 44.7 cycles per K = 16 against 64 for N = 128 (tools/probes/mma_rate.cu).
// With two key regions per step GEMM1 issues M = 64, N = 128 MMAs: 512 instead
// of 614 tensor cycles per kept 64 x 64 block.
//
// Layout. Global step s of a CTA runs on TMEM lane half h = s & 1 (lanes
// {0-15, 32-47, ...} or {16-31, 48-63, ...}); each half holds its own copy of
// Q, its S buffer, its P buffer and its share of O:
//     columns [0,64) Q   [64,192) S   [192,256) P   [256,384) O (items of even
//     parity)   [384,512) O (odd items)
// so consecutive steps never share S / P / O and each barrier has a single
// waiter sequence. Softmax warpgroup h takes the steps of half h and reads its
// 16 lanes per warp with the 16x32bx2 shapes: thread t < 16 holds key region
// 2s of row t, thread t + 16 key region 2s + 1 of the same row
// (tools/probes/tmem16x2.cu). O = O_half0 + O_half1 is summed in the epilogue.
//
// Shared memory: K and V ring slots of two region tiles each (a step); the
// tiles are the pooling pass's GROUPED images (kv_tile_offset_grouped), so two
// adjacent tiles form one 128-row K-major GEMM1 operand.
//
//     GEMM1  S[64 q x 128 k]  = Q . [K_j0 ; K_j1]^T   A = Q (TMEM), B = K slot (smem, K-major, SW128, SBO 2 KB)
//     GEMM2  O[64 q x 128 d] += P . [V_j0 ; V_j1]     A = P (TMEM), B = V tiles (smem, MN-major, SW128)
//
// Roles (384 threads): warp 0 claims items (atomic counter), stages the kept
// list, emits step info and issues K copies; warp 1 GEMM1 issuer + TMEM owner;
// warp 2 V copies; warp 3 GEMM2 issuer; warps 4-7 / 8-11 softmax warpgroups
// for lane half 0 / 1 (each also loads half of Q's features into both halves
// and writes half of the output features).
#include "attn_k4.cuh"
#include "common.cuh"
#include "kernels.h"

// LH_FAKELOAD (probe builds only, tools/probes): bit 0 skips the K copies,
// bit 1 the V copies, bit 2 the softmax work. Results are then wrong; the
// shipped library is built with 0.
// LH_QPRE: the next item's Q rows are loaded during each warpgroup's last
// step of the current item instead of after it
#ifndef LH_QPRE
#define LH_QPRE 0  // measured slower (24.05 vs 23.79 ms interleaved: 161 vs 120 registers)
#endif

#ifndef LH_FAKELOAD
#define LH_FAKELOAD 0
#endif

// LH_PROF: per-CTA cycle accounting of the waits (tools/probes/lh_prof.py),
// written to the da_debug_trace buffer as [CTA][32] int64 at kernel end
#ifdef LH_PROF
#define LH_T0() const long long _t0 = clock64()
#define LH_ACC(k) prof[k] += clock64() - _t0
#else
#define LH_T0() \
  do {          \
  } while (0)
#define LH_ACC(k) \
  do {            \
  } while (0)
#endif

namespace da {
namespace lhk {

constexpr int P = 64;
constexpr int D = 128;
constexpr int TILE = 16384;
constexpr int SLOT = 2 * TILE;  // a step: key regions j0, j1
#ifndef LH_KSL
#define LH_KSL 3
#endif
#ifndef LH_VSL
#define LH_VSL 3
#endif
constexpr int KSL = LH_KSL;
constexpr int VSL = LH_VSL;
// LH_VCP: V tiles move by cp.async (LDGSTS) issued from LH_VCP extra warps
// (warps 12 ..) instead of bulk copies from warp 2, so K (bulk copy engine)
// and V (load/store units) travel L2 -> SM on two paths at once. 0 = both by
// bulk copies.
#ifndef LH_VCP
#define LH_VCP 0
#endif
constexpr int VCP = LH_VCP;
constexpr int THREADS = 384 + 32 * VCP;
constexpr int INFO = 16;  // step-info ring; even, so a slot always holds steps of one lane half
static_assert(INFO % 2 == 0, "info ring parity");
constexpr int RAGW = 512;
#ifndef LH_LISTCAP
#define LH_LISTCAP 4096
#endif
constexpr int LISTCAP = LH_LISTCAP;
constexpr int IR = 8;
constexpr int KBLK = 32;

constexpr int SMEM_K = 0;
constexpr int SMEM_V = SMEM_K + KSL * SLOT;
constexpr int SMEM_END = SMEM_V + VSL * SLOT;

constexpr uint32_t TMEM_COLS = 512;
// wait flavours: 1 = test_wait spin (lowest wake-up latency, but a spinning
// warp takes issue slots from the warps sharing its scheduler), 0 = try_wait
// with a suspend hint (the warp sleeps until the phase completes)
#ifndef LH_SM_SPIN
#define LH_SM_SPIN 1  // the softmax warps' waits (S full, step info, P free)
#endif
#ifndef LH_G_SPIN
#define LH_G_SPIN 1  // the GEMM issuers' waits
#endif
#if LH_SM_SPIN
#define LH_SMWAIT mbar_wait_spin
#else
#define LH_SMWAIT mbar_wait
#endif
#if LH_G_SPIN
#define LH_GWAIT mbar_wait_spin
#else
#define LH_GWAIT mbar_wait
#endif
#ifndef LH_POLY8
#define LH_POLY8 0  // bit k % 8 (k even): exponential pair k on the FMA pipe (degree-3 polynomial) instead of MUFU; 0x40 (one pair in four) measured 1.9 % slower than none (profiles/r02/k4_variants_final.log)
#endif
#ifndef LH_S2
#define LH_S2 0  // 1: two S buffers per lane half (O single-buffered) instead of one (O double-buffered); measured equal
#endif
#if LH_S2
constexpr uint32_t COL_Q = 0, COL_S = 64, COL_P = 320, COL_O = 384;
constexpr int NSB = 2;  // S buffers per lane half
#else
constexpr uint32_t COL_Q = 0, COL_S = 64, COL_P = 192, COL_O = 256;
constexpr int NSB = 1;
#endif
constexpr int NOB = 3 - NSB;  // O buffers (item parity when 2)
constexpr uint32_t LANE_H = 16u << 16;  // TMEM address offset of lane half 1

using k4::Params;
using k4::Item;
using k4::fetch_item;
using k4::item_from_record;
using k4::item_record;
using k4::token_row;
using k4::key_mask;

struct __align__(8) Bars {
  uint64_t k_full[KSL], k_empty[KSL];
  uint64_t v_full[VSL], v_empty[VSL];
  uint64_t s_full[2][NSB], s_free[2][NSB];  // per lane half and S buffer
  uint64_t p_full[2], p_free[2];            // per lane half
  uint64_t o_full[NOB], o_empty[NOB];       // per O buffer
  uint64_t q_full, q_empty;
  uint64_t info_full[INFO], info_empty[INFO];
  uint64_t item_full[IR], item_empty[IR];
};
struct SmemAux {
  Bars bars;
  int4 info[INFO];      // per step: j0, j1, flags (1 j0, 2 j1, 4 j0 ragged, 8 j1 ragged), w (1 last, 2 first)
  int4 items[IR];  // item records (attn_k4.cuh item_record), kept count -1: end
  uint32_t tmem_base;
  float xm[2][64];      // [item parity][row] fixed softmax offset
  float xq[2][2][64];   // [item parity][warpgroup][row] partial |q|^2
  float lsum[2][64];    // [warpgroup][row] partial row sums
  int had[2][64];       // [warpgroup][row] saw a kept valid key
  uint32_t ragged[RAGW];
  int list[LISTCAP];
};
constexpr int SMEM_ALLOC = SMEM_END + (int)sizeof(SmemAux);
static_assert(SMEM_ALLOC <= 227 * 1024, "shared memory budget");

// Per head: query regions by kept count, descending: the dynamic item order
// puts the heaviest items first (the order within a count does not matter:
// every region's output is computed independently). One block per head:
// count histogram, block-wide exclusive scan, atomic placement.
// split: every mask region is two items (its halves 2 i, 2 i + 1, Params::split).
__global__ void __launch_bounds__(1024) region_order_kernel(const int* __restrict__ row_ptr, int g, int mask_h,
                                                            int split, int4* __restrict__ meta) {
  extern __shared__ int bins[];  // [g + 1], key = g - count
  __shared__ int wsum[32];
  const int h = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int* rp = row_ptr + (long long)(h * mask_h) * (g + 1);
  const int nb = g + 1;
  for (int i = t; i < nb; i += blockDim.x) bins[i] = 0;
  __syncthreads();
  for (int i = t; i < g; i += blockDim.x) atomicAdd(&bins[g - min(g, rp[i + 1] - rp[i])], 1 << split);
  __syncthreads();
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int k0 = min(nb, t * per), k1 = min(nb, k0 + per);
  int local = 0;
  for (int k = k0; k < k1; ++k) local += bins[k];
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x / 32;
    int v = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane < nw) wsum[lane] = v;  // inclusive warp totals
  }
  __syncthreads();
  int run = incl - local + (w > 0 ? wsum[w - 1] : 0);
  for (int k = k0; k < k1; ++k) {
    const int v = bins[k];
    bins[k] = run;
    run += v;
  }
  __syncthreads();
  for (int i = t; i < g; i += blockDim.x) {
    const int pos = atomicAdd(&bins[g - min(g, rp[i + 1] - rp[i])], 1 << split);
    const int b = rp[i];
    int4* m = meta + ((long long)h * g << split) + pos;
    for (int s = 0; s < (1 << split); ++s)  // the item records (attn_k4.cuh)
      m[s] = make_int4((i << split) + s, b, rp[i + 1] - b, h);
  }
}

// A warp takes a step-info entry: lane 0 reads it, releases the slot and
// broadcasts it (the slot's release then orders the only read of it).
DA_DEV int4 take_info(const int4* info, uint64_t* empty, int i, int lane) {
  int4 e = make_int4(0, 0, 0, 0);
  if (lane == 0) {
    e = info[i];
    mbar_arrive(empty);
  }
  e.x = __shfl_sync(0xffffffffu, e.x, 0);
  e.y = __shfl_sync(0xffffffffu, e.y, 0);
  e.z = __shfl_sync(0xffffffffu, e.z, 0);
  e.w = __shfl_sync(0xffffffffu, e.w, 0);
  return e;
}

template <bool SPLIT>  // SPLIT: Q / out rows in sequence shards (Params::sh)
__global__ void __launch_bounds__(THREADS, 1) sparse_attn_lh_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  SmemAux& aux = *reinterpret_cast<SmemAux*>(smem + SMEM_END);
  Bars& B = aux.bars;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long items = (long long)p.heads * p.geo.g;
#ifdef LH_PROF
  long long prof[20];
  for (int k = 0; k < 20; ++k) prof[k] = 0;
  const long long t_start = clock64();
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < KSL; ++s) { mbar_init(&B.k_full[s], 1); mbar_init(&B.k_empty[s], 1); }
    for (int s = 0; s < VSL; ++s) { mbar_init(&B.v_full[s], VCP ? 32 * VCP : 1); mbar_init(&B.v_empty[s], 1); }
    for (int h = 0; h < 2; ++h) {
      for (int b = 0; b < NSB; ++b) {
        mbar_init(&B.s_full[h][b], 1);
        mbar_init(&B.s_free[h][b], 128);
      }
      mbar_init(&B.p_full[h], 128);
      mbar_init(&B.p_free[h], 1);
      if (h < NOB) {
        mbar_init(&B.o_full[h], 1);
        mbar_init(&B.o_empty[h], 256);
      }
    }
    mbar_init(&B.q_full, 256);
    mbar_init(&B.q_empty, 1);
    for (int s = 0; s < INFO; ++s) {
      mbar_init(&B.info_full[s], 1);
      // readers of a step entry: the V producer, GEMM1, GEMM2 and the 4 warps of
      // the softmax warpgroup of the step's lane half (INFO is even: a slot
      // always holds steps of one parity)
      mbar_init(&B.info_empty[s], (VCP ? VCP : 1) + 2 + 4);
    }
    for (int s = 0; s < IR; ++s) {
      mbar_init(&B.item_full[s], 1);
      mbar_init(&B.item_empty[s], VCP ? 10 + VCP : 11);  // warps 1, 3, the 8 softmax warps and the V warp(s)
    }
    fence_barrier_init();
  }
  if (LH_FAKELOAD) {
    for (int i = threadIdx.x; i < SMEM_END / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
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
  if (warp == 1) tmem_alloc<TMEM_COLS>(&aux.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = aux.tmem_base;
  uint8_t* sK = smem + SMEM_K;
  uint8_t* sV = smem + SMEM_V;

  int ring_i = 0;
  uint32_t ring_ph = 0;
  auto peek_item = [&]() {
    mbar_wait_spin(&B.item_full[ring_i], ring_ph);
    return aux.items[ring_i];
  };
  auto next_item = [&]() {
    const int4 r = peek_item();
    __syncwarp();
    if (lane == 0) mbar_arrive(&B.item_empty[ring_i]);
    if (++ring_i == IR) { ring_i = 0; ring_ph ^= 1u; }
    return r;
  };

  if (warp == 0 || (warp == 2 && VCP == 0)) {
    // ===================== producers (warp 0: items, step info, K; warp 2: V) =====================
    const bool is_k = warp == 0;
    const int NSL = is_k ? KSL : VSL;
    uint8_t* ring = is_k ? sK : sV;
    uint64_t* full = is_k ? B.k_full : B.v_full;
    uint64_t* empty = is_k ? B.k_empty : B.v_empty;
    const bool bitmap = p.key_valid == nullptr && p.geo.g <= 32 * RAGW;
    int kq = 0, claimed = 0;
    // K producer: claims run two items ahead and item records one ahead, so
    // a new item's first steps follow the previous item's without waiting on
    // global memory; consumers get the record through the item ring
    long long claim = 0;
    int4 rec_next = make_int4(0, 0, -1, 0);
    if (is_k) {
      long long c0 = 0;
      if (lane == 0) {
        c0 = atomicAdd(p.work, 1);
        claim = atomicAdd(p.work, 1);
      }
      rec_next = item_record(p, __shfl_sync(0xffffffffu, c0, 0), items);
    }
    for (;;) {
      Item itm;
      if (is_k) {
        int4 rec;
        for (;;) {
          rec = rec_next;
          long long c = 0;
          if (lane == 0) {
            c = claim;
            claim = atomicAdd(p.work, 1);
          }
          rec_next = item_record(p, __shfl_sync(0xffffffffu, c, 0), items);  // lands while this item streams
          if (rec.z != 0) break;  // kept key regions, or past the last item
          // no kept key region: the region's output rows are zero
          for (int e = lane; e < P * (D / 8); e += 32) {
            const long long row = token_row(p, rec.x, e / (D / 8));
            if (row >= 0)
              reinterpret_cast<uint4*>(shard_at<SPLIT>(p.sh, SH_O, p.out, rec.w * p.oh, row, p.orow))[e % (D / 8)] =
                  make_uint4(0, 0, 0, 0);
          }
        }
        const int slot = claimed % IR;
        if (claimed >= IR) { LH_T0(); mbar_wait(&B.item_empty[slot], (uint32_t)(((claimed / IR) - 1) & 1)); LH_ACC(0); }
        if (lane == 0) {
          aux.items[slot] = rec;
          mbar_arrive(&B.item_full[slot]);
        }
        ++claimed;
        if (!item_from_record(p, rec, itm)) break;
      } else {
        if (!item_from_record(p, next_item(), itm)) break;
      }
      const int nlist = itm.n >> p.split;  // mask entries of the item
      const bool staged = is_k && nlist <= LISTCAP;
      if (staged) {
        __syncwarp();
        for (int e = lane; e < nlist; e += 32) aux.list[e] = __ldg(itm.list + e);
        __syncwarp();
      }
      if (lane == 0) {
        const int n = (itm.n + 1) / 2;
        const uint8_t* hb = (is_k ? p.kt : p.vt) + (long long)itm.h * p.geo.g * TILE;
        for (int t = 0; t < n; ++t) {
          int4 e;
          const int ii = kq % INFO;
          if (is_k) {
            int j0, j1;
            if (p.split) {  // parts 2 sub and 2 sub + 1 of mask entry t >> (split - 1)
              const int e_ = t >> (p.split - 1), sub = t & ((1 << (p.split - 1)) - 1);
              j0 = ((staged ? aux.list[e_] : __ldg(itm.list + e_)) << p.split) + 2 * sub;
              j1 = j0 + 1;
            } else {
              j0 = staged ? aux.list[2 * t] : __ldg(itm.list + 2 * t);
              j1 = 2 * t + 1 < itm.n ? (staged ? aux.list[2 * t + 1] : __ldg(itm.list + 2 * t + 1)) : -1;
            }
            int fl = 1;
            if (bitmap ? (aux.ragged[j0 >> 5] >> (j0 & 31)) & 1 : key_mask(p, j0) != ~0ull) fl |= 4;
            if (j1 >= 0) {
              fl |= 2;
              if (bitmap ? (aux.ragged[j1 >> 5] >> (j1 & 31)) & 1 : key_mask(p, j1) != ~0ull) fl |= 8;
            }
            e = make_int4(j0, j1, fl, (t == n - 1 ? 1 : 0) | (t == 0 ? 2 : 0));
            if (kq >= INFO) mbar_wait(&B.info_empty[ii], (uint32_t)(((kq / INFO) - 1) & 1));
            aux.info[ii] = e;
            mbar_arrive(&B.info_full[ii]);
          } else {
            { LH_T0(); mbar_wait(&B.info_full[ii], (uint32_t)((kq / INFO) & 1)); LH_ACC(18); }
            e = aux.info[ii];
            mbar_arrive(&B.info_empty[ii]);
          }
          const int s = kq % NSL;
          if (kq >= NSL) { LH_T0(); mbar_wait(&empty[s], ((kq / NSL) - 1) & 1); LH_ACC(is_k ? 16 : 17); }
          ++kq;
          if (LH_FAKELOAD & (is_k ? 1 : 2)) {
            mbar_arrive(&full[s]);
            continue;
          }
          uint8_t* st = ring + s * SLOT;
          mbar_expect_tx(&full[s], TILE * (1 + ((e.z >> 1) & 1)));
          bulk_g2s(st, hb + (long long)e.x * TILE, TILE, &full[s], p.pol_kv);
          if (e.z & 2) bulk_g2s(st + TILE, hb + (long long)e.y * TILE, TILE, &full[s], p.pol_kv);
        }
      }
    }
  } else if (warp == 1) {
    // ========================= GEMM1 issuer =========================
    constexpr uint32_t IDESC_N128 = umma_idesc_bf16(64, 128, 0, 0);
    constexpr uint32_t IDESC_N64 = umma_idesc_bf16(64, 64, 0, 0);
    const uint64_t dK = umma_desc_sw128(0, 16, 2048) + (smem_u32(sK) >> 4);
    int gs = 0, iidx = 0;
    uint32_t iph = 0;
    int qi = 0;
    for (;;) {
      Item itm;
      if (!item_from_record(p, next_item(), itm)) break;
      { LH_T0(); mbar_wait(&B.q_full, qi & 1); LH_ACC(1); }
      for (;;) {
        { LH_T0(); LH_GWAIT(&B.info_full[iidx], iph); LH_ACC(2); }
        const int4 e = take_info(aux.info, &B.info_empty[iidx], iidx, lane);
        const int last = e.w & 1;
        const int h = gs & 1;
        // this half's S buffer: the softmax has loaded step gs - 2
        // step gs uses S buffer sb of half h; the softmax has loaded its previous use (step gs - 2 NSB)
        const int sb = (gs >> 1) % NSB;
        if (gs >= 2 * NSB) {
          LH_T0();
          LH_GWAIT(&B.s_free[h][sb], (uint32_t)(((gs / (2 * NSB)) - 1) & 1));
          LH_ACC(3);
        }
        const int s = gs % KSL;
        { LH_T0(); LH_GWAIT(&B.k_full[s], (uint32_t)((gs / KSL) & 1)); LH_ACC(4); }
        tc_fence_after();
        if (elect_one_sync()) {
          const uint32_t lo = h ? LANE_H : 0u;
          const uint32_t idesc = (e.z & 2) ? IDESC_N128 : IDESC_N64;
          const uint64_t bk = dK + (uint64_t)(s * (SLOT >> 4));
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts(tmem + lo + COL_S + 128 * sb, tmem + lo + COL_Q + kk * 8,
                         bk + (uint64_t)((kk >> 2) * (1024 >> 4) + (kk & 3) * 2), idesc, kk > 0 ? 1u : 0u);
          umma_commit(&B.k_empty[s]);
          umma_commit(&B.s_full[h][sb]);
          if (last) umma_commit(&B.q_empty);
        }
        __syncwarp();
        ++gs;
        if (++iidx == INFO) { iidx = 0; iph ^= 1u; }
        if (last) break;
      }
      ++qi;
    }
  } else if (warp == 3) {
    // ========================= GEMM2 issuer =========================
    constexpr uint32_t IDESC2 = umma_idesc_bf16(64, 128, 0, 1);  // B (V) MN-major
    const uint64_t dV = umma_desc_sw128(0, 1024, 2048) + (smem_u32(sV) >> 4);
    int gs = 0, iidx = 0;
    uint32_t iph = 0;
    int qi = 0;
    for (;;) {
      Item itm;
      if (!item_from_record(p, next_item(), itm)) break;
      const int ob = qi % NOB;
      int t = 0;
      for (;;) {
        { LH_T0(); LH_GWAIT(&B.info_full[iidx], iph); LH_ACC(5); }
        const int4 e = take_info(aux.info, &B.info_empty[iidx], iidx, lane);
        const int last = e.w & 1;
        const int h = gs & 1;
        const int s = gs % VSL;
        { LH_T0(); LH_GWAIT(&B.v_full[s], (uint32_t)((gs / VSL) & 1)); LH_ACC(6); }
        { LH_T0(); LH_GWAIT(&B.p_full[h], (uint32_t)((gs >> 1) & 1)); LH_ACC(7); }
        if (t == 0 && qi >= NOB) {
          LH_T0();
          mbar_wait(&B.o_empty[ob], (uint32_t)(((qi / NOB) - 1) & 1));
          LH_ACC(8);
        }
        tc_fence_after();
        if (elect_one_sync()) {
          const uint32_t lo = h ? LANE_H : 0u;
          const uint64_t bv = dV + (uint64_t)(s * (SLOT >> 4));
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            if (c == 1 && !(e.z & 2)) break;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_bf16_ts(tmem + lo + COL_O + 128 * ob, tmem + lo + COL_P + 32 * c + 8 * kk,
                           bv + (uint64_t)((c * TILE + kk * 4096) >> 4), IDESC2,
                           (t < 2 && c == 0 && kk == 0) ? 0u : 1u);
          }
          umma_commit(&B.v_empty[s]);
          umma_commit(&B.p_free[h]);
          if (last) umma_commit(&B.o_full[ob]);
        }
        __syncwarp();
        ++gs;
        ++t;
        if (++iidx == INFO) { iidx = 0; iph ^= 1u; }
        if (last) break;
      }
      ++qi;
    }
  } else if (warp >= 12) {
    // ============ V copiers (LH_VCP > 0): cp.async of the step's V tiles ============
    const int t = threadIdx.x - 384;
    constexpr int NT = 32 * VCP;
    int kq = 0;
    for (;;) {
      Item itm;
      if (!item_from_record(p, next_item(), itm)) break;
      const uint8_t* hb = p.vt + (long long)itm.h * p.geo.g * TILE;
      const int n = (itm.n + 1) / 2;
      for (int st = 0; st < n; ++st) {
        const int ii = kq % INFO;
        mbar_wait_warp(&B.info_full[ii], (uint32_t)((kq / INFO) & 1));
        const int4 e = take_info(aux.info, &B.info_empty[ii], ii, lane);
        const int s = kq % VSL;
        if (kq >= VSL) mbar_wait_warp(&B.v_empty[s], ((kq / VSL) - 1) & 1);
        ++kq;
        const uint32_t dst = smem_u32(sV + s * SLOT);
        const uint8_t* src0 = hb + (long long)e.x * TILE;
#pragma unroll
        for (int c = t; c < TILE / 16; c += NT) cp_async16(dst + 16 * c, src0 + 16 * c, 16);
        if (e.z & 2) {
          const uint8_t* src1 = hb + (long long)e.y * TILE;
#pragma unroll
          for (int c = t; c < TILE / 16; c += NT) cp_async16(dst + TILE + 16 * c, src1 + 16 * c, 16);
        }
        cp_async_arrive_noinc(&B.v_full[s]);
      }
    }
  } else if (warp >= 4) {
    // ============ softmax warpgroup wg = lane half wg; Q loader; epilogue ============
    // Warp w (subpartition sp = w % 4) owns rows 16 sp .. 16 sp + 15: lanes
    // 32 sp + [0,16) of half 0 and 32 sp + 16 + [0,16) of half 1. In a step
    // thread lane (< 16 / >= 16) processes key region j0 / j1 of row
    // 16 sp + lane % 16.
    const int wg = (warp - 4) >> 2;
    const int sp = warp & 3;
    const int c = lane >> 4;            // chunk: key region j0 (0) or j1 (1) of a step
    const int r = 16 * sp + (lane & 15);
    const uint32_t tl = tmem + ((uint32_t)(sp * 32) << 16);    // 32x32b lane base (epilogue, Q)
    const uint32_t th = tl + (wg ? LANE_H : 0u);               // this warpgroup's half (16x32bx2)
    const float sl2 = p.scale_log2;
    int G = 0;   // global step index of the current item's first step
    int qi = 0;
    float qn2_next = 0.f;
    // Q row r, feature half wg, into BOTH lane halves of columns [32 wg, 32 wg + 32)
    // (lane < 16 writes half 0, lane >= 16 half 1: the same row)
    // the next item's Q rows can be fetched early, during this warpgroup's
    // last step of the current item (LH_QPRE), and stored once GEMM1 is done
    // with the current Q
    uint32_t qv[32];
    auto issue_q = [&](const Item& itm) {
      const long long qrow = token_row(p, itm.i, r);
      if (qrow >= 0) {
        const uint4* src = reinterpret_cast<const uint4*>(shard_at<SPLIT>(p.sh, SH_Q, p.q, itm.h * p.qh, qrow, p.qr)) + wg * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint4 w = ldg128_hint(src + k, p.pol_q);
          qv[4 * k] = w.x; qv[4 * k + 1] = w.y; qv[4 * k + 2] = w.z; qv[4 * k + 3] = w.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 32; ++k) qv[k] = 0u;
      }
    };
    auto finish_q = [&](int wait_parity) {
      float s2 = 0.f;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qv[k]));
        s2 = fmaf(f.x, f.x, fmaf(f.y, f.y, s2));
      }
      qn2_next = s2;
      if (wait_parity >= 0) { LH_T0(); mbar_wait(&B.q_empty, (uint32_t)wait_parity); LH_ACC(13); }
      tc_fence_after();
      tmem_st16u(tl + COL_Q + wg * 32, *reinterpret_cast<uint32_t(*)[16]>(&qv[0]));
      tmem_st16u(tl + COL_Q + wg * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(&qv[16]));
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&B.q_full);
    };
    auto load_q = [&](const Item& itm, int wait_parity) {
      issue_q(itm);
      finish_q(wait_parity);
    };
    bool q_issued = false;  // the next item's Q rows are in flight in qv
    bool have_q = false;
    int cur_head = -1;
    float kmax = 0.f;
    for (;;) {
      Item itm;
      if (!item_from_record(p, next_item(), itm)) break;
      const long long row = token_row(p, itm.i, r);
      const int nsteps = (itm.n + 1) / 2;
      const int ob = qi % NOB;
      if (!have_q) load_q(itm, -1);
      const float qn2_own = qn2_next;
      if (itm.h != cur_head) {
        cur_head = itm.h;
        const float* kp = p.kpart + (long long)itm.h * p.kblk;
        float mx = 0.f;
#pragma unroll 8
        for (int k = 0; k < p.kblk; ++k) mx = fmaxf(mx, __ldg(kp + k));
        kmax = mx;
      }
      if (lane < 16) aux.xq[qi & 1][wg][r] = qn2_own;
      { LH_T0(); bar_sync(1, 256); LH_ACC(14); }
      const float qn2 = aux.xq[qi & 1][0][r] + aux.xq[qi & 1][1][r];
      const int first_wg = G & 1;  // the warpgroup that runs the item's first step fixes the offsets
      float m = 0.f, l = 0.f;
      bool had = false;
      bool got_m = false;
      float x[64];
      for (int t = (wg - first_wg) & 1; t < nsteps; t += 2) {
        const int gs = G + t;
#if LH_QPRE
        if (t + 2 >= nsteps && !q_issued &&
            mbar_test_wait(smem_u32(&B.item_full[ring_i]), ring_ph)) {
          // this warpgroup's last step of the item: the next record is out,
          // fetch its Q rows while this step's softmax runs
          Item nx;
          if (item_from_record(p, aux.items[ring_i], nx)) {
            issue_q(nx);
            q_issued = true;
          }
        }
#endif
        const int ii = gs & (INFO - 1);
        { LH_T0(); LH_SMWAIT(&B.info_full[ii], (uint32_t)((gs / INFO) & 1)); LH_ACC(9); }
        const int4 e = take_info(aux.info, &B.info_empty[ii], ii, lane);
        const int sb = (gs >> 1) % NSB;
        { LH_T0(); LH_SMWAIT(&B.s_full[wg][sb], (uint32_t)((gs / (2 * NSB)) & 1)); LH_ACC(10); }
        tc_fence_after();
        const bool kp = ((e.z >> c) & 1) && !(LH_FAKELOAD & 4);
        if (!(LH_FAKELOAD & 4)) {
          tmem_ld16x2_32(th + COL_S + 128 * sb, x);
          tmem_ld16x2_32hi(th + COL_S + 128 * sb + 32, x);
          tmem_ld_wait();
        }
        tc_fence_before();
        mbar_arrive(&B.s_free[wg][sb]);  // scores in registers: GEMM1 may refill this buffer
        if (!(LH_FAKELOAD & 4)) {
          const int j = c ? e.y : e.x;
          const bool rag = (e.z >> (2 + c)) & 1;
          const unsigned long long vm = kp ? (rag ? key_mask(p, j) : ~0ull) : 0ull;
          if (vm != ~0ull) {
#pragma unroll
            for (int k = 0; k < 64; ++k) x[k] = ((vm >> k) & 1ull) ? x[k] : -INFINITY;
          }
          had |= vm != 0ull;
        }
        if (!got_m) {
          if (t == 0) {  // first step of the item: fix the row's offset from its two key regions
            float bm = -INFINITY;
            if (kp) {
              float mx[8];
#pragma unroll
              for (int q = 0; q < 8; ++q)
                mx[q] = fmaxf(fmaxf(fmaxf(x[q], x[q + 8]), fmaxf(x[q + 16], x[q + 24])),
                              fmaxf(fmaxf(x[q + 32], x[q + 40]), fmaxf(x[q + 48], x[q + 56])));
              bm = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                         fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
            }
            bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 16)) * sl2;
            const float bound = sqrtf(qn2) * kmax * sl2 * 1.0001f;
            m = fmaxf(bm, bound - 64.f);
            if (lane < 16) aux.xm[qi & 1][r] = m;
            bar_arrive(2, 256);
          } else {
            { LH_T0(); bar_sync(2, 256); LH_ACC(15); }
            m = aux.xm[qi & 1][r];
          }
          got_m = true;
        }
        uint32_t pk[32];
        {
          const float2 sc = make_float2(sl2, sl2), nm = make_float2(-m, -m);
          float2 acc = make_float2(0.f, 0.f);
#pragma unroll
          for (int k = 0; k < 64; k += 2) {
            const float2 ev = ffma2(make_float2(x[k], x[k + 1]), sc, nm);
            const float2 pe = ((LH_POLY8 >> (k % 8)) & 1) ? exp2_poly2(ev) : make_float2(fast_exp2(ev.x), fast_exp2(ev.y));
            acc = fadd2(acc, pe);
            pk[k / 2] = kp ? pack_bf16(pe.x, pe.y) : 0u;
          }
          if (kp) l += acc.x + acc.y;
        }
        // this half's P buffer: GEMM2 of step gs - 2 has read it
        if (gs >= 2) {
          { LH_T0(); LH_SMWAIT(&B.p_free[wg], (uint32_t)(((gs >> 1) - 1) & 1)); LH_ACC(11); }
          tc_fence_after();
        }
        tmem_st16x2_16(th + COL_P, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
        tmem_st16x2_16(th + COL_P + 16, *reinterpret_cast<uint32_t(*)[16]>(&pk[16]));
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&B.p_full[wg]);
      }
      if (!got_m) {  // this warpgroup had no step: still take part in the offset hand-off
        if (first_wg == wg) bar_arrive(2, 256);
        else bar_sync(2, 256);
      }
      G += nsteps;
      // ---- next item's Q
      have_q = false;
      if (q_issued) {
        finish_q(qi & 1);
        have_q = true;
        q_issued = false;
      } else {
        Item nx;
        if (item_from_record(p, peek_item(), nx)) {
          load_q(nx, qi & 1);
          have_q = true;
        }
      }
      // ------------------------------ epilogue ------------------------------
      l += __shfl_xor_sync(0xffffffffu, l, 16);
      had = __shfl_xor_sync(0xffffffffu, had ? 1 : 0, 16) != 0 || had;
      if (lane < 16) {
        aux.lsum[wg][r] = l;
        aux.had[wg][r] = had ? 1 : 0;
      }
      bar_sync(1, 256);
      const float lt = aux.lsum[0][r] + aux.lsum[1][r];
      const bool bad = (aux.had[0][r] || aux.had[1][r]) && !(lt >= 0x1p-80f);
      { LH_T0(); mbar_wait(&B.o_full[ob], (uint32_t)((qi / NOB) & 1)); LH_ACC(12); }
      tc_fence_after();
      // lane < 16 reads O of half 0, lane >= 16 O of half 1 (same row); a half
      // without any step of this item holds no O for it
      const int myhalf = lane >> 4;
      const bool used = nsteps >= 2 || (G - nsteps + 0) % 2 == myhalf;
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      float o[64];
      tmem_ld32_at<0>(tl + COL_O + 128 * ob + wg * 64, o);
      tmem_ld32_at<32>(tl + COL_O + 128 * ob + wg * 64 + 32, o);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&B.o_empty[ob]);
      uint32_t w[16];
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        // lane < 16 writes features wg*64 + [0,32), lane >= 16 wg*64 + [32,64)
        float a0 = used ? (myhalf ? o[32 + k] : o[k]) : 0.f;
        float a1 = used ? (myhalf ? o[33 + k] : o[k + 1]) : 0.f;
        const float s0 = used ? (myhalf ? o[k] : o[32 + k]) : 0.f;
        const float s1 = used ? (myhalf ? o[k + 1] : o[33 + k]) : 0.f;
        a0 += __shfl_xor_sync(0xffffffffu, s0, 16);
        a1 += __shfl_xor_sync(0xffffffffu, s1, 16);
        w[k / 2] = pack_bf16(a0 * inv, a1 * inv);
      }
      if (row >= 0) {
        uint4* dst = reinterpret_cast<uint4*>(shard_at<SPLIT>(p.sh, SH_O, p.out, itm.h * p.oh, row, p.orow) + wg * 64 + myhalf * 32);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          stg128_hint(dst + k, make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]), p.pol_o);
      }
      if (wg == 0) {  // one push per warp with a bad row; duplicates are harmless
        const unsigned bal = __ballot_sync(0xffffffffu, bad && row >= 0 && lane < 16);
        if (bal != 0u && lane == 0) {
          const int slot = atomicAdd(p.fb_count, 1);
          p.fb_items[slot] = itm.h * (p.geo.g >> p.split) + (itm.i >> p.split);  // (split: the whole region)
        }
      }
      ++qi;
    }
  }
#ifdef LH_PROF
  // lane 0 of warps 0 (K producer), 1 (GEMM1), 2 (V), 3 (GEMM2), 4 and 8 (softmax): sums per CTA
  if (p.trace != nullptr && lane == 0 && (warp <= 4 || warp == 8)) {
    long long* o = p.trace + (long long)blockIdx.x * 32;
    for (int k = 0; k < 20; ++k)
      if (prof[k]) atomicAdd(reinterpret_cast<unsigned long long*>(&o[k]), (unsigned long long)prof[k]);
    if (warp == 1) o[31] = clock64() - t_start;
  }
#endif
  // output rows stored into peer GPUs' shards: made visible system-wide before
  // the kernel ends (the caller's cross-GPU barrier follows it)
  if constexpr (SPLIT) __threadfence_system();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<TMEM_COLS>(tmem);
  }
}

// K and V re-laid out as per-region tiles that are byte-for-byte the
// shared-memory image the MMAs read (GROUPED layout, kv_tile_offset_grouped;
// padding rows zero): the attention kernel fetches each tile with one
// contiguous bulk copy. The pipeline's pooling pass writes these itself; this
// kernel serves the block-sparse seam. grid (g, heads, 2 tensors), 256 threads.
struct KvTileArgs {
  const __nv_bfloat16* x[2];
  long long hs[2], rs[2];
  uint8_t* out[2];
  int layout;
  Shards sh;  // sequence shards of K / V (original layout), or unsplit
};
__global__ void __launch_bounds__(256) kv_tile_kernel(const __grid_constant__ KvTileArgs a, Geo g, RegionDecoder dec) {
#ifdef DA_K4_TK
  __shared__ __align__(16) uint16_t vs[P * D];  // V^T (experimental transposed K4): V rows, transposed on the way out
#endif
  const int j = blockIdx.x, h = blockIdx.y, z = blockIdx.z;
  const RegionXY rc = dec(j);
  // z selects K (0) or V (1) without dynamic parameter indexing (no local-memory copy)
  const __nv_bfloat16* xz = z ? a.x[1] : a.x[0];
  const long long ho = h * (z ? a.hs[1] : a.hs[0]), rs = z ? a.rs[1] : a.rs[0];
  uint8_t* dst = (z ? a.out[1] : a.out[0]) + ((long long)h * g.g + j) * TILE;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = threadIdx.x + 256 * i;
    const int r = idx >> 4, c = idx & 15;
    long long row;
    if (a.layout == DA_LAYOUT_REORDERED) {
      row = (long long)j * P + r;
    } else {
      const int u = r / g.pw, v = r - u * g.pw;
      row = (rc.y0 + u < g.H && rc.x0 + v < g.W) ? ((long long)rc.f * g.H + rc.y0 + u) * g.W + rc.x0 + v : -1;
    }
    const uint4 val =
        row >= 0 ? __ldg(reinterpret_cast<const uint4*>(shard_addr(a.sh, z ? SH_V : SH_K, xz, ho, row, rs)) + c)
                 : make_uint4(0, 0, 0, 0);
#ifndef DA_K4_TK
    *reinterpret_cast<uint4*>(dst + kv_tile_offset_grouped(r, c >> 3, c & 7)) = val;
#else
    if (z == 0) *reinterpret_cast<uint4*>(dst + kv_tile_offset_grouped(r, c >> 3, c & 7)) = val;
    else *reinterpret_cast<uint4*>(vs + r * D + 8 * c) = val;
#endif
  }
#ifdef DA_K4_TK
  if (z == 1) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int o = threadIdx.x + 256 * i;
      const int kc = o >> 7, d = o & 127;  // keys 8 kc .. 8 kc + 7 of feature d
      uint32_t w[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) w[m] = (uint32_t)vs[(8 * kc + 2 * m) * D + d] | ((uint32_t)vs[(8 * kc + 2 * m + 1) * D + d] << 16);
      *reinterpret_cast<uint4*>(dst + kc * 2048 + d * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
#endif
}

// Per-head maximum key row norm as KBLK per-block partial maxima (the bound
// behind the fixed softmax offset), for callers without the pooling pass.
// grid (KBLK, heads), 256 threads: each warp reads two 256-byte rows per load.
__global__ void __launch_bounds__(256) key_norm_kernel(const __nv_bfloat16* __restrict__ k, long long kh, long long kr,
                                                       long long rows, float* __restrict__ kpart,
                                                       const __grid_constant__ Shards sh) {
  __shared__ float red[8];
  const int h = blockIdx.y;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int sub = lane >> 4, c = lane & 15;
  const long long step = (long long)KBLK * 8 * 2;
  float mx = 0.f;
  for (long long r0 = ((long long)blockIdx.x * 8 + w) * 2 + sub; r0 < rows; r0 += 4 * step) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long rr = r0 + u * step;
      v[u] = rr < rows ? __ldg(reinterpret_cast<const uint4*>(shard_addr(sh, SH_K, k, h * kh, rr, kr)) + c)
                       : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t wv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
      float s2 = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[e]));
        s2 = fmaf(f.x, f.x, fmaf(f.y, f.y, s2));
      }
#pragma unroll
      for (int o = 8; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      mx = fmaxf(mx, s2);
    }
  }
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
  if (lane == 0) red[w] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = red[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) b = fmaxf(b, red[i]);
    kpart[(long long)h * KBLK + blockIdx.x] = sqrtf(b);
  }
}

}  // namespace lhk

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static long long* g_trace = nullptr;  // LH_PROF builds only (da_debug_trace)
void set_tc_trace(void* buf) { g_trace = static_cast<long long*>(buf); }

static inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// Attention workspace: [counters 256 B | key norm maxima (heads x KBLK floats)
// | fallback items (4 per item) | region order (heads x g) | K tiles | V tiles]
static size_t ws_norms() { return 256; }
static size_t ws_items(int heads) { return ws_norms() + align256(sizeof(float) * heads * lhk::KBLK); }
static size_t ws_order(int heads, const Geo& g) { return ws_items(heads) + align256(sizeof(int) * 4 * (size_t)heads * g.g); }
static size_t ws_tiles(int heads, const Geo& g) { return ws_order(heads, g) + align256(sizeof(int4) * (size_t)heads * g.g); }

// The geometry K4 runs on: 64-token regions as they are; 64 x 2^s-token
// regions as their 2^s column parts (Params::split = s), so the paper's 8x16
// pools run as 8x8 half-regions on the same kernel.
Geo attn_geo(const Geo& g) {
  const int s = region_parts_shift(g);
  if (s <= 0) return g;
  Geo v = g;
  v.pw = g.pw >> s;
  v.Pw = g.Pw << s;  // parts of padding-only columns stay (all keys invalid, no output rows)
  v.p = 64;
  v.g = g.g << s;
  return v;
}

uint8_t* attn_tiles(void* ws, int heads, const Geo& g0, int which) {
  const Geo g = attn_geo(g0);
  return static_cast<uint8_t*>(ws) + ws_tiles(heads, g) + (size_t)which * heads * g.g * lhk::TILE;
}

size_t attn_workspace_size(int heads, const Geo& g0) {
  const Geo g = attn_geo(g0);
  return ws_tiles(heads, g) + 2 * (size_t)heads * g.g * lhk::TILE;
}

// The lane-half kernel is the shipped K4; DA_K4_TK builds the transposed
// TMEM-fed kernel instead (A/B experiments, tools/probes/k4_variants.py)
bool attn_uses_tk() {
#ifdef DA_K4_TK
  return true;
#else
  return false;
#endif
}

bool tc_supported(const da_attn_args& a, const Geo& g) {
  if (a.d != 128 || a.dv != 128 || region_parts_shift(g) < 0) return false;
  if (!(a.scale > 0.0)) return false;  // the fixed softmax offset bounds scale * |q| |k| from above
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  if (!al16(a.q) || !al16(a.k) || !al16(a.v) || !al16(a.out)) return false;
  if (a.layout == DA_LAYOUT_ORIGINAL && a.shard_count > 1)
    for (int s = 0; s < a.shard_count; ++s)
      if (!al16(a.q_shards[s]) || !al16(a.k_shards[s]) || !al16(a.v_shards[s]) || !al16(a.out_shards[s])) return false;
  if (a.q_row_stride % 8 || a.k_row_stride % 8 || a.v_row_stride % 8) return false;
  if (a.q_head_stride % 8 || a.k_head_stride % 8 || a.v_head_stride % 8) return false;
  if (a.o_row_stride % 8 || a.o_head_stride % 8) return false;
  return (long long)a.heads * g.g < (1ll << 31);
}

cudaError_t launch_tc_attn(const da_attn_args& a, const Geo& gm, cudaStream_t st, const float* kpart, int kblk,
                           bool tiles_ready) {
  const Geo g = attn_geo(gm);  // gm: the mask's geometry; g: K4's (half-regions when split)
  lhk::Params p;
  p.split = region_parts_shift(gm) > 0 ? region_parts_shift(gm) : 0;
  p.trace = g_trace;
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
  p.per_head = make_fastdiv((uint32_t)g.g);
  p.sh = make_shards(a);
#ifndef LH_L2POL
#define LH_L2POL 6  // bit 0: K/V tiles evict_last, bit 1: Q rows evict_first, bit 2: output rows evict_first (6: DRAM reads 11.0 -> 9.9 GB per HV720 launch, K4 -0.6 %, profiles/r02/l2pol)
#endif
  p.pol_kv = (LH_L2POL & 1) ? L2_EVICT_LAST : L2_EVICT_NORMAL;
  p.pol_q = (LH_L2POL & 2) ? L2_EVICT_FIRST : L2_EVICT_NORMAL;
  p.pol_o = (LH_L2POL & 4) ? L2_EVICT_FIRST : L2_EVICT_NORMAL;
  char* ws = static_cast<char*>(a.workspace);
  p.fb_count = reinterpret_cast<int*>(ws);
  p.work = reinterpret_cast<int*>(ws + 4);
  p.fb_items = reinterpret_cast<int*>(ws + ws_items(a.heads));
  int4* meta = reinterpret_cast<int4*>(ws + ws_order(a.heads, g));
  cudaMemsetAsync(ws, 0, 2 * sizeof(int), st);  // fallback counter, item counter
  if (kpart != nullptr) {  // norms from the pooling pass
    p.kpart = kpart;
    p.kblk = kblk;
  } else {
    float* kp = reinterpret_cast<float*>(ws + ws_norms());
    const long long key_rows = a.layout == DA_LAYOUT_REORDERED ? g.n_pad : g.n_real;
    lhk::key_norm_kernel<<<dim3(lhk::KBLK, a.heads), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(a.k),
                                                                  a.k_head_stride, a.k_row_stride, key_rows, kp, p.sh);
    p.kpart = kp;
    p.kblk = lhk::KBLK;
  }
  cudaError_t e;
  {
    const size_t smem = sizeof(int) * ((size_t)gm.g + 1);
    if (smem <= 200 * 1024 && ensure_smem_optin((const void*)lhk::region_order_kernel, (int)smem) == cudaSuccess) {
      lhk::region_order_kernel<<<a.heads, 1024, smem, st>>>(a.row_ptr, gm.g, a.shared_mask ? 0 : 1, p.split, meta);
      p.meta = meta;
    } else {
      cudaGetLastError();
      p.meta = nullptr;  // natural region order
    }
  }
  if (!tiles_ready) {
    lhk::KvTileArgs ta;
    ta.x[0] = static_cast<const __nv_bfloat16*>(a.k);
    ta.x[1] = static_cast<const __nv_bfloat16*>(a.v);
    ta.hs[0] = a.k_head_stride; ta.hs[1] = a.v_head_stride;
    ta.rs[0] = a.k_row_stride; ta.rs[1] = a.v_row_stride;
    ta.out[0] = attn_tiles(a.workspace, a.heads, g, 0);
    ta.out[1] = attn_tiles(a.workspace, a.heads, g, 1);
    ta.layout = a.layout;
    ta.sh = p.sh;
    lhk::kv_tile_kernel<<<dim3(g.g, a.heads, 2), 256, 0, st>>>(ta, g, p.dec);
  }
  p.kt = attn_tiles(a.workspace, a.heads, g, 0);
  p.vt = attn_tiles(a.workspace, a.heads, g, 1);
  const int sms = device_sms();
  const long long items = (long long)a.heads * g.g;
  const int grid = (int)(items < sms ? items : sms);
#ifdef DA_K4_TK
  if (attn_uses_tk() && p.sh.n <= 1 && !p.split) {  // (the experiment addresses neither shards nor halves)
    if ((e = launch_tk_kernel(p, grid, st)) != cudaSuccess) return e;
  } else
#endif
  {
    if (p.sh.n > 1) {
      if ((e = ensure_smem_optin((const void*)lhk::sparse_attn_lh_kernel<true>, lhk::SMEM_ALLOC)) != cudaSuccess) return e;
      lhk::sparse_attn_lh_kernel<true><<<grid, lhk::THREADS, lhk::SMEM_ALLOC, st>>>(p);
    } else {
      if ((e = ensure_smem_optin((const void*)lhk::sparse_attn_lh_kernel<false>, lhk::SMEM_ALLOC)) != cudaSuccess) return e;
      lhk::sparse_attn_lh_kernel<false><<<grid, lhk::THREADS, lhk::SMEM_ALLOC, st>>>(p);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // rows whose fixed softmax offset underflowed: redo their regions exactly
  return launch_portable_list(a, gm, st, p.fb_items, p.fb_count, 2 * sms);
}

}  // namespace da
