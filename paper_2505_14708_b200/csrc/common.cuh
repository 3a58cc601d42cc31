// Shared device helpers for the sm_100a kernels: geometry, mbarriers, TMA,
// tcgen05 (UMMA descriptors, MMA issue, TMEM load/store).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/draftattn_b200.h"

#define DA_DEV __device__ __forceinline__

namespace da {

// ---------------------------------------------------------------------------
// Grid geometry (closed forms of layout.py:106-123 and padding.py:45-56).
// A reordered position pos = i*p + r sits in region i = (f*Ph + a)*Pw + b at
// in-patch offset r = u*pw + v, i.e. padded token (f, a*ph + u, b*pw + v).
// ---------------------------------------------------------------------------
struct Geo {
  int F, H, W, ph, pw;   // real extent and pool size
  int Ph, Pw;            // patches per column / row on the padded grid
  int p;                 // region size ph*pw
  int g;                 // regions F*Ph*Pw
  long long n_real, n_pad;
};

inline Geo make_geo(const da_grid& gr) {
  Geo g;
  g.F = gr.frames; g.H = gr.height; g.W = gr.width; g.ph = gr.patch_h; g.pw = gr.patch_w;
  g.Ph = (g.H + g.ph - 1) / g.ph;
  g.Pw = (g.W + g.pw - 1) / g.pw;
  g.p = g.ph * g.pw;
  g.g = g.F * g.Ph * g.Pw;
  g.n_real = (long long)g.F * g.H * g.W;
  g.n_pad = (long long)g.g * g.p;
  return g;
}

// 64-token regions run on the tcgen05 kernel as they are (0); 64 x 2^s-token
// regions whose pool width 2^s divides run as 2^s column parts of 64 tokens
// (s = 1..3: e.g. the paper's 8x16 pools as two 8x8 halves); -1: neither.
__host__ __device__ inline int region_parts_shift(const Geo& g) {
  for (int s = 0; s <= 3; ++s)
    if (g.p == (64 << s) && g.pw % (1 << s) == 0) return s;
  return -1;
}

// Division by a runtime constant with a precomputed multiplier
// (q = (umulhi(n, mul) + n) >> shift; exact for n < 2^31).
struct FastDiv {
  uint32_t d, mul, shift;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  f.shift = 0;
  while ((1ull << f.shift) < d) ++f.shift;
  f.mul = (uint32_t)(((1ull << 32) * ((1ull << f.shift) - d)) / d + 1);
  return f;
}
DA_DEV uint32_t fdiv(uint32_t n, const FastDiv& f) { return (__umulhi(n, f.mul) + n) >> f.shift; }

// Token rows split over shard buffers (da_attn_args' sequence shards, possibly
// peer GPUs' memory reached over NVLink): row r is local row r - s*rows of
// shard s = r / rows. Kernels holding one take it as a __grid_constant__
// parameter, so the table is indexed in the parameter bank (no local copy).
struct Shards {
  const char* base[4][DA_MAX_SHARDS];  // q, k, v, out
  int n;                               // shard count; <= 1: unsplit (tables unused)
  int rows;
  FastDiv div;
};
enum { SH_Q = 0, SH_K = 1, SH_V = 2, SH_O = 3 };

// Address of element (ho + row * rs) of tensor t: `plain` + that offset when
// unsplit, else the same offset from row's shard with its local row.
template <class T>
DA_DEV T* shard_addr(const Shards& s, int t, T* plain, long long ho, long long row, long long rs) {
  if (s.n <= 1) return plain + ho + row * rs;
  const int part = (int)fdiv((uint32_t)row, s.div);
  T* b = reinterpret_cast<T*>(const_cast<char*>(s.base[t][part]));
  return b + ho + (row - (long long)part * s.rows) * rs;
}

// shard_addr when SPLIT, else the plain address (kernels instantiated both ways
// keep the unsplit build's registers and code)
template <bool SPLIT, class T>
DA_DEV T* shard_at(const Shards& s, int t, T* plain, long long ho, long long row, long long rs) {
  if constexpr (SPLIT) return shard_addr(s, t, plain, ho, row, rs);
  else return plain + ho + row * rs;
}

inline Shards no_shards() {
  Shards s = {};
  s.n = 1;
  s.rows = 1;
  s.div = make_fastdiv(1);
  return s;
}

inline Shards make_shards(const da_attn_args& a) {
  Shards s;
  s.n = a.layout == DA_LAYOUT_ORIGINAL && a.shard_count > 1 ? a.shard_count : 1;
  s.rows = s.n > 1 ? (int)a.shard_rows : 1;
  s.div = make_fastdiv((uint32_t)s.rows);
  for (int i = 0; i < DA_MAX_SHARDS; ++i) {
    const bool on = s.n > 1 && i < s.n;
    s.base[SH_Q][i] = on ? static_cast<const char*>(a.q_shards[i]) : nullptr;
    s.base[SH_K][i] = on ? static_cast<const char*>(a.k_shards[i]) : nullptr;
    s.base[SH_V][i] = on ? static_cast<const char*>(a.v_shards[i]) : nullptr;
    s.base[SH_O][i] = on ? static_cast<const char*>(a.out_shards[i]) : nullptr;
  }
  return s;
}

// Region coordinates: frame, first padded row and column of region i.
struct RegionXY {
  int f, y0, x0;
};
struct RegionDecoder {
  FastDiv per_frame;  // Ph*Pw
  FastDiv per_row;    // Pw
  int ph, pw;
  DA_DEV RegionXY operator()(int i) const {
    int f = (int)fdiv((uint32_t)i, per_frame);
    int rest = i - f * (int)per_frame.d;
    int a = (int)fdiv((uint32_t)rest, per_row);
    int b = rest - a * (int)per_row.d;
    return {f, a * ph, b * pw};
  }
};
inline RegionDecoder make_decoder(const Geo& g) {
  RegionDecoder d;
  d.per_frame = make_fastdiv((uint32_t)(g.Ph * g.Pw));
  d.per_row = make_fastdiv((uint32_t)g.Pw);
  d.ph = g.ph;
  d.pw = g.pw;
  return d;
}

// Order-preserving 64-bit key of a float64 selection score: larger score <=>
// larger key; -0.0 folded onto +0.0 (they tie, as numpy compares them); NaN
// below everything (a stable descending argsort puts NaN last).
DA_DEV unsigned long long score_key(double s) {
  if (s != s) return 0ull;
  if (s == 0.0) s = 0.0;
  unsigned long long b = (unsigned long long)__double_as_longlong(s);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Real-token row of reordered position (region i, offset r), or -1 for padding.
DA_DEV long long real_row(const Geo& g, int i, int r) {
  int f = i / (g.Ph * g.Pw);
  int rest = i - f * g.Ph * g.Pw;
  int a = rest / g.Pw, b = rest - a * g.Pw;
  int u = r / g.pw, v = r - u * g.pw;
  int y = a * g.ph + u, x = b * g.pw + v;
  if (y >= g.H || x >= g.W) return -1;
  return ((long long)f * g.H + y) * g.W + x;
}

DA_DEV bool key_is_valid(const Geo& g, int i, int r) {
  int rest = i % (g.Ph * g.Pw);
  int a = rest / g.Pw, b = rest - a * g.Pw;
  int u = r / g.pw, v = r - u * g.pw;
  return (a * g.ph + u) < g.H && (b * g.pw + v) < g.W;
}

// ---------------------------------------------------------------------------
// mbarrier
// ---------------------------------------------------------------------------
DA_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

DA_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
DA_DEV void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
DA_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
DA_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
DA_DEV bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  // with a suspend-time hint the warp sleeps in hardware until the phase
  // completes (or the hint expires) instead of spinning on issue slots
#ifdef DA_MBAR_NOHINT
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, 1000000;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
#endif
  return ok != 0;
}
// Blocking wait with a watchdog: a pipeline bug traps (kernel error) after
// ~2^34 cycles (~9 s) instead of hanging the device.
DA_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(addr, parity)) {
    if (clock64() - t0 > (1ll << 34)) __trap();
  }
}

// Latency-critical wait: non-blocking test_wait in a tight loop (no suspend),
// for waits on the MMA <-> softmax critical path.
DA_DEV bool mbar_test_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
DA_DEV void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_test_wait(addr, parity)) return;
  const long long t0 = clock64();
  while (!mbar_test_wait(addr, parity)) {
    if (clock64() - t0 > (1ll << 34)) __trap();
  }
}

// Warp-wide wait: one lane polls the barrier, __syncwarp publishes the
// acquired state to the rest of the (converged) warp. 32 lanes polling the same
// mbarrier cost far more than one.
DA_DEV void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  if ((threadIdx.x & 31) == 0) mbar_wait_spin(bar, parity);
  __syncwarp();
}
// Same, but the polling lane sleeps in try_wait (suspend-time hint) instead of
// spinning: for waits off the critical path, so that waiting warps leave the
// issue slots to the warps that compute.
DA_DEV void mbar_wait_warp_sleep(uint64_t* bar, uint32_t parity) {
  if ((threadIdx.x & 31) == 0) mbar_wait(bar, parity);
  __syncwarp();
}

// ---------------------------------------------------------------------------
// TMA
// ---------------------------------------------------------------------------
DA_DEV void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// L2 cache-policy operands for .L2::cache_hint (same encodings CUTLASS uses).
constexpr uint64_t L2_EVICT_NORMAL = 0x1000000000000000ull;
constexpr uint64_t L2_EVICT_FIRST = 0x12F0000000000000ull;
constexpr uint64_t L2_EVICT_LAST = 0x14F0000000000000ull;

DA_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                        uint64_t policy = L2_EVICT_NORMAL) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
DA_DEV void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3, int c4,
                        uint64_t policy = L2_EVICT_NORMAL) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "l"(policy)
      : "memory");
}
// 16-byte global load / store with an L2 cache-policy operand (L1 bypassed on the load).
DA_DEV uint4 ldg128_hint(const void* p, uint64_t policy) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(policy));
  return v;
}
DA_DEV void stg128_hint(void* p, uint4 v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(policy)
               : "memory");
}
// 16-byte cp.async (L2 only); src_bytes = 0 zero-fills the destination.
DA_DEV void cp_async16(uint32_t saddr, const void* g, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes) : "memory");
}
DA_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// The mbarrier receives one arrival (counted in its init count) once every
// cp.async this thread issued before the call has landed in shared memory.
DA_DEV void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
template <int N>
DA_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// Contiguous global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0).
DA_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy = L2_EVICT_NORMAL) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
DA_DEV void sts128(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// ---------------------------------------------------------------------------
// tcgen05 / UMMA
// ---------------------------------------------------------------------------
// Byte offset of (row r, feature half h, 16-byte chunk c of the half) in a
// 64 x 128 bf16 key/value region tile in the GROUPED layout: [8-row group]
// [half][8 rows x 128 B] with the 128-byte swizzle. Group stride 2048 B, so
// two tiles 16 KB apart read as one 128-row MMA operand (N = 128 GEMM1 of
// the lane-half kernel); the halves sit 1 KB apart.
DA_DEV uint32_t kv_tile_offset_grouped(int r, int h, int c) {
  return (uint32_t)((((r >> 3) * 2 + h) << 10) + ((r & 7) << 7) + (((c ^ r) & 7) << 4));
}
// Shared-memory matrix descriptor (SM100 "version 1"), SWIZZLE_128B.
//   start address >> 4 in [0,14), LBO >> 4 in [16,30), SBO >> 4 in [32,46),
//   version 1 at bit 46, layout type SWIZZLE_128B (2) in [61,64).
DA_DEV uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor for kind::f16 with BF16 inputs and F32 accumulate.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                       // c_format = F32
         | (1u << 7)                     // a_format = BF16
         | (1u << 10)                    // b_format = BF16
         | ((uint32_t)a_mn_major << 15)  // a major
         | ((uint32_t)b_mn_major << 16)  // b major
         | ((uint32_t)(N >> 3) << 17)    // n_dim
         | ((uint32_t)(M >> 4) << 24);   // m_dim
}

DA_DEV void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// A operand from TMEM (K-major, packed bf16x2 per 32-bit column), B from shared memory.
DA_DEV void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(0u));
}

// One lane of a converged warp (elect.sync): lets a whole warp run the MMA
// issue loop (descriptors stay warp-uniform, in uniform registers) while one
// lane issues.
DA_DEV bool elect_one_sync() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "elect.sync _|P1, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}

DA_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

DA_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DA_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
DA_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int NCOLS>
DA_DEV void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
DA_DEV void tmem_free(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns per warp: thread gets 32 registers.
DA_DEV void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
DA_DEV void tmem_st16u(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
DA_DEV void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// Same load into v[OFF .. OFF+31] of a larger register array.
template <int OFF, int N>
DA_DEV void tmem_ld32_at(uint32_t taddr, float (&v)[N]) {
  static_assert(OFF + 32 <= N, "range");
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[OFF + i] = __uint_as_float(r[i]);
}
// 16x32bx2 shapes (tools/probes/tmem16x2.cu): threads 0-15 access TMEM lanes
// base + t at columns [c, c + N), threads 16-31 lanes base + t - 16 at columns
// [c + split, c + split + N). Used on M = 64 tiles, whose 64 rows occupy 16
// lanes of each warp's 32-lane slice.
DA_DEV void tmem_ld16x2_32(uint32_t taddr, float (&v)[64]) {  // split 64: 32 columns -> v[0..31]
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], 64;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
DA_DEV void tmem_ld16x2_32hi(uint32_t taddr, float (&v)[64]) {  // split 64: 32 columns -> v[32..63]
  uint32_t* r = reinterpret_cast<uint32_t*>(v) + 32;
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], 64;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
DA_DEV void tmem_st16x2_16(uint32_t taddr, const uint32_t (&r)[16]) {  // split 32: 16 columns
  asm volatile(
      "tcgen05.st.sync.aligned.16x32bx2.x16.b32 [%0], 32, "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
DA_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
DA_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Named barrier with an OR-vote over the participating threads.
DA_DEV bool bar_red_or(int id, int nthreads, bool pred) {
  uint32_t out;
  asm volatile(
      "{\n"
      ".reg .pred pi, po;\n"
      "setp.ne.u32 pi, %1, 0;\n"
      "barrier.red.or.pred po, %2, %3, pi;\n"
      "selp.u32 %0, 1, 0, po;\n"
      "}\n"
      : "=r"(out)
      : "r"((uint32_t)pred), "r"(id), "r"(nthreads)
      : "memory");
  return out != 0;
}
DA_DEV void bar_arrive(int id, int nthreads) {
  asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
DA_DEV void bar_sync(int id, int nthreads) { asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }

DA_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

DA_DEV float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32x2 FMA (Blackwell FFMA2): d = a * b + c, lane-wise.
DA_DEV float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}

// Packed fp32x2 add (Blackwell FADD2).
DA_DEV float2 fadd2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}

// 2^x for a pair, on the FMA pipe (no MUFU): round-to-nearest split
// x = j + f (|f| <= 1/2) by the 1.5 * 2^23 trick, degree-3 near-minimax
// polynomial for 2^f (relative error < 7.5e-5, far below the bf16 rounding of
// P), exponent add. Inputs are clamped at -125 (2^-125 for -inf scores:
// below every kept term by > 60 binades, so it only perturbs sums at ~1e-19).
DA_DEV float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 t = fadd2(x, make_float2(12582912.f, 12582912.f));
  const float2 j = fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = fadd2(x, make_float2(-j.x, -j.y));
  float2 p = ffma2(f, make_float2(0.05517167f, 0.05517167f), make_float2(0.24261115f, 0.24261115f));
  p = ffma2(p, f, make_float2(0.69326097f, 0.69326097f));
  p = ffma2(p, f, make_float2(0.99992806f, 0.99992806f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

}  // namespace da
