// K3b: global top-m selection per head (masking.py:59-91), force-row-keep
// (masking.py:84-88), dead key-region drop (masking.py:94-105), packed bitmap
// (masking.py:168-170) and per-row ascending column lists for K4.
//
// Ranking key: descending score, ties to the smaller flat index i*g + j. Scores
// map to order-preserving 64-bit keys (-0.0 folded onto +0.0 so they tie, NaN
// below everything, as in a stable descending argsort). The m-th key T is found
// by a most-significant-digit radix select with 11-bit digits:
//   digit 0 (bits 53..63) and digit 1 (bits 42..52): histograms over all g*g
//     scores of the head (digit 0 can be fused into the draft GEMM epilogue);
//   then the entries sharing the resolved 22-bit prefix (typically a few
//     thousand) are compacted and one CTA per head resolves the remaining 42
//     bits in shared memory. If that bucket is too large (massive ties) the
//     remaining digits run as full passes instead.
// One pass per row then marks  key > T,  or key == T among the first `need`
// equal keys in flat order,  or the row's first argmax (force_row_keep),  minus
// dead columns, into a word-aligned bitmap; a scan of the row counts places
// each row's columns.
#include "common.cuh"
#include "kernels.h"

namespace da {

constexpr int RB = 11;           // radix digit bits
constexpr int NB = 1 << RB;      // bins
constexpr int NPASS = 6;         // 5 * 11 + 9 = 64 bits
constexpr int CAND_CAP = 1 << 16;

struct SelState {
  unsigned long long prefix;     // resolved high bits of T
  long long remaining;           // entries still to take from the current bucket
  long long gt;                  // entries above the current bucket (kept)
  long long eq_total;            // entries with key == T (after the last digit)
  long long bucket;              // size of the current bucket
  unsigned long long T;
  int compact;                   // candidates compacted after digit 1
  unsigned int cand_count;
};

// Launch gate: with `gate` set, a kernel runs only when (*gate != 0) == want
// (the fp32 selection runs when its fallback flag is clear, the fp64 one when set).
DA_DEV bool gated_off(const int* gate, int want) { return gate != nullptr && ((*gate != 0) != (want != 0)); }

DA_DEV double key_score(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

DA_DEV int pass_hi(int pass) { return 64 - RB * pass; }
DA_DEV int pass_lo(int pass) { int lo = 64 - RB * (pass + 1); return lo < 0 ? 0 : lo; }

__global__ void sel_init_kernel(SelState* st, unsigned int* hist, long long m, const int* __restrict__ gate = nullptr, int want = 1) {
  if (gated_off(gate, want)) return;
  const int h = blockIdx.x;
  if (threadIdx.x == 0) {
    SelState s;
    s.prefix = 0; s.remaining = m; s.gt = 0; s.eq_total = 0; s.bucket = 0; s.T = 0;
    s.compact = 0; s.cand_count = 0;
    st[h] = s;
  }
  for (int b = threadIdx.x; b < NB; b += blockDim.x) hist[(long long)h * NB + b] = 0;
}

// Histogram of digit `pass` over the full score array of each head (keys that
// still match the resolved prefix). grid: (chunks, heads).
__global__ void __launch_bounds__(256) sel_hist_kernel(const double* __restrict__ scores, long long n,
                                                       const SelState* __restrict__ st, unsigned int* hist,
                                                       int pass, const int* __restrict__ gate = nullptr, int want = 1) {
  if (gated_off(gate, want)) return;
  const int h = blockIdx.y;
  if (pass >= 2 && st[h].compact) return;
  __shared__ unsigned int sh[NB];
  for (int b = threadIdx.x; b < NB; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const int hi = pass_hi(pass), lo = pass_lo(pass);
  const unsigned long long prefix = st[h].prefix;
  const unsigned long long dmask = (1ull << (hi - lo)) - 1;
  const double* s = scores + (long long)h * n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
    const unsigned long long k = score_key(__ldg(s + e));
    if (hi == 64 || (k >> hi) == prefix) atomicAdd(&sh[(unsigned)((k >> lo) & dmask)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < NB; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[(long long)h * NB + b], sh[b]);
}

// Warp-level walk over a histogram from the top bucket: find the bucket
// holding the rem-th entry. Returns (bucket, count above it, bucket size).
DA_DEV void pick_bucket(const unsigned int* H, int nb, long long rem, int lane, int& chosen, long long& above_out,
                        long long& cnt_out) {
  long long above = 0;
  chosen = -1;
  above_out = 0;
  cnt_out = 0;
  for (int top = nb - 1; top >= 0 && chosen < 0; top -= 32) {
    const int b = top - lane;
    const long long c = (b >= 0) ? (long long)H[b] : 0;
    long long incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const long long excl = incl - c;
    const bool hit = b >= 0 && (above + excl < rem) && (above + incl >= rem);
    const unsigned mask = __ballot_sync(0xffffffffu, hit);
    if (mask) {
      const int src = __ffs(mask) - 1;
      chosen = __shfl_sync(0xffffffffu, b, src);
      above_out = above + __shfl_sync(0xffffffffu, excl, src);
      cnt_out = __shfl_sync(0xffffffffu, c, src);
    }
    above += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// One warp per head: resolve digit `pass` from the global histogram.
__global__ void sel_scan_kernel(SelState* st, unsigned int* hist, int pass, const int* __restrict__ gate = nullptr, int want = 1) {
  if (gated_off(gate, want)) return;
  const int h = blockIdx.x;
  const int lane = threadIdx.x;
  if (pass >= 2 && st[h].compact) return;
  const int hi = pass_hi(pass), lo = pass_lo(pass);
  unsigned int* H = hist + (long long)h * NB;
  const long long rem = st[h].remaining;
  int chosen;
  long long above, cnt;
  pick_bucket(H, 1 << (hi - lo), rem, lane, chosen, above, cnt);
  __syncwarp();
  for (int b = lane; b < NB; b += 32) H[b] = 0;
  if (lane == 0) {
    SelState s = st[h];
    s.gt += above;
    s.remaining = rem - above;
    s.prefix = (s.prefix << (hi - lo)) | (unsigned long long)chosen;
    s.bucket = cnt;
    if (lo == 0) {
      s.T = s.prefix;
      s.eq_total = cnt;
    }
    if (pass == 1) s.compact = cnt <= CAND_CAP;
    st[h] = s;
  }
}

// Gather the entries of the 22-bit bucket (key, flat index) when it is small.
__global__ void __launch_bounds__(256) sel_compact_kernel(const double* __restrict__ scores, long long n,
                                                          SelState* st, unsigned long long* cand_key,
                                                          unsigned int* cand_idx, const int* __restrict__ gate = nullptr, int want = 1) {
  if (gated_off(gate, want)) return;
  const int h = blockIdx.y;
  if (!st[h].compact) return;
  const unsigned long long prefix = st[h].prefix;
  const int hi = pass_lo(1);
  const double* s = scores + (long long)h * n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += stride) {
    const long long e = base + threadIdx.x;
    unsigned long long k = 0;
    bool hit = false;
    if (e < n) {
      k = score_key(__ldg(s + e));
      hit = (k >> hi) == prefix;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, hit);
    if (mask) {
      unsigned slot0 = 0;
      if (lane == 0) slot0 = atomicAdd(&st[h].cand_count, (unsigned)__popc(mask));
      slot0 = __shfl_sync(0xffffffffu, slot0, 0);
      if (hit) {
        const unsigned slot = slot0 + __popc(mask & ((1u << lane) - 1));
        cand_key[(long long)h * CAND_CAP + slot] = k;
        cand_idx[(long long)h * CAND_CAP + slot] = (unsigned)e;
      }
    }
  }
}

// One CTA per head: digits 2..5 over the compacted candidates, in shared memory.
__global__ void __launch_bounds__(1024) sel_cand_finish_kernel(SelState* st, const unsigned long long* cand_key, const int* __restrict__ gate = nullptr, int want = 1) {
  if (gated_off(gate, want)) return;
  const int h = blockIdx.x;
  if (!st[h].compact) return;
  __shared__ unsigned int sh[NB];
  __shared__ unsigned long long s_prefix;
  __shared__ long long s_rem;
  const unsigned n = st[h].cand_count;
  const unsigned long long* K = cand_key + (long long)h * CAND_CAP;
  if (threadIdx.x == 0) {
    s_prefix = st[h].prefix;
    s_rem = st[h].remaining;
  }
  long long gt_add = 0, last_cnt = 0;
  for (int pass = 2; pass < NPASS; ++pass) {
    for (int b = threadIdx.x; b < NB; b += blockDim.x) sh[b] = 0;
    __syncthreads();
    const int hi = pass_hi(pass), lo = pass_lo(pass);
    const unsigned long long prefix = s_prefix;
    const unsigned long long dmask = (1ull << (hi - lo)) - 1;
    for (unsigned e = threadIdx.x; e < n; e += blockDim.x) {
      const unsigned long long k = K[e];
      if ((k >> hi) == prefix) atomicAdd(&sh[(unsigned)((k >> lo) & dmask)], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      int chosen;
      long long above, cnt;
      pick_bucket(sh, 1 << (hi - lo), s_rem, threadIdx.x, chosen, above, cnt);
      if (threadIdx.x == 0) {
        s_prefix = (prefix << (hi - lo)) | (unsigned long long)chosen;
        s_rem -= above;
        gt_add += above;
        last_cnt = cnt;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    SelState s = st[h];
    s.gt += gt_add;
    s.remaining = s_rem;
    s.prefix = s_prefix;
    s.T = s_prefix;
    s.eq_total = last_cnt;
    st[h] = s;
  }
}

// Per-row equal-key counts (only needed when ties at T straddle the cut).
__global__ void __launch_bounds__(256) sel_rowcount_eq_kernel(const double* __restrict__ scores, int g,
                                                              const SelState* __restrict__ st, int* eq_rows, const int* __restrict__ gate = nullptr, int want = 1) {
  if (gated_off(gate, want)) return;
  const int h = blockIdx.y;
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= g) return;
  const SelState s = st[h];
  if (s.eq_total == s.remaining) return;  // every tied entry is kept: no ranks needed
  const double* S = scores + ((long long)h * g + row) * g;
  int cnt = 0;
  for (int j = lane; j < g; j += 32) cnt += score_key(__ldg(S + j)) == s.T;
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) eq_rows[(long long)h * g + row] = cnt;
}

// Exclusive scan of int rows per head (one CTA per head); out[g] = total.
// If `extra` is given, its per-row values are summed into extra_total[h].
__global__ void __launch_bounds__(1024) scan_rows_kernel(const int* __restrict__ in, int* __restrict__ out, int g,
                                                         int out_stride, const SelState* st, int only_if_ties,
                                                         const int* __restrict__ extra, long long* extra_total,
                                                         const int* __restrict__ gate = nullptr, int want = 1) {
  if (gated_off(gate, want)) return;
  const int h = blockIdx.x;
  if (only_if_ties && st[h].eq_total == st[h].remaining) return;
  __shared__ int warp_tot[32];
  __shared__ int carry;
  __shared__ long long ex_sum;
  const int* I = in + (long long)h * g;
  int* O = out + (long long)h * out_stride;
  if (threadIdx.x == 0) { carry = 0; ex_sum = 0; }
  __syncthreads();
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  long long ex_local = 0;
  for (int base = 0; base < g; base += blockDim.x) {
    const int idx = base + threadIdx.x;
    const int v = idx < g ? I[idx] : 0;
    if (extra && idx < g) ex_local += extra[(long long)h * g + idx];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
      const int nw = blockDim.x / 32;
      const int t = lane < nw ? warp_tot[lane] : 0;
      int ti = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, ti, o);
        if (lane >= o) ti += u;
      }
      if (lane < nw) warp_tot[lane] = ti - t;
    }
    __syncthreads();
    const int excl = carry + warp_tot[w] + incl - v;
    if (idx < g) O[idx] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (extra) {
    ex_local += __shfl_xor_sync(0xffffffffu, ex_local, 16);
    ex_local += __shfl_xor_sync(0xffffffffu, ex_local, 8);
    ex_local += __shfl_xor_sync(0xffffffffu, ex_local, 4);
    ex_local += __shfl_xor_sync(0xffffffffu, ex_local, 2);
    ex_local += __shfl_xor_sync(0xffffffffu, ex_local, 1);
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&ex_sum), (unsigned long long)ex_local);
    __syncthreads();
    if (threadIdx.x == 0) extra_total[h] = ex_sum;
  }
  if (threadIdx.x == 0) O[g] = carry;
}

// Mark one row per warp into the word-aligned bitmap (bit j%32 of word j/32),
// with the first argmax forced in (force_row_keep) and dead columns dropped.
__global__ void __launch_bounds__(256) sel_mark_kernel(const double* __restrict__ scores, int g, const SelState* st,
                                                       const int* __restrict__ eq_prefix, int force_row_keep,
                                                       const uint8_t* __restrict__ dead, unsigned int* bm, int w32,
                                                       int* row_counts, int* row_forced, const int* __restrict__ gate = nullptr, int want = 1) {
  if (gated_off(gate, want)) return;
  const int h = blockIdx.y;
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= g) return;
  const SelState s = st[h];
  const bool all_eq = s.eq_total == s.remaining;
  const double* S = scores + ((long long)h * g + row) * g;
  unsigned int* B = bm + ((long long)h * g + row) * w32;
  const int eq0 = all_eq ? 0 : eq_prefix[(long long)h * (g + 1) + row];
  int eq_run = eq0;
  int cnt = 0;
  int best = -1;
  double bv = 0.0;
  bool bnan = false;
  for (int j0 = 0; j0 < g; j0 += 32) {
    const int j = j0 + lane;
    bool kept = false, eq = false;
    if (j < g) {
      const double v = __ldg(S + j);
      const unsigned long long k = score_key(v);
      kept = k > s.T;
      eq = k == s.T;
      const bool vnan = v != v;
      if (best < 0 || (!bnan && (vnan || v > bv))) { best = j; bv = v; bnan = vnan; }
    }
    const unsigned eqb = __ballot_sync(0xffffffffu, eq);
    if (eq) kept = all_eq || (eq_run + __popc(eqb & ((1u << lane) - 1))) < s.remaining;
    eq_run += __popc(eqb);
    if (kept && dead != nullptr && dead[j]) kept = false;
    const unsigned word = __ballot_sync(0xffffffffu, kept);
    if (lane == 0) B[j0 >> 5] = word;
    cnt += __popc(word);
  }
  int forced = 0;
  if (force_row_keep) {
    // first argmax across lanes (np.argmax: first max; first NaN wins)
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int ob = __shfl_xor_sync(0xffffffffu, best, o);
      const bool onan = __shfl_xor_sync(0xffffffffu, (int)bnan, o) != 0;
      bool take;
      if (ob < 0) take = false;
      else if (best < 0) take = true;
      else if (bnan != onan) take = onan;
      else if (!bnan && ov != bv) take = ov > bv;
      else take = ob < best;
      if (take) { bv = ov; best = ob; bnan = onan; }
    }
    __syncwarp();
    if (lane == 0 && best >= 0) {
      // was it kept by the global rule (before the dead-column drop)?
      const unsigned long long kb = score_key(bv);
      bool global_kept = kb > s.T;
      if (kb == s.T) {
        if (all_eq) {
          global_kept = true;
        } else {
          int before = 0;  // equal keys of this row left of `best`
          for (int j = 0; j < best; ++j) before += score_key(__ldg(S + j)) == s.T;
          global_kept = eq0 + before < s.remaining;
        }
      }
      if (!global_kept) {
        forced = 1;
        if (!(dead != nullptr && dead[best])) {
          B[best >> 5] |= 1u << (best & 31);
          ++cnt;
        }
      }
    }
  }
  if (lane == 0) {
    row_counts[(long long)h * g + row] = cnt;
    row_forced[(long long)h * g + row] = forced;
  }
}

// Expand bitmap rows into ascending column lists at row_ptr offsets.
__global__ void __launch_bounds__(256) sel_collect_kernel(const unsigned int* __restrict__ bm, int g, int w32,
                                                          const int* __restrict__ row_ptr, int* col_idx,
                                                          long long cap, const int* __restrict__ gate = nullptr, int want = 1) {
  if (gated_off(gate, want)) return;
  const int h = blockIdx.y;
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= g) return;
  const unsigned int* B = bm + ((long long)h * g + row) * w32;
  int out = row_ptr[(long long)h * (g + 1) + row];
  int* C = col_idx + (long long)h * cap;
  // 32 words per round, one per lane (independent loads), warp prefix sum of
  // their popcounts, then each lane expands its own word: ascending columns
  for (int c0 = 0; c0 < w32; c0 += 32) {
    const int c = c0 + lane;
    const unsigned word = c < w32 ? __ldg(B + c) : 0u;
    const int cnt = __popc(word);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int pos = out + incl - cnt;
    for (unsigned wv = word; wv; wv &= wv - 1) C[pos++] = c * 32 + __ffs(wv) - 1;
    out += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// np.packbits(kept) (masking.py:168-170): one output byte per thread.
__global__ void __launch_bounds__(256) sel_packbits_kernel(const unsigned int* __restrict__ bm, int g, int w32,
                                                           FastDiv gdiv, long long bytes_per_head, uint8_t* out,
                                                           const int* __restrict__ gate = nullptr, int want = 1) {
  if (gated_off(gate, want)) return;
  const int h = blockIdx.y;
  const long long byte = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (byte >= bytes_per_head) return;
  const long long n = (long long)g * g;
  const unsigned int* B = bm + (long long)h * g * w32;
  unsigned v = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const long long b = byte * 8 + t;
    unsigned bit = 0;
    if (b < n) {
      const int i = (int)fdiv((uint32_t)b, gdiv);
      const int j = (int)(b - (long long)i * g);
      bit = (__ldg(B + (long long)i * w32 + (j >> 5)) >> (j & 31)) & 1u;
    }
    v |= bit << (7 - t);
  }
  out[(long long)h * bytes_per_head + byte] = (uint8_t)v;
}

__global__ void sel_finish_kernel(const SelState* st, int heads, double* threshold, const int* __restrict__ gate = nullptr, int want = 1) {
  if (gated_off(gate, want)) return;
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h < heads) threshold[h] = key_score(st[h].T);
}

__global__ void copy_total_kernel(const int* row_ptr, int g, int heads, int64_t* kept, const int* __restrict__ gate = nullptr, int want = 1) {
  if (gated_off(gate, want)) return;
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h < heads) kept[h] = row_ptr[(long long)h * (g + 1) + g];
}

// ---------------------------------------------------------------------------
struct SelWs {
  SelState* state;
  unsigned int* hist;
  unsigned long long* cand_key;
  unsigned int* cand_idx;
  int* eq_rows;
  int* eq_prefix;
  int* row_counts;
  int* row_forced;
  unsigned int* bm;
  size_t total;
};

static SelWs carve_sel(void* base, int heads, int g) {
  SelWs w;
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) { char* r = p ? p + off : nullptr; off += (bytes + 255) & ~size_t(255); return r; };
  const int w32 = (g + 31) / 32;
  w.state = reinterpret_cast<SelState*>(take(sizeof(SelState) * heads));
  w.hist = reinterpret_cast<unsigned int*>(take(sizeof(unsigned int) * NB * heads));
  w.cand_key = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * CAND_CAP * heads));
  w.cand_idx = reinterpret_cast<unsigned int*>(take(sizeof(unsigned int) * CAND_CAP * heads));
  w.eq_rows = reinterpret_cast<int*>(take(sizeof(int) * (size_t)heads * g));
  w.eq_prefix = reinterpret_cast<int*>(take(sizeof(int) * (size_t)heads * (g + 1)));
  w.row_counts = reinterpret_cast<int*>(take(sizeof(int) * (size_t)heads * g));
  w.row_forced = reinterpret_cast<int*>(take(sizeof(int) * (size_t)heads * g));
  w.bm = reinterpret_cast<unsigned int*>(take(sizeof(unsigned int) * (size_t)heads * g * w32));
  w.total = off;
  return w;
}

size_t select_workspace_size(int heads, int g) { return carve_sel(nullptr, heads, g).total; }

long long bitmap_bytes_per_head(int g) { return ((long long)g * g + 7) / 8; }

unsigned int* select_hist_buffer(void* ws, int heads, int g) { return carve_sel(ws, heads, g).hist; }

cudaError_t launch_select(const double* scores, int heads, int g, long long m, int force, const uint8_t* dead,
                          void* ws, int* row_ptr, int* col_idx, uint8_t* bitmap, double* threshold,
                          int64_t* forced, int64_t* kept, long long cap, cudaStream_t st, bool digit0_done,
                          const int* gate) {
  SelWs w = carve_sel(ws, heads, g);
  const long long n = (long long)g * g;
  const int w32 = (g + 31) / 32;
  if (!digit0_done) sel_init_kernel<<<heads, 256, 0, st>>>(w.state, w.hist, m, gate);
  int chunks = (int)((n + 256 * 16 - 1) / (256 * 16));
  if (chunks > 256) chunks = 256;
  if (chunks < 1) chunks = 1;
  for (int pass = 0; pass < NPASS; ++pass) {
    if (!(pass == 0 && digit0_done))
      sel_hist_kernel<<<dim3(chunks, heads), 256, 0, st>>>(scores, n, w.state, w.hist, pass, gate);
    sel_scan_kernel<<<heads, 32, 0, st>>>(w.state, w.hist, pass, gate);
    if (pass == 1) {
      sel_compact_kernel<<<dim3(chunks, heads), 256, 0, st>>>(scores, n, w.state, w.cand_key, w.cand_idx, gate);
      sel_cand_finish_kernel<<<heads, 1024, 0, st>>>(w.state, w.cand_key, gate);
    }
  }
  dim3 rows_grid((g + 7) / 8, heads);
  sel_rowcount_eq_kernel<<<rows_grid, 256, 0, st>>>(scores, g, w.state, w.eq_rows, gate);
  scan_rows_kernel<<<heads, 1024, 0, st>>>(w.eq_rows, w.eq_prefix, g, g + 1, w.state, 1, nullptr, nullptr, gate);
  sel_mark_kernel<<<rows_grid, 256, 0, st>>>(scores, g, w.state, w.eq_prefix, force, dead, w.bm, w32, w.row_counts,
                                             w.row_forced, gate);
  scan_rows_kernel<<<heads, 1024, 0, st>>>(w.row_counts, row_ptr, g, g + 1, w.state, 0, w.row_forced,
                                           reinterpret_cast<long long*>(forced), gate);
  sel_collect_kernel<<<rows_grid, 256, 0, st>>>(w.bm, g, w32, row_ptr, col_idx, cap, gate);
  sel_finish_kernel<<<(heads + 127) / 128, 128, 0, st>>>(w.state, heads, threshold, gate);
  copy_total_kernel<<<(heads + 127) / 128, 128, 0, st>>>(row_ptr, g, heads, kept, gate);
  if (bitmap != nullptr) {
    const long long bph = bitmap_bytes_per_head(g);
    sel_packbits_kernel<<<dim3((unsigned)((bph + 255) / 256), heads), 256, 0, st>>>(w.bm, g, w32, make_fastdiv(g),
                                                                                     bph, bitmap, gate);
  }
  return cudaGetLastError();
}

// Fused digit-0 histogram support for the draft GEMM epilogue.
void select_init(void* ws, int heads, int g, long long m, cudaStream_t st, const int* gate) {
  SelWs w = carve_sel(ws, heads, g);
  sel_init_kernel<<<heads, 256, 0, st>>>(w.state, w.hist, m, gate);
}


// ===========================================================================
// fp32 draft scores with an exact fp64 guard band (the pipeline's default).
//
// The ranking must equal the reference's float64 argsort. Scores are computed
// in fp32 (FFMA GEMM, 4x the fp64 rate), and every fp32 score is within
// eps = (d + 8) 2^-24 max|q~| max|k~| |scale| of the fp64 score (Cauchy-Schwarz
// over the fp32 input rounding, FMA accumulation and the scale multiply). With
// T32 the m-th largest fp32 score, the m-th largest fp64 score t lies in
// [T32 - eps, T32 + eps], so
//   s32 > T32 + 2 eps   -> kept (s64 > t),
//   s32 < T32 - 2 eps   -> dropped (s64 < t),
// and only the band in between (a few hundred entries per head for real data)
// is rescored in fp64 and ranked exactly (descending score, ties to the smaller
// flat index). The row argmax (force_row_keep) is resolved the same way among
// the entries within 2 eps of the row's fp32 maximum. Non-finite inputs or a
// band larger than S32_CAP set a flag, and the fp64 GEMM + radix selection
// then run for the call (their launches are no-ops otherwise).
// ===========================================================================
constexpr int S32_CAP = 8192;    // band candidates per head resolved in one CTA

struct Sel32State {
  unsigned int prefix;           // resolved high bits of T32's key
  int pad0;                      // explicit padding: the state is copied whole (initcheck-clean)
  long long remaining;           // entries still to take from the current bucket
  unsigned long long nq2, nk2;   // largest pooled row norms^2 (double bits; non-negative so uint order)
  double eps;
  long long count_hi;            // sure-kept entries
  int cand_count;
  int pad1;
};

DA_DEV unsigned int key32(float s) {
  if (s != s) return 0u;
  if (s == 0.f) s = 0.f;
  const unsigned int b = __float_as_uint(s);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
DA_DEV float key32_score(unsigned int k) {
  const unsigned int b = (k >> 31) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(b);
}

// fp64 dot product of two feature rows in the fp64 GEMM's order
// (draft_gemm_kernel, prep.cu: one sequential FMA chain over the features,
// starting from 0.0), by ONE thread: band rescoring and the argmax rescoring
// therefore rank exactly as the fp64 fallback path does. Callers give each
// lane its own candidate so a warp runs 32 chains at once.
DA_DEV double dot64_seq(const double* __restrict__ q, const double* __restrict__ k, int d) {
  double acc = 0.0;
  int c = 0;
  if (((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k)) & 15) == 0) {
    // 16 features per batch: all 16 loads in flight, then the FMAs in order
    for (; c + 16 <= d; c += 16) {
      double2 qa[8], ka[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        qa[u] = __ldg(reinterpret_cast<const double2*>(q + c) + u);
        ka[u] = __ldg(reinterpret_cast<const double2*>(k + c) + u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc = fma(qa[u].x, ka[u].x, acc);
        acc = fma(qa[u].y, ka[u].y, acc);
      }
    }
  }
  for (; c + 4 <= d; c += 4) {
    const double q0 = __ldg(q + c), q1 = __ldg(q + c + 1), q2 = __ldg(q + c + 2), q3 = __ldg(q + c + 3);
    const double k0 = __ldg(k + c), k1 = __ldg(k + c + 1), k2 = __ldg(k + c + 2), k3 = __ldg(k + c + 3);
    acc = fma(q0, k0, acc);
    acc = fma(q1, k1, acc);
    acc = fma(q2, k2, acc);
    acc = fma(q3, k3, acc);
  }
  for (; c < d; ++c) acc = fma(__ldg(q + c), __ldg(k + c), acc);
  return acc;
}

__global__ void s32_init_kernel(Sel32State* st, unsigned int* hist, unsigned int* rowmax, int g, long long m,
                                int* fallback, const unsigned long long* __restrict__ pnorm) {
  const int h = blockIdx.x;
  if (threadIdx.x == 0) {
    Sel32State s;
    s.prefix = 0; s.pad0 = 0; s.remaining = m; s.eps = 0.0; s.count_hi = 0; s.cand_count = 0; s.pad1 = 0;
    s.nq2 = pnorm ? pnorm[2 * h] : 0;  // norms from the pooling pass, else s32_norm_kernel
    s.nk2 = pnorm ? pnorm[2 * h + 1] : 0;
    st[h] = s;
    if (h == 0) *fallback = 0;
  }
  for (int b = threadIdx.x; b < NB; b += blockDim.x) hist[(long long)h * NB + b] = 0;
  for (int i = threadIdx.x; i < g; i += blockDim.x) rowmax[(long long)h * g + i] = 0u;
}

// Largest pooled row norms per head (fp64), for eps; grid (heads, EPSB).
constexpr int EPSB = 16;
__global__ void __launch_bounds__(256) s32_norm_kernel(const double* __restrict__ qp, const double* __restrict__ kp,
                                                       int g, int d, Sel32State* st) {
  const int h = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int t = 0; t < 2; ++t) {
    const double* X = (t ? kp : qp) + (long long)h * g * d;
    double mx = 0.0;
    for (int i = blockIdx.y * 8 + w; i < g; i += 8 * EPSB) {
      double s2 = 0.0;
      for (int c = lane; c < d; c += 32) { const double v = __ldg(X + (long long)i * d + c); s2 = fma(v, v, s2); }
#pragma unroll
      for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      mx = (s2 != s2) ? s2 : fmax(mx, s2);  // keep NaN visible
    }
    if (lane == 0) {
      const unsigned long long bits = (unsigned long long)__double_as_longlong(mx);
      atomicMax(t ? &st[h].nk2 : &st[h].nq2, bits);  // NaN / inf bits sort above every finite value
    }
  }
}

DA_DEV void s32_set_eps(Sel32State& s, int d, double scale, int* fallback) {
  const double a = __longlong_as_double((long long)s.nq2), b = __longlong_as_double((long long)s.nk2);
  const double e = (double)(d + 8) * 0x1p-24 * sqrt(a) * sqrt(b) * fabs(scale) * 1.0625 + 1e-300;
  s.eps = e;
  if (!(a <= 1e300) || !(b <= 1e300) || !(e <= 1e30)) atomicOr(fallback, 1);
}

// fp32 draft scores: 128 x 128 tiles, 8 x 8 outputs per thread; epilogue keeps
// the digit-0 histogram of the 32-bit keys and each row's largest key.
// Operands come pre-packed by s32_pack_kernel: fp32, transposed and zero
// padded, [heads][dp][gp] (dp = d rounded up to DK32, gp = g rounded up to
// DT32), so each k-chunk is DK32 contiguous 512-byte rows per operand, moved
// by cp.async through a G32_STAGES-deep ring with no bounds checks.
constexpr int DT32 = 128, DK32 = 16, G32_TS = DT32 + 4, G32_STAGES = 3;
constexpr int G32_STAGE_FLOATS = 2 * DK32 * DT32;
constexpr int G32_SMEM = (DT32 * G32_TS > G32_STAGES * G32_STAGE_FLOATS ? DT32 * G32_TS : G32_STAGES * G32_STAGE_FLOATS) * 4;
__host__ __device__ inline long long g32_pad(long long x, int to) { return (x + to - 1) / to * to; }
// per-head stride of the fp32 score planes: g * g rounded up to 4 floats, so
// every plane starts 16-byte aligned (odd g)
__host__ __device__ inline long long s32_plane(int g) { return g32_pad((long long)g * g, 4); }

// fp64 pooled [heads][g][d] -> fp32 [heads][dp][gp] (zero padded); grid
// (gp / 32, dp / 32, 2 * heads), block (32, 8)
__global__ void __launch_bounds__(256) s32_pack_kernel(const double* __restrict__ qp, const double* __restrict__ kp,
                                                       int g, int d, float* __restrict__ qt, float* __restrict__ kt) {
  __shared__ float tile[32][33];
  const int h = blockIdx.z >> 1, which = blockIdx.z & 1;
  const int gp = (int)g32_pad(g, DT32), dp = (int)g32_pad(d, DK32);
  const double* X = (which ? kp : qp) + (long long)h * g * d;
  float* Y = (which ? kt : qt) + (long long)h * dp * gp;
  const int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int r = r0 + y, c = c0 + threadIdx.x;
    tile[y][threadIdx.x] = (r < g && c < d) ? (float)__ldg(X + (long long)r * d + c) : 0.f;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int c = c0 + y, r = r0 + threadIdx.x;
    if (c < dp) Y[(long long)c * gp + r] = tile[threadIdx.x][y];
  }
}

__global__ void __launch_bounds__(256, 2) draft32_gemm_kernel(const float* __restrict__ qt, const float* __restrict__ kt,
                                                              float* __restrict__ scores, int g, int d, float scale,
                                                              unsigned int* __restrict__ hist0,
                                                              unsigned int* __restrict__ rowmax) {
  // dynamic shared memory: the operand ring during the main loop, then the
  // 128 x 128 score tile, which the epilogue writes out row by row (coalesced
  // 16-byte stores, row maxima and the digit-0 histogram per row)
  extern __shared__ __align__(16) float g32s[];
  float (*T)[G32_TS] = reinterpret_cast<float (*)[G32_TS]>(g32s);  // [DT32][G32_TS]
  __shared__ unsigned int sh[NB];
  const int h = blockIdx.z;
  const int i0 = blockIdx.y * DT32, j0 = blockIdx.x * DT32;
  const int gp = (int)g32_pad(g, DT32), dp = (int)g32_pad(d, DK32);
  const float* Q = qt + (long long)h * dp * gp + i0;
  const float* K = kt + (long long)h * dp * gp + j0;
  const int tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;
  for (int b = tid; b < NB; b += 256) sh[b] = 0;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(g32s);
  const int nk = dp / DK32;
  // chunk kc -> stage kc % G32_STAGES: [operand][DK32][DT32] floats; each
  // thread moves 4 x 16 bytes (row c = tid / 32 + 8 t, 16-byte column tid % 32)
  auto issue = [&](int kc) {
    if (kc < nk) {
      const uint32_t s = sbase + (uint32_t)((kc % G32_STAGES) * G32_STAGE_FLOATS * 4);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int op = t >> 1, c = (tid >> 5) + 8 * (t & 1), col = (tid & 31) * 4;
        const float* src = (op ? K : Q) + (long long)(kc * DK32 + c) * gp + col;
        cp_async16(s + (uint32_t)(((op * DK32 + c) * DT32 + col) * 4), src, 16);
      }
    }
    cp_async_commit();
  };
  // thread (ty, tx) owns rows 4 ty + {0..3} and 64 + 4 ty + {0..3} (u = 0..7),
  // columns 4 tx + {0..3} and 64 + 4 tx + {0..3}; acc[u][v2] = column pair v2
  float2 acc[8][4];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = make_float2(0.f, 0.f);
#pragma unroll
  for (int s = 0; s < G32_STAGES - 1; ++s) issue(s);
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<G32_STAGES - 2>();
    __syncthreads();  // chunk kc visible to all; stage (kc - 1) % STAGES free
    issue(kc + G32_STAGES - 1);
    const float* sq = g32s + (kc % G32_STAGES) * G32_STAGE_FLOATS;
    const float* sk = sq + DK32 * DT32;
#pragma unroll
    for (int c = 0; c < DK32; ++c) {
      const float4 a0 = *reinterpret_cast<const float4*>(sq + c * DT32 + 4 * ty);
      const float4 a1 = *reinterpret_cast<const float4*>(sq + c * DT32 + 64 + 4 * ty);
      const float4 b0 = *reinterpret_cast<const float4*>(sk + c * DT32 + 4 * tx);
      const float4 b1 = *reinterpret_cast<const float4*>(sk + c * DT32 + 64 + 4 * tx);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float2 b[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                           make_float2(b1.z, b1.w)};
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = ffma2(make_float2(a[u], a[u]), b[v], acc[u][v]);
    }
  }
  cp_async_wait<0>();
  float* S = scores + (long long)h * s32_plane(g);
  // each row's largest key, from registers: per thread over its 8 columns,
  // then across the 16 threads of the row group (8 independent chains)
  {
    unsigned int rk[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      rk[u] = 0u;
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int col = (v < 4 ? 0 : 64) + 4 * tx + (v & 3);
        const float2 a2 = acc[u][v >> 1];
        const float val = ((v & 1) ? a2.y : a2.x) * scale;
        if (j0 + col < g) rk[u] = max(rk[u], key32(val));
      }
    }
#pragma unroll
    for (int o2 = 8; o2; o2 >>= 1)
#pragma unroll
      for (int u = 0; u < 8; ++u) rk[u] = max(rk[u], __shfl_xor_sync(0xffffffffu, rk[u], o2));
    if (tx == 0) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int gi = i0 + (u < 4 ? 0 : 60) + 4 * ty + u;
        if (gi < g) atomicMax(&rowmax[(long long)h * g + gi], rk[u]);
      }
    }
  }
  __syncthreads();  // operands no longer needed: the tile reuses the space
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int r = (u < 4 ? 0 : 60) + 4 * ty + u;
    *reinterpret_cast<float4*>(&T[r][4 * tx]) =
        make_float4(acc[u][0].x * scale, acc[u][0].y * scale, acc[u][1].x * scale, acc[u][1].y * scale);
    *reinterpret_cast<float4*>(&T[r][64 + 4 * tx]) =
        make_float4(acc[u][2].x * scale, acc[u][2].y * scale, acc[u][3].x * scale, acc[u][3].y * scale);
  }
  __syncthreads();
  const int lane = tid & 31, wp = tid >> 5;
  const bool vec = (g & 3) == 0;  // 16-byte aligned rows
  for (int rr = wp; rr < DT32; rr += 8) {
    const int gi = i0 + rr;
    if (gi >= g) break;
    const float4 o = *reinterpret_cast<const float4*>(&T[rr][4 * lane]);
    const int gj = j0 + 4 * lane;
    const float ov[4] = {o.x, o.y, o.z, o.w};
#ifdef DA_G32_NOSTORE
    if (o.x == 12345.f)
#endif
    if (vec && gj + 3 < g) {
      *reinterpret_cast<float4*>(S + (long long)gi * g + gj) = o;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (gj + q < g) S[(long long)gi * g + gj + q] = ov[q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // digit-0 histogram: plain shared-memory atomics (measured faster than
      // warp-aggregating equal bins with match.any, whose latency dominated)
#ifndef DA_G32_NOHIST
      if (gj + q < g) atomicAdd(&sh[key32(ov[q]) >> 21], 1u);
#endif
    }
  }
  __syncthreads();
  for (int b = tid; b < NB; b += 256)
    if (sh[b]) atomicAdd(&hist0[(long long)h * NB + b], sh[b]);
}

// digits: 0 = bits 21..31 (fused in the GEMM), 1 = bits 10..20, 2 = bits 0..9.
// Only digits 0 and 1 are resolved: the 22-bit key bucket of the m-th score
// spans 2^10 fp32 ulps (2^-13 relative), so the guard band simply covers it.
constexpr int S32_PASSES = 2;
DA_DEV int p32_hi(int pass) { return pass == 0 ? 32 : pass == 1 ? 21 : 10; }
DA_DEV int p32_lo(int pass) { return pass == 0 ? 21 : pass == 1 ? 10 : 0; }

__global__ void __launch_bounds__(256) s32_hist_kernel(const float* __restrict__ scores, long long n,
                                                       const Sel32State* __restrict__ st, unsigned int* hist, int pass,
                                                       const int* __restrict__ fallback) {
  if (*fallback) return;
  const int h = blockIdx.y;
  __shared__ unsigned int sh[NB];
  for (int b = threadIdx.x; b < NB; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const int hi = p32_hi(pass), lo = p32_lo(pass);
  const unsigned int prefix = st[h].prefix;
  const unsigned int dmask = (1u << (hi - lo)) - 1u;
  const float* plane = scores + (long long)h * g32_pad(n, 4);
  const float4* s4 = reinterpret_cast<const float4*>(plane);
  const long long n4 = n / 4;
  // each CTA streams a contiguous range of 16-byte groups, 4 loads in flight per thread
  const long long per = (n4 + gridDim.x - 1) / gridDim.x;
  const long long b0 = (long long)blockIdx.x * per, b1 = min(n4, b0 + per);
  auto count = [&](float x) {
    const unsigned int k = key32(x);
    if ((k >> hi) == prefix) atomicAdd(&sh[(k >> lo) & dmask], 1u);
  };
  for (long long e0 = b0 + threadIdx.x; e0 < b1; e0 += 4 * blockDim.x) {
    float4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long e = e0 + (long long)u * blockDim.x;
      if (e < b1) x[u] = __ldg(s4 + e);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (e0 + (long long)u * blockDim.x < b1) {
        count(x[u].x); count(x[u].y); count(x[u].z); count(x[u].w);
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (int)(n - n4 * 4)) count(__ldg(plane + n4 * 4 + threadIdx.x));  // tail
  __syncthreads();
  for (int b = threadIdx.x; b < NB; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[(long long)h * NB + b], sh[b]);
}

// One block (1024 threads) per head: resolve digit `pass` from the global
// histogram. Bins are walked from the top: thread t owns bins nb-1-2t and
// nb-2-2t, a block-wide scan of the pair sums gives every bin's count above
// it, and the bin where that count first reaches `remaining` is chosen (the
// warp-serial pick_bucket walk took 15-22 us).
__global__ void __launch_bounds__(1024) s32_scan_kernel(Sel32State* st, unsigned int* hist, int pass, int* fallback,
                                                        int d, double scale) {
  __shared__ long long wsum[32];
  __shared__ int s_chosen;
  __shared__ long long s_above;
  if (*fallback) return;
  const int h = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int hi = p32_hi(pass), lo = p32_lo(pass);
  const int nb = 1 << (hi - lo);
  unsigned int* H = hist + (long long)h * NB;
  const long long rem = st[h].remaining;
  const int b0 = nb - 1 - 2 * t, b1 = b0 - 1;  // descending
  const long long c0 = b0 >= 0 ? (long long)H[b0] : 0, c1 = b1 >= 0 ? (long long)H[b1] : 0;
  const long long local = c0 + c1;
  long long incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  if (t == 0) s_chosen = -1;
  __syncthreads();
  if (w == 0) {
    long long v = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    wsum[lane] = v;  // inclusive over warps
  }
  __syncthreads();
  const long long excl = incl - local + (w > 0 ? wsum[w - 1] : 0);  // count in bins above b0
  // exactly one bin satisfies above < rem <= above + count
  if (b0 >= 0 && excl < rem && excl + c0 >= rem) {
    s_chosen = b0;
    s_above = excl;
  } else if (b1 >= 0 && excl + c0 < rem && excl + c0 + c1 >= rem) {
    s_chosen = b1;
    s_above = excl + c0;
  }
  __syncthreads();
  for (int b = t; b < NB; b += blockDim.x) H[b] = 0;
  if (t == 0) {
    Sel32State s = st[h];
    const int chosen = s_chosen;
    const long long above = chosen >= 0 ? s_above : 0;
    s.remaining = rem - above;
    s.prefix = (pass == 0 ? 0u : (s.prefix << (hi - lo))) | (unsigned int)chosen;
    if (pass == S32_PASSES - 1) s32_set_eps(s, d, scale, fallback);
    st[h] = s;
  }
}

// One warp per row: sure-kept bits into the word-aligned bitmap, band entries
// into the candidate list, and the row's exact first argmax.
__global__ void __launch_bounds__(256) s32_mark_kernel(const float* __restrict__ scores, const double* __restrict__ qp,
                                                       const double* __restrict__ kp, int g, int d, double scale,
                                                       Sel32State* st, unsigned int* bm, int w32,
                                                       const unsigned int* __restrict__ rowmax, int* argmax,
                                                       int* cand, const int* __restrict__ fallback) {
  if (*fallback) return;
  const int h = blockIdx.y;
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= g) return;
  const double eps = st[h].eps;
  // the m-th largest fp32 score lies in the 22-bit key bucket the two radix
  // passes resolved (key bits 10..31); the band spans that bucket plus the
  // 2 eps guard
  const unsigned int kb = st[h].prefix << p32_lo(S32_PASSES - 1);
  const double t_lo = (double)key32_score(kb), t_hi = (double)key32_score(kb | ((1u << p32_lo(S32_PASSES - 1)) - 1u));
  const float hi_f = __double2float_ru(t_hi + 2.0 * eps);
  const float lo_f = __double2float_rd(t_lo - 2.0 * eps);
  const float rmax = key32_score(rowmax[(long long)h * g + row]);
  const float rlo = __double2float_rd((double)rmax - 2.0 * eps);
  const float* S = scores + (long long)h * s32_plane(g) + (long long)row * g;
  unsigned int* B = bm + ((long long)h * g + row) * w32;
  int* C = cand + (long long)h * S32_CAP;
  long long hi_cnt = 0;
  int best = -1;
  double bv = 0.0;
  const double* qrow = qp + ((long long)h * g + row) * d;
  // Row argmax candidates (within 2 eps of the fp32 row max) are collected in
  // ascending column order, 32 at a time, and rescored in fp64 (the fp64
  // GEMM's summation order) one candidate per lane; the first maximum in
  // ascending column order wins, as np.argmax's does.
  __shared__ int acand[8][32];
  int* ac = acand[threadIdx.x / 32];
  int na = 0;  // warp-uniform
  auto flush_candidates = [&]() {
    __syncwarp();
    double sv = 0.0;
    int col = 0x7fffffff;
    if (lane < na) {
      col = ac[lane];
      sv = dot64_seq(qrow, kp + ((long long)h * g + col) * d, d) * scale;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double s2 = __shfl_xor_sync(0xffffffffu, sv, o);
      const int c2 = __shfl_xor_sync(0xffffffffu, col, o);
      if (c2 != 0x7fffffff && (col == 0x7fffffff || s2 > sv || (s2 == sv && c2 < col))) { sv = s2; col = c2; }
    }
    if (best < 0 || sv > bv) { best = col; bv = sv; }  // later batches hold larger columns
    na = 0;
    __syncwarp();
  };
  auto argmax_candidate = [&](int jj) {
    if (lane == 0) ac[na] = jj;
    if (++na == 32) flush_candidates();
  };
  if ((g & 3) == 0) {
    // 16-byte path: lane holds columns j0 + 4 lane .. + 3 (128 per step, the
    // next step's load in flight); bitmap word w of the step is assembled
    // from the 4-bit masks of lanes 8 w .. 8 w + 7
    const float4 ninf = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    float4 nxt = 4 * lane < g ? __ldg(reinterpret_cast<const float4*>(S + 4 * lane)) : ninf;
    for (int j0 = 0; j0 < g; j0 += 128) {
      const float4 x = nxt;
      const int j = j0 + 4 * lane;
      nxt = j + 128 < g ? __ldg(reinterpret_cast<const float4*>(S + j + 128)) : ninf;
      const float v[4] = {x.x, x.y, x.z, x.w};
      unsigned int sn = 0, bn = 0, an = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool sure = v[q] > hi_f;
        sn |= (unsigned)sure << q;
        bn |= (unsigned)(!sure && v[q] >= lo_f) << q;
        an |= (unsigned)(j < g && v[q] >= rlo) << q;
      }
      hi_cnt += __popc(sn);
      unsigned int word = sn << (4 * (lane & 7));
      word |= __shfl_xor_sync(0xffffffffu, word, 1);
      word |= __shfl_xor_sync(0xffffffffu, word, 2);
      word |= __shfl_xor_sync(0xffffffffu, word, 4);
      const int wi = (j0 >> 5) + (lane >> 3);
      if ((lane & 7) == 0 && wi < w32) B[wi] = word;
      if (__any_sync(0xffffffffu, bn != 0)) {
        const int c = __popc(bn);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        int base = 0;
        if (lane == 31) base = atomicAdd(&st[h].cand_count, incl);
        base = __shfl_sync(0xffffffffu, base, 31);
        int slot = base + incl - c;
        for (unsigned int b = bn; b; b &= b - 1, ++slot)
          if (slot < S32_CAP) C[slot] = row * g + j + __ffs(b) - 1;
      }
      unsigned int aw = __ballot_sync(0xffffffffu, an != 0);
      while (aw) {
        const int src = __ffs(aw) - 1;
        aw &= aw - 1;
        for (unsigned int nib = __shfl_sync(0xffffffffu, an, src); nib; nib &= nib - 1)
          argmax_candidate(j0 + 4 * src + __ffs(nib) - 1);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) hi_cnt += __shfl_xor_sync(0xffffffffu, hi_cnt, o);  // per-lane counts above
  } else {
    for (int j0 = 0; j0 < g; j0 += 32) {
      const int j = j0 + lane;
      const float v = j < g ? __ldg(S + j) : -INFINITY;
      const bool sure = v > hi_f;
      const bool band = !sure && v >= lo_f;
      const unsigned sw = __ballot_sync(0xffffffffu, sure);
      if (lane == 0) B[j0 >> 5] = sw;
      hi_cnt += __popc(sw);
      const unsigned bw = __ballot_sync(0xffffffffu, band);
      if (bw) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&st[h].cand_count, __popc(bw));
        base = __shfl_sync(0xffffffffu, base, 0);
        const int slot = base + __popc(bw & ((1u << lane) - 1));
        if (band && slot < S32_CAP) C[slot] = row * g + j;
      }
      // row argmax candidates (within 2 eps of the fp32 row max), resolved in fp64
      unsigned aw = __ballot_sync(0xffffffffu, j < g && v >= rlo);
      while (aw) {
        const int src = __ffs(aw) - 1;
        aw &= aw - 1;
        argmax_candidate(j0 + src);
      }
    }
  }
  if (na > 0) {
    __syncwarp();
    if (best < 0 && na == 1) best = ac[0];  // the row's only candidate is its argmax: nothing to rescore
    else flush_candidates();
  }
  if (lane == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&st[h].count_hi), (unsigned long long)hi_cnt);
    argmax[(long long)h * g + row] = best;
  }
}

// One CTA per head: sort the band (fp64 keys from s32_band_score_kernel) into
// the reference order - descending score, ties to the smaller flat index -
// with a bitonic sort in shared memory, keep the first `need`, set their bits
// and emit the threshold.
// fp64 rescoring of the band, one thread per candidate (the fp64 GEMM's
// summation order): keys into bkey[head][S32_CAP]; grid (S32_SCORE_CTAS, heads)
constexpr int S32_SCORE_CTAS = 64;
__global__ void __launch_bounds__(256) s32_band_score_kernel(const double* __restrict__ qp,
                                                             const double* __restrict__ kp, int g, int d, double scale,
                                                             const Sel32State* __restrict__ st,
                                                             const int* __restrict__ cand,
                                                             unsigned long long* __restrict__ bkey,
                                                             const int* __restrict__ fallback) {
  if (*fallback) return;
  const int h = blockIdx.y;
  const int cnt = min(st[h].cand_count, S32_CAP);
  const int* C = cand + (long long)h * S32_CAP;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cnt; c += gridDim.x * blockDim.x) {
    const int f = C[c];
    const int i = f / g, j = f - i * g;
    const double sc = dot64_seq(qp + ((long long)h * g + i) * d, kp + ((long long)h * g + j) * d, d) * scale;
    bkey[(long long)h * S32_CAP + c] = score_key(sc);
  }
}

__global__ void __launch_bounds__(1024) s32_finish_kernel(const double* __restrict__ qp,
                                                          const double* __restrict__ kp, int g, int d, double scale,
                                                          long long m, Sel32State* st, const int* __restrict__ cand,
                                                          const unsigned long long* __restrict__ bkey,
                                                          unsigned int* bm, int w32, double* threshold,
                                                          int* fallback) {
  extern __shared__ unsigned char smraw[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smraw);  // [S32_CAP]
  int* idx = reinterpret_cast<int*>(key + S32_CAP);                         // [S32_CAP]
  __shared__ int bad;
  const int h = blockIdx.x;
  if (*fallback) return;
  const int cnt = st[h].cand_count;
  const long long need = m - st[h].count_hi;
  if (threadIdx.x == 0) bad = (cnt > S32_CAP || need < 1 || need > cnt) ? 1 : 0;
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) atomicOr(fallback, 1);
    return;
  }
  const int* C = cand + (long long)h * S32_CAP;
  const unsigned long long* K = bkey + (long long)h * S32_CAP;  // fp64 band scores (s32_band_score_kernel)
  int np = 1;
  while (np < cnt) np <<= 1;
  for (int c = threadIdx.x; c < np; c += blockDim.x) {  // padding sorts last (key 0, index INT_MAX)
    key[c] = c < cnt ? K[c] : 0ull;
    idx[c] = c < cnt ? C[c] : 0x7fffffff;
  }
  __syncthreads();
  // bitonic sort into reference order: descending score, ties by ascending flat index
  for (int k = 2; k <= np; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < np / 2; t += blockDim.x) {
        const int a = 2 * t - (t & (j - 1));  // lower element of the pair (bit j clear)
        const int b = a + j;
        const bool desc = (a & k) == 0;       // this run's direction
        const unsigned long long ka = key[a], kb = key[b];
        const int ia = idx[a], ib = idx[b];
        const bool a_first = ka > kb || (ka == kb && ia < ib);
        if (a_first != desc) {
          key[a] = kb; key[b] = ka;
          idx[a] = ib; idx[b] = ia;
        }
      }
      __syncthreads();
    }
  }
  unsigned int* Bh = bm + (long long)h * g * w32;
  for (int c = threadIdx.x; c < need; c += blockDim.x) {
    const int fc = idx[c];
    const int i = fc / g, j = fc - i * g;
    atomicOr(&Bh[(long long)i * w32 + (j >> 5)], 1u << (j & 31));
  }
  if (threadIdx.x == 0) threshold[h] = key_score(key[need - 1]);
}

// Per row: force the first argmax in (force_row_keep) and count the row.
__global__ void __launch_bounds__(256) s32_force_kernel(unsigned int* bm, int g, int w32,
                                                        const int* __restrict__ argmax, int force, int* row_counts,
                                                        int* row_forced, const int* __restrict__ fallback) {
  if (*fallback) return;
  const int h = blockIdx.y;
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= g) return;
  unsigned int* B = bm + ((long long)h * g + row) * w32;
  int forced = 0;
  if (force && lane == 0) {
    const int a = argmax[(long long)h * g + row];
    if (a >= 0 && !((B[a >> 5] >> (a & 31)) & 1u)) {
      B[a >> 5] |= 1u << (a & 31);
      forced = 1;
    }
  }
  __syncwarp();
  int cnt = 0;
  for (int c = lane; c < w32; c += 32) cnt += __popc(B[c]);
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) {
    row_counts[(long long)h * g + row] = cnt;
    row_forced[(long long)h * g + row] = forced;
  }
}

__global__ void copy_total_guarded_kernel(const int* row_ptr, int g, int heads, int64_t* kept,
                                          const int* __restrict__ fallback) {
  if (*fallback) return;
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h < heads) kept[h] = row_ptr[(long long)h * (g + 1) + g];
}

struct Sel32Ws {
  Sel32State* state;
  unsigned int* hist;
  unsigned int* rowmax;
  int* argmax;
  int* cand;
  unsigned long long* bkey;  // fp64 keys of the band candidates, [heads][S32_CAP]
  int* row_counts;
  int* row_forced;
  unsigned int* bm;
  int* fallback;
  float* qt;  // packed fp32 operands of the draft GEMM, [heads][dp][gp]
  float* kt;
  size_t total;
};

static Sel32Ws carve_sel32(void* base, int heads, int g, int d) {
  Sel32Ws w;
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) { char* r = p ? p + off : nullptr; off += (bytes + 255) & ~size_t(255); return r; };
  const int w32 = (g + 31) / 32;
  w.state = reinterpret_cast<Sel32State*>(take(sizeof(Sel32State) * heads));
  w.hist = reinterpret_cast<unsigned int*>(take(sizeof(unsigned int) * NB * heads));
  w.rowmax = reinterpret_cast<unsigned int*>(take(sizeof(unsigned int) * (size_t)heads * g));
  w.argmax = reinterpret_cast<int*>(take(sizeof(int) * (size_t)heads * g));
  w.cand = reinterpret_cast<int*>(take(sizeof(int) * (size_t)heads * S32_CAP));
  w.bkey = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * (size_t)heads * S32_CAP));
  w.row_counts = reinterpret_cast<int*>(take(sizeof(int) * (size_t)heads * g));
  w.row_forced = reinterpret_cast<int*>(take(sizeof(int) * (size_t)heads * g));
  w.bm = reinterpret_cast<unsigned int*>(take(sizeof(unsigned int) * (size_t)heads * g * w32));
  w.fallback = reinterpret_cast<int*>(take(sizeof(int)));
  const size_t packed = sizeof(float) * (size_t)heads * g32_pad(d, DK32) * g32_pad(g, DT32);
  w.qt = reinterpret_cast<float*>(take(packed));
  w.kt = reinterpret_cast<float*>(take(packed));
  w.total = off;
  return w;
}

size_t select32_workspace_size(int heads, int g, int d) { return carve_sel32(nullptr, heads, g, d).total; }
const int* select32_fallback_flag(void* ws, int heads, int g) { return carve_sel32(ws, heads, g, 0).fallback; }

cudaError_t launch_select32(const double* qp, const double* kp, float* scores32, int heads, int g, int d,
                            double scale, long long m, int force, void* ws, int* row_ptr, int* col_idx,
                            uint8_t* bitmap, double* threshold, int64_t* forced, int64_t* kept, long long cap,
                            cudaStream_t st, const unsigned long long* pnorm) {
  Sel32Ws w = carve_sel32(ws, heads, g, d);
  const long long n = (long long)g * g;
  const int w32 = (g + 31) / 32;
  s32_init_kernel<<<heads, 256, 0, st>>>(w.state, w.hist, w.rowmax, g, m, w.fallback, pnorm);
  if (pnorm == nullptr) s32_norm_kernel<<<dim3(heads, EPSB), 256, 0, st>>>(qp, kp, g, d, w.state);
  dim3 ggrid((g + DT32 - 1) / DT32, (g + DT32 - 1) / DT32, heads);
  {
    cudaError_t e = ensure_smem_optin((const void*)draft32_gemm_kernel, G32_SMEM);
    if (e != cudaSuccess) return e;
  }
  s32_pack_kernel<<<dim3((unsigned)(g32_pad(g, DT32) / 32), (unsigned)g32_pad(d, 32) / 32, 2 * heads), dim3(32, 8), 0,
                    st>>>(qp, kp, g, d, w.qt, w.kt);
  draft32_gemm_kernel<<<ggrid, 256, G32_SMEM, st>>>(w.qt, w.kt, scores32, g, d, (float)scale, w.hist, w.rowmax);
#ifndef S32_HIST_EPT
#define S32_HIST_EPT 32  // 16-byte groups per thread per CTA of the digit-histogram pass
#endif
  int chunks = (int)((n / 4 + 256 * S32_HIST_EPT - 1) / (256 * S32_HIST_EPT));
  if (chunks > 512) chunks = 512;
  if (chunks < 1) chunks = 1;
  for (int pass = 0; pass < S32_PASSES; ++pass) {
    if (pass > 0) s32_hist_kernel<<<dim3(chunks, heads), 256, 0, st>>>(scores32, n, w.state, w.hist, pass, w.fallback);
    s32_scan_kernel<<<heads, 1024, 0, st>>>(w.state, w.hist, pass, w.fallback, d, scale);
  }
  dim3 rows_grid((g + 7) / 8, heads);
  s32_mark_kernel<<<rows_grid, 256, 0, st>>>(scores32, qp, kp, g, d, scale, w.state, w.bm, w32, w.rowmax, w.argmax,
                                             w.cand, w.fallback);
  const size_t fsmem = (sizeof(unsigned long long) + sizeof(int)) * S32_CAP;
  {
    cudaError_t e = ensure_smem_optin((const void*)s32_finish_kernel, (int)fsmem);
    if (e != cudaSuccess) return e;
  }
  s32_band_score_kernel<<<dim3(S32_SCORE_CTAS, heads), 256, 0, st>>>(qp, kp, g, d, scale, w.state, w.cand, w.bkey,
                                                                    w.fallback);
  s32_finish_kernel<<<heads, 1024, fsmem, st>>>(qp, kp, g, d, scale, m, w.state, w.cand, w.bkey,
                                                                      w.bm, w32, threshold, w.fallback);
  s32_force_kernel<<<rows_grid, 256, 0, st>>>(w.bm, g, w32, w.argmax, force, w.row_counts, w.row_forced, w.fallback);
  scan_rows_kernel<<<heads, 1024, 0, st>>>(w.row_counts, row_ptr, g, g + 1, nullptr, 0, w.row_forced,
                                           reinterpret_cast<long long*>(forced), w.fallback, 0);
  sel_collect_kernel<<<rows_grid, 256, 0, st>>>(w.bm, g, w32, row_ptr, col_idx, cap, w.fallback, 0);
  copy_total_guarded_kernel<<<(heads + 127) / 128, 128, 0, st>>>(row_ptr, g, heads, kept, w.fallback);
  if (bitmap != nullptr) {
    const long long bph = bitmap_bytes_per_head(g);
    sel_packbits_kernel<<<dim3((unsigned)((bph + 255) / 256), heads), 256, 0, st>>>(w.bm, g, w32, make_fastdiv(g),
                                                                                     bph, bitmap, w.fallback, 0);
  }
  return cudaGetLastError();
}

}  // namespace da
