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

DA_DEV double key_score(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

DA_DEV int pass_hi(int pass) { return 64 - RB * pass; }
DA_DEV int pass_lo(int pass) { int lo = 64 - RB * (pass + 1); return lo < 0 ? 0 : lo; }

__global__ void sel_init_kernel(SelState* st, unsigned int* hist, long long m) {
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
                                                       int pass) {
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
__global__ void sel_scan_kernel(SelState* st, unsigned int* hist, int pass) {
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
                                                          unsigned int* cand_idx) {
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
__global__ void __launch_bounds__(1024) sel_cand_finish_kernel(SelState* st, const unsigned long long* cand_key) {
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
                                                              const SelState* __restrict__ st, int* eq_rows) {
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
                                                         const int* __restrict__ extra, long long* extra_total) {
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
                                                       int* row_counts, int* row_forced) {
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
                                                          long long cap) {
  const int h = blockIdx.y;
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= g) return;
  const unsigned int* B = bm + ((long long)h * g + row) * w32;
  int out = row_ptr[(long long)h * (g + 1) + row];
  int* C = col_idx + (long long)h * cap;
  for (int c = 0; c < w32; ++c) {
    const unsigned word = __ldg(B + c);
    if ((word >> lane) & 1u) C[out + __popc(word & ((1u << lane) - 1))] = c * 32 + lane;
    out += __popc(word);
  }
}

// np.packbits(kept) (masking.py:168-170): one output byte per thread.
__global__ void __launch_bounds__(256) sel_packbits_kernel(const unsigned int* __restrict__ bm, int g, int w32,
                                                           FastDiv gdiv, long long bytes_per_head, uint8_t* out) {
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

__global__ void sel_finish_kernel(const SelState* st, int heads, double* threshold) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h < heads) threshold[h] = key_score(st[h].T);
}

__global__ void copy_total_kernel(const int* row_ptr, int g, int heads, int64_t* kept) {
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
                          int64_t* forced, int64_t* kept, long long cap, cudaStream_t st, bool digit0_done) {
  SelWs w = carve_sel(ws, heads, g);
  const long long n = (long long)g * g;
  const int w32 = (g + 31) / 32;
  if (!digit0_done) sel_init_kernel<<<heads, 256, 0, st>>>(w.state, w.hist, m);
  int chunks = (int)((n + 256 * 16 - 1) / (256 * 16));
  if (chunks > 256) chunks = 256;
  if (chunks < 1) chunks = 1;
  for (int pass = 0; pass < NPASS; ++pass) {
    if (!(pass == 0 && digit0_done))
      sel_hist_kernel<<<dim3(chunks, heads), 256, 0, st>>>(scores, n, w.state, w.hist, pass);
    sel_scan_kernel<<<heads, 32, 0, st>>>(w.state, w.hist, pass);
    if (pass == 1) {
      sel_compact_kernel<<<dim3(chunks, heads), 256, 0, st>>>(scores, n, w.state, w.cand_key, w.cand_idx);
      sel_cand_finish_kernel<<<heads, 1024, 0, st>>>(w.state, w.cand_key);
    }
  }
  dim3 rows_grid((g + 7) / 8, heads);
  sel_rowcount_eq_kernel<<<rows_grid, 256, 0, st>>>(scores, g, w.state, w.eq_rows);
  scan_rows_kernel<<<heads, 1024, 0, st>>>(w.eq_rows, w.eq_prefix, g, g + 1, w.state, 1, nullptr, nullptr);
  sel_mark_kernel<<<rows_grid, 256, 0, st>>>(scores, g, w.state, w.eq_prefix, force, dead, w.bm, w32, w.row_counts,
                                             w.row_forced);
  scan_rows_kernel<<<heads, 1024, 0, st>>>(w.row_counts, row_ptr, g, g + 1, w.state, 0, w.row_forced,
                                           reinterpret_cast<long long*>(forced));
  sel_collect_kernel<<<rows_grid, 256, 0, st>>>(w.bm, g, w32, row_ptr, col_idx, cap);
  sel_finish_kernel<<<(heads + 127) / 128, 128, 0, st>>>(w.state, heads, threshold);
  copy_total_kernel<<<(heads + 127) / 128, 128, 0, st>>>(row_ptr, g, heads, kept);
  if (bitmap != nullptr) {
    const long long bph = bitmap_bytes_per_head(g);
    sel_packbits_kernel<<<dim3((unsigned)((bph + 255) / 256), heads), 256, 0, st>>>(w.bm, g, w32, make_fastdiv(g),
                                                                                     bph, bitmap);
  }
  return cudaGetLastError();
}

// Fused digit-0 histogram support for the draft GEMM epilogue.
void select_init(void* ws, int heads, int g, long long m, cudaStream_t st) {
  SelWs w = carve_sel(ws, heads, g);
  sel_init_kernel<<<heads, 256, 0, st>>>(w.state, w.hist, m);
}

}  // namespace da
