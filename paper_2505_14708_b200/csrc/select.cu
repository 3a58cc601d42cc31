// K3b: global top-m selection per head (masking.py:59-91), force-row-keep
// (masking.py:84-88), dead key-region drop (masking.py:94-105), packed bitmap
// (masking.py:168-170) and per-row ascending column lists.
//
// Ranking key: descending score, ties to the smaller flat index i*g + j. Scores
// map to order-preserving 64-bit keys (-0.0 folded onto +0.0 so they tie, NaN
// below everything as in a stable descending argsort). The m-th key T is found
// with a most-significant-digit radix select (11-bit digits, 6 passes, each a
// histogram of the keys that still match the resolved prefix). Then one pass
// per row marks  key > T,  or key == T and among the first `need` equal keys in
// flat order,  or the row's first argmax  (if force_row_keep),  minus dead
// columns; a scan of the per-row counts places each row's columns.
#include "common.cuh"
#include "kernels.h"

namespace da {

constexpr int RB = 11;            // radix digit bits
constexpr int NB = 1 << RB;       // bins
constexpr int NPASS = 6;          // 5*11 + 9 = 64 bits

struct SelState {
  unsigned long long prefix;      // resolved high bits of T
  long long remaining;            // entries still to take from the current prefix bucket
  long long gt;                   // entries with key > prefix bucket (already kept)
  long long eq_total;             // entries with key == T (after the last pass)
  unsigned long long T;
  long long forced;
  long long kept;
};

DA_DEV unsigned long long score_key(double s) {
  if (s != s) return 0ull;  // NaN ranks last
  if (s == 0.0) s = 0.0;    // -0.0 ties +0.0
  unsigned long long b = (unsigned long long)__double_as_longlong(s);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
DA_DEV double key_score(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

DA_DEV int pass_hi(int pass) { return 64 - RB * pass; }
DA_DEV int pass_lo(int pass) { int lo = 64 - RB * (pass + 1); return lo < 0 ? 0 : lo; }

__global__ void sel_init_kernel(SelState* st, unsigned int* hist, int heads, long long m) {
  int h = blockIdx.x;
  if (threadIdx.x == 0) {
    st[h].prefix = 0; st[h].remaining = m; st[h].gt = 0; st[h].eq_total = 0; st[h].T = 0;
    st[h].forced = 0; st[h].kept = 0;
  }
  for (int b = threadIdx.x; b < NB; b += blockDim.x) hist[(long long)h * NB + b] = 0;
}

// grid: (chunks, heads), 256 threads.
__global__ void __launch_bounds__(256) sel_hist_kernel(const double* __restrict__ scores, long long n,
                                                       const SelState* __restrict__ st, unsigned int* hist,
                                                       int pass) {
  __shared__ unsigned int sh[NB];
  const int h = blockIdx.y;
  for (int b = threadIdx.x; b < NB; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const int hi = pass_hi(pass), lo = pass_lo(pass);
  const unsigned long long prefix = st[h].prefix;
  const double* s = scores + (long long)h * n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
    unsigned long long k = score_key(__ldg(s + e));
    bool match = (hi == 64) ? true : ((k >> hi) == prefix);
    if (match) atomicAdd(&sh[(unsigned)((k >> lo) & ((1ull << (hi - lo)) - 1))], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < NB; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[(long long)h * NB + b], sh[b]);
}

// one CTA (1 warp) per head: pick the bucket holding the remaining-th entry.
__global__ void sel_scan_kernel(SelState* st, unsigned int* hist, int pass) {
  const int h = blockIdx.x;
  const int lane = threadIdx.x;
  const int hi = pass_hi(pass), lo = pass_lo(pass);
  const int nb = 1 << (hi - lo);
  unsigned int* H = hist + (long long)h * NB;
  __shared__ long long s_rem;
  if (lane == 0) s_rem = st[h].remaining;
  __syncwarp();
  long long rem = s_rem;
  long long above = 0;  // running count of buckets above the current chunk
  int chosen = -1;
  long long chosen_above = 0, chosen_cnt = 0;
  // walk buckets from the top, 32 at a time
  for (int top = nb - 1; top >= 0 && chosen < 0; top -= 32) {
    int b = top - lane;
    long long c = (b >= 0) ? (long long)H[b] : 0;
    // inclusive prefix over lanes (lane 0 = highest bucket)
    long long incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    long long excl = incl - c;
    bool hit = (above + excl < rem) && (above + incl >= rem) && b >= 0;
    unsigned mask = __ballot_sync(0xffffffffu, hit);
    if (mask) {
      int src = __ffs(mask) - 1;
      chosen = __shfl_sync(0xffffffffu, b, src);
      chosen_above = above + __shfl_sync(0xffffffffu, excl, src);
      chosen_cnt = __shfl_sync(0xffffffffu, c, src);
    }
    above += __shfl_sync(0xffffffffu, incl, 31);
  }
  __syncwarp();
  // reset the histogram for the next pass
  for (int b = lane; b < NB; b += 32) H[b] = 0;
  if (lane == 0) {
    SelState s = st[h];
    s.gt += chosen_above;
    s.remaining = rem - chosen_above;
    s.prefix = (s.prefix << (hi - lo)) | (unsigned long long)chosen;
    if (lo == 0) {
      s.T = s.prefix;
      s.eq_total = chosen_cnt;
    }
    st[h] = s;
  }
}

// Per-row equal-key counts (only needed when ties at T straddle the cut).
// grid: (ceil(g/8), heads), 256 threads, one warp per row.
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

// Exclusive scan of an int array of length g per head (one CTA per head).
__global__ void __launch_bounds__(1024) scan_rows_kernel(const int* __restrict__ in, int* __restrict__ out, int g,
                                                         int out_stride, const SelState* st, int only_if_ties) {
  const int h = blockIdx.x;
  if (only_if_ties && st[h].eq_total == st[h].remaining) return;
  __shared__ int warp_tot[32];
  __shared__ int carry;
  const int* I = in + (long long)h * g;
  int* O = out + (long long)h * out_stride;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  for (int base = 0; base < g; base += blockDim.x) {
    int idx = base + threadIdx.x;
    int v = idx < g ? I[idx] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
      int nw = blockDim.x / 32;
      int t = lane < nw ? warp_tot[lane] : 0;
      int ti = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int u = __shfl_up_sync(0xffffffffu, ti, o);
        if (lane >= o) ti += u;
      }
      if (lane < nw) warp_tot[lane] = ti - t;  // exclusive warp offsets
    }
    __syncthreads();
    int excl = carry + warp_tot[w] + incl - v;
    if (idx < g) O[idx] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) O[g] = carry;
}

// Mark kept entries of each row: bitmap bits + per-row counts.
// grid: (ceil(g/8), heads), 256 threads, one warp per row. bitmap zeroed.
__global__ void __launch_bounds__(256) sel_mark_kernel(const double* __restrict__ scores, int g, SelState* st,
                                                       const int* __restrict__ eq_prefix, int force_row_keep,
                                                       const uint8_t* __restrict__ dead, unsigned int* bitmap_words,
                                                       long long bitmap_bytes_per_head, int* row_counts) {
  const int h = blockIdx.y;
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= g) return;
  const SelState s = st[h];
  const bool all_eq = s.eq_total == s.remaining;
  const double* S = scores + ((long long)h * g + row) * g;
  // first argmax of the row (np.argmax: first max; first NaN wins)
  int best = -1;
  if (force_row_keep) {
    double bv = 0.0;
    bool bnan = false;
    for (int j = lane; j < g; j += 32) {
      double v = __ldg(S + j);
      bool vnan = v != v;
      if (best < 0 || (!bnan && (vnan || v > bv))) { best = j; bv = v; bnan = vnan; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int ob = __shfl_xor_sync(0xffffffffu, best, o);
      bool onan = __shfl_xor_sync(0xffffffffu, (int)bnan, o) != 0;
      bool take;
      if (ob < 0) take = false;
      else if (best < 0) take = true;
      else if (bnan != onan) take = onan;                 // NaN beats numbers
      else if (!bnan && ov != bv) take = ov > bv;          // larger value
      else take = ob < best;                               // tie: smaller column
      if (take) { bv = ov; best = ob; bnan = onan; }
    }
  }
  int eq_run = all_eq ? 0 : eq_prefix[(long long)h * g + row];
  int cnt = 0;
  bool forced_here = false;
  const long long flat0 = (long long)row * g;
  unsigned int* words = bitmap_words + (long long)h * (bitmap_bytes_per_head / 4);
  for (int j0 = 0; j0 < g; j0 += 32) {
    int j = j0 + lane;
    bool kept = false, eq = false;
    if (j < g) {
      unsigned long long k = score_key(__ldg(S + j));
      kept = k > s.T;
      eq = k == s.T;
    }
    unsigned eqb = __ballot_sync(0xffffffffu, eq);
    if (eq) {
      if (all_eq) kept = true;
      else kept = (eq_run + __popc(eqb & ((1u << lane) - 1))) < s.remaining;
    }
    eq_run += __popc(eqb);
    if (j == best && j < g) {
      if (!kept) forced_here = true;
      kept = true;
    }
    if (kept && dead != nullptr && dead[j]) kept = false;
    cnt += kept;
    // bitmap: bit b -> byte b/8, MSB first; word = b/32 (little-endian bytes)
    unsigned w0m = 0, w1m = 0;
    long long b = flat0 + j;
    long long wbase = (flat0 + j0) >> 5;
    if (kept) {
      long long word = b >> 5;
      unsigned pos = (unsigned)(((b >> 3) & 3) * 8 + (7 - (b & 7)));
      if (word == wbase) w0m = 1u << pos; else w1m = 1u << pos;
    }
    w0m = __reduce_or_sync(0xffffffffu, w0m);
    w1m = __reduce_or_sync(0xffffffffu, w1m);
    if (lane == 0) {
      if (w0m) atomicOr(words + wbase, w0m);
      if (w1m) atomicOr(words + wbase + 1, w1m);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  unsigned fb = __ballot_sync(0xffffffffu, forced_here);
  if (lane == 0) {
    row_counts[(long long)h * g + row] = cnt;
    atomicAdd(reinterpret_cast<unsigned long long*>(&st[h].kept), (unsigned long long)cnt);
    if (fb) atomicAdd(reinterpret_cast<unsigned long long*>(&st[h].forced), 1ull);
  }
}

// Expand bitmap rows into ascending column lists at row_ptr offsets.
__global__ void __launch_bounds__(256) sel_collect_kernel(const unsigned int* __restrict__ bitmap_words, int g,
                                                          long long bitmap_bytes_per_head,
                                                          const int* __restrict__ row_ptr, int* col_idx,
                                                          long long cap) {
  const int h = blockIdx.y;
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= g) return;
  const uint8_t* bytes = reinterpret_cast<const uint8_t*>(bitmap_words) + (long long)h * bitmap_bytes_per_head;
  int out = row_ptr[(long long)h * (g + 1) + row];
  int* C = col_idx + (long long)h * cap;
  const long long flat0 = (long long)row * g;
  for (int j0 = 0; j0 < g; j0 += 32) {
    int j = j0 + lane;
    bool kept = false;
    if (j < g) {
      long long b = flat0 + j;
      kept = (bytes[b >> 3] >> (7 - (b & 7))) & 1;
    }
    unsigned kb = __ballot_sync(0xffffffffu, kept);
    if (kept) C[out + __popc(kb & ((1u << lane) - 1))] = j;
    out += __popc(kb);
  }
}

__global__ void sel_finish_kernel(const SelState* st, int heads, double* threshold, int64_t* forced,
                                  int64_t* kept) {
  int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= heads) return;
  threshold[h] = key_score(st[h].T);
  forced[h] = st[h].forced;
  kept[h] = st[h].kept;
}

// ---------------------------------------------------------------------------
size_t select_workspace_size(int heads, int g) {
  size_t n = 0;
  auto take = [&](size_t bytes) { n += (bytes + 255) & ~size_t(255); };
  take(sizeof(SelState) * heads);
  take(sizeof(unsigned int) * NB * heads);
  take(sizeof(int) * (size_t)heads * g);        // eq per row
  take(sizeof(int) * (size_t)heads * (g + 1));  // eq prefix
  take(sizeof(int) * (size_t)heads * g);        // row counts
  take(bitmap_bytes_per_head(g) * heads);       // internal bitmap
  return n;
}

long long bitmap_bytes_per_head(int g) {
  long long bits = (long long)g * g;
  long long bytes = (bits + 7) / 8;
  return (bytes + 3) / 4 * 4;  // word aligned rows of the workspace copy
}

cudaError_t launch_select(const double* scores, int heads, int g, long long m, int force, const uint8_t* dead,
                          void* ws, int* row_ptr, int* col_idx, uint8_t* bitmap, double* threshold,
                          int64_t* forced, int64_t* kept, long long cap, cudaStream_t st) {
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) { char* r = p; p += (bytes + 255) & ~size_t(255); return r; };
  SelState* state = reinterpret_cast<SelState*>(take(sizeof(SelState) * heads));
  unsigned int* hist = reinterpret_cast<unsigned int*>(take(sizeof(unsigned int) * NB * heads));
  int* eq_rows = reinterpret_cast<int*>(take(sizeof(int) * (size_t)heads * g));
  int* eq_prefix = reinterpret_cast<int*>(take(sizeof(int) * (size_t)heads * (g + 1)));
  int* row_counts = reinterpret_cast<int*>(take(sizeof(int) * (size_t)heads * g));
  const long long bpb = bitmap_bytes_per_head(g);
  unsigned int* bm = reinterpret_cast<unsigned int*>(take(bpb * heads));

  const long long n = (long long)g * g;
  sel_init_kernel<<<heads, 256, 0, st>>>(state, hist, heads, m);
  int chunks = (int)((n + 256 * 16 - 1) / (256 * 16));
  if (chunks > 512) chunks = 512;
  if (chunks < 1) chunks = 1;
  for (int pass = 0; pass < NPASS; ++pass) {
    sel_hist_kernel<<<dim3(chunks, heads), 256, 0, st>>>(scores, n, state, hist, pass);
    sel_scan_kernel<<<heads, 32, 0, st>>>(state, hist, pass);
  }
  dim3 rows_grid((g + 7) / 8, heads);
  sel_rowcount_eq_kernel<<<rows_grid, 256, 0, st>>>(scores, g, state, eq_rows);
  scan_rows_kernel<<<heads, 1024, 0, st>>>(eq_rows, eq_prefix, g, g + 1, state, 1);
  cudaMemsetAsync(bm, 0, bpb * heads, st);
  sel_mark_kernel<<<rows_grid, 256, 0, st>>>(scores, g, state, eq_prefix, force, dead, bm, bpb, row_counts);
  scan_rows_kernel<<<heads, 1024, 0, st>>>(row_counts, row_ptr, g, g + 1, state, 0);
  sel_collect_kernel<<<rows_grid, 256, 0, st>>>(bm, g, bpb, row_ptr, col_idx, cap);
  sel_finish_kernel<<<(heads + 127) / 128, 128, 0, st>>>(state, heads, threshold, forced, kept);
  if (bitmap != nullptr) {
    long long packed = (n + 7) / 8;
    cudaMemcpy2DAsync(bitmap, packed, bm, bpb, packed, heads, cudaMemcpyDeviceToDevice, st);
  }
  return cudaGetLastError();
}

}  // namespace da
