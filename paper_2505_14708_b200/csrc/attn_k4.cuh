// Shared pieces of the K4 kernels (attn_lh.cu, attn_tk.cu): launch
// parameters, the work item (one query region of one head with its kept key
// list) and token / key geometry in either tensor layout.
#pragma once

#include "common.cuh"

namespace da {
namespace k4 {

constexpr int P = 64;         // region rows (8x8 pool)
constexpr int D = 128;        // head dim
constexpr int TILE = 16384;   // one region of K or V, bf16
constexpr int KBLK = 32;      // key_norm_kernel blocks per head
constexpr int RAGW = 512;     // ragged-region bitmap words (g <= 16384)
constexpr int LISTCAP = 4096; // staged kept-list entries per item (else read from global)

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
  FastDiv per_head;  // g
  const uint8_t* kt;
  const uint8_t* vt;
  // [heads][g] item records in claim order (query regions by kept count,
  // descending): {region i, list offset rp[i], kept count, head}, or null
  // (natural region order, records computed from row_ptr)
  const int4* meta;
  const float* kpart;
  int kblk;
  int* fb_count;
  int* fb_items;
  int* work;
  uint64_t pol_kv, pol_q, pol_o;
  long long* trace;  // LH_PROF output ([CTA][32]) or null
  Shards sh;         // sequence shards of Q / out (original layout), or unsplit
  // s > 0: 64 x 2^s-token regions run as their 2^s column parts of 64 tokens
  // (geo is the part geometry, attn_geo): item i_v = 2^s i + part of region i
  // takes region i's mask list, each kept key region j as 2^(s-1) steps over
  // the parts 2^s j .. 2^s j + 2^s - 1, two per step (row_ptr / col_idx / cap
  // stay the mask's). s = 1: the paper's 8x16 pools as two 8x8 halves.
  int split;
};

struct Item {
  int h, i;
  const int* list;
  int n;
};

// The record of claimed item ``it``: {region, list offset, kept count, head};
// kept count -1 past the last item. One 16-byte load with the region-order
// pass's records, else two dependent row_ptr loads.
DA_DEV int4 item_record(const Params& p, long long it, long long items) {
  if (it < 0 || it >= items) return make_int4(0, 0, -1, 0);
  if (p.meta != nullptr) return __ldg(p.meta + it);
  const int g = p.geo.g;
  const int h = (int)fdiv((uint32_t)it, p.per_head);
  const int i = (int)(it - (long long)h * g);
  const int gm = g >> p.split;  // regions of the mask
  const int* rp = p.row_ptr + (long long)(h * p.mask_h) * (gm + 1);
  const int b = rp[i >> p.split];
  return make_int4(i, b, rp[(i >> p.split) + 1] - b, h);
}

DA_DEV bool item_from_record(const Params& p, const int4 r, Item& o) {
  if (r.z < 0) return false;
  o.h = r.w;
  o.i = r.x;
  o.list = p.col_idx + (long long)(r.w * p.mask_h) * p.cap + r.y;
  o.n = r.z << p.split;  // key regions of the item (split: two halves per mask entry)
  return true;
}

DA_DEV bool fetch_item(const Params& p, long long it, long long items, Item& o) {
  return item_from_record(p, item_record(p, it, items), o);
}

DA_DEV long long token_row(const Params& p, int region, int r) {
  if (p.layout == DA_LAYOUT_REORDERED) return (long long)region * P + r;
  const RegionXY rc = p.dec(region);
  const int u = r / p.geo.pw, v = r - u * p.geo.pw;
  const int y = rc.y0 + u, x = rc.x0 + v;
  if (y >= p.geo.H || x >= p.geo.W) return -1;
  return ((long long)rc.f * p.geo.H + y) * p.geo.W + x;
}

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
  if (vy <= 0 || vx <= 0) return 0ull;  // a half of a 128-token region can lie wholly in the padding
  const unsigned long long rowm = (1ull << vx) - 1ull;
  unsigned long long m = 0;
  for (int u = 0; u < vy; ++u) m |= rowm << (u * p.geo.pw);
  return m;
}

// Is key row r of key region j a real (unmasked) key?
DA_DEV bool key_row_valid(const Params& p, int j, int r) {
  if (p.key_valid != nullptr) return p.key_valid[(long long)j * P + r] != 0;
  const RegionXY rc = p.dec(j);
  const int u = r / p.geo.pw, v = r - u * p.geo.pw;
  return rc.y0 + u < p.geo.H && rc.x0 + v < p.geo.W;
}

}  // namespace k4
}  // namespace da
