/*
 * c_abi_demo.c — the whole DraftAttention call through the C ABI alone
 * (include/draftattn_b200.h): no Python, no torch. What a C / C++ / Go (cgo)
 * host that replaces the reference's padded_sparse_attention
 * (padding.py:95-165) per head batch would do.
 *
 *   gcc -O2 -I include examples/c_abi_demo.c -o c_abi_demo \
 *       -L paper_2505_14708_b200 -ldraftattn_b200 -L /usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$PWD/paper_2505_14708_b200 -Wl,-rpath,/usr/local/cuda/lib64
 *   ./c_abi_demo frames height width patch_h patch_w heads d sparsity DIR
 *
 * DIR/q.bin, k.bin, v.bin: bf16 (heads, n, d) row-major, n = frames*height*width
 * tokens in (f, y, x) order. Writes DIR/out.bin (bf16, same layout) and
 * DIR/kept.bin (int64 kept count per head). Exit 0 on success.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "draftattn_b200.h"

static void* read_file(const char* dir, const char* name, size_t bytes) {
  char path[4096];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  void* buf = malloc(bytes);
  size_t got = fread(buf, 1, bytes, f);
  fclose(f);
  if (got != bytes) {
    free(buf);
    return NULL;
  }
  return buf;
}

static int write_file(const char* dir, const char* name, const void* buf, size_t bytes) {
  char path[4096];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE* f = fopen(path, "wb");
  if (!f) return 1;
  size_t put = fwrite(buf, 1, bytes, f);
  fclose(f);
  return put != bytes;
}

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                     \
      return 3;                                                                    \
    }                                                                              \
  } while (0)

int main(int argc, char** argv) {
  if (argc != 10) {
    fprintf(stderr, "usage: %s frames height width patch_h patch_w heads d sparsity DIR\n", argv[0]);
    return 1;
  }
  da_grid grid = {atoi(argv[1]), atoi(argv[2]), atoi(argv[3]), atoi(argv[4]), atoi(argv[5])};
  const int heads = atoi(argv[6]), d = atoi(argv[7]);
  const double sparsity = atof(argv[8]);
  const char* dir = argv[9];
  const int32_t g = da_num_regions(&grid);
  if (g < 1 || heads < 1 || d < 8) return 1;
  const int64_t n = (int64_t)grid.frames * grid.height * grid.width;
  const size_t bytes = (size_t)heads * n * d * 2;

  /* m = top_fraction_count(g*g, 1 - sparsity) (masking.py:49-56): the same double expression */
  const int64_t entries = (int64_t)g * g;
  int64_t m = (int64_t)ceil((1.0 - sparsity) * (double)entries - 1e-9);
  if (m < 1) m = 1;
  if (m > entries) m = entries;
  const int64_t cap = da_mask_capacity(g, m);

  void* hq = read_file(dir, "q.bin", bytes);
  void* hk = read_file(dir, "k.bin", bytes);
  void* hv = read_file(dir, "v.bin", bytes);
  if (!hq || !hk || !hv) {
    fprintf(stderr, "cannot read %s/{q,k,v}.bin (%zu bytes each)\n", dir, bytes);
    return 1;
  }
  void *q, *k, *v, *out, *ws;
  int32_t *row_ptr, *col_idx;
  double* thr;
  int64_t *forced, *kept;
  const size_t ws_bytes = da_pipeline_workspace_size(&grid, heads, d);
  CK(cudaMalloc(&q, bytes));
  CK(cudaMalloc(&k, bytes));
  CK(cudaMalloc(&v, bytes));
  CK(cudaMalloc(&out, bytes));
  CK(cudaMalloc(&ws, ws_bytes));
  CK(cudaMalloc((void**)&row_ptr, sizeof(int32_t) * heads * (g + 1)));
  CK(cudaMalloc((void**)&col_idx, sizeof(int32_t) * heads * cap));
  CK(cudaMalloc((void**)&thr, sizeof(double) * heads));
  CK(cudaMalloc((void**)&forced, sizeof(int64_t) * heads));
  CK(cudaMalloc((void**)&kept, sizeof(int64_t) * heads));
  CK(cudaMemcpy(q, hq, bytes, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(k, hk, bytes, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(v, hv, bytes, cudaMemcpyHostToDevice));

  da_pipeline_args pa;
  memset(&pa, 0, sizeof pa);
  pa.attn.q = q;
  pa.attn.k = k;
  pa.attn.v = v;
  pa.attn.out = out;
  /* (heads, n, d): head stride n*d, row stride d (elements) */
  pa.attn.q_head_stride = pa.attn.k_head_stride = pa.attn.v_head_stride = pa.attn.o_head_stride = n * d;
  pa.attn.q_row_stride = pa.attn.k_row_stride = pa.attn.v_row_stride = pa.attn.o_row_stride = d;
  pa.attn.heads = heads;
  pa.attn.d = d;
  pa.attn.dv = d;
  pa.attn.layout = DA_LAYOUT_ORIGINAL;
  pa.attn.scale = 1.0 / sqrt((double)d); /* head_dim_scale (core.py:13-17) */
  pa.m = m;
  pa.force_row_keep = 1; /* the reference default */
  pa.pool_mode = 0;      /* average */
  pa.select_softmax = 0; /* select_on="logits" */
  pa.shared_head_mask = 0;
  pa.row_ptr = row_ptr;
  pa.col_idx = col_idx;
  pa.bitmap = NULL;
  pa.threshold = thr;
  pa.forced = forced;
  pa.kept = kept;
  pa.workspace = ws;
  const int rc = da_sparse_attention(&pa, &grid, NULL);
  if (rc != DA_OK) {
    fprintf(stderr, "da_sparse_attention: %d %s\n", rc, da_last_error());
    return 2;
  }
  CK(cudaDeviceSynchronize());
  void* hout = malloc(bytes);
  int64_t* hkept = (int64_t*)malloc(sizeof(int64_t) * heads);
  CK(cudaMemcpy(hout, out, bytes, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hkept, kept, sizeof(int64_t) * heads, cudaMemcpyDeviceToHost));
  if (write_file(dir, "out.bin", hout, bytes) || write_file(dir, "kept.bin", hkept, sizeof(int64_t) * heads)) return 1;
  printf("ok: %d heads x %lld tokens, g = %d, m = %lld, kept[0] = %lld\n", heads, (long long)n, g, (long long)m,
         (long long)hkept[0]);
  return 0;
}
