/*
 * draftattn_b200.h — C ABI of the B200 (sm_100a) DraftAttention sparse-attention path.
 *
 * The reference (arXiv 2505.14708, /root/reference/pkg/src/draftattn) is a pure
 * Python/numpy package with no FFI; each entry point below replaces one stage of
 * its padded_sparse_attention pipeline (padding.py:95-165) and is what a
 * ctypes / cffi binding of that package would call. Reference interfaces
 * replaced are cited per entry point (paths relative to pkg/src/draftattn/).
 *
 * Conventions
 *  - Plain device pointers, element strides and sizes; no torch types.
 *  - Token matrices are bf16 with the feature dimension contiguous. A tensor of
 *    `heads` heads x `rows` tokens is addressed as base + h*head_stride +
 *    row*row_stride (strides in ELEMENTS), which covers (heads, n, d) as well as
 *    the DiT (n, heads, d) layout.
 *  - The caller owns every buffer, including `workspace`. No entry point
 *    allocates, frees or synchronises; all work is ordered on `stream`
 *    (a cudaStream_t; NULL = legacy default stream).
 *  - Return 0 on success, DA_EINVAL for invalid arguments, DA_ECUDA for a CUDA
 *    launch/driver error. da_last_error() returns a thread-local message.
 */
#ifndef DRAFTATTN_B200_H
#define DRAFTATTN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DA_OK 0
#define DA_EINVAL 1
#define DA_ECUDA 2

/* Real token grid and pool size. Regions are patch_h x patch_w tiles of the
 * grid padded up to multiples of the pool size (padding.py:45-56 pad_plan;
 * layout.py:10-60 LatentLayout). */
typedef struct da_grid {
  int32_t frames;
  int32_t height;
  int32_t width;
  int32_t patch_h;
  int32_t patch_w;
} da_grid;

/* Derived sizes: number of regions g, region size p, padded token count. */
int32_t da_num_regions(const da_grid* grid);
int32_t da_region_size(const da_grid* grid);
int64_t da_padded_tokens(const da_grid* grid);

/* ABI version (major*100 + minor) and last error message of this thread. */
int32_t da_version(void);
const char* da_last_error(void);

/* Mask capacity per head for `m` globally kept entries: m + g (force_row_keep
 * adds at most one entry per row, masking.py:84-88). */
int64_t da_mask_capacity(int32_t g, int64_t m);

/* ---- K1 permute-in ---------------------------------------------------------
 * x_r[h, pos, :] = valid(pos) ? x[h, src(pos), :] : 0 for pos in [0, n_pad).
 * Replaces permute_rows(embed_rows(x, plan), perm) (padding.py:140-142,
 * padding.py:59-66, layout.py:133-141). Bit-exact copy. x_r is dense
 * (heads, n_pad, d). d must be a multiple of 8. */
int da_permute_in(const void* x, int64_t head_stride, int64_t row_stride, void* x_r, int32_t heads,
                  int32_t d, const da_grid* grid, void* stream);

/* ---- K5 permute-out --------------------------------------------------------
 * out[h, src(pos), :] = o_r[h, pos, :] for valid pos. Replaces
 * extract_rows(permute_rows(o_r, perm.inverse), plan) (padding.py:157,
 * padding.py:69-75). Bit-exact. o_r is dense (heads, n_pad, d). */
int da_permute_out(const void* o_r, void* out, int64_t head_stride, int64_t row_stride, int32_t heads,
                   int32_t d, const da_grid* grid, void* stream);

/* ---- K2 pool ---------------------------------------------------------------
 * pooled[h, i, :] (float64) = sum of valid rows of region i / max(count, 1)
 * (mode 0, average: padding.py:78-92 / pooling.py:29-30) or coordinatewise
 * max (mode 1: pooling.py:31-32; divisible grids only). Reads x in ORIGINAL
 * token order; sums are exact in float64 for bf16 inputs. */
int da_pool(const void* x, int64_t head_stride, int64_t row_stride, double* pooled, int32_t heads, int32_t d,
            const da_grid* grid, int32_t mode, void* stream);

/* ---- K3a draft scores ------------------------------------------------------
 * scores[h, i, j] = (qp[h, i, :] . kp[h, j, :]) * scale in float64
 * (pooling.py:35-56 draft_logits -> core.py:20-35 logits: product first,
 * then multiply by scale). If softmax != 0, rows are then softmaxed
 * (core.py:38-54; select_on="softmax", padding.py:148-149). */
int da_draft_scores(const double* qp, const double* kp, double* scores, int32_t heads, int32_t g, int32_t d,
                    double scale, int32_t softmax, void* stream);

/* ---- K3b selection ---------------------------------------------------------
 * Global top-m per head with ties to the smaller flat index, optional
 * per-row argmax keep, then dead key-region columns dropped
 * (masking.py:59-91 select_top_fraction, masking.py:94-105 drop_key_regions,
 * padding.py:150-153). m comes from the host (masking.py:49-56).
 * Outputs per head h (cap = da_mask_capacity(g, m)):
 *   row_ptr[h*(g+1) + i]     offsets into col_idx[h*cap ...], ascending columns
 *   col_idx[h*cap + k]       kept key regions of each row, ascending
 *   bitmap[h*ceil(g*g/8)]    np.packbits(kept) layout (masking.py:168-170), may be NULL
 *   threshold[h]             score of the m-th ranked entry (masking.py:84)
 *   forced[h], kept[h]       forced_row_keeps and kept_count
 * dead_cols: optional uint8[g], nonzero = all-padding key region.
 * workspace: da_select_workspace_size(heads, g) bytes. */
size_t da_select_workspace_size(int32_t heads, int32_t g);
int da_select(const double* scores, int32_t heads, int32_t g, int64_t m, int32_t force_row_keep,
              const uint8_t* dead_cols, void* workspace, int32_t* row_ptr, int32_t* col_idx, uint8_t* bitmap,
              double* threshold, int64_t* forced, int64_t* kept, void* stream);

/* ---- K4 block-sparse attention forward ----------------------------------
 * For every head h and query region i: softmax over the valid keys of the kept
 * key regions (ascending) of scale * q k^T, times v (sparse.py:88-166
 * block_sparse_attention with key_valid). Rows of regions with no kept valid
 * key are zero (sparse.py:137-138, 164-165).
 * layout 0 (REORDERED): q/k/v/out are (heads, n_pad, d) in reordered order
 *   (the block_sparse_attention seam). key_valid: optional uint8[n_pad], shared
 *   by all heads (nonzero = valid key); NULL = the grid's own validity.
 * layout 1 (ORIGINAL): q/k/v/out hold real tokens only, in original order,
 *   with the given strides; permutation and padding happen inside the kernel
 *   (padding.py:139-157 fused). key_valid must be NULL.
 * d == dv == 128 with p == 64 (any pool shape), or p == 64 x 2^s (s <= 3)
 * with a pool width divisible by 2^s (e.g. the paper's 8x16, run as two
 * 64-token column halves), take the tcgen05/TMEM lane-half kernel (da_sparse_attention feeds it the K/V
 * region tiles its pooling pass writes; da_block_sparse_fwd writes them first);
 * any other shape takes the portable CUDA-core kernel (same semantics). */
#define DA_LAYOUT_REORDERED 0
#define DA_LAYOUT_ORIGINAL 1
#define DA_MAX_SHARDS 8
typedef struct da_attn_args {
  const void* q;
  const void* k;
  const void* v;
  void* out;
  int64_t q_head_stride, q_row_stride;
  int64_t k_head_stride, k_row_stride;
  int64_t v_head_stride, v_row_stride;
  int64_t o_head_stride, o_row_stride;
  int32_t heads;
  int32_t d;
  int32_t dv;
  int32_t layout;
  double scale;
  const int32_t* row_ptr; /* per head: g+1 offsets */
  const int32_t* col_idx; /* per head base h*mask_cap */
  int64_t mask_cap;
  const uint8_t* key_valid;
  int32_t shared_mask;    /* nonzero: every head uses head 0's row_ptr/col_idx
                             (multi_head_sparse_attention shared_head_mask, sparse.py:281-301) */
  int32_t force_portable; /* nonzero: use the CUDA-core kernel even when tcgen05 applies */
  void* workspace;        /* da_attn_workspace_size(heads, grid) bytes of device memory (caller-owned;
                             required by the tcgen05 path, ignored by the portable one) */
  /* Sequence shards (layout ORIGINAL only; no reference counterpart: the
     reference is single-process). shard_count >= 2: the tokens are split into
     row blocks held in separate buffers, typically the sequence shards of a
     group of ranks in peer GPUs' memory (mapped with da_ipc_open), which the
     kernels then read and write over NVLink directly, with no all-to-all.
     Token row r (original order) is row r - s*shard_rows of shard
     s = r / shard_rows, at q_shards[s] + h*q_head_stride + (r - s*shard_rows)*q_row_stride
     (likewise k, v, out; all shards share the strides); every shard but the
     last holds shard_rows rows, and q/k/v/out are unused.
     shard_count 0 or 1: plain tensors at q/k/v/out. */
  int32_t shard_count;
  int64_t shard_rows;
  const void* q_shards[DA_MAX_SHARDS];
  const void* k_shards[DA_MAX_SHARDS];
  const void* v_shards[DA_MAX_SHARDS];
  void* out_shards[DA_MAX_SHARDS];
} da_attn_args;
size_t da_attn_workspace_size(int32_t heads, const da_grid* grid);
int da_block_sparse_fwd(const da_attn_args* args, const da_grid* grid, void* stream);

/* ---- Whole pipeline ---------------------------------------------------------
 * padded_sparse_attention (padding.py:95-165) / draft_sparse_attention
 * (sparse.py:193-246) for `heads` independent heads in one call: pool,
 * draft scores, selection, block-sparse attention with the permutation fused,
 * output in original order. workspace: da_pipeline_workspace_size(...) bytes.
 * The mask outputs (row_ptr/col_idx/bitmap/threshold/forced/kept, as in
 * da_select) are written into caller buffers so return_details can read them;
 * bitmap may be NULL. */
typedef struct da_pipeline_args {
  da_attn_args attn; /* layout must be ORIGINAL; row_ptr/col_idx/mask_cap/key_valid ignored */
  int64_t m;         /* top_fraction_count(g*g, 1 - sparsity) */
  int32_t force_row_keep;
  int32_t pool_mode; /* 0 average, 1 max (divisible grids only, padding.py:131-132) */
  int32_t select_softmax;
  int32_t shared_head_mask; /* one mask from the head-mean of the bases (sparse.py:281-297) */
  int32_t* row_ptr;
  int32_t* col_idx;
  uint8_t* bitmap;
  double* threshold;
  int64_t* forced;
  int64_t* kept;
  void* workspace;
  void* ev_attn_begin; /* optional cudaEvent_t recorded around the K4 launch (timing hook) */
  void* ev_attn_end;
} da_pipeline_args;
size_t da_pipeline_workspace_size(const da_grid* grid, int32_t heads, int32_t d);
/* Byte offset, inside the pipeline workspace, of the int the fp32 guard-band
 * selection sets when the exact fp64 selection had to run instead (non-finite
 * inputs, massive ties); 0 after a call means the fast path decided the mask.
 * Diagnostics / tests; -1 on invalid arguments. */
int64_t da_pipeline_fallback_offset(const da_grid* grid, int32_t heads, int32_t d);
/* Kernel launches one da_sparse_attention call issues (for launch accounting). */
int32_t da_pipeline_launches(int32_t select_softmax, int32_t shared_head_mask);
int da_sparse_attention(const da_pipeline_args* args, const da_grid* grid, void* stream);

/* ---- Peer memory (sequence shards over NVLink) ------------------------------
 * CUDA IPC for da_attn_args' shard tables. da_ipc_export: the 64-byte handle
 * of the device allocation holding dev_ptr and dev_ptr's byte offset in it
 * (any pointer into a cudaMalloc allocation, e.g. a caching allocator's).
 * da_ipc_open (in another process): maps that allocation into the current
 * device, enabling peer access when it lives on another GPU, and returns the
 * exported pointer's address here. da_ipc_close unmaps (the pointer
 * da_ipc_open returned and the same offset). A process cannot open its own
 * exports (use the pointer itself). */
#define DA_IPC_HANDLE_BYTES 64
int da_ipc_export(const void* dev_ptr, void* handle, int64_t* offset);
int da_ipc_open(const void* handle, int64_t offset, void** dev_ptr);
int da_ipc_close(void* dev_ptr, int64_t offset);

/* ---- Diagnostics -------------------------------------------------------------
 * While set, the tcgen05 kernel of CTA 0 records clock64() stamps of its
 * pipeline events (24 event rows x 1024 steps, int64) into this device buffer.
 * NULL disables. Not thread-safe; for profiling only. */
int da_debug_trace(void* device_buffer);

#ifdef __cplusplus
}
#endif

#endif /* DRAFTATTN_B200_H */
