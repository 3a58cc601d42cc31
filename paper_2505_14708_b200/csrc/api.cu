// C-ABI entry points (include/draftattn_b200.h): argument validation, error
// reporting, workspace carving and the whole-pipeline driver. Validation
// mirrors the reference's ValueError conditions where they apply to raw
// buffers; the Python host layer raises the reference's own messages first.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return DA_OK;
  return fail(DA_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

bool grid_ok(const da_grid* g) {
  return g && g->frames > 0 && g->height > 0 && g->width > 0 && g->patch_h > 0 && g->patch_w > 0;
}

size_t align256(size_t n) { return (n + 255) & ~size_t(255); }

}  // namespace

namespace da {

// Per-device facts, filled once per device and never changed afterwards.
namespace {
constexpr int kMaxDevices = 64;
std::atomic<int> g_sms[kMaxDevices];
std::mutex g_optin_mu;
struct OptIn {
  const void* kernel;
  int dev;
  int bytes;
};
std::vector<OptIn> g_optin;
}  // namespace

int device_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 1;
  }
  int n = g_sms[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 1;
    g_sms[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

cudaError_t ensure_smem_optin(const void* kernel, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_optin_mu);
  for (OptIn& o : g_optin)
    if (o.kernel == kernel && o.dev == dev) {
      if (o.bytes >= bytes) return cudaSuccess;
      cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      if (e == cudaSuccess) o.bytes = bytes;
      return e;
    }
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) g_optin.push_back({kernel, dev, bytes});
  return e;
}

}  // namespace da

extern "C" {

int32_t da_version(void) { return 101; }  // 1.01: sequence shards, IPC

// ---------------------------------------------------------------------------
// CUDA IPC for the sequence-shard tables (peer GPUs' shards over NVLink)
// ---------------------------------------------------------------------------
static_assert(sizeof(cudaIpcMemHandle_t) == DA_IPC_HANDLE_BYTES, "IPC handle size");

// cuMemGetAddressRange through the runtime's driver entry point (no libcuda link)
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

int da_ipc_export(const void* dev_ptr, void* handle, int64_t* offset) {
  if (!dev_ptr || !handle || !offset) return fail(DA_EINVAL, "ipc_export: null argument");
  static AddrRangeFn range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return fail(DA_ECUDA, "ipc_export: cuMemGetAddressRange unavailable");
    range = reinterpret_cast<AddrRangeFn>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(DA_EINVAL, "ipc_export: not a device allocation");
  cudaIpcMemHandle_t h;
  if (int rc = cuda_status(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "ipc_export")) return rc;
  memcpy(handle, &h, sizeof(h));
  *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return DA_OK;
}

int da_ipc_open(const void* handle, int64_t offset, void** dev_ptr) {
  if (!handle || !dev_ptr || offset < 0) return fail(DA_EINVAL, "ipc_open: bad argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  if (int rc = cuda_status(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "ipc_open")) return rc;
  *dev_ptr = static_cast<char*>(base) + offset;
  return DA_OK;
}

int da_ipc_close(void* dev_ptr, int64_t offset) {
  if (!dev_ptr || offset < 0) return fail(DA_EINVAL, "ipc_close: bad argument");
  return cuda_status(cudaIpcCloseMemHandle(static_cast<char*>(dev_ptr) - offset), "ipc_close");
}

int da_debug_trace(void* device_buffer) {
  da::set_tc_trace(device_buffer);
  return DA_OK;
}

const char* da_last_error(void) { return g_err.c_str(); }

int32_t da_num_regions(const da_grid* grid) {
  if (!grid_ok(grid)) return -1;
  return da::make_geo(*grid).g;
}

int32_t da_region_size(const da_grid* grid) {
  if (!grid_ok(grid)) return -1;
  return grid->patch_h * grid->patch_w;
}

int64_t da_padded_tokens(const da_grid* grid) {
  if (!grid_ok(grid)) return -1;
  return da::make_geo(*grid).n_pad;
}

int64_t da_mask_capacity(int32_t g, int64_t m) { return m + g; }

int da_permute_in(const void* x, int64_t head_stride, int64_t row_stride, void* x_r, int32_t heads, int32_t d,
                  const da_grid* grid, void* stream) {
  if (!grid_ok(grid)) return fail(DA_EINVAL, "all grid dimensions must be positive");
  if (!x || !x_r || heads < 1 || d < 8 || d % 8) return fail(DA_EINVAL, "permute_in: need d %% 8 == 0, heads >= 1");
  if (head_stride % 8 || row_stride % 8 || (reinterpret_cast<uintptr_t>(x) & 15) ||
      (reinterpret_cast<uintptr_t>(x_r) & 15))
    return fail(DA_EINVAL, "permute_in: 16-byte aligned rows required");
  da::Geo g = da::make_geo(*grid);
  return cuda_status(da::launch_permute_in(x, head_stride, row_stride, x_r, heads, d, g, (cudaStream_t)stream),
                     "permute_in");
}

int da_permute_out(const void* o_r, void* out, int64_t head_stride, int64_t row_stride, int32_t heads, int32_t d,
                   const da_grid* grid, void* stream) {
  if (!grid_ok(grid)) return fail(DA_EINVAL, "all grid dimensions must be positive");
  if (!o_r || !out || heads < 1 || d < 8 || d % 8) return fail(DA_EINVAL, "permute_out: need d %% 8 == 0");
  if (head_stride % 8 || row_stride % 8 || (reinterpret_cast<uintptr_t>(out) & 15) ||
      (reinterpret_cast<uintptr_t>(o_r) & 15))
    return fail(DA_EINVAL, "permute_out: 16-byte aligned rows required");
  da::Geo g = da::make_geo(*grid);
  return cuda_status(da::launch_permute_out(o_r, out, head_stride, row_stride, heads, d, g, (cudaStream_t)stream),
                     "permute_out");
}

int da_pool(const void* x, int64_t head_stride, int64_t row_stride, double* pooled, int32_t heads, int32_t d,
            const da_grid* grid, int32_t mode, void* stream) {
  if (!grid_ok(grid)) return fail(DA_EINVAL, "all grid dimensions must be positive");
  if (!x || !pooled || heads < 1 || d < 8 || d % 8 || d > 2048) return fail(DA_EINVAL, "pool: need d %% 8 == 0");
  if (mode != 0 && mode != 1) return fail(DA_EINVAL, "pool mode must be 0 (average) or 1 (max)");
  if (mode == 1 && (grid->height % grid->patch_h || grid->width % grid->patch_w))
    return fail(DA_EINVAL, "padded grids support average pooling only");
  if (head_stride % 8 || row_stride % 8 || (reinterpret_cast<uintptr_t>(x) & 15))
    return fail(DA_EINVAL, "pool: 16-byte aligned rows required");
  da::Geo g = da::make_geo(*grid);
  return cuda_status(da::launch_pool(x, head_stride, row_stride, pooled, heads, d, mode, g, (cudaStream_t)stream),
                     "pool");
}

int da_draft_scores(const double* qp, const double* kp, double* scores, int32_t heads, int32_t g, int32_t d,
                    double scale, int32_t softmax, void* stream) {
  if (!qp || !kp || !scores || heads < 1 || g < 1 || d < 1) return fail(DA_EINVAL, "draft_scores: bad arguments");
  return cuda_status(da::launch_draft_scores(qp, kp, scores, heads, g, d, scale, softmax, (cudaStream_t)stream),
                     "draft_scores");
}

size_t da_select_workspace_size(int32_t heads, int32_t g) {
  if (heads < 1 || g < 1) return 0;
  return da::select_workspace_size(heads, g);
}

int da_select(const double* scores, int32_t heads, int32_t g, int64_t m, int32_t force_row_keep,
              const uint8_t* dead_cols, void* workspace, int32_t* row_ptr, int32_t* col_idx, uint8_t* bitmap,
              double* threshold, int64_t* forced, int64_t* kept, void* stream) {
  if (!scores || !workspace || !row_ptr || !col_idx || !threshold || !forced || !kept)
    return fail(DA_EINVAL, "select: null buffer");
  if (heads < 1 || g < 1 || (int64_t)g * g > 0x7fffffffLL) return fail(DA_EINVAL, "select: bad g");
  if (m < 1 || m > (int64_t)g * g) return fail(DA_EINVAL, "select: m must be in [1, g*g]");
  return cuda_status(da::launch_select(scores, heads, g, m, force_row_keep, dead_cols, workspace, row_ptr, col_idx,
                                       bitmap, threshold, forced, kept, da_mask_capacity(g, m),
                                       (cudaStream_t)stream),
                     "select");
}

// Sequence shards: 2..DA_MAX_SHARDS non-null, 16-byte aligned buffers whose
// row blocks cover exactly the grid's real tokens (every shard non-empty).
static int check_shards(const da_attn_args& a, const da_grid* grid, const char* what) {
  if (a.shard_count <= 1) return DA_OK;
  if (a.layout != DA_LAYOUT_ORIGINAL) return fail(DA_EINVAL, "%s: sequence shards need the original layout", what);
  if (a.shard_count > DA_MAX_SHARDS) return fail(DA_EINVAL, "%s: at most %d shards", what, DA_MAX_SHARDS);
  const long long n = (long long)grid->frames * grid->height * grid->width;
  if (a.shard_rows < 1 || a.shard_rows >= (1ll << 31) || (long long)(a.shard_count - 1) * a.shard_rows >= n ||
      (long long)a.shard_count * a.shard_rows < n)
    return fail(DA_EINVAL, "%s: %d shards of %lld rows do not cover %lld tokens", what, a.shard_count,
                (long long)a.shard_rows, n);
  for (int s = 0; s < a.shard_count; ++s) {
    const void* ptrs[4] = {a.q_shards[s], a.k_shards[s], a.v_shards[s], a.out_shards[s]};
    for (const void* ptr : ptrs)
      if (!ptr || (reinterpret_cast<uintptr_t>(ptr) & 15))
        return fail(DA_EINVAL, "%s: shard %d has a null or unaligned buffer", what, s);
  }
  return DA_OK;
}

// Point q/k/v/out at shard 0 when sharded (the plain pointers are unused then;
// this keeps the null / alignment checks meaningful).
static da_attn_args with_shard_bases(const da_attn_args& a) {
  da_attn_args b = a;
  if (a.layout == DA_LAYOUT_ORIGINAL && a.shard_count > 1) {
    b.q = a.q_shards[0]; b.k = a.k_shards[0]; b.v = a.v_shards[0]; b.out = a.out_shards[0];
  }
  return b;
}

static int check_attn(const da_attn_args* a, const da_grid* grid) {
  if (!a || !grid_ok(grid)) return fail(DA_EINVAL, "block_sparse_fwd: bad arguments");
  if (int rc = check_shards(*a, grid, "block_sparse_fwd")) return rc;
  if (!a->q || !a->k || !a->v || !a->out || !a->row_ptr || !a->col_idx)
    return fail(DA_EINVAL, "block_sparse_fwd: null buffer");
  if (a->heads < 1 || a->d < 1 || a->dv < 1) return fail(DA_EINVAL, "block_sparse_fwd: bad sizes");
  if (a->layout != DA_LAYOUT_REORDERED && a->layout != DA_LAYOUT_ORIGINAL)
    return fail(DA_EINVAL, "block_sparse_fwd: unknown layout");
  if (a->layout == DA_LAYOUT_ORIGINAL && a->key_valid)
    return fail(DA_EINVAL, "block_sparse_fwd: key_valid requires the reordered layout");
  return DA_OK;
}

size_t da_attn_workspace_size(int32_t heads, const da_grid* grid) {
  if (!grid_ok(grid) || heads < 1) return 0;
  return da::attn_workspace_size(heads, da::make_geo(*grid));
}

static int block_sparse_fwd_impl(const da_attn_args* args, const da_grid* grid, void* stream, const float* kpart,
                                 int kblk, bool tiles_ready);

int da_block_sparse_fwd(const da_attn_args* args, const da_grid* grid, void* stream) {
  if (!args) return fail(DA_EINVAL, "block_sparse_fwd: bad arguments");
  const da_attn_args a = with_shard_bases(*args);
  return block_sparse_fwd_impl(&a, grid, stream, nullptr, 0, false);
}

static int block_sparse_fwd_impl(const da_attn_args* args, const da_grid* grid, void* stream, const float* kpart,
                                 int kblk, bool tiles_ready) {
  int rc = check_attn(args, grid);
  if (rc) return rc;
  da::Geo g = da::make_geo(*grid);
  cudaStream_t st = (cudaStream_t)stream;
  if (!args->force_portable && da::tc_supported(*args, g)) {
    if (!args->workspace)
      return fail(DA_EINVAL, "block_sparse_fwd: the tcgen05 path needs a workspace (da_attn_workspace_size)");
    return cuda_status(da::launch_tc_attn(*args, g, st, kpart, kblk, tiles_ready), "block_sparse_fwd (tcgen05)");
  }
  if (da::portable_smem_bytes(g.p, args->d, args->dv) > 227 * 1024)
    return fail(DA_EINVAL, "block_sparse_fwd: region size %d with d=%d, dv=%d exceeds the portable kernel's "
                           "shared-memory tile", g.p, args->d, args->dv);
  return cuda_status(da::launch_portable_attn(*args, g, st), "block_sparse_fwd (portable)");
}

// ---------------------------------------------------------------------------
// whole pipeline
// ---------------------------------------------------------------------------
struct PipeWs {
  double* qp;
  double* kp;
  double* scores;
  void* sel;
  void* attn;
  void* sel32;
  float* kpart;
  unsigned long long* pnorm;  // [heads][2] pooled row norm^2 maxima (pooling pass -> fp32 selection)
  size_t total;
};

static PipeWs carve(void* base, const da::Geo& g, int heads, int d) {
  PipeWs w;
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) { char* r = p ? p + off : nullptr; off += align256(bytes); return r; };
  w.qp = reinterpret_cast<double*>(take(sizeof(double) * (size_t)heads * g.g * d));
  w.kp = reinterpret_cast<double*>(take(sizeof(double) * (size_t)heads * g.g * d));
  // fp64 scores, or the fp32 planes of the guard-band path (per-head stride g * g rounded up to 4)
  w.scores = reinterpret_cast<double*>(take(sizeof(double) * (size_t)heads * ((size_t)g.g * g.g + 2)));
  w.sel = take(da::select_workspace_size(heads, g.g));
  w.attn = take(da::attn_workspace_size(heads, g));
  w.sel32 = take(da::select32_workspace_size(heads, g.g, d));
  w.kpart = reinterpret_cast<float*>(take(sizeof(float) * (size_t)heads * (da::pool_norm_blocks(d, g) + 1)));
  w.pnorm = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * 2 * (size_t)heads));
  w.total = off;
  return w;
}

__global__ void head_mean_kernel(const double* __restrict__ scores, double* __restrict__ out, int heads,
                                 long long n) {
  // basis_sum = basis_0 + basis_1 + ... (left fold), then / heads (sparse.py:296-297)
  long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double s = scores[e];
  for (int h = 1; h < heads; ++h) s = s + scores[(long long)h * n + e];
  out[e] = s / (double)heads;
}

int64_t da_pipeline_fallback_offset(const da_grid* grid, int32_t heads, int32_t d) {
  if (!grid_ok(grid) || heads < 1 || d < 1) return -1;
  da::Geo g = da::make_geo(*grid);
  // carve a notional workspace at a non-null base (a null base carves to null pointers)
  char* const base = reinterpret_cast<char*>(uintptr_t(1) << 20);
  const PipeWs w = carve(base, g, heads, d);
  const char* flag = reinterpret_cast<const char*>(da::select32_fallback_flag(w.sel32, heads, g.g));
  return (int64_t)(flag - base);
}

size_t da_pipeline_workspace_size(const da_grid* grid, int32_t heads, int32_t d) {
  if (!grid_ok(grid) || heads < 1 || d < 1) return 0;
  da::Geo g = da::make_geo(*grid);
  // + one extra g x g buffer for the shared-head mean
  return carve(nullptr, g, heads, d).total + align256(sizeof(double) * (size_t)g.g * g.g);
}

int32_t da_pipeline_launches(int32_t select_softmax, int32_t shared_head_mask) {
  // pool (Q and K), draft GEMM (+ row softmax) [+ head mean], selection: init,
  // digit histograms (digit 0 fused into the GEMM on the per-head logits path)
  // and scans, candidate compaction + finish, tie counts + scan, mark, row
  // scan, collect, threshold, kept totals, packbits (bitmap requested);
  // attention: region order, tcgen05 kernel, fallback list (key norms come from pooling)
  // (per-head logits path, average pooling: the fp32 guard-band selection — init, operand pack, GEMM,
  // 1 digit histogram + 2 scans, mark, band rescoring + finish, force, row scan, collect,
  // kept totals, packbits — followed by the gated fp64 launches, which exit
  // at once unless the fp32 path flagged a fallback)
  const int fused = (!select_softmax && !shared_head_mask) ? 1 : 0;
  const int fp64_path = 1 + (select_softmax ? 1 : 0) + (shared_head_mask ? 1 : 0) + 1 + (6 - fused) + 6 + 2 + 7 + 1;
  return 1 + (fused ? 14 : 0) + fp64_path + 3;  // + region order, tcgen05 kernel, fallback list (tiles come from pooling)
}

int da_sparse_attention(const da_pipeline_args* pa, const da_grid* grid, void* stream) {
  if (!pa || !grid_ok(grid)) return fail(DA_EINVAL, "sparse_attention: bad arguments");
  const da_attn_args a = with_shard_bases(pa->attn);
  if (a.layout != DA_LAYOUT_ORIGINAL) return fail(DA_EINVAL, "sparse_attention: inputs must be in original order");
  if (int rc = check_shards(a, grid, "sparse_attention")) return rc;
  if (!pa->workspace || !pa->row_ptr || !pa->col_idx || !pa->threshold || !pa->forced || !pa->kept)
    return fail(DA_EINVAL, "sparse_attention: null buffer");
  const bool divisible = grid->height % grid->patch_h == 0 && grid->width % grid->patch_w == 0;
  if (pa->pool_mode == 1 && !divisible) return fail(DA_EINVAL, "padded grids support average pooling only");
  da::Geo g = da::make_geo(*grid);
  if (pa->m < 1 || pa->m > (int64_t)g.g * g.g) return fail(DA_EINVAL, "sparse_attention: m out of range");
  cudaStream_t st = (cudaStream_t)stream;
  PipeWs w = carve(pa->workspace, g, a.heads, a.d);
  int rc;
  if (a.d % 8 || a.d > 2048 || a.q_head_stride % 8 || a.q_row_stride % 8 || a.k_head_stride % 8 ||
      a.k_row_stride % 8 || (reinterpret_cast<uintptr_t>(a.q) & 15) || (reinterpret_cast<uintptr_t>(a.k) & 15))
    return fail(DA_EINVAL, "sparse_attention: q/k need d %% 8 == 0 and 16-byte aligned rows");
  // K2: pool Q and K in one launch
  // (average pooling also records K's row-norm maxima for the attention kernel)
  // (and, on the tcgen05 shape, writes K and V as the attention kernel's region tiles)
  const int kblk = pa->pool_mode == 0 ? da::pool_norm_blocks(a.d, g) : 0;
  // (64-token regions, or 64 x 2^s-token ones as K4's column-part tiles)
  const bool tiles = kblk > 0 && a.d == 128 && a.dv == 128 && da::region_parts_shift(g) >= 0 &&
                     a.v_row_stride % 8 == 0 && (reinterpret_cast<uintptr_t>(a.v) & 15) == 0 &&
                     da::tc_supported(a, g) && !a.force_portable;
  // (the averaging kernel also records the pooled rows' largest norms for the fp32 selection)
  if (kblk > 0) cudaMemsetAsync(w.pnorm, 0, sizeof(unsigned long long) * 2 * a.heads, st);
  const da::Shards shards = da::make_shards(a);
  if ((rc = cuda_status(da::launch_pool2(a.q, a.q_head_stride, a.q_row_stride, w.qp, a.k, a.k_head_stride,
                                         a.k_row_stride, w.kp, a.heads, a.d, pa->pool_mode, g, st,
                                         kblk > 0 ? w.kpart : nullptr, tiles ? a.v : nullptr, a.v_head_stride,
                                         a.v_row_stride, tiles ? da::attn_tiles(w.attn, a.heads, g, 0) : nullptr,
                                         tiles ? da::attn_tiles(w.attn, a.heads, g, 1) : nullptr,
                                         kblk > 0 ? w.pnorm : nullptr, &shards),
                        "pool")))
    return rc;
  // K3: per-head selection on raw logits (the default) runs on fp32 draft
  // scores with an exact fp64 guard band (launch_select32); the fp64 GEMM and
  // radix selection below then only run (gated on the device) if that path
  // flags non-finite inputs or an oversized band. softmax selection and the
  // shared-head mask always take the fp64 path.
  const bool fuse_digit0 = !pa->select_softmax && !pa->shared_head_mask;
  const int* gate = nullptr;
  if (fuse_digit0) {
    if ((rc = cuda_status(da::launch_select32(w.qp, w.kp, reinterpret_cast<float*>(w.scores), a.heads, g.g, a.d,
                                              a.scale, pa->m, pa->force_row_keep, w.sel32, pa->row_ptr, pa->col_idx,
                                              pa->bitmap, pa->threshold, pa->forced, pa->kept,
                                              da_mask_capacity(g.g, pa->m), st, kblk > 0 ? w.pnorm : nullptr),
                          "select32")))
      return rc;
    gate = da::select32_fallback_flag(w.sel32, a.heads, g.g);
  }
  // fp64 draft scores; on the per-head logits path the GEMM epilogue also
  // histograms digit 0 of the selection keys
  if (fuse_digit0) da::select_init(w.sel, a.heads, g.g, pa->m, st, gate);
  if ((rc = cuda_status(da::launch_draft_scores(w.qp, w.kp, w.scores, a.heads, g.g, a.d, a.scale, pa->select_softmax,
                                                st, fuse_digit0 ? da::select_hist_buffer(w.sel, a.heads, g.g) : nullptr,
                                                gate),
                        "draft_scores")))
    return rc;
  const double* sel_scores = w.scores;
  int sel_heads = a.heads;
  if (pa->shared_head_mask) {
    double* mean = reinterpret_cast<double*>(static_cast<char*>(pa->workspace) + w.total);
    long long n = (long long)g.g * g.g;
    head_mean_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w.scores, mean, a.heads, n);
    if ((rc = cuda_status(cudaGetLastError(), "head_mean"))) return rc;
    sel_scores = mean;
    sel_heads = 1;
  }
  // a padded grid never has an all-padding region (the last patch of each axis
  // starts inside the real extent), so no dead columns (padding.py:151-153)
  if ((rc = cuda_status(da::launch_select(sel_scores, sel_heads, g.g, pa->m, pa->force_row_keep, nullptr, w.sel,
                                          pa->row_ptr, pa->col_idx, pa->bitmap, pa->threshold, pa->forced, pa->kept,
                                          da_mask_capacity(g.g, pa->m), st, fuse_digit0, gate),
                        "select")))
    return rc;
  da_attn_args aa = a;
  aa.row_ptr = pa->row_ptr;
  aa.col_idx = pa->col_idx;
  aa.mask_cap = da_mask_capacity(g.g, pa->m);
  aa.key_valid = nullptr;
  aa.shared_mask = pa->shared_head_mask ? 1 : 0;
  aa.workspace = w.attn;
  if (pa->ev_attn_begin) cudaEventRecord((cudaEvent_t)pa->ev_attn_begin, st);
  rc = block_sparse_fwd_impl(&aa, grid, stream, kblk > 0 ? w.kpart : nullptr, kblk, tiles);
  if (pa->ev_attn_end) cudaEventRecord((cudaEvent_t)pa->ev_attn_end, st);
  return rc;
}

}  // extern "C"
