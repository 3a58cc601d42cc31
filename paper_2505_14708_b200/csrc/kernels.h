// Internal launcher declarations (host side) shared by the .cu files.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/draftattn_b200.h"

namespace da {

struct Geo;
struct Shards;

cudaError_t launch_permute_in(const void* x, long long hs, long long rs, void* x_r, int heads, int d, const Geo& g,
                              cudaStream_t st);
cudaError_t launch_permute_out(const void* o_r, void* out, long long hs, long long rs, int heads, int d,
                               const Geo& g, cudaStream_t st);
cudaError_t launch_pool(const void* x, long long hs, long long rs, double* pooled, int heads, int d, int mode,
                        const Geo& g, cudaStream_t st);
// pools two tensors (Q and K) in one launch; kpart (optional, average mode with
// pool_norm_blocks(d, g) > 0) receives per-block maxima of K's row norms,
// [heads][pool_norm_blocks(d, g)]
// x2/ktile/vtile (optional, d = 128 and 8x8 pools): the same pass also writes
// K and V as the attention kernel's region tiles (attn_tiles)
cudaError_t launch_pool2(const void* x0, long long hs0, long long rs0, double* out0, const void* x1, long long hs1,
                         long long rs1, double* out1, int heads, int d, int mode, const Geo& g, cudaStream_t st,
                         float* kpart, const void* x2 = nullptr, long long hs2 = 0, long long rs2 = 0,
                         uint8_t* ktile = nullptr, uint8_t* vtile = nullptr, unsigned long long* pnorm = nullptr,
                         const Shards* sh = nullptr);  // sh: sequence shards of x0 / x1 / x2 (Q / K / V)
// K / V tile buffers inside the attention workspace ([heads][g][16 KB] each),
// in the GROUPED layout of kv_tile_offset_grouped (the K4 shared-memory image)
uint8_t* attn_tiles(void* ws, int heads, const Geo& g, int which);
// The library's K4 for d = 128, 8x8 pools: the transposed TMEM-fed kernel
// (attn_tk.cu; its own tile layouts) or the lane-half kernel (attn_lh.cu).
bool attn_uses_tk();
int pool_norm_blocks(int d, const Geo& g);
// hist0 (optional): per-head 2048-bin histogram of the top 11 key bits, filled in the epilogue
cudaError_t launch_draft_scores(const double* qp, const double* kp, double* scores, int heads, int g, int d,
                                double scale, int softmax, cudaStream_t st, unsigned int* hist0 = nullptr,
                                const int* gate = nullptr);

size_t select_workspace_size(int heads, int g);
long long bitmap_bytes_per_head(int g);
unsigned int* select_hist_buffer(void* ws, int heads, int g);
void select_init(void* ws, int heads, int g, long long m, cudaStream_t st, const int* gate = nullptr);
cudaError_t launch_select(const double* scores, int heads, int g, long long m, int force, const uint8_t* dead,
                          void* ws, int* row_ptr, int* col_idx, uint8_t* bitmap, double* threshold,
                          int64_t* forced, int64_t* kept, long long cap, cudaStream_t st, bool digit0_done = false,
                          const int* gate = nullptr);
// fp32 draft scores + exact fp64 guard-band selection (the pipeline default);
// sets the flag select32_fallback_flag() points to when the fp64 path must run
size_t select32_workspace_size(int heads, int g, int d);
const int* select32_fallback_flag(void* ws, int heads, int g);
// pnorm (optional): [heads][2] largest pooled row norms^2 (double bits) from
// the pooling pass; null = computed here
cudaError_t launch_select32(const double* qp, const double* kp, float* scores32, int heads, int g, int d,
                            double scale, long long m, int force, void* ws, int* row_ptr, int* col_idx,
                            uint8_t* bitmap, double* threshold, int64_t* forced, int64_t* kept, long long cap,
                            cudaStream_t st, const unsigned long long* pnorm = nullptr);

size_t portable_smem_bytes(int p, int d, int dv);
cudaError_t launch_portable_attn(const da_attn_args& args, const Geo& geo, cudaStream_t st);
// regions listed in items[0 .. *count) (entries h * g + i; count read on the device)
cudaError_t launch_portable_list(const da_attn_args& args, const Geo& geo, cudaStream_t st, const int* items,
                                 const int* count, int blocks);
size_t attn_workspace_size(int heads, const Geo& g);

void set_tc_trace(void* buf);
bool tc_supported(const da_attn_args& a, const Geo& g);
// kpart/kblk: per-head key row norm maxima already computed by the pooling
// pass ([heads][kblk]); null = the attention launch computes them itself.
// tiles_ready: the pooling pass already wrote the K/V region tiles.
cudaError_t launch_tc_attn(const da_attn_args& a, const Geo& g, cudaStream_t st, const float* kpart = nullptr,
                           int kblk = 0, bool tiles_ready = false);

namespace k4 {
struct Params;
}
// K4 transposed TMEM-fed kernel (attn_tk.cu), launched by launch_tc_attn
cudaError_t launch_tk_kernel(const k4::Params& p, int grid, cudaStream_t st);

// Per-device facts cached once per device (the library keeps no other state):
// the SM count, and the dynamic shared-memory opt-in of a kernel.
int device_sms();  // of the current device
cudaError_t ensure_smem_optin(const void* kernel, int bytes);

}  // namespace da
