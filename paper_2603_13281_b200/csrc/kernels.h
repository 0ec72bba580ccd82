// Internal kernel launch interface (not part of the public C ABI).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace icr {

struct GemmParams;

// --------------------------------------------------------------- GEMM (gemm.cu)
cudaError_t gemm_launch(const CUtensorMap& tw, const CUtensorMap& tx, const GemmParams& p,
                        int x_row0, int nt, int num_sms, cudaStream_t s);
int gemm_pick_nt(int rows);
size_t gemm_ws_floats(int num_sms);

// --------------------------------------------------------------- attention (attention.cu)
struct AttnItem {
  int chunk_start;  // absolute key position of the chunk's first page
  int n_pages;      // pages to visit
  int page_off;     // into item_pages
  int row_off;      // into item_rows
  int n_rows;       // query rows (<= 64)
  int chunk_idx;    // chunk index c (partial slot)
};

struct AttnLaunch {
  const __nv_bfloat16* q;
  int q_ld;
  const __nv_bfloat16* k_pages;
  const __nv_bfloat16* v_pages;
  int num_kv_heads, num_heads, group, head_dim;
  const AttnItem* items;
  const int* item_pages;
  const int2* item_rows;
  const int* n_items_dev;
  int n_items_cap;
  const int* row_pos;
  const int* row_kind;
  int n_rows;
  int max_chunks, chunk_tokens;
  float scale;
  float* part_o;
  float2* part_ml;
  __nv_bfloat16* out;
  int out_ld;
};
cudaError_t attn_launch(const AttnLaunch& a, cudaStream_t s);

// --------------------------------------------------------------- row ops (rowops.cu)
// x_out[r] = embed[tok[r]] (if embed != null) else x_in; h[r] = bf16(x * rsqrt(mean(x^2)+eps))
cudaError_t rmsnorm_launch(const float* x_in, const int* tokens, const __nv_bfloat16* embed,
                           float* x_out, __nv_bfloat16* h_out, const int* row_kind,
                           const int* row_map, int n_rows, int d, float eps, cudaStream_t s);

// LoRA shrink (SGMV): for each adapter slot a and each row n of segment a,
//   U[n][t][j] = scale * sum_k h[n][k] * A_t[a][j][k]          (t < n_targets <= 2)
cudaError_t lora_shrink_launch(const __nv_bfloat16* h, int ld_h, int K,
                               const __nv_bfloat16* A0, const __nv_bfloat16* A1, int n_targets,
                               int slots, int rank, float scale, const int* seg_off,
                               const int* seg_rows, float* U, cudaStream_t s);

// Final argmax over LM-head tiles (lowest index on ties, src/engine.py:75-76).
cudaError_t argmax_reduce_launch(const float2* tile_best, int tiles, int stride, int n_rows,
                                 int* out_tokens, cudaStream_t s);

}  // namespace icr
