// Weight-streaming GEMM for the multi-model decode step (and prefill), sm_100a.
//
//   D[m, n] = sum_k W[m, k] * X[n, k]      (swap-AB: weight rows on the MMA M axis,
//                                          token rows -- encoder + decoder -- on N)
//
// Reference op: `base_linear` / `icarus_linear` (src/model.py:334-371) whose inner
// product is `_mm` (src/tensor.py:151-156). The reference stores W as [in, out];
// the device copy is [out, in] (K-major) so both MMA operands are K-major.
//
// Design (B200-first):
//  * persistent stream-K over (m_tile, k_chunk) units: grid = #SMs, every CTA gets the
//    same number of 64-wide K chunks (+-1), so all 148 SMs stream weights to the end;
//  * warp-specialised: warp0 = TMA producer, warp1 = tcgen05.mma issuer,
//    warp2 = TMEM allocator, warps4..7 = epilogue (one TMEM lane = one output feature);
//  * TMA 128B-swizzled tiles W[128 x 64] + X[N x 64] into a deep smem ring;
//    accumulator [128 x N] fp32 in TMEM, read back with tcgen05.ld;
//  * split tiles are reduced deterministically: every segment writes its fp32 partial,
//    the last arriving segment sums them in segment order (fixed by (M, K, grid) only,
//    never by N) -- so a token row's result does not depend on batch composition;
//  * fused epilogues: LoRA expand on decoder rows only (SGMV, CUDA cores, B read once),
//    RoPE + paged-KV write (encoder rows only), residual add, SiLU*up, LM-head argmax.
#pragma once
#include "ptx.cuh"

namespace icr {

enum EpiMode : int {
  EPI_F32 = 0,     // out_f32[n, m] = acc                       (tests / debug logits)
  EPI_QKV = 1,     // RoPE(q,k); q -> q_out bf16; k,v of encoder rows -> KV pages
  EPI_RESID = 2,   // resid[n, m] += acc                       (wo, down)
  EPI_SILU = 3,    // rows interleaved (gate_j, up_j): f[n, j] = silu(g) * u
  EPI_ARGMAX = 4,  // per-tile (max, argmax) over m for every row n (LM head)
};

struct GemmParams {
  int mode;
  int M;        // rows of W (multiple of 128)
  int K;        // multiple of 64
  int n_rows;   // valid token rows in this launch (<= N tile)
  int m_valid;  // features >= m_valid are masked (LM head vocab padding)
  // per-row metadata (already offset to this row group)
  const int* row_kind;     // 0 encoder, 1 decoder, <0 padding
  const int* row_adapter;  // adapter slot for decoder rows
  const int* row_pos;      // absolute position
  const int* row_seq;      // sequence slot (block-table row)
  // LoRA expand (decoder rows only): delta[m] = sum_j U[n, uidx, j] * Bs[slot, m, j]
  const __nv_bfloat16* lora_b;  // [slots][lora_m][rank], scaling folded in; null = none
  const float* lora_u;          // [rows][n_u][rank]
  int lora_m;                   // rows of W that carry an adapter (q_dim for qkv)
  int rank;
  int n_u;                      // 1, or 2 for interleaved gate/up
  // outputs
  float* out_f32;               // EPI_F32
  int ld_out;
  float* resid;                 // EPI_RESID, [rows][M]
  __nv_bfloat16* out_bf16;      // EPI_QKV: q [rows][q_dim]; EPI_SILU: f [rows][M/2]
  // EPI_QKV specifics
  int q_dim, kv_dim, head_dim, num_kv_heads;
  const float2* rope;           // [max_pos][head_dim/2] (cos, sin), fp64-derived
  __nv_bfloat16* k_pages;       // [num_pages][H_kv][16][hd] for this layer
  __nv_bfloat16* v_pages;
  const int* block_table;       // [num_seq_slots][max_pages_per_seq]
  int bt_stride;
  // EPI_ARGMAX
  float2* tile_best;            // [m_tiles][rows_total] (value, index-as-float-bits)
  int best_stride;
  // stream-K bookkeeping (scratch, zero-initialised once; counters self-reset)
  float* ws;                    // [m_tiles][max_segs][N][128]
  int* counters;                // [m_tiles]
  int max_segs;
};

}  // namespace icr
