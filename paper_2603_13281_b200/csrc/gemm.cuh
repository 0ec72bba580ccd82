// Weight-streaming GEMM for the multi-model decode step (and prefill), sm_100a.
//
//   D[m, n] = sum_k W[m, k] * X[n, k]      (swap-AB: weight rows on the MMA M axis,
//                                          token rows -- encoder + decoder -- on N)
//
// Reference op: `base_linear` / `icarus_linear` (src/model.py:334-371) whose inner
// product is `_mm` (src/tensor.py:151-156). The reference stores W as [in, out];
// the device copy is [out, in] (K-major), tile-major [M/128][K/64][128][64].
//
// Design (B200-first):
//  * persistent stream-K over (m_tile, k_chunk) units: grid = #SMs, every CTA gets the
//    same number of 64-wide K chunks (+-1), so all 148 SMs stream weights to the end;
//  * warp-specialised: warp0 = TMA producer, warp1 = tcgen05.mma issuer,
//    warp2 = TMEM allocator, warps4..7 = epilogue (one TMEM lane = one output feature);
//  * programmatic dependent launch: the producer streams the first ring of WEIGHT tiles
//    before `griddepcontrol.wait`, i.e. while the previous kernel is still draining --
//    only the activation tiles depend on it;
//  * split tiles are reduced deterministically: the CTA holding a tile's first K segment
//    (its last tile) folds its own TMEM accumulator + the partials the other segments'
//    CTAs published (polled until not WS_EMPTY), in segment order -- fixed by (M, K, grid)
//    only, never by N -- so a token row's result does not depend on batch composition;
//  * two TMEM accumulator buffers: a CTA's tiles alternate, so its last tile accumulates
//    while its first tile's partial is still being published;
//  * RMSNorm folded in: X is bf16(x) (the raw residual stream); the epilogue scales row n
//    by inv_n = 1/sqrt(mean(x_n^2)+eps) from per-128-feature sum-of-squares partials that
//    the residual-producing epilogue wrote (gain folded into W on upload);
//  * LoRA shrink (SGMV, U = x A^T per decoder row) is computed by the otherwise idle warps
//    2-3 of every CTA while the weights stream; the expand (B_cat U) runs as extra tcgen05
//    K-chunks, U being zero on encoder rows;
//  * fused epilogues: RoPE + paged-KV write (encoder rows only), residual add (+ bf16 copy
//    + sum-of-squares partials for the next norm), SiLU*up, LM-head per-tile argmax.
#pragma once
#include "ptx.cuh"

namespace icr {

enum EpiMode : int {
  EPI_F32 = 0,     // out_f32[n, m] = acc                       (tests / debug logits)
  EPI_QKV = 1,     // RoPE(q,k); q -> q_out bf16; k,v of encoder rows -> KV pages
  EPI_RESID = 2,   // x[n, m] += acc; xb = bf16(x); ssq partial of x^2 per 128-feature tile
  EPI_SILU = 3,    // rows interleaved (gate_j, up_j): f[n, j] = silu(g) * u
  EPI_ARGMAX = 4,  // per-tile (max, argmax) over m for every row n (LM head)
};

struct GemmParams {
  int mode;
  int w_blocked;  // 1: W stored tile-major [M/128][K/64][128][64] (3-D tensor map)
  int M;          // rows of W (multiple of 128)
  int K;          // multiple of 64
  int n_rows;     // valid token rows in this launch (<= N tile)
  int row0;       // global index of this launch's first row (row groups of <= 256)
  int rows_total; // padded rows of the whole forward (stride of global-row scratch)
  int m_valid;    // features >= m_valid are masked (LM head vocab padding)
  // per-row metadata, GLOBAL row indexing (this launch reads [row0, row0 + n_rows))
  const int* row_kind;     // 0 encoder, 1 decoder, <0 padding; null = all encoder
  const int* row_adapter;  // adapter slot for decoder rows (-1 = none)
  const int* row_pos;      // absolute position
  const int* row_seq;      // sequence slot (block-table row)
  // RMSNorm of the input rows: inv_n from partial sums of squares [ss_tiles][ss_stride]
  const float* in_ssq;     // null = no scaling
  int ss_tiles, ss_stride;
  float ss_d, eps;         // feature count d (mean = sum / d) and RMSNorm eps
  // LoRA (decoder rows only), SGMV as extra tcgen05 K-chunks: each tile accumulates
  // B_cat[m, :] . Ubd[n, :] over lora_chunks 64-wide chunks, where B_cat concatenates every
  // slot's (alpha/r) * B along K (tile-major like W) and Ubd is block-diagonal: row n holds
  // its adapter's U = X_n A^T in its own slot columns, zeros elsewhere (encoder rows: 0).
  int lora_chunks;              // 0 = no LoRA in this launch
  // in-kernel LoRA shrink (warps 2-3): Ubd[n][t*slots*rank + a*rank + j] = X_sh[n] . A_t[a][j]
  const __nv_bfloat16* sh_x;    // bf16 [rows_total][sh_ld]; null = no shrink
  int sh_ld, sh_K, sh_targets;  // sh_targets 1 or 2
  const __nv_bfloat16* sh_a0;   // [slots][rank][sh_K]
  const __nv_bfloat16* sh_a1;
  int rank;
  const int* seg_off;           // [slots + 1] decoder rows grouped by adapter slot
  const int* seg_rows;          // global row indices
  int slots;
  __nv_bfloat16* ubd;           // block-diagonal U [rows_total][ubd_ld] (bf16, TMA operand)
  int ubd_ld;
  int* sync;                    // shrink-done counter: 2 shrink warps x grid per launch
  int sync_round;               // 1-based launch index within this projection (row groups of
                                // <= 256 share the counter, so launch g waits for g x 2 x grid)
  int* reset_sync;              // counter of an EARLIER launch to zero after griddepcontrol.wait
  float* sh_part;               // [SHRINK_SPLITS][rows_total][2][rank] K-split partials
  int* sh_cnt;                  // [2][slots][rank] split arrivals per adapter row (self-resetting)
  // outputs (GLOBAL row indexing)
  float* out_f32;               // EPI_F32
  int ld_out;
  float* resid;                 // EPI_RESID x [rows_total][M]
  __nv_bfloat16* resid_bf16;    // EPI_RESID bf16 copy of x (next GEMM's X operand)
  float* out_ssq;               // EPI_RESID partial sums of squares [M/128][ss_stride]
  __nv_bfloat16* out_bf16;      // EPI_QKV: q [rows][q_dim]; EPI_SILU: f [rows][M/2]
  // EPI_QKV specifics
  int q_dim, kv_dim, head_dim, num_kv_heads;
  const float2* rope;           // [max_pos][head_dim/2] (cos, sin), fp64-derived
  __nv_bfloat16* k_pages;       // [num_pages][H_kv][16][hd] for this layer
  __nv_bfloat16* v_pages;
  const int* block_table;       // [num_seq_slots][max_pages_per_seq]
  int bt_stride;
  // EPI_ARGMAX
  float2* tile_best;            // [m_tiles][best_stride] (value, index-as-float-bits)
  int best_stride;
  // stream-K bookkeeping: ws = [grid][N/16 chunks][4 float4][128] published partials, each
  // word WS_EMPTY when unpublished (cleared once at allocation, re-armed by the finalizer);
  // counters: unused by the current exchange (kept for the C ABI's scratch layout)
  float* ws;
  int* counters;
  int max_segs;
  // tuning / diagnostics (0 = defaults)
  unsigned long long* trace;  // per-CTA %globaltimer stamps [grid][16] (null = off)
  int stages;     // smem ring depth actually used (<= compiled maximum)
  int preissue_cap;  // weight stages issued before griddepcontrol.wait: 0 all, <0 none, k>0 min(k, ring)
  int skip_mma;   // 1: consume stages without tcgen05.mma (pure TMA streaming rate)
};

}  // namespace icr
