/* icarus_b200.h -- C ABI of the B200-native ICaRus multi-model decode hot path.
 *
 * The reference (arxiv 2603.13281, `icarus` numpy package) has no FFI: its hot path is
 * the Python module API below. Each entry point names the reference function it replaces
 * (paths relative to /root/reference/pkg/src/icarus/). The Python shim
 * paper_2603_13281_b200/_lib.py binds these with ctypes and re-exposes the reference's
 * names, argument meaning and exception classes.
 *
 * Conventions
 *  - Plain pointers + sizes only. "dev" pointers are CUDA device pointers owned by the
 *    caller (torch tensors on the Python side); "host" pointers are host memory.
 *  - Every call is asynchronous on the given stream unless documented otherwise.
 *  - Status codes map 1:1 onto the reference's exception classes (errors.py:8-38):
 *      ICR_OK 0, ICR_SHAPE 1 (ShapeError), ICR_CONFIG 2 (ConfigError), ICR_MODE 3
 *      (ModeError), ICR_STATE 4 (StateError), ICR_CAPACITY 5 (CapacityError),
 *      ICR_CONTRACT 6 (ContractViolationError), ICR_CUDA 7 (device error), ICR_INDEX 8
 *      (IndexError: token id outside the vocabulary, engine.py:66-72).
 *  - icr_last_error() returns a thread-local message for the last non-zero status.
 */
#ifndef ICARUS_B200_H
#define ICARUS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int icr_status;
enum {
  ICR_OK = 0,
  ICR_SHAPE = 1,
  ICR_CONFIG = 2,
  ICR_MODE = 3,
  ICR_STATE = 4,
  ICR_CAPACITY = 5,
  ICR_CONTRACT = 6,
  ICR_CUDA = 7,
  ICR_INDEX = 8
};

typedef struct icr_model icr_model; /* opaque */

/* Shape constants: ModelConfig (model.py:36-85) plus the device-side capacities. */
typedef struct icr_model_config {
  int num_layers, hidden_dim, num_heads, num_kv_heads, head_dim, ffn_dim, vocab_size;
  float rms_eps;
  double rope_theta;
  int max_positions;     /* RoPE table rows; >= max context                        */
  int num_pages;         /* KV page arena capacity (16 tokens per page = BLOCK_TOKENS) */
  int max_seqs;          /* block-table rows                                      */
  int max_pages_per_seq; /* block-table columns                                   */
  int max_rows;          /* token rows per forward call (encoder + decoder)      */
  int adapter_slots;     /* resident LoRA adapters                                */
  int lora_rank;         /* rank r of every resident adapter (0 = no adapters)    */
  int chunk_pages;       /* attention chunk length in pages (fixed per model)     */
} icr_model_config;

/* Device weights of one layer. Layouts are the transpose of the reference's [in, out]
 * (model.py:10-14) so every GEMM operand is K-major; RMSNorm gains are folded in.
 *   w_qkv  [q_dim + 2*kv_dim, d]  rows: wq^T | wk^T | wv^T          (attn_gain folded)
 *   w_o    [d, q_dim]
 *   w_gu   [2*ffn, d]             rows interleaved gate_0, up_0, gate_1, up_1 ...  (ffn_gain)
 *   w_down [d, ffn]
 * LoRA (AdapterSet, model.py:180-256; only DECODER_TARGETS q, o, gate, up, down):
 *   a_*    [slots][r][in]         the reference's A exactly ([rank, in_dim])
 *   b_q    [slots][q_dim][r]      reference B ([out_dim, rank])
 *   b_o    [slots][d][r]
 *   b_gu   [slots][2*ffn][r]      gate/up rows interleaved like w_gu
 *   b_down [slots][d][r]
 * KV pages (this layer): k_pages, v_pages [num_pages][num_kv_heads][16][head_dim].
 * All bf16. The four projection matrices and lm_head are stored TILE-MAJOR: the [M, K]
 * matrix above is laid out as [M/128][K/64][128][64] so every 128x64 GEMM tile is one
 * contiguous 16 KB block (runtime.py: tile_major). The reference has no slot for k/v
 * adapters: there is none here either. */
typedef struct icr_layer_weights {
  const void* w_qkv;
  const void* w_o;
  const void* w_gu;
  const void* w_down;
  const void* a_q;
  const void* b_q;
  const void* a_o;
  const void* b_o;
  const void* a_gate;
  const void* a_up;
  const void* b_gu;
  const void* a_down;
  const void* b_down;
  void* k_pages;
  void* v_pages;
} icr_layer_weights;

/* Replaces BaseWeights/AdapterSet residency (model.py:88-256): binds device weights,
 * builds TMA descriptors, allocates scratch sized by cfg->max_rows.
 * embed [vocab, d] bf16; lm_head [ceil(vocab/128)*128, d] bf16 tile-major, final_gain folded,
 * zero rows past vocab. lora_scaling is
 * AdapterSet.scaling = alpha / rank (model.py:220-222), identical for all slots. */
icr_status icr_model_create(const icr_model_config* cfg, const icr_layer_weights* layers,
                            const void* embed, const void* lm_head, float lora_scaling,
                            icr_model** out);
icr_status icr_model_destroy(icr_model* m);

/* One batch of token rows for a forward pass. A decode step of N adapted sessions is
 * 2N rows -- the fused pair of decode_step_fused (engine.py:179-193) per session:
 * an encoder row (kind 0, base weights, writes K/V) and a decoder row (kind 1,
 * base + LoRA of `row_adapter`, reads K/V). A prefill (engine.py:84-153) is S encoder rows.
 * Rows may share sequences; sequences may share pages (cross-model prefix cache). */
typedef struct icr_batch {
  int n_rows;
  const int32_t* tokens;      /* host [n_rows]                                         */
  const int32_t* row_kind;    /* host [n_rows] 0 encoder, 1 decoder                    */
  const int32_t* row_seq;     /* host [n_rows] block-table row                         */
  const int32_t* row_pos;     /* host [n_rows] absolute position                       */
  const int32_t* row_adapter; /* host [n_rows] adapter slot for decoder rows, else -1  */
  const int32_t* row_emit;    /* host [n_rows] 1 = run the LM head + argmax on this row (and
                                 keep its final hidden for icr_seq_logits), 2 = the same
                                 without keeping it, 0 = no LM head                       */
  const int32_t* block_table; /* host [max_seqs][max_pages_per_seq] page ids           */
  int n_seqs;                 /* block-table rows referenced                           */
} icr_batch;

/* One forward pass over the batch: L fused layers (model.py:441-506) + final norm +
 * LM head + greedy argmax (engine.py:75-81). Writes, for the i-th row with
 * row_emit != 0, the argmax token to out_tokens_host[i] and (if logits_dev != NULL) the
 * fp32 logits to logits_dev[i * vocab_pad ...]. Synchronises the stream before return. */
icr_status icr_forward(icr_model* m, const icr_batch* b, int32_t* out_tokens_host,
                       float* logits_dev, void* stream);

/* Device-resident decode loop for throughput measurement: runs `steps` forward passes of
 * the same row layout, position += 1 per step, feeding each sequence's decoder-row
 * output (feedback_src[r] = index of the emitting row whose token row r consumes next)
 * back on the device. Pages for every step must already be in block_table. Per-step
 * device times are written to step_ms_host (may be NULL). Synchronises at the end. */
icr_status icr_decode_loop(icr_model* m, const icr_batch* first, const int32_t* feedback_src,
                           int steps, int32_t* out_tokens_host_last, float* step_ms_host,
                           void* stream);

/* --- instrumentation ------------------------------------------------------------- */

/* out3 = {kernel launches, metadata bytes uploaded, attention work items} of the last
 * icr_forward / icr_decode_loop step. */
icr_status icr_model_stats(icr_model* m, int64_t* out3);

/* Invariant check of the GEMM's split-tile exchange: *out = the number of stream-K scratch
 * words of the model that do not hold the "unpublished" pattern (0 after every completed
 * forward: each published partial is consumed and re-armed by its tile's finalizer).
 * Synchronises the stream. */
icr_status icr_debug_ws_check(icr_model* m, int64_t* out, void* stream);

/* Per-kernel-kind device time of the last forward, replayed without the graph with an
 * event after every launch: kind_ms[0..8] = embed, qkv, attention, o, gate|up, down,
 * LM gather, LM head, argmax; kind_ms[9] = total (ms). Recomputes identical K/V. */
icr_status icr_profile_step(icr_model* m, float* kind_ms, void* stream);

/* Average device time of one projection-GEMM launch (which: 0 wo, 1 gate|up, 2 down,
 * 3 lm_head) re-run `iters` times over all layers with the last forward's rows. */
icr_status icr_profile_gemm(icr_model* m, int which, int iters, float* avg_ms, void* stream);
/* Diagnostic: average ms of the last forward replayed as a graph with kernel kinds
 * (bit k = kind k of icr_profile_step) left out. */
icr_status icr_profile_ablate(icr_model* m, int skip_mask, int iters, float* avg_ms, void* stream);
/* Instrumentation: host time split of icr_forward calls [calls, prep us, launch us, wait us]. */
icr_status icr_host_timing(double* out4, int reset);
/* Diagnostic: per-CTA timestamps of every GEMM launch of the last forward -> CSV. */
icr_status icr_profile_trace(icr_model* m, const char* path, void* stream);

/* Weight-streaming GEMM micro-benchmark (tuning): cycles n_mats matrices [n_mats][M][K]
 * (tile-major if blocked) against `rows` token rows; stages / ctas_per_sm / skip_mma
 * override the ring depth, CTAs per SM and bypass tcgen05.mma (0 = defaults). */
icr_status icr_bench_gemm(const void* w, const void* x, int M, int K, int rows, int n_mats,
                          int blocked, int stages, int ctas_per_sm, int skip_mma, int iters,
                          float* avg_ms, void* stream);

/* Paged-attention micro-benchmark (C4 sweep): plan once, time `iters` launches of the
 * partial + merge kernels (a read of flush_dev between launches evicts L2 when non-NULL).
 * alt_page_offset > 0: pipelined mode -- `iters` launches back to back (PDL, no flush), odd
 * launches reading the same plan with every page id + alt_page_offset (a second copy of the
 * K/V, so no launch finds its pages in L2); avg_ms = total / iters. span_us (may be NULL):
 * cold mode's average device span of the kernels themselves -- first partial CTA start to
 * last partial / merge CTA end by %globaltimer, i.e. without the event/launch overhead. */
icr_status icr_bench_attention(const void* q_dev, const void* k_pages, const void* v_pages,
                               int num_heads, int num_kv_heads, int head_dim, int chunk_pages,
                               int n_rows, const int32_t* row_seq_host, const int32_t* row_pos_host,
                               const int32_t* block_table_host, int n_seqs, int max_pages_per_seq,
                               void* out_dev, void* flush_dev, long long flush_bytes, int iters,
                               int alt_page_offset, float* avg_ms, int32_t* n_items_out,
                               float* span_us, void* stream);

/* --- building blocks, exported for parity tests -------------------------------- */

/* out_f32[n, m] = sum_k W[m, k] X[n, k]; W [M, K] bf16 (dev), X [n_rows, K] bf16 (dev).
 * M % 128 == 0, K % 64 == 0. The tcgen05 stream-K kernel behind every projection. */
icr_status icr_gemm_bf16(const void* w_dev, const void* x_dev, float* out_dev, int M, int K,
                         int n_rows, void* stream);

/* Paged attention for explicit rows (layer_attention, model.py:384-425):
 * q [n_rows][num_heads*hd] bf16, out [n_rows][num_heads*hd] bf16, pages as above. */
icr_status icr_paged_attention(const void* q_dev, const void* k_pages, const void* v_pages,
                               int num_heads, int num_kv_heads, int head_dim, int chunk_pages,
                               int n_rows, const int32_t* row_seq_host,
                               const int32_t* row_pos_host, const int32_t* block_table_host,
                               int n_seqs, int max_pages_per_seq, void* out_dev,
                               int32_t* n_items_out, void* stream);

/* --- the reference's module-level model functions (model.py:334-538) ------------- */

/* One transformer layer of the hot path (block_forward, model.py:441-506, and
 * decoder_block_readonly, :511-538) over explicit fp32 input rows x_in_dev [n_rows][d]
 * (device), writing the layer output rows to x_out_dev [n_rows][d]. Rows as in icr_batch
 * (tokens are ignored; row_emit must be 0): prefill = S encoder rows, fused decode = an
 * encoder row + a decoder row, read-only decoder pass = one decoder row. Encoder rows write
 * their K/V into this layer's pages. The same kernels, in the same order, as icr_forward's
 * layer `layer`. Synchronises the stream. */
icr_status icr_layer_forward(icr_model* m, const icr_batch* b, int layer, const float* x_in_dev,
                             float* x_out_dev, void* stream);

/* session.last_logits (engine.py:190-192) on demand: fp32 logits [n][vocab_pad] of the final
 * hidden states kept by the last forward that emitted them -- store slot 2*seq + kind
 * (kind 0 encoder row, 1 decoder row) holds the last row of that sequence and kind with
 * row_emit == 1 (row_emit == 2 emits without replacing the stored hidden). Bitwise equal to
 * the logits icr_forward writes when given logits_dev. Synchronises the stream. */
icr_status icr_seq_logits(icr_model* m, const int32_t* slots_host, int n, float* logits_dev,
                          void* stream);

/* base_linear / adapted_linear / icarus_linear (model.py:334-371) for arbitrary weights:
 * out_dev[n][m] = sum_k W[m][k] x[n][k], plus on rows with row_adapted_host[n] != 0 the
 * low-rank term sum_j (x[n] . A[j]) * Bs[m][j] (LoRA shrink + expand inside the same tcgen05
 * GEMM, as in the decode step). W [M][K] bf16 row-major (dev), x [n_rows][K] bf16 (dev),
 * A [rank][K] bf16 (dev), Bs = scaling * B stored tile-major [M/128][1][128][64] bf16 (dev,
 * columns >= rank zero). M % 128 == 0, K % 64 == 0, rank <= 32 (0 = no low-rank term).
 * Synchronises the stream. */
icr_status icr_linear_bf16(const void* w_dev, const void* x_dev, float* out_dev, int M, int K,
                           int n_rows, const void* a_dev, const void* bs_blocked_dev, int rank,
                           const int32_t* row_adapted_host, void* stream);

const char* icr_last_error(void);
int icr_abi_version(void);
int icr_num_sms(void);

#ifdef __cplusplus
}
#endif
#endif /* ICARUS_B200_H */
