// Internal kernel launch interface (not part of the public C ABI).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace icr {

struct GemmParams;

// Programmatic dependent launch for every kernel of the step: the next kernel may start
// (prologue, weight prefetch) while this one drains; kernels call griddepcontrol.wait
// before touching their predecessor's outputs. g_pdl = 0 disables it (ICR_NO_PDL=1).
extern int g_pdl;
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// --------------------------------------------------------------- GEMM (gemm.cu)
// tlb / tlu: LoRA expand operands (B_cat tile-major 3-D map, block-diagonal U 2-D map);
// may be null when p.lora_chunks == 0.
cudaError_t gemm_launch(const CUtensorMap& tw, const CUtensorMap& tx, const CUtensorMap* tlb,
                        const CUtensorMap* tlu, const GemmParams& p, int x_row0, int nt,
                        int num_sms, cudaStream_t s);
int gemm_pick_nt(int rows);
int gemm_stages(int nt);
size_t gemm_ws_floats(int num_sms);
// stream-K scratch starts (and is always left) holding the "unpublished" pattern
cudaError_t gemm_ws_clear(float* ws, int num_sms, cudaStream_t s);

// --------------------------------------------------------------- attention (attention.cu)
struct AttnItem {
  int chunk_start;  // absolute key position of the chunk's first page
  int n_pages;      // pages to visit
  int page_off;     // into item_pages
  int row_off;      // into item_rows
  int n_rows;       // query rows (<= 64)
  int chunk_idx;    // chunk index c (partial slot)
  int n_pre;        // leading pages entirely below every row's position: written by earlier
                    // steps, so the producer may load them before griddepcontrol.wait
};

struct AttnLaunch {
  const __nv_bfloat16* q;
  int q_ld;
  const __nv_bfloat16* k_pages;
  const __nv_bfloat16* v_pages;
  int num_kv_heads, num_heads, group, head_dim;
  const AttnItem* items;
  const int* sched_off;    // tcgen05 path: persistent CTA c runs units [sched_off[c], sched_off[c+1])
  const int* sched_units;  //   unit = item * num_kv_heads + KV head
  int num_sms;             //   grid = min(num_sms, n_items_cap * num_kv_heads)
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
  int* merge_cnt;  // tcgen05 long-chunk path: 64-bit launch counter of the in-kernel merge (zeroed once, 8-byte aligned)
  CUtensorMap tm_k, tm_v;  // page-arena maps: one 64-dim half page of one KV head per box
  CUtensorMap tm_k8, tm_v8;  // the same arena as runs: 8 consecutive page ids of one KV head,
                             // both halves, in one box (32 KB, [half][page][key][128 B])
  const uint8_t* pf_base;  // L2 prefetch of the next projection's weights (null = none)
  long long pf_bytes;
  __nv_bfloat16* out;
  int out_ld;
  unsigned long long* trace;  // diagnostic per-CTA stamps [2 launches][4096][8] (null = off)
  unsigned long long* span;   // bench: {min CTA start, max CTA end} %globaltimer (null = off)
};
cudaError_t attn_launch(const AttnLaunch& a, cudaStream_t s);
// tcgen05 partial kernel (attention_tc.cu), head_dim 128, chunks of <= 16 pages.
cudaError_t attn_tc_partial_launch(const AttnLaunch& a, int chunk_pages, cudaStream_t s);
// Query entries (row, head-in-group) per work item: 128 = the tcgen05 M (head_dim 128
// unless ICR_ATTN_MMA=1), 64 for the mma.sync kernel.
int attn_entries_per_item(int head_dim);

// --------------------------------------------------------------- row ops (rowops.cu)
// Layer-0 input: x[r] = embed[tok[r]] (fp32 residual stream), xb = bf16(x), and the
// per-128-feature sums of squares ssq[c][r] that the first GEMM turns into RMSNorm scales.
cudaError_t embed_launch(const int* tokens, const int* row_kind, const __nv_bfloat16* embed,
                         float* x, __nv_bfloat16* xb, float* ssq, int ss_stride, int n_rows,
                         int d, const uint8_t* pf_base, long long pf_bytes, __nv_bfloat16* ubd,
                         int ubd_ld, cudaStream_t s);

// Each CTA of a latency-bound kernel prefetches its slice of [base, base + bytes) into L2.
__device__ __forceinline__ void prefetch_slice_l2(const uint8_t* base, long long bytes, int part,
                                                  int nparts) {
  if (base == nullptr) return;
  const long long units = bytes >> 14;  // 16 KB pieces
  const long long b = (long long)part * units / nparts, e = (long long)(part + 1) * units / nparts;
  for (long long u = b + threadIdx.x; u < e; u += blockDim.x)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], 16384;\n" ::"l"(base + (u << 14)) : "memory");
}

// Emitting rows for the LM head: hlm[i] = xb[lm_rows[i]], ssq_lm[c][i] = ssq[c][lm_rows[i]];
// rows n_lm..n_pad-1 are zero. store_slot[i] >= 0 also keeps row i in the per-sequence hidden
// store (hid, hid_ssq); from_store = 1 gathers from the store instead (lm_rows = store slots).
cudaError_t lm_gather_launch(const __nv_bfloat16* xb, const float* ssq, int ss_stride,
                             const int* lm_rows, int n_lm, int n_pad, int d,
                             __nv_bfloat16* hlm, float* ssq_lm, const int* store_slot,
                             __nv_bfloat16* hid, float* hid_ssq, int hid_stride, int from_store,
                             cudaStream_t s);

// Layer input from an explicit fp32 residual stream (same outputs as embed_launch).
cudaError_t resid_load_launch(const float* x_in, int n_valid, int n_rows, float* x,
                              __nv_bfloat16* xb, float* ssq, int ss_stride, int d,
                              __nv_bfloat16* ubd, int ubd_ld, cudaStream_t s);

// Final argmax over LM-head tiles (lowest index on ties, src/engine.py:75-76).
cudaError_t argmax_reduce_launch(const float2* tile_best, int tiles, int stride, int n_rows,
                                 int* out_tokens, cudaStream_t s);

// tokens[r] = out_tok[src[r]] for src[r] >= 0 (device-side greedy feedback).
cudaError_t feedback_launch(int* tokens, const int* out_tok, const int* src, int n,
                            cudaStream_t s);

}  // namespace icr
