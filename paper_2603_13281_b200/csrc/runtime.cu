// Native runtime behind the C ABI (include/icarus_b200.h): model residency, TMA
// descriptors, the shared-page attention planner, and the per-step kernel schedule.
//
// One forward pass (= one fused multi-model decode step, or one prefill chunk) is:
//   per layer (src/model.py:480-506 fused decode, :463-478 prefill):
//     rmsnorm(+embed) -> LoRA shrink(q) -> GEMM qkv [RoPE, q out, encoder K/V -> pages]
//     -> paged attention partials + fixed-order merge -> LoRA shrink(o) -> GEMM o [+= x]
//     -> rmsnorm -> LoRA shrink(gate, up) -> GEMM gate|up [silu*up] -> LoRA shrink(down)
//     -> GEMM down [+= x]
//   final rmsnorm on emitting rows -> GEMM lm_head [per-tile argmax] -> argmax reduce.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/icarus_b200.h"
#include "gemm.cuh"
#include "kernels.h"

namespace icr {
__global__ void feedback_kernel(int* tokens, const int* out_tok, const int* src, int n) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n && src[r] >= 0) tokens[r] = out_tok[src[r]];
}
}  // namespace icr

using namespace icr;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static icr_status fail(icr_status code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(ICR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),    \
                  __FILE__, __LINE__);                                                  \
  } while (0)

// ------------------------------------------------------------------ TMA descriptors
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static icr_status get_encode() {
  if (g_encode) return ICR_OK;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || fn == nullptr)
    return fail(ICR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return ICR_OK;
}

// bf16 matrix [rows, cols] row-major (cols contiguous), box {64, box_rows}, 128B swizzle.
static icr_status make_map(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols,
                           uint32_t box_rows) {
  icr_status st = get_encode();
  if (st) return st;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(ICR_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu box=%u", (int)r,
                (unsigned long long)rows, (unsigned long long)cols, box_rows);
  return ICR_OK;
}

static int nt_index(int nt) {
  switch (nt) {
    case 16: return 0;
    case 32: return 1;
    case 64: return 2;
    case 128: return 3;
    default: return 4;
  }
}
static const int kNts[5] = {16, 32, 64, 128, 256};

static int query_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// ------------------------------------------------------------------ attention planner
struct AttnPlan {
  std::vector<AttnItem> items;
  std::vector<int> pages;
  std::vector<int2> rows;
};

// Group (sequence, chunk) pairs that map to identical physical pages, so each shared page
// is read once per KV head for every query row attached to it.
static icr_status build_attn_plan(int n_rows, const int* kind, const int* seq, const int* pos,
                                  const int* bt, int n_seqs, int bt_stride, int num_pages,
                                  int group, int chunk_pages, AttnPlan& plan) {
  const int CT = chunk_pages * 16;
  plan.items.clear();
  plan.pages.clear();
  plan.rows.clear();
  std::vector<std::vector<int>> seq_rows(n_seqs);
  std::vector<int> maxpos(n_seqs, -1);
  for (int r = 0; r < n_rows; ++r) {
    if (kind[r] < 0) continue;
    const int s = seq[r];
    if (s < 0 || s >= n_seqs) return fail(ICR_SHAPE, "row %d: sequence slot %d outside [0,%d)", r, s, n_seqs);
    seq_rows[s].push_back(r);
    maxpos[s] = std::max(maxpos[s], pos[r]);
  }
  struct Group {
    int c;
    std::vector<int> pages;
    std::vector<int> seqs;
  };
  std::vector<Group> groups;
  std::map<std::pair<int, std::vector<int>>, int> index;
  for (int s = 0; s < n_seqs; ++s) {
    if (maxpos[s] < 0) continue;
    if ((maxpos[s] >> 4) >= bt_stride)
      return fail(ICR_CAPACITY, "sequence %d position %d exceeds block table (%d pages)", s, maxpos[s], bt_stride);
    for (int c = 0; c * CT <= maxpos[s]; ++c) {
      const int last = std::min(maxpos[s], (c + 1) * CT - 1) >> 4;
      std::vector<int> pg;
      for (int p = c * chunk_pages; p <= last; ++p) {
        const int id = bt[(size_t)s * bt_stride + p];
        if (id < 0 || id >= num_pages)
          return fail(ICR_STATE, "sequence %d page %d is unmapped (id %d)", s, p, id);
        pg.push_back(id);
      }
      auto key = std::make_pair(c, pg);
      auto it = index.find(key);
      if (it == index.end()) {
        index.emplace(key, (int)groups.size());
        groups.push_back(Group{c, std::move(pg), {s}});
      } else {
        groups[it->second].seqs.push_back(s);
      }
    }
  }
  for (const Group& gr : groups) {
    const int c0 = gr.c * CT, c1 = (gr.c + 1) * CT - 1;
    std::vector<int2> entries;
    std::vector<int> entry_pos;
    for (int s : gr.seqs)
      for (int r : seq_rows[s])
        if (pos[r] >= c0)
          for (int hg = 0; hg < group; ++hg) {
            entries.push_back(make_int2(r, hg));
            entry_pos.push_back(pos[r]);
          }
    for (size_t e0 = 0; e0 < entries.size(); e0 += 64) {
      const size_t e1 = std::min(entries.size(), e0 + 64);
      int npages = 0;
      for (size_t e = e0; e < e1; ++e)
        npages = std::max(npages, ((std::min(entry_pos[e], c1) - c0) >> 4) + 1);
      AttnItem it;
      it.chunk_start = c0;
      it.n_pages = npages;
      it.page_off = (int)plan.pages.size();
      it.row_off = (int)plan.rows.size();
      it.n_rows = (int)(e1 - e0);
      it.chunk_idx = gr.c;
      plan.items.push_back(it);
      plan.pages.insert(plan.pages.end(), gr.pages.begin(), gr.pages.begin() + npages);
      plan.rows.insert(plan.rows.end(), entries.begin() + e0, entries.begin() + e1);
    }
  }
  return ICR_OK;
}

// Device-side view of one forward's metadata (offsets into meta_dev).
struct Meta {
  int n_rows, rp, n_lm, n_dec, n_items;
  size_t o_tokens, o_kind, o_seq, o_pos, o_adapter, o_lm_rows, o_seg_off, o_seg_rows, o_bt,
      o_items, o_item_pages, o_item_rows, o_n_items, o_feedback, total;
};

// ------------------------------------------------------------------ model
struct LayerMaps {
  CUtensorMap qkv, o, gu, down;
};

struct icr_model {
  icr_model_config cfg;
  std::vector<icr_layer_weights> layers;
  std::vector<LayerMaps> maps;
  CUtensorMap lm_map;
  const __nv_bfloat16* embed;
  const __nv_bfloat16* lm_head;
  float scaling;
  int num_sms;
  int q_dim, kv_dim, vpad, rp, max_chunks;
  // scratch
  float* x;
  __nv_bfloat16 *h, *qb, *att, *f, *hlm;
  float* U;
  float2* tile_best;
  int* out_tok;
  float* part_o;
  float2* part_ml;
  float2* rope;
  float* ws;
  int* counters;
  int* zero_kind;
  CUtensorMap xmap_h[5], xmap_att[5], xmap_f[5], xmap_hlm[5];
  // metadata staging
  int* meta_dev = nullptr;
  size_t meta_cap = 0;  // ints
  int* staging[2] = {nullptr, nullptr};
  size_t staging_cap = 0;
  cudaEvent_t staging_ev[2];
  cudaEvent_t step_ev[2];
  // instrumentation of the last forward
  long long last_launches = 0;
  long long last_meta_bytes = 0;
  long long last_items = 0;
  Meta last_mt{};
  bool has_last = false;
};

static icr_status ensure_meta(icr_model* m, size_t ints) {
  if (ints <= m->meta_cap) return ICR_OK;
  size_t cap = std::max(ints, m->meta_cap * 2 + 4096);
  if (m->meta_dev) cudaFree(m->meta_dev);
  for (int i = 0; i < 2; ++i)
    if (m->staging[i]) cudaFreeHost(m->staging[i]);
  CUDA_TRY(cudaMalloc(&m->meta_dev, cap * sizeof(int)));
  for (int i = 0; i < 2; ++i) CUDA_TRY(cudaMallocHost(&m->staging[i], cap * sizeof(int)));
  m->meta_cap = cap;
  return ICR_OK;
}

// Packs host batch metadata into `stage` (capacity checked by caller via sizing pass).
static icr_status pack_meta(icr_model* m, const icr_batch* b, const int* pos_override,
                            const int* feedback, int* stage, Meta& mt, AttnPlan& plan,
                            bool size_only) {
  const icr_model_config& c = m->cfg;
  const int n = b->n_rows;
  const int rp = (n + 15) & ~15;
  const int* pos = pos_override ? pos_override : b->row_pos;
  mt.n_rows = n;
  mt.rp = rp;
  if (!size_only) {
    icr_status st = build_attn_plan(n, b->row_kind, b->row_seq, pos, b->block_table, b->n_seqs,
                                    c.max_pages_per_seq, c.num_pages,
                                    c.num_heads / c.num_kv_heads, c.chunk_pages, plan);
    if (st) return st;
  }
  mt.n_items = (int)plan.items.size();
  int n_lm = 0, n_dec = 0;
  for (int r = 0; r < n; ++r) {
    if (b->row_emit && b->row_emit[r]) ++n_lm;
    if (b->row_kind[r] == 1) ++n_dec;
  }
  mt.n_lm = n_lm;
  mt.n_dec = n_dec;
  size_t off = 0;
  auto take = [&](size_t count) {
    size_t o = off;
    off += (count + 3) & ~size_t(3);  // 16-byte alignment
    return o;
  };
  mt.o_tokens = take(rp);
  mt.o_kind = take(rp);
  mt.o_seq = take(rp);
  mt.o_pos = take(rp);
  mt.o_adapter = take(rp);
  mt.o_lm_rows = take(rp);
  mt.o_seg_off = take(c.adapter_slots + 1);
  mt.o_seg_rows = take(rp);
  mt.o_bt = take((size_t)b->n_seqs * c.max_pages_per_seq);
  mt.o_items = take(plan.items.size() * (sizeof(AttnItem) / sizeof(int)));
  mt.o_item_pages = take(plan.pages.size());
  mt.o_item_rows = take(plan.rows.size() * 2);
  mt.o_n_items = take(1);
  mt.o_feedback = take(rp);
  mt.total = off;
  if (size_only) return ICR_OK;

  int* t = stage;
  for (int r = 0; r < rp; ++r) {
    const bool valid = r < n;
    t[mt.o_tokens + r] = valid ? b->tokens[r] : 0;
    t[mt.o_kind + r] = valid ? b->row_kind[r] : -1;
    t[mt.o_seq + r] = valid ? b->row_seq[r] : 0;
    t[mt.o_pos + r] = valid ? pos[r] : 0;
    t[mt.o_adapter + r] = valid ? b->row_adapter[r] : -1;
    t[mt.o_feedback + r] = (valid && feedback) ? feedback[r] : -1;
  }
  int li = 0;
  for (int r = 0; r < n; ++r)
    if (b->row_emit && b->row_emit[r]) t[mt.o_lm_rows + li++] = r;
  // decoder rows grouped by adapter slot (SGMV segments)
  int* seg_off = t + mt.o_seg_off;
  int* seg_rows = t + mt.o_seg_rows;
  int k = 0;
  for (int a = 0; a < c.adapter_slots; ++a) {
    seg_off[a] = k;
    for (int r = 0; r < n; ++r)
      if (b->row_kind[r] == 1 && b->row_adapter[r] == a) seg_rows[k++] = r;
  }
  seg_off[c.adapter_slots] = k;
  memcpy(t + mt.o_bt, b->block_table, sizeof(int) * (size_t)b->n_seqs * c.max_pages_per_seq);
  memcpy(t + mt.o_items, plan.items.data(), plan.items.size() * sizeof(AttnItem));
  memcpy(t + mt.o_item_pages, plan.pages.data(), plan.pages.size() * sizeof(int));
  memcpy(t + mt.o_item_rows, plan.rows.data(), plan.rows.size() * sizeof(int2));
  t[mt.o_n_items] = mt.n_items;
  return ICR_OK;
}

static icr_status validate_batch(icr_model* m, const icr_batch* b, const int* pos_override) {
  const icr_model_config& c = m->cfg;
  if (b->n_rows < 1) return fail(ICR_SHAPE, "batch needs at least one row");
  if (b->n_rows > c.max_rows)
    return fail(ICR_CAPACITY, "batch of %d rows exceeds max_rows %d", b->n_rows, c.max_rows);
  if (b->n_seqs < 1 || b->n_seqs > c.max_seqs)
    return fail(ICR_CAPACITY, "n_seqs %d outside [1, %d]", b->n_seqs, c.max_seqs);
  const int* pos = pos_override ? pos_override : b->row_pos;
  for (int r = 0; r < b->n_rows; ++r) {
    if (b->tokens[r] < 0 || b->tokens[r] >= c.vocab_size)
      return fail(ICR_INDEX, "token %d outside vocab [0, %d)", b->tokens[r], c.vocab_size);
    const int k = b->row_kind[r];
    if (k != 0 && k != 1) return fail(ICR_MODE, "row %d kind %d must be 0 (encoder) or 1 (decoder)", r, k);
    if (k == 1) {
      if (b->row_adapter[r] >= 0 && (c.lora_rank == 0 || b->row_adapter[r] >= c.adapter_slots))
        return fail(ICR_CONFIG, "row %d adapter slot %d outside [0, %d)", r, b->row_adapter[r], c.adapter_slots);
    }
    if (pos[r] < 0 || pos[r] >= c.max_positions)
      return fail(ICR_CAPACITY, "row %d position %d outside [0, %d)", r, pos[r], c.max_positions);
  }
  return ICR_OK;
}

// Enqueue the whole forward on `s` using metadata already resident at m->meta_dev.
static icr_status enqueue_forward(icr_model* m, const Meta& mt, float* logits_dev, cudaStream_t s) {
  const icr_model_config& c = m->cfg;
  int* md = m->meta_dev;
  const int* tokens = md + mt.o_tokens;
  const int* kind = md + mt.o_kind;
  const int* seq = md + mt.o_seq;
  const int* pos = md + mt.o_pos;
  const int* adapter = md + mt.o_adapter;
  const int* lm_rows = md + mt.o_lm_rows;
  const int* seg_off = md + mt.o_seg_off;
  const int* seg_rows = md + mt.o_seg_rows;
  const int* bt = md + mt.o_bt;
  const bool lora = c.lora_rank > 0 && mt.n_dec > 0;
  const int d = c.hidden_dim, rp = mt.rp;
  long long launches = 0;

  auto gemm = [&](const CUtensorMap& wmap, CUtensorMap* xmaps, GemmParams p, int rows,
                  int row_stride_out) -> icr_status {
    for (int g0 = 0; g0 < rows; g0 += 256) {
      const int gr = std::min(256, rows - g0);
      const int nt = gemm_pick_nt(gr);
      GemmParams q = p;
      q.n_rows = gr;
      if (p.row_kind) q.row_kind = p.row_kind + g0;
      if (p.row_adapter) q.row_adapter = p.row_adapter + g0;
      if (p.row_pos) q.row_pos = p.row_pos + g0;
      if (p.row_seq) q.row_seq = p.row_seq + g0;
      if (p.lora_u) q.lora_u = p.lora_u + (size_t)g0 * p.n_u * p.rank;
      if (p.out_f32) q.out_f32 = p.out_f32 + (size_t)g0 * p.ld_out;
      if (p.resid) q.resid = p.resid + (size_t)g0 * p.M;
      if (p.out_bf16) q.out_bf16 = p.out_bf16 + (size_t)g0 * row_stride_out;
      if (p.tile_best) q.tile_best = p.tile_best + g0;
      cudaError_t e = gemm_launch(wmap, xmaps[nt_index(nt)], q, g0, nt, m->num_sms, s);
      if (e != cudaSuccess) return fail(ICR_CUDA, "gemm launch: %s", cudaGetErrorString(e));
      ++launches;
    }
    return ICR_OK;
  };

  GemmParams base{};
  base.ws = m->ws;
  base.counters = m->counters;
  base.rank = c.lora_rank;
  base.n_u = 1;
  base.m_valid = 1 << 30;

  AttnLaunch al{};
  al.q = m->qb;
  al.q_ld = m->q_dim;
  al.num_kv_heads = c.num_kv_heads;
  al.num_heads = c.num_heads;
  al.group = c.num_heads / c.num_kv_heads;
  al.head_dim = c.head_dim;
  al.items = reinterpret_cast<const AttnItem*>(md + mt.o_items);
  al.item_pages = md + mt.o_item_pages;
  al.item_rows = reinterpret_cast<const int2*>(md + mt.o_item_rows);
  al.n_items_dev = md + mt.o_n_items;
  al.n_items_cap = mt.n_items;
  al.row_pos = pos;
  al.row_kind = kind;
  al.n_rows = rp;
  al.max_chunks = m->max_chunks;
  al.chunk_tokens = c.chunk_pages * 16;
  al.scale = (float)(1.0 / std::sqrt((double)c.head_dim));
  al.part_o = m->part_o;
  al.part_ml = m->part_ml;
  al.out = m->att;
  al.out_ld = m->q_dim;

  icr_status st;
  for (int l = 0; l < c.num_layers; ++l) {
    const icr_layer_weights& w = m->layers[l];
    const LayerMaps& lm = m->maps[l];
    ++launches;
    CUDA_TRY(rmsnorm_launch(m->x, tokens, l == 0 ? m->embed : nullptr, m->x, m->h, kind, nullptr,
                            rp, d, c.rms_eps, s));
    if (lora) {
      ++launches;
      CUDA_TRY(lora_shrink_launch(m->h, d, d, (const __nv_bfloat16*)w.a_q, nullptr, 1,
                                  c.adapter_slots, c.lora_rank, m->scaling, seg_off, seg_rows,
                                  m->U, s));
    }
    {
      GemmParams p = base;
      p.mode = EPI_QKV;
      p.M = m->q_dim + 2 * m->kv_dim;
      p.K = d;
      p.row_kind = kind;
      p.row_adapter = adapter;
      p.row_pos = pos;
      p.row_seq = seq;
      p.lora_b = lora ? (const __nv_bfloat16*)w.b_q : nullptr;
      p.lora_u = m->U;
      p.lora_m = m->q_dim;
      p.out_bf16 = m->qb;
      p.q_dim = m->q_dim;
      p.kv_dim = m->kv_dim;
      p.head_dim = c.head_dim;
      p.num_kv_heads = c.num_kv_heads;
      p.rope = m->rope;
      p.k_pages = (__nv_bfloat16*)w.k_pages;
      p.v_pages = (__nv_bfloat16*)w.v_pages;
      p.block_table = bt;
      p.bt_stride = c.max_pages_per_seq;
      if ((st = gemm(lm.qkv, m->xmap_h, p, rp, m->q_dim))) return st;
    }
    al.k_pages = (const __nv_bfloat16*)w.k_pages;
    al.v_pages = (const __nv_bfloat16*)w.v_pages;
    {
      cudaError_t e = attn_launch(al, s);
      launches += 2;
      if (e != cudaSuccess) return fail(ICR_CUDA, "attention launch: %s", cudaGetErrorString(e));
    }
    if (lora) {
      ++launches;
      CUDA_TRY(lora_shrink_launch(m->att, m->q_dim, m->q_dim, (const __nv_bfloat16*)w.a_o, nullptr,
                                  1, c.adapter_slots, c.lora_rank, m->scaling, seg_off, seg_rows,
                                  m->U, s));
    }
    {
      GemmParams p = base;
      p.mode = EPI_RESID;
      p.M = d;
      p.K = m->q_dim;
      p.row_kind = kind;
      p.row_adapter = adapter;
      p.lora_b = lora ? (const __nv_bfloat16*)w.b_o : nullptr;
      p.lora_u = m->U;
      p.lora_m = d;
      p.resid = m->x;
      if ((st = gemm(lm.o, m->xmap_att, p, rp, 0))) return st;
    }
    ++launches;
    CUDA_TRY(rmsnorm_launch(m->x, nullptr, nullptr, m->x, m->h, kind, nullptr, rp, d, c.rms_eps, s));
    if (lora) {
      ++launches;
      CUDA_TRY(lora_shrink_launch(m->h, d, d, (const __nv_bfloat16*)w.a_gate,
                                  (const __nv_bfloat16*)w.a_up, 2, c.adapter_slots, c.lora_rank,
                                  m->scaling, seg_off, seg_rows, m->U, s));
    }
    {
      GemmParams p = base;
      p.mode = EPI_SILU;
      p.M = 2 * c.ffn_dim;
      p.K = d;
      p.row_kind = kind;
      p.row_adapter = adapter;
      p.lora_b = lora ? (const __nv_bfloat16*)w.b_gu : nullptr;
      p.lora_u = m->U;
      p.lora_m = 2 * c.ffn_dim;
      p.n_u = 2;
      p.out_bf16 = m->f;
      if ((st = gemm(lm.gu, m->xmap_h, p, rp, c.ffn_dim))) return st;
    }
    if (lora) {
      ++launches;
      CUDA_TRY(lora_shrink_launch(m->f, c.ffn_dim, c.ffn_dim, (const __nv_bfloat16*)w.a_down,
                                  nullptr, 1, c.adapter_slots, c.lora_rank, m->scaling, seg_off,
                                  seg_rows, m->U, s));
    }
    {
      GemmParams p = base;
      p.mode = EPI_RESID;
      p.M = d;
      p.K = c.ffn_dim;
      p.row_kind = kind;
      p.row_adapter = adapter;
      p.lora_b = lora ? (const __nv_bfloat16*)w.b_down : nullptr;
      p.lora_u = m->U;
      p.lora_m = d;
      p.resid = m->x;
      if ((st = gemm(lm.down, m->xmap_f, p, rp, 0))) return st;
    }
  }
  // final norm (emitting rows only) + LM head + argmax (src/engine.py:188-193)
  if (mt.n_lm > 0) {
    const int nlm_p = (mt.n_lm + 15) & ~15;
    ++launches;
    CUDA_TRY(rmsnorm_launch(m->x, nullptr, nullptr, nullptr, m->hlm, nullptr, lm_rows, mt.n_lm, d,
                            c.rms_eps, s));
    if (nlm_p > mt.n_lm)
      CUDA_TRY(cudaMemsetAsync(m->hlm + (size_t)mt.n_lm * d, 0,
                               sizeof(__nv_bfloat16) * (size_t)(nlm_p - mt.n_lm) * d, s));
    GemmParams p = base;
    p.mode = EPI_ARGMAX;
    p.M = m->vpad;
    p.K = d;
    p.m_valid = c.vocab_size;
    p.tile_best = m->tile_best;
    p.best_stride = rp;
    if ((st = gemm(m->lm_map, m->xmap_hlm, p, mt.n_lm, 0))) return st;
    ++launches;
    CUDA_TRY(argmax_reduce_launch(m->tile_best, m->vpad / 128, rp, mt.n_lm, m->out_tok, s));
    if (logits_dev) {
      GemmParams q = base;
      q.mode = EPI_F32;
      q.M = m->vpad;
      q.K = d;
      q.out_f32 = logits_dev;
      q.ld_out = m->vpad;
      if ((st = gemm(m->lm_map, m->xmap_hlm, q, mt.n_lm, 0))) return st;
    }
  }
  m->last_launches = launches;
  m->last_items = mt.n_items;
  m->last_mt = mt;
  m->has_last = true;
  return ICR_OK;
}

// ------------------------------------------------------------------ C ABI
extern "C" {

const char* icr_last_error(void) { return g_err.c_str(); }
int icr_abi_version(void) { return 1; }
int icr_num_sms(void) { return query_sms(); }

icr_status icr_model_create(const icr_model_config* cfg, const icr_layer_weights* layers,
                            const void* embed, const void* lm_head, float lora_scaling,
                            icr_model** out) {
  if (!cfg || !layers || !embed || !lm_head || !out) return fail(ICR_CONFIG, "null argument");
  const icr_model_config& c = *cfg;
  if (c.num_layers < 1 || c.hidden_dim < 1 || c.num_heads < 1 || c.num_kv_heads < 1 ||
      c.head_dim < 1 || c.ffn_dim < 1 || c.vocab_size < 1)
    return fail(ICR_CONFIG, "shape constants must be positive");
  if (c.num_heads % c.num_kv_heads)
    return fail(ICR_CONFIG, "num_heads %d not divisible by num_kv_heads %d", c.num_heads, c.num_kv_heads);
  if (c.hidden_dim != c.num_heads * c.head_dim)
    return fail(ICR_CONFIG, "hidden_dim %d != num_heads*head_dim", c.hidden_dim);
  if (c.head_dim != 64 && c.head_dim != 128)
    return fail(ICR_CONFIG, "B200 attention kernel supports head_dim 64 or 128, got %d", c.head_dim);
  const int q_dim = c.num_heads * c.head_dim, kv_dim = c.num_kv_heads * c.head_dim;
  if ((q_dim + 2 * kv_dim) % 128 || c.hidden_dim % 128 || (2 * c.ffn_dim) % 128 || c.ffn_dim % 64)
    return fail(ICR_CONFIG, "B200 GEMM tiles need hidden_dim %% 128 == 0, ffn_dim %% 64 == 0 and "
                "(q_dim + 2 kv_dim) %% 128 == 0");
  if (c.lora_rank < 0 || (c.lora_rank > 0 && (c.lora_rank % 8 || c.adapter_slots < 1)))
    return fail(ICR_CONFIG, "lora_rank must be 0 or a multiple of 8 with adapter_slots >= 1");
  if (c.chunk_pages < 1 || c.max_rows < 1 || c.max_positions < 1 || c.num_pages < 1 ||
      c.max_seqs < 1 || c.max_pages_per_seq < 1)
    return fail(ICR_CONFIG, "capacities must be positive");

  icr_model* m = new icr_model();
  m->cfg = c;
  m->layers.assign(layers, layers + c.num_layers);
  m->embed = (const __nv_bfloat16*)embed;
  m->lm_head = (const __nv_bfloat16*)lm_head;
  m->scaling = lora_scaling;
  m->num_sms = query_sms();
  m->q_dim = q_dim;
  m->kv_dim = kv_dim;
  m->vpad = (c.vocab_size + 127) / 128 * 128;
  m->rp = (c.max_rows + 15) & ~15;
  const int CT = c.chunk_pages * 16;
  m->max_chunks = (c.max_positions + CT - 1) / CT;
  const size_t rp = m->rp;
  auto bail = [&](icr_status s) {
    icr_model_destroy(m);
    return s;
  };
#define ALLOC(ptr, bytes)                                                         \
  do {                                                                            \
    cudaError_t _e = cudaMalloc(&(ptr), (bytes));                                 \
    if (_e != cudaSuccess)                                                        \
      return bail(fail(ICR_CUDA, "cudaMalloc %zu: %s", (size_t)(bytes),           \
                       cudaGetErrorString(_e)));                                  \
    cudaMemset((ptr), 0, (bytes));                                                \
  } while (0)
  ALLOC(m->x, rp * c.hidden_dim * sizeof(float));
  ALLOC(m->h, rp * c.hidden_dim * 2);
  ALLOC(m->qb, rp * q_dim * 2);
  ALLOC(m->att, rp * q_dim * 2);
  ALLOC(m->f, rp * c.ffn_dim * 2);
  ALLOC(m->hlm, rp * c.hidden_dim * 2);
  ALLOC(m->U, rp * 2 * std::max(c.lora_rank, 8) * sizeof(float));
  ALLOC(m->tile_best, (size_t)(m->vpad / 128) * rp * sizeof(float2));
  ALLOC(m->out_tok, rp * sizeof(int));
  ALLOC(m->part_o, rp * c.num_heads * m->max_chunks * c.head_dim * sizeof(float));
  ALLOC(m->part_ml, rp * c.num_heads * m->max_chunks * sizeof(float2));
  ALLOC(m->rope, (size_t)c.max_positions * (c.head_dim / 2) * sizeof(float2));
  ALLOC(m->ws, gemm_ws_floats(m->num_sms) * sizeof(float));
  {
    const int max_tiles = std::max({m->vpad, 2 * c.ffn_dim, q_dim + 2 * kv_dim, c.hidden_dim}) / 128;
    ALLOC(m->counters, (size_t)max_tiles * sizeof(int));
  }
  ALLOC(m->zero_kind, rp * sizeof(int));
#undef ALLOC
  // RoPE table, float64 angles cast once (src/tensor.py:270-279).
  {
    const int half = c.head_dim / 2;
    std::vector<float2> tab((size_t)c.max_positions * half);
    for (int p = 0; p < c.max_positions; ++p)
      for (int i = 0; i < half; ++i) {
        const double inv_freq = std::pow(c.rope_theta, (-(double)i * 2.0) / (double)c.head_dim);
        const double ang = (double)p * inv_freq;
        tab[(size_t)p * half + i] = make_float2((float)std::cos(ang), (float)std::sin(ang));
      }
    cudaError_t e = cudaMemcpy(m->rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return bail(fail(ICR_CUDA, "rope upload: %s", cudaGetErrorString(e)));
  }
  icr_status st;
  m->maps.resize(c.num_layers);
  for (int l = 0; l < c.num_layers; ++l) {
    const icr_layer_weights& w = layers[l];
    if (!w.w_qkv || !w.w_o || !w.w_gu || !w.w_down || !w.k_pages || !w.v_pages)
      return bail(fail(ICR_CONFIG, "layer %d: missing weight or page pointer", l));
    if (c.lora_rank > 0 && (!w.a_q || !w.b_q || !w.a_o || !w.b_o || !w.a_gate || !w.a_up ||
                            !w.b_gu || !w.a_down || !w.b_down))
      return bail(fail(ICR_CONFIG, "layer %d: missing adapter pointer", l));
    if ((st = make_map(&m->maps[l].qkv, w.w_qkv, q_dim + 2 * kv_dim, c.hidden_dim, 128))) return bail(st);
    if ((st = make_map(&m->maps[l].o, w.w_o, c.hidden_dim, q_dim, 128))) return bail(st);
    if ((st = make_map(&m->maps[l].gu, w.w_gu, 2 * c.ffn_dim, c.hidden_dim, 128))) return bail(st);
    if ((st = make_map(&m->maps[l].down, w.w_down, c.hidden_dim, c.ffn_dim, 128))) return bail(st);
  }
  if ((st = make_map(&m->lm_map, lm_head, m->vpad, c.hidden_dim, 128))) return bail(st);
  for (int i = 0; i < 5; ++i) {
    if ((st = make_map(&m->xmap_h[i], m->h, rp, c.hidden_dim, kNts[i]))) return bail(st);
    if ((st = make_map(&m->xmap_att[i], m->att, rp, q_dim, kNts[i]))) return bail(st);
    if ((st = make_map(&m->xmap_f[i], m->f, rp, c.ffn_dim, kNts[i]))) return bail(st);
    if ((st = make_map(&m->xmap_hlm[i], m->hlm, rp, c.hidden_dim, kNts[i]))) return bail(st);
  }
  for (int i = 0; i < 2; ++i) {
    cudaEventCreateWithFlags(&m->staging_ev[i], cudaEventDisableTiming);
    cudaEventCreate(&m->step_ev[i]);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return bail(fail(ICR_CUDA, "model create: %s", cudaGetErrorString(e)));
  *out = m;
  return ICR_OK;
}

icr_status icr_model_destroy(icr_model* m) {
  if (!m) return ICR_OK;
  cudaDeviceSynchronize();
  void* bufs[] = {m->x, m->h, m->qb, m->att, m->f, m->hlm, m->U, m->tile_best, m->out_tok,
                  m->part_o, m->part_ml, m->rope, m->ws, m->counters, m->zero_kind, m->meta_dev};
  for (void* p : bufs)
    if (p) cudaFree(p);
  for (int i = 0; i < 2; ++i)
    if (m->staging[i]) cudaFreeHost(m->staging[i]);
  delete m;
  return ICR_OK;
}

icr_status icr_forward(icr_model* m, const icr_batch* b, int32_t* out_tokens_host,
                       float* logits_dev, void* stream) {
  if (!m || !b) return fail(ICR_CONFIG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  icr_status st = validate_batch(m, b, nullptr);
  if (st) return st;
  Meta mt;
  AttnPlan plan;
  // plan first (needs no staging), then size, then pack
  st = build_attn_plan(b->n_rows, b->row_kind, b->row_seq, b->row_pos, b->block_table, b->n_seqs,
                       m->cfg.max_pages_per_seq, m->cfg.num_pages,
                       m->cfg.num_heads / m->cfg.num_kv_heads, m->cfg.chunk_pages, plan);
  if (st) return st;
  pack_meta(m, b, nullptr, nullptr, nullptr, mt, plan, true);
  if ((st = ensure_meta(m, mt.total))) return st;
  CUDA_TRY(cudaEventSynchronize(m->staging_ev[0]));
  if ((st = pack_meta(m, b, nullptr, nullptr, m->staging[0], mt, plan, false))) return st;
  CUDA_TRY(cudaMemcpyAsync(m->meta_dev, m->staging[0], mt.total * sizeof(int), cudaMemcpyHostToDevice, s));
  m->last_meta_bytes = (long long)mt.total * sizeof(int);
  CUDA_TRY(cudaEventRecord(m->staging_ev[0], s));
  if ((st = enqueue_forward(m, mt, logits_dev, s))) return st;
  if (mt.n_lm > 0 && out_tokens_host) {
    int* pin = m->staging[1];
    CUDA_TRY(cudaEventSynchronize(m->staging_ev[1]));
    CUDA_TRY(cudaMemcpyAsync(pin, m->out_tok, mt.n_lm * sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    memcpy(out_tokens_host, pin, mt.n_lm * sizeof(int));
  } else {
    CUDA_TRY(cudaStreamSynchronize(s));
  }
  return ICR_OK;
}

icr_status icr_decode_loop(icr_model* m, const icr_batch* first, const int32_t* feedback_src,
                           int steps, int32_t* out_tokens_host_last, float* step_ms_host,
                           void* stream) {
  if (!m || !first || !feedback_src || steps < 1) return fail(ICR_CONFIG, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  const int n = first->n_rows;
  std::vector<int> pos(first->row_pos, first->row_pos + n);
  std::vector<cudaEvent_t> evs(steps + 1);
  for (auto& e : evs) CUDA_TRY(cudaEventCreate(&e));
  icr_status st = ICR_OK;
  Meta mt{};
  int n_lm = 0;
  for (int i = 0; i < steps && st == ICR_OK; ++i) {
    if (i > 0)
      for (int r = 0; r < n; ++r) pos[r] += 1;
    if ((st = validate_batch(m, first, pos.data()))) break;
    AttnPlan plan;
    if ((st = build_attn_plan(n, first->row_kind, first->row_seq, pos.data(), first->block_table,
                              first->n_seqs, m->cfg.max_pages_per_seq, m->cfg.num_pages,
                              m->cfg.num_heads / m->cfg.num_kv_heads, m->cfg.chunk_pages, plan)))
      break;
    pack_meta(m, first, pos.data(), feedback_src, nullptr, mt, plan, true);
    // Growing the buffers would free memory the in-flight steps still read: size once.
    if (mt.total > m->meta_cap) {
      cudaStreamSynchronize(s);
      if ((st = ensure_meta(m, mt.total * 2))) break;
    }
    const int slot = i & 1;
    cudaEventSynchronize(m->staging_ev[slot]);
    if ((st = pack_meta(m, first, pos.data(), feedback_src, m->staging[slot], mt, plan, false))) break;
    // Step 0 uploads everything; later steps keep the device-fed tokens.
    const size_t from = (i == 0) ? 0 : mt.o_kind;
    cudaMemcpyAsync(m->meta_dev + from, m->staging[slot] + from, (mt.total - from) * sizeof(int),
                    cudaMemcpyHostToDevice, s);
    m->last_meta_bytes = (long long)(mt.total - from) * sizeof(int);
    cudaEventRecord(m->staging_ev[slot], s);
    cudaEventRecord(evs[i], s);
    if ((st = enqueue_forward(m, mt, nullptr, s))) break;
    n_lm = mt.n_lm;
    feedback_kernel<<<(mt.rp + 127) / 128, 128, 0, s>>>(m->meta_dev + mt.o_tokens, m->out_tok,
                                                        m->meta_dev + mt.o_feedback, mt.rp);
  }
  if (st == ICR_OK) {
    cudaEventRecord(evs[steps], s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = fail(ICR_CUDA, "decode loop: %s", cudaGetErrorString(e));
  }
  if (st == ICR_OK && step_ms_host)
    for (int i = 0; i < steps; ++i) cudaEventElapsedTime(&step_ms_host[i], evs[i], evs[i + 1]);
  if (st == ICR_OK && out_tokens_host_last && n_lm > 0)
    cudaMemcpy(out_tokens_host_last, m->out_tok, n_lm * sizeof(int), cudaMemcpyDeviceToHost);
  for (auto& e : evs) cudaEventDestroy(e);
  return st;
}

// Instrumentation: [launches, metadata bytes, attention items] of the last forward.
icr_status icr_model_stats(icr_model* m, int64_t* out3) {
  if (!m || !out3) return fail(ICR_CONFIG, "null argument");
  out3[0] = m->last_launches;
  out3[1] = m->last_meta_bytes;
  out3[2] = m->last_items;
  return ICR_OK;
}

// Re-launch one projection GEMM family of the last forward `iters` times, cycling through
// all layers so no weight tile is served from L2, and return the average device time per
// launch (CUDA events on the launch stream). which: 0 wo, 1 gate|up, 2 down, 3 lm_head.
// Side effects are confined to scratch buffers (residual stream, f, tile maxima).
icr_status icr_profile_gemm(icr_model* m, int which, int iters, float* avg_ms, void* stream) {
  if (!m || !avg_ms || iters < 1) return fail(ICR_CONFIG, "bad arguments");
  if (!m->has_last) return fail(ICR_STATE, "profile needs a previous forward");
  cudaStream_t s = (cudaStream_t)stream;
  const icr_model_config& c = m->cfg;
  const Meta& mt = m->last_mt;
  int* md = m->meta_dev;
  const bool lora = c.lora_rank > 0 && mt.n_dec > 0;
  GemmParams p{};
  p.ws = m->ws;
  p.counters = m->counters;
  p.rank = c.lora_rank;
  p.n_u = 1;
  p.m_valid = 1 << 30;
  p.row_kind = md + mt.o_kind;
  p.row_adapter = md + mt.o_adapter;
  p.lora_u = m->U;
  int rows = mt.rp;
  CUtensorMap* xmaps = m->xmap_att;
  const void* bptr_off = nullptr;
  (void)bptr_off;
  switch (which) {
    case 0: p.mode = EPI_RESID; p.M = c.hidden_dim; p.K = m->q_dim; p.lora_m = c.hidden_dim;
            p.resid = m->x; xmaps = m->xmap_att; break;
    case 1: p.mode = EPI_SILU; p.M = 2 * c.ffn_dim; p.K = c.hidden_dim; p.lora_m = 2 * c.ffn_dim;
            p.n_u = 2; p.out_bf16 = m->f; xmaps = m->xmap_h; break;
    case 2: p.mode = EPI_RESID; p.M = c.hidden_dim; p.K = c.ffn_dim; p.lora_m = c.hidden_dim;
            p.resid = m->x; xmaps = m->xmap_f; break;
    case 3: p.mode = EPI_ARGMAX; p.M = m->vpad; p.K = c.hidden_dim; p.m_valid = c.vocab_size;
            p.tile_best = m->tile_best; p.best_stride = mt.rp; rows = mt.n_lm; xmaps = m->xmap_hlm;
            p.row_kind = nullptr; break;
    default: return fail(ICR_MODE, "which must be 0..3");
  }
  if (rows > 256) return fail(ICR_SHAPE, "profile supports <= 256 rows");
  p.n_rows = rows;
  const int nt = gemm_pick_nt(rows);
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  const int L = which == 3 ? 1 : c.num_layers;
  CUDA_TRY(cudaEventRecord(e0, s));
  for (int it = 0; it < iters; ++it)
    for (int l = 0; l < L; ++l) {
      const icr_layer_weights& w = m->layers[l];
      GemmParams q = p;
      const CUtensorMap* wm = &m->lm_map;
      if (which == 0) { wm = &m->maps[l].o; q.lora_b = lora ? (const __nv_bfloat16*)w.b_o : nullptr; }
      if (which == 1) { wm = &m->maps[l].gu; q.lora_b = lora ? (const __nv_bfloat16*)w.b_gu : nullptr; }
      if (which == 2) { wm = &m->maps[l].down; q.lora_b = lora ? (const __nv_bfloat16*)w.b_down : nullptr; }
      cudaError_t e = gemm_launch(*wm, xmaps[nt_index(nt)], q, 0, nt, m->num_sms, s);
      if (e != cudaSuccess) return fail(ICR_CUDA, "gemm: %s", cudaGetErrorString(e));
    }
  CUDA_TRY(cudaEventRecord(e1, s));
  CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  *avg_ms = ms / (float)(iters * L);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ICR_OK;
}

// ---- building blocks for parity tests ----
static float* g_ws = nullptr;
static int* g_counters = nullptr;
static int g_counters_n = 0;

icr_status icr_gemm_bf16(const void* w_dev, const void* x_dev, float* out_dev, int M, int K,
                         int n_rows, void* stream) {
  if (M % 128 || K % 64 || M <= 0 || K <= 0 || n_rows <= 0)
    return fail(ICR_SHAPE, "icr_gemm_bf16 needs M %% 128 == 0, K %% 64 == 0 (M=%d K=%d rows=%d)", M, K, n_rows);
  cudaStream_t s = (cudaStream_t)stream;
  const int sms = query_sms();
  if (!g_ws) CUDA_TRY(cudaMalloc(&g_ws, gemm_ws_floats(sms) * sizeof(float)));
  if (g_counters_n < M / 128) {
    if (g_counters) cudaFree(g_counters);
    CUDA_TRY(cudaMalloc(&g_counters, (M / 128) * sizeof(int)));
    CUDA_TRY(cudaMemset(g_counters, 0, (M / 128) * sizeof(int)));
    g_counters_n = M / 128;
  }
  CUtensorMap wm;
  icr_status st = make_map(&wm, w_dev, M, K, 128);
  if (st) return st;
  for (int g0 = 0; g0 < n_rows; g0 += 256) {
    const int gr = std::min(256, n_rows - g0);
    const int nt = gemm_pick_nt(gr);
    CUtensorMap xm;
    if ((st = make_map(&xm, x_dev, n_rows, K, nt))) return st;
    GemmParams p{};
    p.mode = EPI_F32;
    p.M = M;
    p.K = K;
    p.n_rows = gr;
    p.m_valid = M;
    p.out_f32 = out_dev + (size_t)g0 * M;
    p.ld_out = M;
    p.ws = g_ws;
    p.counters = g_counters;
    cudaError_t e = gemm_launch(wm, xm, p, g0, nt, sms, s);
    if (e != cudaSuccess) return fail(ICR_CUDA, "gemm: %s", cudaGetErrorString(e));
  }
  return ICR_OK;
}

icr_status icr_paged_attention(const void* q_dev, const void* k_pages, const void* v_pages,
                               int num_heads, int num_kv_heads, int head_dim, int chunk_pages,
                               int n_rows, const int32_t* row_seq_host, const int32_t* row_pos_host,
                               const int32_t* block_table_host, int n_seqs, int max_pages_per_seq,
                               void* out_dev, int32_t* n_items_out, void* stream) {
  if (head_dim != 64 && head_dim != 128) return fail(ICR_CONFIG, "head_dim must be 64 or 128");
  if (num_heads % num_kv_heads) return fail(ICR_CONFIG, "num_heads %% num_kv_heads != 0");
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<int> kind(n_rows, 0);
  AttnPlan plan;
  icr_status st = build_attn_plan(n_rows, kind.data(), row_seq_host, row_pos_host, block_table_host,
                                  n_seqs, max_pages_per_seq, 1 << 30, num_heads / num_kv_heads,
                                  chunk_pages, plan);
  if (st) return st;
  if (n_items_out) *n_items_out = (int)plan.items.size();
  int maxpos = 0;
  for (int r = 0; r < n_rows; ++r) maxpos = std::max(maxpos, row_pos_host[r]);
  const int max_chunks = maxpos / (chunk_pages * 16) + 1;
  int *d_pos, *d_kind, *d_pages, *d_n;
  AttnItem* d_items;
  int2* d_rows;
  float* d_po;
  float2* d_pml;
  const size_t np = std::max<size_t>(plan.pages.size(), 1), nr = std::max<size_t>(plan.rows.size(), 1),
               ni = std::max<size_t>(plan.items.size(), 1);
  CUDA_TRY(cudaMalloc(&d_pos, n_rows * sizeof(int)));
  CUDA_TRY(cudaMalloc(&d_kind, n_rows * sizeof(int)));
  CUDA_TRY(cudaMalloc(&d_pages, np * sizeof(int)));
  CUDA_TRY(cudaMalloc(&d_n, sizeof(int)));
  CUDA_TRY(cudaMalloc(&d_items, ni * sizeof(AttnItem)));
  CUDA_TRY(cudaMalloc(&d_rows, nr * sizeof(int2)));
  CUDA_TRY(cudaMalloc(&d_po, (size_t)n_rows * num_heads * max_chunks * head_dim * sizeof(float)));
  CUDA_TRY(cudaMalloc(&d_pml, (size_t)n_rows * num_heads * max_chunks * sizeof(float2)));
  int nitems = (int)plan.items.size();
  CUDA_TRY(cudaMemcpyAsync(d_pos, row_pos_host, n_rows * sizeof(int), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_kind, kind.data(), n_rows * sizeof(int), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_pages, plan.pages.data(), plan.pages.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_items, plan.items.data(), plan.items.size() * sizeof(AttnItem), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_rows, plan.rows.data(), plan.rows.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_n, &nitems, sizeof(int), cudaMemcpyHostToDevice, s));
  AttnLaunch a{};
  a.q = (const __nv_bfloat16*)q_dev;
  a.q_ld = num_heads * head_dim;
  a.k_pages = (const __nv_bfloat16*)k_pages;
  a.v_pages = (const __nv_bfloat16*)v_pages;
  a.num_kv_heads = num_kv_heads;
  a.num_heads = num_heads;
  a.group = num_heads / num_kv_heads;
  a.head_dim = head_dim;
  a.items = d_items;
  a.item_pages = d_pages;
  a.item_rows = d_rows;
  a.n_items_dev = d_n;
  a.n_items_cap = nitems;
  a.row_pos = d_pos;
  a.row_kind = d_kind;
  a.n_rows = n_rows;
  a.max_chunks = max_chunks;
  a.chunk_tokens = chunk_pages * 16;
  a.scale = (float)(1.0 / std::sqrt((double)head_dim));
  a.part_o = d_po;
  a.part_ml = d_pml;
  a.out = (__nv_bfloat16*)out_dev;
  a.out_ld = num_heads * head_dim;
  cudaError_t e = attn_launch(a, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  void* bufs[] = {d_pos, d_kind, d_pages, d_n, d_items, d_rows, d_po, d_pml};
  for (void* p : bufs) cudaFree(p);
  if (e != cudaSuccess) return fail(ICR_CUDA, "attention: %s", cudaGetErrorString(e));
  if (e2 != cudaSuccess) return fail(ICR_CUDA, "attention sync: %s", cudaGetErrorString(e2));
  return ICR_OK;
}

}  // extern "C"
