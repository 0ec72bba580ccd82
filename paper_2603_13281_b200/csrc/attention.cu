// Shared-KV paged decode attention (reference: `layer_attention`, src/model.py:384-425,
// with the fused 2H query heads of `block_forward` decode, src/model.py:495-501).
//
// Work decomposition (built on the host by runtime.cu build_attn_plan):
//   * each sequence's keys are cut into fixed chunks of CHUNK_PAGES pages at ABSOLUTE
//     positions [c*CHUNK, (c+1)*CHUNK);
//   * sequences whose chunk c maps to the SAME physical pages (a cross-model shared
//     prefix) are grouped into one work item, so each shared page is staged into shared
//     memory once and reused by the encoder and every adapter's decoder queries;
//   * a work item x one KV head = one CTA; up to 64 query rows (4 warps x 16).
// Per (row, head, chunk) the kernel emits an unnormalised partial (o, m, l) -- m in the log2
// domain (scores scaled by log2 e, exp2 throughout); the merge
// kernel folds chunks 0..last in fixed order. Partials depend only on the row's own query, the chunk's keys and the row's position, never on which other rows share the
// CTA -- the batch-invariance the reference gets from its per-head loop (2H == H||H,
// tests/test_model.py:225-239) and that makes prefill / decode KV bytes identical.
#include <algorithm>
#include <cstdlib>

#include "attn_merge.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace icr {

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4],
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Row-major [rows][HD] bf16 tile with 16-byte chunks XOR-swizzled by (row & 7):
// conflict-free ldmatrix for both K (non-trans) and V (trans) reads.
template <int HD>
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * HD * 2 + ((chunk ^ (row & 7)) << 4));
}

constexpr int PAGE_STAGES = 16;  // K/V pages in flight per CTA (TMA ring, 8 KB each)
constexpr int ATTN_THREADS = 288;  // warp 0: TMA producer; warps 1..8: consumers

template <int HD>
__host__ __device__ constexpr uint32_t page_bytes() { return 16 * HD * 2; }  // one K (or V) page of one head
template <int HD>
constexpr size_t attn_smem() {
  return 1024 + (size_t)PAGE_STAGES * 2 * page_bytes<HD>() + (size_t)64 * HD * 2 + 256;
}

// Page tile in smem as written by TMA with 128-byte swizzle: HD/64 halves of [16 keys][128 B],
// 16-byte chunk c of key row r at (c ^ (r & 7)) -- exactly what ldmatrix reads conflict-free.
template <int HD>
__device__ __forceinline__ uint32_t page_off(int key, int ch) {
  return (uint32_t)((ch >> 3) * 2048 + key * 128 + (((ch & 7) ^ (key & 7)) << 4));
}

// Warp-specialised shared-page attention. The producer warp streams each page of the chunk
// (K and V for this KV head) into a PAGE_STAGES-deep smem ring with TMA; 8 consumer warps
// -- 4 query-row groups x 2 page parities -- read every staged page for ALL rows of the
// item (the encoder and decoder heads of every sequence sharing the pages), with per-stage
// mbarriers instead of block barriers. The two page-parity states are combined at the end
// in a fixed order, so a row's partial depends only on its own query, the chunk's keys and
// its position.
template <int HD>
__global__ void __launch_bounds__(ATTN_THREADS, 1)
    attn_partial_kernel(const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const __nv_bfloat16* __restrict__ q,
                        int q_ld, int num_kv_heads, int group, const AttnItem* __restrict__ items,
                        const int* __restrict__ item_pages, const int2* __restrict__ item_rows,
                        const int* __restrict__ row_pos, int num_heads, int max_chunks, float scale,
                        float* __restrict__ part_o, float2* __restrict__ part_ml,
                        const int* __restrict__ n_items_dev, const uint8_t* __restrict__ pf_base,
                        long long pf_bytes, unsigned long long* __restrict__ trace) {
  constexpr int CH = HD / 8;  // 16-byte chunks per row
  constexpr uint32_t PB = page_bytes<HD>();
  extern __shared__ uint8_t attn_smem_raw[];
  const int cta_id = blockIdx.y * gridDim.x + blockIdx.x;
  if (trace != nullptr && threadIdx.x == 0 && cta_id < 4096)
    trace[(size_t)cta_id * 16 + 6] = globaltimer();
  if (trace != nullptr && threadIdx.x == 0 && cta_id < 4096) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    trace[(size_t)cta_id * 16 + 8] = smid + 1;
  }
  uint8_t* base = attn_smem_raw + ((1024 - (smem_u32(attn_smem_raw) & 1023)) & 1023);
  uint8_t* ring = base;                                   // [stage][K | V] pages
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(ring + PAGE_STAGES * 2 * PB);
  uint64_t* full = reinterpret_cast<uint64_t*>(sQ + 64 * HD);
  uint64_t* empty = full + PAGE_STAGES;

  // attention moves few bytes: use the idle HBM to pull the o-projection weights into L2
  prefetch_slice_l2(pf_base, pf_bytes, blockIdx.y * gridDim.x + blockIdx.x, gridDim.x * gridDim.y);
  pdl_launch();
  const int item_id = blockIdx.y;  // grid (KV head, item): long items' heads in the first wave
  if (item_id >= *n_items_dev) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < PAGE_STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 4); }
    fence_barrier_init();
  }
  __syncthreads();
  // the plan (items, pages) was uploaded before the forward: readable before the wait
  const AttnItem it = items[item_id];
  const int g = blockIdx.x;

  if (warp == 0) {
    // ---------------- producer: TMA page ring ----------------
    if (elect_one()) {
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      // pages written by earlier steps stream in while the q/k/v GEMM is still finishing
      const int pre = min(it.n_pre, PAGE_STAGES);
      for (int pi = 0; pi < it.n_pages; ++pi) {
        if (pi == pre) {
          pdl_wait();
          if (trace != nullptr && cta_id < 4096) trace[(size_t)cta_id * 16 + 7] = globaltimer();
        }
        const int st = pi % PAGE_STAGES;
        mbar_wait(&empty[st], ((pi / PAGE_STAGES) & 1) ^ 1);
        const int plane = item_pages[it.page_off + pi] * num_kv_heads + g;
        uint8_t* kd = ring + (size_t)st * 2 * PB;
        mbar_expect_tx(&full[st], 2 * PB);
#pragma unroll
        for (int h = 0; h < HD / 64; ++h) {
          tma_load_4d(kd + h * 2048, &tm_k, &full[st], 0, 0, h, plane);
          tma_load_4d(kd + PB + h * 2048, &tm_v, &full[st], 0, 0, h, plane);
        }
      }
      if (it.n_pages <= pre) pdl_wait();
    }
    return;
  }

  // ---------------- consumers ----------------
  pdl_wait();  // q comes from the q/k/v GEMM
  const int cw = warp - 1, rg = cw & 3, kg = cw >> 2;
  const int ctid = tid - 32;
  for (int idx = ctid; idx < 64 * CH; idx += 256) {
    const int row = idx / CH, ch = idx % CH;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (row < it.n_rows) {
      const int2 rr = item_rows[it.row_off + row];
      const int head = g * group + rr.y;
      val = *reinterpret_cast<const uint4*>(q + (size_t)rr.x * q_ld + head * HD + ch * 8);
    }
    *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sQ) + swz<HD>(row, ch)) = val;
  }
  named_bar_sync(1, 256);

  const int r_lo = rg * 16 + (lane >> 2);  // rows r_lo and r_lo + 8 of the item
  const bool active = rg * 16 < it.n_rows;
  int pos_lo = -1, pos_hi = -1;
  if (r_lo < it.n_rows) pos_lo = row_pos[item_rows[it.row_off + r_lo].x];
  if (r_lo + 8 < it.n_rows) pos_hi = row_pos[item_rows[it.row_off + r_lo + 8].x];

  uint32_t qa[HD / 16][4];
  if (active) {
    const uint32_t qbase = smem_u32(sQ);
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      const int row = rg * 16 + (lane & 15);
      const int ch = kk * 2 + (lane >> 4);
      ldsm_x4(qbase + swz<HD>(row, ch), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
    }
  }

  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  // running max in the log2 domain (scores pre-multiplied by scale * log2(e))
  float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;
  const float sl2 = scale * 1.4426950408889634f;

  // Key groups of 4 pages (64 keys): group kb belongs to page parity kg = kb & 1.
  for (int kb = kg; kb * 4 < it.n_pages; kb += 2) {
    const int p0 = kb * 4;
    const int np = min(4, it.n_pages - p0);
    for (int j = 0; j < np; ++j) mbar_wait(&full[(p0 + j) % PAGE_STAGES], ((p0 + j) / PAGE_STAGES) & 1);
    if (active) {
      // S = Q K^T for up to 64 keys: 8 n8 tiles, independent accumulation chains
      float s[8][4];
#pragma unroll
      for (int t = 0; t < 8; ++t) s[t][0] = s[t][1] = s[t][2] = s[t][3] = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j < np) {
          const uint32_t kbase = smem_u32(ring + (size_t)((p0 + j) % PAGE_STAGES) * 2 * PB);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const int key = (lane & 7) + ((lane >> 4) << 3);
            const int ch = kk * 2 + ((lane >> 3) & 1);
            uint32_t b0, b1, b2, b3;
            ldsm_x4(kbase + page_off<HD>(key, ch), b0, b1, b2, b3);
            mma_bf16_16816(s[2 * j], qa[kk], b0, b1);
            mma_bf16_16816(s[2 * j + 1], qa[kk], b2, b3);
          }
        }
      }
      // scale into the log2 domain, mask (src/model.py:415-423), block row max
      const int kpos0 = it.chunk_start + p0 * 16;
      float mx_lo = m_lo, mx_hi = m_hi;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int kp = kpos0 + t * 8 + (lane & 3) * 2 + e;
          const bool inb = t < 2 * np;
          float a = __fmul_rn(s[t][e], sl2);
          float b = __fmul_rn(s[t][2 + e], sl2);
          a = (inb && kp <= pos_lo) ? a : -INFINITY;
          b = (inb && kp <= pos_hi) ? b : -INFINITY;
          s[t][e] = a;
          s[t][2 + e] = b;
          mx_lo = fmaxf(mx_lo, a);
          mx_hi = fmaxf(mx_hi, b);
        }
      }
      mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
      mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
      mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
      mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
      const float corr_lo = (mx_lo == -INFINITY) ? 1.f : exp2f(m_lo - mx_lo);
      const float corr_hi = (mx_hi == -INFINITY) ? 1.f : exp2f(m_hi - mx_hi);
      float sum_lo = 0.f, sum_hi = 0.f;
      uint32_t pa[4][4];  // P as bf16 A-fragments, one per 16-key page
#pragma unroll
      for (int t = 0; t < 8; ++t) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float a = (s[t][e] == -INFINITY) ? 0.f : exp2f(s[t][e] - mx_lo);
          const float b = (s[t][2 + e] == -INFINITY) ? 0.f : exp2f(s[t][2 + e] - mx_hi);
          s[t][e] = a;
          s[t][2 + e] = b;
          sum_lo += a;
          sum_hi += b;
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        pa[j][0] = pack_bf16(s[2 * j][0], s[2 * j][1]);
        pa[j][1] = pack_bf16(s[2 * j][2], s[2 * j][3]);
        pa[j][2] = pack_bf16(s[2 * j + 1][0], s[2 * j + 1][1]);
        pa[j][3] = pack_bf16(s[2 * j + 1][2], s[2 * j + 1][3]);
      }
      sum_lo += __shfl_xor_sync(0xffffffffu, sum_lo, 1);
      sum_lo += __shfl_xor_sync(0xffffffffu, sum_lo, 2);
      sum_hi += __shfl_xor_sync(0xffffffffu, sum_hi, 1);
      sum_hi += __shfl_xor_sync(0xffffffffu, sum_hi, 2);
      l_lo = l_lo * corr_lo + sum_lo;
      l_hi = l_hi * corr_hi + sum_hi;
      m_lo = mx_lo;
      m_hi = mx_hi;
      // rescale O only when some row's running max moved (rare on long contexts)
      if (__any_sync(0xffffffffu, corr_lo != 1.f || corr_hi != 1.f)) {
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
          o[i][0] *= corr_lo; o[i][1] *= corr_lo;
          o[i][2] *= corr_hi; o[i][3] *= corr_hi;
        }
      }
      // O += P V, page by page
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j < np) {
          const uint32_t vbase = smem_u32(ring + (size_t)((p0 + j) % PAGE_STAGES) * 2 * PB) + PB;
#pragma unroll
          for (int dt = 0; dt < HD / 16; ++dt) {
            const int key = (lane & 7) + (((lane >> 3) & 1) << 3);
            const int ch = dt * 2 + (lane >> 4);
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(vbase + page_off<HD>(key, ch), b0, b1, b2, b3);
            mma_bf16_16816(o[dt * 2], pa[j], b0, b1);
            mma_bf16_16816(o[dt * 2 + 1], pa[j], b2, b3);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0)
      for (int j = 0; j < np; ++j) mbar_arrive(&empty[(p0 + j) % PAGE_STAGES]);
  }

  // ---- combine the odd-page state into the even-page state (fixed order) ----
  named_bar_sync(1, 256);  // every consumer is done with the ring
  float* so = reinterpret_cast<float*>(ring);  // [64 rows][HD] from the odd-page warps
  float2* sml = reinterpret_cast<float2*>(so + 64 * HD);
  if (kg == 1 && active) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int r = r_lo + half * 8;
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) {
        const int col = i * 8 + (lane & 3) * 2;
        *reinterpret_cast<float2*>(so + r * HD + col) =
            half == 0 ? make_float2(o[i][0], o[i][1]) : make_float2(o[i][2], o[i][3]);
      }
      if ((lane & 3) == 0) sml[r] = half == 0 ? make_float2(m_lo, l_lo) : make_float2(m_hi, l_hi);
    }
  }
  named_bar_sync(1, 256);
  if (trace != nullptr && tid == 32 && cta_id < 4096) trace[(size_t)cta_id * 16 + 5] = globaltimer();
  if (kg == 1 || !active) return;
  const int chunk = it.chunk_idx;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int r = r_lo + half * 8;
    if (r >= it.n_rows) continue;
    const float m0 = half == 0 ? m_lo : m_hi, l0 = half == 0 ? l_lo : l_hi;
    const float2 ml1 = sml[r];
    const float M = fmaxf(m0, ml1.x);
    const float w0 = (m0 == -INFINITY) ? 0.f : exp2f(m0 - M);
    const float w1 = (ml1.x == -INFINITY) ? 0.f : exp2f(ml1.x - M);
    const int2 rr = item_rows[it.row_off + r];
    const int head = g * group + rr.y;
    const size_t slot = ((size_t)rr.x * num_heads + head) * max_chunks + chunk;
    float* dst = part_o + slot * HD;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      const int col = i * 8 + (lane & 3) * 2;
      const float2 o1 = *reinterpret_cast<const float2*>(so + r * HD + col);
      const float a0 = half == 0 ? o[i][0] : o[i][2], a1 = half == 0 ? o[i][1] : o[i][3];
      *reinterpret_cast<float2*>(dst + col) =
          make_float2(fmaf(o1.x, w1, a0 * w0), fmaf(o1.y, w1, a1 * w0));
    }
    if ((lane & 3) == 0) part_ml[slot] = make_float2(M, fmaf(ml1.y, w1, l0 * w0));
  }
}

// Fixed-order merge of chunk partials (attn_merge.cuh) for the mma.sync path: one CTA per
// (row, KV group), one thread per (head-in-group, 4 dims), no shared memory. (The tcgen05
// partial kernel merges in-kernel with the same merge_unit.)
constexpr int MERGE_THREADS = 128;

template <int HD>
__global__ void __launch_bounds__(MERGE_THREADS)
    attn_merge_kernel(const float* __restrict__ part_o, const float2* __restrict__ part_ml,
                      const int* __restrict__ row_pos, const int* __restrict__ row_kind,
                      int num_heads, int group, int max_chunks, int chunk_tokens,
                      __nv_bfloat16* __restrict__ out, int out_ld,
                      unsigned long long* __restrict__ trace, unsigned long long* __restrict__ span) {
  const int cta_id = blockIdx.y * gridDim.x + blockIdx.x;
  if (trace != nullptr && threadIdx.x == 0 && cta_id < 4096) trace[(size_t)cta_id * 16 + 6] = globaltimer();
  pdl_launch();
  // the row table is uploaded before the forward: read it while the partials run
  const int kind = row_kind[blockIdx.x], nch = row_pos[blockIdx.x] / chunk_tokens + 1;
  pdl_wait();
  if (trace != nullptr && threadIdx.x == 0 && cta_id < 4096) trace[(size_t)cta_id * 16 + 7] = globaltimer();
  merge_unit<HD>(part_o, part_ml, kind, nch, blockIdx.x, blockIdx.y, num_heads, group, max_chunks,
                 out, out_ld, threadIdx.x, blockDim.x);
  if (trace != nullptr && threadIdx.x == 0 && cta_id < 4096) trace[(size_t)cta_id * 16 + 5] = globaltimer();
  if (span != nullptr) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(span + 1, globaltimer());
  }
}

static bool use_tc(int head_dim) {
  static const bool mma_only = getenv("ICR_ATTN_MMA") != nullptr;
  return head_dim == 128 && !mma_only;
}

int attn_entries_per_item(int head_dim) { return use_tc(head_dim) ? 128 : 64; }

template <int HD>
static cudaError_t attn_launch_hd(const AttnLaunch& a, cudaStream_t s) {
  if (use_tc(HD)) {
    cudaError_t e = attn_tc_partial_launch(a, a.chunk_tokens / 16, s);
    // long chunks (>= 32 pages) merge inside the partial kernel; short-chunk (decode)
    // launches keep the compact merge kernel: its small CTAs share SMs with the next GEMM's,
    // which streams its weights meanwhile (measured: in-kernel costs the C2 step +0.06 ms)
    if (e != cudaSuccess || a.chunk_tokens >= 32 * 16) return e;
    const int mthreads = std::min(MERGE_THREADS, ((a.group * HD / 4 + 31) / 32) * 32);
    return launch_pdl(attn_merge_kernel<HD>, dim3(a.n_rows, a.num_kv_heads), dim3(mthreads), 0, s,
                      a.part_o, a.part_ml, a.row_pos, a.row_kind, a.num_heads, a.group,
                      a.max_chunks, a.chunk_tokens, a.out, a.out_ld,
                      a.trace ? a.trace + 4096 * 16 : nullptr, a.span);
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_partial_kernel<HD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)attn_smem<HD>());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(a.num_kv_heads, a.n_items_cap);
  cudaError_t e = launch_pdl(attn_partial_kernel<HD>, grid, dim3(ATTN_THREADS), attn_smem<HD>(), s,
                             a.tm_k, a.tm_v, a.q, a.q_ld, a.num_kv_heads, a.group, a.items,
                             a.item_pages, a.item_rows, a.row_pos, a.num_heads, a.max_chunks,
                             a.scale, a.part_o, a.part_ml, a.n_items_dev, a.pf_base, a.pf_bytes, a.trace);
  if (e != cudaSuccess) return e;
  const int mthreads = std::min(MERGE_THREADS, ((a.group * HD / 4 + 31) / 32) * 32);
  return launch_pdl(attn_merge_kernel<HD>,
                    dim3(a.n_rows, a.num_kv_heads), dim3(mthreads), 0, s,
                    a.part_o, a.part_ml, a.row_pos, a.row_kind, a.num_heads, a.group,
                    a.max_chunks, a.chunk_tokens, a.out, a.out_ld,
                    a.trace ? a.trace + 4096 * 16 : nullptr, a.span);
}

cudaError_t attn_launch(const AttnLaunch& a, cudaStream_t s) {
  if (a.n_items_cap <= 0) return cudaSuccess;
  if (a.head_dim == 128) return attn_launch_hd<128>(a, s);
  if (a.head_dim == 64) return attn_launch_hd<64>(a, s);
  return cudaErrorInvalidValue;
}

}  // namespace icr
