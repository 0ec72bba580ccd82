// Shared-KV paged decode attention on the 5th-generation tensor cores (head_dim 128).
// Reference semantics: `layer_attention` (src/model.py:384-425) over the fused 2H query
// heads of `block_forward` decode (src/model.py:495-501): scores = (q . k) * 1/sqrt(hd) with
// the causal mask, softmax, weights @ V -- per (row, head), batch-invariant.
//
// One CTA = one work item (a chunk of <= MAXP pages at fixed absolute positions, shared by
// every sequence whose block table maps the same physical pages) x one KV head. The up to 128
// query entries (row, head-in-group) attached to those pages -- the encoder and decoder heads
// of every model sharing the prefix -- are the M = 128 rows of two tcgen05 MMAs:
//   S[128 x 16P]  = Q[128 x 128] . K[16P x 128]^T      (K-major Q and K, fp32 in TMEM)
//   softmax       : one epilogue thread per entry reads its S row from TMEM (exp2 domain,
//                   causal mask), writes P as bf16 into the SW128 K-major layout over the
//                   now-dead K buffer
//   O[128 x 128]  = P[128 x 16P] . V[16P x 128]         (V consumed MN-major, straight from
//                                                        the TMA-written pages)
// and the unnormalised partial (O, m, l) per (row, head, chunk) goes to the same fixed-order
// merge kernel as the mma.sync path. Each K/V page is staged in shared memory once per KV
// head for all entries: HBM bytes scale with context, not with the number of models.
#include "kernels.h"
#include "ptx.cuh"

namespace icr {

constexpr int TC_THREADS = 256;  // w0 TMA, w1 MMA + TMEM, w2-3 Q loaders, w4-7 softmax/epilogue
constexpr int TC_ROWS = 128;     // MMA M: query entries per item

template <int MAXP>
struct TcLayout {
  static constexpr uint32_t Q_BYTES = TC_ROWS * 256;            // 2 K-blocks x [128 x 128 B]
  static constexpr uint32_t HALF = MAXP * 16 * 128;             // one 64-dim half of K or V
  static constexpr uint32_t KV_BYTES = 2 * HALF;
  static constexpr uint32_t Q_OFF = 0, K_OFF = Q_BYTES, V_OFF = K_OFF + KV_BYTES;
  static constexpr uint32_t BAR_OFF = V_OFF + KV_BYTES;
  static constexpr size_t SMEM = 1024 + BAR_OFF + 64 + 2 * 128 * 4;
  static constexpr uint32_t S_COLS = MAXP * 16;
  static constexpr uint32_t TMEM_COLS = (S_COLS + 128) <= 256 ? 256 : 512;
};

// MN-major, 128-byte-swizzle shared-memory descriptor (B operand of P.V): 64 consecutive
// N elements (one 128-byte row) per K index, 8 K rows per 1024-byte atom; SBO = bytes
// between 8-row K groups, LBO = bytes between 64-element N blocks.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint64_t sdesc_mnmajor_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

template <int MAXP>
__global__ void __launch_bounds__(TC_THREADS, MAXP <= 8 ? 2 : 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                   const __nv_bfloat16* __restrict__ q, int q_ld, int num_kv_heads, int group,
                   const AttnItem* __restrict__ items, const int* __restrict__ item_pages,
                   const int2* __restrict__ item_rows, const int* __restrict__ row_pos,
                   int num_heads, int max_chunks, float scale, float* __restrict__ part_o,
                   float2* __restrict__ part_ml, const int* __restrict__ n_items_dev,
                   unsigned long long* __restrict__ trace) {
  using L = TcLayout<MAXP>;
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* smem = tc_smem_raw + ((1024 - (smem_u32(tc_smem_raw) & 1023)) & 1023);
  uint8_t* sQ = smem + L::Q_OFF;
  uint8_t* sK = smem + L::K_OFF;  // becomes P after the S MMA has read it
  uint8_t* sV = smem + L::V_OFF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = bars + 2;
  uint64_t* s_full = bars + 3;
  uint64_t* o_full = bars + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6);

  const int cta_id = blockIdx.y * gridDim.x + blockIdx.x;
  auto stamp = [&](int k) {
    if (trace != nullptr && cta_id < 4096) trace[(size_t)cta_id * 16 + k] = globaltimer();
  };
  if (threadIdx.x == 0) stamp(6);
  pdl_launch();
  const int item_id = blockIdx.x;
  if (item_id >= *n_items_dev) return;
  const int warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    mbar_init(q_full, 192);
    mbar_init(k_full, 1);
    mbar_init(v_full, 1);
    mbar_init(s_full, 1);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<L::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_s = *tmem_slot;
  const uint32_t tmem_o = tmem_s + L::S_COLS;
  const AttnItem it = items[item_id];  // uploaded before the forward
  const int g = blockIdx.y;
  const int np = it.n_pages;

  if (warp == 0) {
    // ---------------- producer: K and V pages of this KV head ----------------
    if (elect_one()) {
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      mbar_expect_tx(k_full, (uint32_t)np * 2 * 2048);
      mbar_expect_tx(v_full, (uint32_t)np * 2 * 2048);
      const int pre = it.n_pre;  // pages no kernel of this forward writes
      for (int pi = 0; pi < np; ++pi) {
        if (pi == pre) {
          pdl_wait();
          stamp(7);
        }
        const int plane = item_pages[it.page_off + pi] * num_kv_heads + g;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tma_load_3d(sK + h * L::HALF + pi * 2048, &tm_k, k_full, h * 64, 0, plane);
          tma_load_3d(sV + h * L::HALF + pi * 2048, &tm_v, v_full, h * 64, 0, plane);
        }
      }
      if (np <= pre) pdl_wait();
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- S = Q K^T ----------------
    mbar_wait(q_full, 0);
    if (lane == 0) stamp(1);
    mbar_wait(k_full, 0);
    if (lane == 0) stamp(2);
    tc_fence_after();
    if (elect_one()) {
      const uint32_t idesc_s = idesc_bf16_f32(TC_ROWS, (uint32_t)np * 16);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t a = smem_u32(sQ) + (kk >> 2) * (TC_ROWS * 128) + (kk & 3) * 32;
        const uint32_t b = smem_u32(sK) + (kk >> 2) * L::HALF + (kk & 3) * 32;
        tc_mma_bf16(tmem_s, sdesc_kmajor_sw128(a), sdesc_kmajor_sw128(b), idesc_s, kk > 0 ? 1u : 0u);
      }
      tc_commit(s_full);
    }
    __syncwarp();
  } else {
    // ---------------- Q gather (warps 2-7) ----------------
    pdl_wait();  // q comes from the q/k/v GEMM
    const int t = threadIdx.x - 64;  // 0..191
    // entry e sits in M row / TMEM lane r(e) = (e % 4) * 32 + e / 4, so the entries of a
    // partly filled item spread over all four lane quarters
    for (int idx = t; idx < TC_ROWS * 16; idx += 192) {
      const int e = idx >> 4, c = idx & 15;
      const int r = (e & 3) * 32 + (e >> 2);
      uint4 val = make_uint4(0, 0, 0, 0);
      if (e < it.n_rows) {
        const int2 rr = item_rows[it.row_off + e];
        val = *reinterpret_cast<const uint4*>(q + (size_t)rr.x * q_ld + (g * group + rr.y) * 128 + c * 8);
      }
      *reinterpret_cast<uint4*>(sQ + (c >> 3) * (TC_ROWS * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = val;
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_arrive(q_full);
  }

  // ---------------- softmax on all 8 warps ----------------
  // TMEM lane quarter w % 4 is readable by warps w and w + 4: each row's key columns are split
  // between the two (16-column groups [0, h) and [h, np)); row max and sum are combined through
  // shared memory in a fixed order.
  float* red = reinterpret_cast<float*>(bars + 8);  // [2][128] partial max, then partial sum
  const int r = (warp & 3) * 32 + lane;             // TMEM lane = M row
  const int e = (r & 31) * 4 + (r >> 5);            // the query entry held in that row
  const int half = warp >> 2;
  const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
  const bool valid = e < it.n_rows;
  int2 rr = make_int2(0, 0);
  int pos = -1;
  if (valid) {
    rr = item_rows[it.row_off + e];
    pos = row_pos[rr.x];
  }
  const float sl2 = scale * 1.4426950408889634f;
  const int hsplit = (np + 1) >> 1;
  const int c_lo = half == 0 ? 0 : hsplit * 16, c_hi = half == 0 ? hsplit * 16 : np * 16;
  mbar_wait(s_full, 0);
  tc_fence_after();
  if (r == 0 && half == 1) stamp(3);
  float m = -INFINITY;
  for (int c0 = c_lo; c0 < c_hi; c0 += 64) {
    uint32_t v[4][16];
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4)
      if (c0 + q4 * 16 < c_hi) tmem_ld16_nowait(tmem_s + lane_base + c0 + q4 * 16, v[q4]);
    tmem_wait_ld();
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      tmem_reg_fence(v[q4]);
      if (c0 + q4 * 16 < c_hi) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (it.chunk_start + c0 + q4 * 16 + j <= pos) m = fmaxf(m, __fmul_rn(__uint_as_float(v[q4][j]), sl2));
      }
    }
  }
  red[half * 128 + r] = m;
  named_bar_sync(1, TC_THREADS);
  m = fmaxf(red[r], red[128 + r]);
  named_bar_sync(1, TC_THREADS);  // red is reused for the sums
  // P = exp2(s - m) as bf16 into the K-major SW128 layout (over the dead K buffer)
  float l = 0.f;
  for (int c0 = c_lo; c0 < c_hi; c0 += 64) {
    uint32_t v[4][16];
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4)
      if (c0 + q4 * 16 < c_hi) tmem_ld16_nowait(tmem_s + lane_base + c0 + q4 * 16, v[q4]);
    tmem_wait_ld();
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      tmem_reg_fence(v[q4]);
      const int c = c0 + q4 * 16;
      if (c < c_hi) {
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          float p0 = 0.f, p1 = 0.f;
          if (it.chunk_start + c + j <= pos) p0 = ex2_approx(__fmul_rn(__uint_as_float(v[q4][j]), sl2) - m);
          if (it.chunk_start + c + j + 1 <= pos) p1 = ex2_approx(__fmul_rn(__uint_as_float(v[q4][j + 1]), sl2) - m);
          l += p0;
          l += p1;
          __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
          pk[j >> 1] = *reinterpret_cast<uint32_t*>(&h2);
        }
        const int blk = c >> 6, ch = (c & 63) >> 3;  // 64-key block, 8-key chunk
        uint8_t* rowp = sK + blk * (TC_ROWS * 128) + r * 128;
        *reinterpret_cast<uint4*>(rowp + (((ch) ^ (r & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(rowp + (((ch + 1) ^ (r & 7)) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  }
  red[half * 128 + r] = l;
  tc_fence_before();
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  named_bar_sync(1, TC_THREADS);
  if (r == 0 && half == 1) stamp(4);

  if (warp == 1) {
    // ---------------- O = P V ----------------
    mbar_wait(v_full, 0);
    tc_fence_after();
    if (elect_one()) {
      const uint32_t idesc_o = idesc_bf16_f32(TC_ROWS, 128) | (1u << 16);  // B (V) MN-major
      for (int kk = 0; kk < np; ++kk) {  // 16 keys (one page) per instruction
        const uint32_t a = smem_u32(sK) + (kk >> 2) * (TC_ROWS * 128) + (kk & 3) * 32;
        const uint32_t b = smem_u32(sV) + kk * 2048;
        tc_mma_bf16(tmem_o, sdesc_kmajor_sw128(a), sdesc_mnmajor_sw128(b, L::HALF, 1024), idesc_o,
                    kk > 0 ? 1u : 0u);
      }
      tc_commit(o_full);
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------- epilogue: unnormalised partial O and (m, l) per (row, head, chunk) ------
    l = red[r] + red[128 + r];
    mbar_wait(o_full, 0);
    tc_fence_after();
    if (r == 0) stamp(0);
    const size_t slot = valid ? ((size_t)rr.x * num_heads + g * group + rr.y) * max_chunks + it.chunk_idx : 0;
    float* dst = part_o + slot * 128;
#pragma unroll 1
    for (int c0 = 0; c0 < 128; c0 += 64) {
      uint32_t v[4][16];
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) tmem_ld16_nowait(tmem_o + lane_base + c0 + q4 * 16, v[q4]);
      tmem_wait_ld();
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        tmem_reg_fence(v[q4]);
        if (valid) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4*>(dst + c0 + q4 * 16 + j) =
                make_float4(__uint_as_float(v[q4][j]), __uint_as_float(v[q4][j + 1]),
                            __uint_as_float(v[q4][j + 2]), __uint_as_float(v[q4][j + 3]));
        }
      }
    }
    if (valid) part_ml[slot] = make_float2(m, l);
    if (r == 0) stamp(5);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<L::TMEM_COLS>(tmem_s);
}

template <int MAXP>
static cudaError_t launch_tc(const AttnLaunch& a, cudaStream_t s) {
  using L = TcLayout<MAXP>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<MAXP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(attn_tc_kernel<MAXP>, dim3(a.n_items_cap, a.num_kv_heads), dim3(TC_THREADS), L::SMEM, s,
                    a.tm_k, a.tm_v, a.q, a.q_ld, a.num_kv_heads, a.group, a.items, a.item_pages,
                    a.item_rows, a.row_pos, a.num_heads, a.max_chunks, a.scale, a.part_o, a.part_ml,
                    a.n_items_dev, a.trace);
}

cudaError_t attn_tc_partial_launch(const AttnLaunch& a, int chunk_pages, cudaStream_t s) {
  if (chunk_pages <= 8) return launch_tc<8>(a, s);
  if (chunk_pages <= 16) return launch_tc<16>(a, s);
  return cudaErrorInvalidValue;
}

}  // namespace icr
