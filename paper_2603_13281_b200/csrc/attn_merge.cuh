// Fixed-order merge of per-chunk attention partials (O unnormalised, m in the log2 domain, l).
// Reference semantics: the single softmax over all keys of `layer_attention`
// (src/model.py:415-424) equals sum_c O_c 2^(m_c - M) / sum_c l_c 2^(m_c - M), M = max_c m_c.
//
// Two passes so the arithmetic never depends on how the loads are batched: pass 1 takes the
// exact maximum M (order-free), pass 2 folds the chunks in chunk order with fma against that M.
// Used by the tcgen05 attention kernel (merged in-kernel by its last CTAs) and by the
// standalone merge kernel of the mma.sync path -- the same function, so a row's output bits
// depend only on its own partials.
#pragma once
#include "ptx.cuh"

namespace icr {

// One thread: 4 consecutive dims [d, d + 4) of one (row, head); base = the slot of chunk 0.
template <int HD>
__device__ __forceinline__ void store4(__nv_bfloat16* dst, float4 O, float L) {
  // one correctly rounded reciprocal, four multiplies (no division slow paths on the tail)
  const float r = __frcp_rn(L);
  __nv_bfloat162 lo = __floats2bfloat162_rn(__fmul_rn(O.x, r), __fmul_rn(O.y, r));
  __nv_bfloat162 hi = __floats2bfloat162_rn(__fmul_rn(O.z, r), __fmul_rn(O.w, r));
  uint2 pk;
  pk.x = *reinterpret_cast<uint32_t*>(&lo);
  pk.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(dst) = pk;
}

__device__ __forceinline__ void fold4(float& L, float4& O, float2 ml, float4 po, float M) {
  // MUFU exp2 (~2 ulp; the partials' own softmax uses it): exp2(-inf) = 0 for absent chunks
  float w;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(w) : "f"(ml.x - M));
  L = fmaf(ml.y, w, L);
  O.x = fmaf(po.x, w, O.x);
  O.y = fmaf(po.y, w, O.y);
  O.z = fmaf(po.z, w, O.z);
  O.w = fmaf(po.w, w, O.w);
}

template <int HD>
__device__ __forceinline__ void merge_slice4(const float* __restrict__ part_o,
                                             const float2* __restrict__ part_ml, size_t base,
                                             int nch, int d, __nv_bfloat16* __restrict__ dst) {
  constexpr int B0 = 24, B1 = 16, B2 = 8;
  if (nch <= B0) {
    // the common case: every load in one round trip, then the same two passes in registers,
    // branch-free -- chunks past nch carry (m, l, O) = (-inf, 0, 0), i.e. weight exp2(-inf) = 0
    // and fma(0, 0, x) = x -- so the exponentials of all chunks issue back to back (measured:
    // the C4 merge 2.3 -> 1.6 us against a per-chunk branch around each fold)
    float2 ml[B0];
    float4 po[B0];
#pragma unroll
    for (int k = 0; k < B0; ++k) {
      const bool in = k < nch;
      ml[k] = in ? __ldcg(&part_ml[base + k]) : make_float2(-INFINITY, 0.f);
      po[k] = in ? __ldcg(reinterpret_cast<const float4*>(part_o + (base + k) * HD + d))
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float M = -INFINITY;
#pragma unroll
    for (int k = 0; k < B0; ++k) M = fmaxf(M, ml[k].x);
    float L = 0.f;
    float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < B0; ++k) fold4(L, O, ml[k], po[k], M);
    store4<HD>(dst, O, L);
    return;
  }
  float M = -INFINITY;
  for (int c0 = 0; c0 < nch; c0 += B1) {
    float mk[B1];
#pragma unroll
    for (int k = 0; k < B1; ++k) mk[k] = (c0 + k < nch) ? __ldcg(&part_ml[base + c0 + k]).x : -INFINITY;
#pragma unroll
    for (int k = 0; k < B1; ++k) M = fmaxf(M, mk[k]);
  }
  float L = 0.f;
  float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c0 = 0; c0 < nch; c0 += B2) {
    float2 ml[B2];
    float4 po[B2];
#pragma unroll
    for (int k = 0; k < B2; ++k) {
      const bool in = c0 + k < nch;
      ml[k] = in ? __ldcg(&part_ml[base + c0 + k]) : make_float2(-INFINITY, 0.f);
      po[k] = in ? __ldcg(reinterpret_cast<const float4*>(part_o + (base + c0 + k) * HD + d))
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < B2; ++k)
      if (c0 + k < nch) fold4(L, O, ml[k], po[k], M);
  }
  store4<HD>(dst, O, L);
}

// The merge of one (row r, KV group g) unit by `nthr` threads (thread lt): every head of the
// group, HD / 4 threads per head. Padding rows (kind < 0) have no output.
// (kind, nch = chunks of the row) come from the row table, which the caller may read early.
template <int HD>
__device__ __forceinline__ void merge_unit(const float* __restrict__ part_o,
                                           const float2* __restrict__ part_ml, int kind, int nch,
                                           int r, int g, int num_heads, int group, int max_chunks,
                                           __nv_bfloat16* __restrict__ out, int out_ld, int lt,
                                           int nthr) {
  if (kind < 0) return;
  constexpr int V = HD / 4;
  for (int idx = lt; idx < group * V; idx += nthr) {
    const int hg = idx / V, d = (idx % V) * 4;
    const int head = g * group + hg;
    const size_t base = ((size_t)r * num_heads + head) * max_chunks;
    merge_slice4<HD>(part_o, part_ml, base, nch, d, out + (size_t)r * out_ld + head * HD + d);
  }
}

}  // namespace icr
