// Row-wise kernels of the decode step: embedding gather (+ RMSNorm statistics), LM-row
// gather, the cross-tile LM-head argmax, and the on-device greedy token feedback.
#include "kernels.h"
#include "ptx.cuh"

namespace icr {

int g_pdl = 1;

// One CTA (8 warps) per token row. Reference: gather_rows, src/tensor.py:321-332; the
// sums of squares feed rms_norm (src/tensor.py:217-246) inside the first projection GEMM.
// Warp w owns 128-feature chunks w, w+8, ...: no block barriers, all loads in flight.
__global__ void __launch_bounds__(256)
    embed_kernel(const int* __restrict__ tokens, const int* __restrict__ row_kind,
                 const __nv_bfloat16* __restrict__ embed, float* __restrict__ x,
                 __nv_bfloat16* __restrict__ xb, float* __restrict__ ssq, int ss_stride, int d,
                 const uint8_t* __restrict__ pf_base, long long pf_bytes,
                 __nv_bfloat16* __restrict__ ubd, int ubd_ld) {
  pdl_launch();
  prefetch_slice_l2(pf_base, pf_bytes, blockIdx.x, gridDim.x);
  pdl_wait();
  const int r = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the block-diagonal LoRA U row starts the step all zero (the shrinks fill own slots)
  for (int i = threadIdx.x * 8; i < ubd_ld; i += 256 * 8)
    *reinterpret_cast<uint4*>(ubd + (size_t)r * ubd_ld + i) = make_uint4(0, 0, 0, 0);
  const bool valid = row_kind[r] >= 0;
  const __nv_bfloat16* e = embed + (size_t)(valid ? tokens[r] : 0) * d;
  for (int c = w; c < d / 128; c += 8) {
    const int i = c * 128 + lane * 4;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (valid) {
      const uint2 raw = *reinterpret_cast<const uint2*>(e + i);
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
      const float2 a = __bfloat1622float2(h2[0]), b = __bfloat1622float2(h2[1]);
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
    *reinterpret_cast<float4*>(x + (size_t)r * d + i) = make_float4(v[0], v[1], v[2], v[3]);
    __nv_bfloat162 o0 = __floats2bfloat162_rn(v[0], v[1]), o1 = __floats2bfloat162_rn(v[2], v[3]);
    uint2 ob;
    ob.x = *reinterpret_cast<uint32_t*>(&o0);
    ob.y = *reinterpret_cast<uint32_t*>(&o1);
    *reinterpret_cast<uint2*>(xb + (size_t)r * d + i) = ob;
    float sq = __fadd_rn(__fadd_rn(__fmul_rn(v[0], v[0]), __fmul_rn(v[1], v[1])),
                         __fadd_rn(__fmul_rn(v[2], v[2]), __fmul_rn(v[3], v[3])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) ssq[(size_t)c * ss_stride + r] = sq;
  }
}

cudaError_t embed_launch(const int* tokens, const int* row_kind, const __nv_bfloat16* embed,
                         float* x, __nv_bfloat16* xb, float* ssq, int ss_stride, int n_rows,
                         int d, const uint8_t* pf_base, long long pf_bytes, __nv_bfloat16* ubd,
                         int ubd_ld, cudaStream_t s) {
  if (n_rows <= 0) return cudaSuccess;
  return launch_pdl(embed_kernel, dim3(n_rows), dim3(256), 0, s, tokens, row_kind, embed, x, xb,
                    ssq, ss_stride, d, pf_base, pf_bytes, ubd, ubd_ld);
}

// Layer input from an explicit fp32 residual stream (icr_layer_forward: the module-level
// block_forward / decoder_block_readonly of the reference, src/model.py:441-538): same outputs
// as embed_kernel -- x, xb = bf16(x), per-128-feature sums of squares, zeroed LoRA U row --
// so the layer's first GEMM sees exactly what it sees inside a full forward.
__global__ void __launch_bounds__(256)
    resid_load_kernel(const float* __restrict__ x_in, int n_valid, float* __restrict__ x,
                      __nv_bfloat16* __restrict__ xb, float* __restrict__ ssq, int ss_stride, int d,
                      __nv_bfloat16* __restrict__ ubd, int ubd_ld) {
  pdl_launch();
  pdl_wait();
  const int r = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x * 8; i < ubd_ld; i += 256 * 8)
    *reinterpret_cast<uint4*>(ubd + (size_t)r * ubd_ld + i) = make_uint4(0, 0, 0, 0);
  const bool valid = r < n_valid;
  for (int c = w; c < d / 128; c += 8) {
    const int i = c * 128 + lane * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) v = *reinterpret_cast<const float4*>(x_in + (size_t)r * d + i);
    *reinterpret_cast<float4*>(x + (size_t)r * d + i) = v;
    __nv_bfloat162 o0 = __floats2bfloat162_rn(v.x, v.y), o1 = __floats2bfloat162_rn(v.z, v.w);
    uint2 ob;
    ob.x = *reinterpret_cast<uint32_t*>(&o0);
    ob.y = *reinterpret_cast<uint32_t*>(&o1);
    *reinterpret_cast<uint2*>(xb + (size_t)r * d + i) = ob;
    float sq = __fadd_rn(__fadd_rn(__fmul_rn(v.x, v.x), __fmul_rn(v.y, v.y)),
                         __fadd_rn(__fmul_rn(v.z, v.z), __fmul_rn(v.w, v.w)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) ssq[(size_t)c * ss_stride + r] = sq;
  }
}

cudaError_t resid_load_launch(const float* x_in, int n_valid, int n_rows, float* x,
                              __nv_bfloat16* xb, float* ssq, int ss_stride, int d,
                              __nv_bfloat16* ubd, int ubd_ld, cudaStream_t s) {
  if (n_rows <= 0) return cudaSuccess;
  return launch_pdl(resid_load_kernel, dim3(n_rows), dim3(256), 0, s, x_in, n_valid, x, xb, ssq,
                    ss_stride, d, ubd, ubd_ld);
}

// LM-head input rows. hlm[i] = xb[src_i], ssq_lm[c][i] = ssq[c][src_i] for i < n_lm, zero rows
// up to n_pad. src_i = lm_rows[i] (a row of the forward) or, with from_store, a slot of the
// per-sequence hidden store (icr_seq_logits). store_slot[i] >= 0 additionally keeps row i's
// final hidden (+ its sums of squares) in the store: the last emitting row of each
// (sequence, row kind), from which session.last_logits is recomputed on demand -- bitwise the
// logits the forward would have produced (the same LM-head GEMM over the same inputs).
__global__ void __launch_bounds__(128)
    lm_gather_kernel(const __nv_bfloat16* __restrict__ xb, const float* __restrict__ ssq,
                     int ss_stride, const int* __restrict__ lm_rows, int n_lm, int n_pad, int d,
                     __nv_bfloat16* __restrict__ hlm, float* __restrict__ ssq_lm,
                     const int* __restrict__ store_slot, __nv_bfloat16* __restrict__ hid,
                     float* __restrict__ hid_ssq, int hid_stride, int from_store) {
  pdl_launch();
  pdl_wait();
  const int i = blockIdx.x, t = threadIdx.x;
  const bool valid = i < n_lm;
  const int src = valid ? lm_rows[i] : 0;
  const __nv_bfloat16* xsrc = from_store ? hid : xb;
  const float* ssrc = from_store ? hid_ssq : ssq;
  const int sstride = from_store ? hid_stride : ss_stride;
  const int keep = (valid && store_slot != nullptr) ? store_slot[i] : -1;
  for (int k = t * 8; k < d; k += 128 * 8) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (valid) v = *reinterpret_cast<const uint4*>(xsrc + (size_t)src * d + k);
    *reinterpret_cast<uint4*>(hlm + (size_t)i * d + k) = v;
    if (keep >= 0) *reinterpret_cast<uint4*>(hid + (size_t)keep * d + k) = v;
  }
  for (int c = t; c < d / 128; c += 128) {
    const float v = valid ? ssrc[(size_t)c * sstride + src] : 0.f;
    ssq_lm[(size_t)c * ss_stride + i] = v;
    if (keep >= 0) hid_ssq[(size_t)c * hid_stride + keep] = v;
  }
}

cudaError_t lm_gather_launch(const __nv_bfloat16* xb, const float* ssq, int ss_stride,
                             const int* lm_rows, int n_lm, int n_pad, int d, __nv_bfloat16* hlm,
                             float* ssq_lm, const int* store_slot, __nv_bfloat16* hid,
                             float* hid_ssq, int hid_stride, int from_store, cudaStream_t s) {
  if (n_pad <= 0) return cudaSuccess;
  return launch_pdl(lm_gather_kernel, dim3(n_pad), dim3(128), 0, s, xb, ssq, ss_stride, lm_rows,
                    n_lm, n_pad, d, hlm, ssq_lm, store_slot, hid, hid_ssq, hid_stride, from_store);
}

// One CTA per row. (value, index) is a total order (value desc, index asc), so the result
// is the first maximum regardless of scan order -- np.argmax semantics.
__device__ __forceinline__ void argmax_take(float& bv, int& bi, float ov, int oi) {
  if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
}
__global__ void __launch_bounds__(256)
    argmax_reduce_kernel(const float2* __restrict__ tile_best, int tiles, int stride, int n_rows,
                         int* __restrict__ out_tokens) {
  pdl_launch();
  pdl_wait();
  const int r = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  __shared__ float sv[8];
  __shared__ int si[8];
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int t = tid; t < tiles; t += 256) {
    const float2 e = tile_best[(size_t)t * stride + r];
    argmax_take(bv, bi, e.x, __float_as_int(e.y));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    argmax_take(bv, bi, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bi, o));
  if (lane == 0) { sv[tid >> 5] = bv; si[tid >> 5] = bi; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < 8; ++w) argmax_take(bv, bi, sv[w], si[w]);
    out_tokens[r] = bi;
  }
}

cudaError_t argmax_reduce_launch(const float2* tile_best, int tiles, int stride, int n_rows,
                                 int* out_tokens, cudaStream_t s) {
  if (n_rows <= 0) return cudaSuccess;
  return launch_pdl(argmax_reduce_kernel, dim3(n_rows), dim3(256), 0, s, tile_best, tiles, stride,
                    n_rows, out_tokens);
}

__global__ void feedback_kernel(int* tokens, const int* out_tok, const int* src, int n) {
  pdl_launch();
  pdl_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n && src[r] >= 0) tokens[r] = out_tok[src[r]];
}

cudaError_t feedback_launch(int* tokens, const int* out_tok, const int* src, int n,
                            cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(feedback_kernel, dim3((n + 127) / 128), dim3(128), 0, s, tokens, out_tok, src,
                    n);
}

}  // namespace icr
