// Row-wise kernels of the decode step: embedding gather + RMSNorm, LoRA shrink (SGMV),
// and the cross-tile LM-head argmax.
#include "kernels.h"
#include "ptx.cuh"

namespace icr {

// One CTA per token row. Reference: rms_norm, src/tensor.py:217-246 (gain folded into the
// next weight on upload, see runtime.cu); embedding gather, src/tensor.py:321-332.
__global__ void __launch_bounds__(256)
    rmsnorm_kernel(const float* __restrict__ x_in, const int* __restrict__ tokens,
                   const __nv_bfloat16* __restrict__ embed, float* __restrict__ x_out,
                   __nv_bfloat16* __restrict__ h_out, const int* __restrict__ row_kind,
                   const int* __restrict__ row_map, int d, float eps) {
  const int r = blockIdx.x;
  const int src_row = row_map != nullptr ? row_map[r] : r;
  const int tid = threadIdx.x;
  __shared__ float red[8];
  __nv_bfloat16* h = h_out + (size_t)r * d;
  if (row_kind != nullptr && row_kind[r] < 0) {
    for (int i = tid; i < d; i += 256) h[i] = __float2bfloat16_rn(0.f);
    return;
  }
  const float* x = x_in + (size_t)src_row * d;
  float* xo = x_out + (size_t)src_row * d;
  float ss = 0.f;
  if (embed != nullptr) {
    const __nv_bfloat16* e = embed + (size_t)tokens[src_row] * d;
    for (int i = tid; i < d; i += 256) {
      const float v = __bfloat162float(e[i]);
      xo[i] = v;
      ss = fmaf(v, v, ss);
    }
  } else {
    for (int i = tid; i < d; i += 256) {
      const float v = x[i];
      ss = fmaf(v, v, ss);
    }
  }
  ss = warp_sum(ss);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  __syncthreads();
  if (tid < 32) {
    float t = tid < 8 ? red[tid] : 0.f;
    t = warp_sum(t);
    if (tid == 0) red[0] = t;
  }
  __syncthreads();
  const float mean = __fdiv_rn(red[0], (float)d);
  const float inv = __fdiv_rn(1.f, sqrtf(__fadd_rn(mean, eps)));
  const float* src = embed != nullptr ? xo : x;
  for (int i = tid; i < d; i += 256) h[i] = __float2bfloat16_rn(__fmul_rn(src[i], inv));
}

cudaError_t rmsnorm_launch(const float* x_in, const int* tokens, const __nv_bfloat16* embed,
                           float* x_out, __nv_bfloat16* h_out, const int* row_kind,
                           const int* row_map, int n_rows, int d, float eps, cudaStream_t s) {
  if (n_rows <= 0) return cudaSuccess;
  rmsnorm_kernel<<<n_rows, 256, 0, s>>>(x_in, tokens, embed, x_out, h_out, row_kind, row_map, d,
                                        eps);
  return cudaGetLastError();
}

// grid = (rank, slots, n_targets). Each CTA owns one A row (adapter a, rank index j) and
// produces U[n][t][j] for every row of segment a (reference: _lowrank_delta's first
// product x @ A^T, src/model.py:340-343; A stored [rank, in] exactly as the reference).
constexpr int SHRINK_ROWS = 16;
__global__ void __launch_bounds__(256)
    lora_shrink_kernel(const __nv_bfloat16* __restrict__ h, int ld_h, int K,
                       const __nv_bfloat16* __restrict__ A0, const __nv_bfloat16* __restrict__ A1,
                       int n_targets, int rank, float scale, const int* __restrict__ seg_off,
                       const int* __restrict__ seg_rows, float* __restrict__ U) {
  const int j = blockIdx.x, a = blockIdx.y, t = blockIdx.z;
  const int r0 = seg_off[a], r1 = seg_off[a + 1];
  if (r0 == r1) return;
  const __nv_bfloat16* A = (t == 0 ? A0 : A1) + ((size_t)a * rank + j) * K;
  const int tid = threadIdx.x;
  __shared__ float red[8][SHRINK_ROWS];
  for (int rb = r0; rb < r1; rb += SHRINK_ROWS) {
    const int nr = min(SHRINK_ROWS, r1 - rb);
    float acc[SHRINK_ROWS];
#pragma unroll
    for (int i = 0; i < SHRINK_ROWS; ++i) acc[i] = 0.f;
    for (int k = tid * 8; k < K; k += 256 * 8) {
      const uint4 araw = *reinterpret_cast<const uint4*>(A + k);
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&araw);
      float af[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(a2[q]);
        af[2 * q] = f.x;
        af[2 * q + 1] = f.y;
      }
#pragma unroll
      for (int i = 0; i < SHRINK_ROWS; ++i) {
        if (i < nr) {
          const int n = seg_rows[rb + i];
          const uint4 hraw = *reinterpret_cast<const uint4*>(h + (size_t)n * ld_h + k);
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&hraw);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f = __bfloat1622float2(h2[q]);
            acc[i] = fmaf(f.x, af[2 * q], acc[i]);
            acc[i] = fmaf(f.y, af[2 * q + 1], acc[i]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < SHRINK_ROWS; ++i) {
      const float v = warp_sum(acc[i]);
      if ((tid & 31) == 0) red[tid >> 5][i] = v;
    }
    __syncthreads();
    if (tid < nr) {
      float v = 0.f;
      for (int w = 0; w < 8; ++w) v += red[w][tid];
      const int n = seg_rows[rb + tid];
      U[((size_t)n * n_targets + t) * rank + j] = __fmul_rn(v, scale);
    }
    __syncthreads();
  }
}

cudaError_t lora_shrink_launch(const __nv_bfloat16* h, int ld_h, int K, const __nv_bfloat16* A0,
                               const __nv_bfloat16* A1, int n_targets, int slots, int rank,
                               float scale, const int* seg_off, const int* seg_rows, float* U,
                               cudaStream_t s) {
  if (slots <= 0) return cudaSuccess;
  dim3 grid(rank, slots, n_targets);
  lora_shrink_kernel<<<grid, 256, 0, s>>>(h, ld_h, K, A0, A1, n_targets, rank, scale, seg_off,
                                          seg_rows, U);
  return cudaGetLastError();
}

// One warp per row. (value, index) is a total order (value desc, index asc), so the
// result is the first maximum regardless of scan order -- np.argmax semantics.
__global__ void argmax_reduce_kernel(const float2* __restrict__ tile_best, int tiles, int stride,
                                     int n_rows, int* __restrict__ out_tokens) {
  const int r = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n_rows) return;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int t = lane; t < tiles; t += 32) {
    const float2 e = tile_best[(size_t)t * stride + r];
    const int ei = __float_as_int(e.y);
    if (e.x > bv || (e.x == bv && ei < bi)) { bv = e.x; bi = ei; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if (lane == 0) out_tokens[r] = bi;
}

cudaError_t argmax_reduce_launch(const float2* tile_best, int tiles, int stride, int n_rows,
                                 int* out_tokens, cudaStream_t s) {
  if (n_rows <= 0) return cudaSuccess;
  argmax_reduce_kernel<<<(n_rows + 3) / 4, 128, 0, s>>>(tile_best, tiles, stride, n_rows,
                                                         out_tokens);
  return cudaGetLastError();
}

}  // namespace icr
