// Standalone timing of the attention merge (tuning tool, not product code): C4 shape, 16 rows x
// 32 heads x 17 chunks of L2-resident partials, one CTA per (row, KV head) as the product
// launches it; %globaltimer span of the kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2603_13281_b200/csrc -o merge_probe merge_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "attn_merge.cuh"
using namespace icr;
__global__ void k(const float* po_, const float2* pml, int nch, int H, int G, int mc, __nv_bfloat16* out,
                  unsigned long long* span, int variant) {
  if (threadIdx.x == 0) atomicMin(span, globaltimer());
  if (variant == 0) {
    merge_unit<128>(po_, pml, 0, nch, blockIdx.x, blockIdx.y, H, G, mc, out, H * 128, threadIdx.x, blockDim.x);
  } else if (variant == 3) {  // branch-free fold: masked chunks weigh 0
    const int hg = threadIdx.x / 32, d = (threadIdx.x % 32) * 4, head = blockIdx.y * G + hg;
    const size_t base = ((size_t)blockIdx.x * H + head) * mc;
    float4 po[24]; float2 ml[24];
#pragma unroll
    for (int c = 0; c < 24; ++c) {
      const bool in = c < nch;
      po[c] = in ? __ldcg(reinterpret_cast<const float4*>(po_ + (base + c) * 128 + d)) : make_float4(0, 0, 0, 0);
      ml[c] = in ? __ldcg(&pml[base + c]) : make_float2(-INFINITY, 0.f);
    }
    float M = -INFINITY;
#pragma unroll
    for (int c = 0; c < 24; ++c) M = fmaxf(M, ml[c].x);
    float w[24];
#pragma unroll
    for (int c = 0; c < 24; ++c) w[c] = exp2f(ml[c].x - M);
    float L = 0.f; float4 O = make_float4(0, 0, 0, 0);
#pragma unroll
    for (int c = 0; c < 24; ++c) fold4(L, O, ml[c], po[c], M);
    store4<128>(out + (size_t)blockIdx.x * H * 128 + head * 128 + d, O, L);
  } else if (variant == 1) {  // the same loads, a plain sum
    const int hg = threadIdx.x / 32, d = (threadIdx.x % 32) * 4, head = blockIdx.y * G + hg;
    const size_t base = ((size_t)blockIdx.x * H + head) * mc;
    float4 acc = make_float4(0, 0, 0, 0); float l = 0;
    float4 v[24]; float2 m[24];
#pragma unroll
    for (int c = 0; c < 24; ++c) if (c < nch) { v[c] = __ldcg(reinterpret_cast<const float4*>(po_ + (base + c) * 128 + d)); m[c] = __ldcg(&pml[base + c]); }
#pragma unroll
    for (int c = 0; c < 24; ++c) if (c < nch) { acc.x += v[c].x; acc.y += v[c].y; acc.z += v[c].z; acc.w += v[c].w; l += m[c].y; }
    out[(size_t)blockIdx.x * H * 128 + head * 128 + d] = __float2bfloat16(acc.x + acc.y + acc.z + acc.w + l);
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(span + 1, globaltimer());
}
int main() {
  const int R = 16, H = 32, Hkv = 8, G = 4, NCH = 17, MC = 17;
  float* po; float2* pml; __nv_bfloat16* out; unsigned long long* sp;
  cudaMalloc(&po, (size_t)R * H * MC * 128 * 4); cudaMalloc(&pml, (size_t)R * H * MC * 8);
  cudaMalloc(&out, (size_t)R * H * 128 * 2); cudaMalloc(&sp, 16);
  cudaMemset(po, 0, (size_t)R * H * MC * 128 * 4); cudaMemset(pml, 0, (size_t)R * H * MC * 8);
  for (int it = 0; it < 16; ++it) {
    const int variant = it % 4;
    unsigned long long init[2] = {~0ull, 0};
    cudaMemcpy(sp, init, 16, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<dim3(R, Hkv), 128>>>(po, pml, NCH, H, G, MC, out, sp, variant);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[2]; cudaMemcpy(h, sp, 16, cudaMemcpyDeviceToHost);
    printf("variant %d: span %.2f us, events %.2f us\n", variant, (h[1] - h[0]) / 1000.0, ms * 1000);
  }
  return 0;
}
