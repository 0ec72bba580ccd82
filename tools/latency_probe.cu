// L2 round-trip latency under HBM streaming load (tuning tool, not product code).
// 148 CTAs: CTAs [0, n_lat) chase pointers through an L2-resident buffer (and time a global
// atomic), the others stream a 2 GB buffer with cp.async.bulk (like the weight-streaming GEMM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o latency_probe latency_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
constexpr int STAGES = 12, STAGE_BYTES = 16384;

__global__ void __launch_bounds__(128, 1)
    probe(const uint8_t* __restrict__ src, long long bytes, int n_lat, const int* __restrict__ chain,
          int* atom, long long* out, int streaming, int use_cg) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  if ((int)blockIdx.x < n_lat) {
    if (threadIdx.x != 0) return;
    // warm: touch the chain once
    int p = 0;
    for (int i = 0; i < 64; ++i) p = chain[p];
    __syncwarp(1);
    if (streaming) {  // let the streaming CTAs run for a while (TLB / queue pressure)
      const long long w = clock64();
      while (clock64() - w < 40000) {}
    }
    long long t0 = clock64();
    for (int i = 0; i < 64; ++i) p = use_cg ? __ldcg(chain + p) : *(volatile const int*)(chain + p);
    long long t1 = clock64();
    int v = 0;
    for (int i = 0; i < 16; ++i) v += atomicAdd(atom + blockIdx.x * 32, 1);
    long long t2 = clock64();
    out[blockIdx.x * 4 + 0] = (t1 - t0) / 64;
    out[blockIdx.x * 4 + 1] = (t2 - t1) / 16;
    out[blockIdx.x * 4 + 2] = p + v;
    return;
  }
  if (!streaming) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int G = gridDim.x - n_lat, c = blockIdx.x - n_lat;
  const long long units = bytes / STAGE_BYTES;
  const long long b = (long long)c * units / G, e = (long long)(c + 1) * units / G;
  const int warp = threadIdx.x >> 5;
  if (warp == 0 && (threadIdx.x & 31) == 0) {
    int st = 0;
    uint32_t ph = 0;
    for (long long u = b; u < e; ++u) {
      if (u - b >= STAGES)
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                         smem_u32(&empty[st])), "r"(ph ^ 1));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&full[st])),
                   "r"(STAGE_BYTES));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       smem_u32(sm + st * STAGE_BYTES)), "l"(src + u * STAGE_BYTES), "r"(STAGE_BYTES),
                   "r"(smem_u32(&full[st]))
                   : "memory");
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1 && (threadIdx.x & 31) == 0) {
    int st = 0;
    uint32_t ph = 0;
    for (long long u = b; u < e; ++u) {
      asm volatile("{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(
                       smem_u32(&full[st])), "r"(ph));
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[st])));
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
  }
}

int main() {
  const size_t total = 2ull << 30;
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  // pointer chains: (a) 4 KB stride within 1 MB; (b) one hop per 2 MB page over 256 MB
  const int N = 1 << 26;  // 256 MB of ints
  int* h = new int[N];
  for (int i = 0; i < N; ++i) h[i] = 0;
  const int small_n = 1 << 18;
  for (int i = 0; i < small_n; ++i) h[i] = (i + 1031) % small_n;
  int *chain, *atom;
  cudaMalloc(&chain, (size_t)N * sizeof(int));
  int* chain_far;
  {
    // far chain lives in the same allocation at offset 16 MB: hop = 2 MB + 4 KB, 64 hops
    const int base = 1 << 22, hop = (1 << 19) + 1024;
    for (int k = 0; k < 100; ++k) {
      const long long a = base + (long long)k * hop, b = base + (long long)(k + 1) * hop;
      if (b < N) h[a] = (int)(b - base);
    }
    chain_far = chain + base;
  }
  cudaMemcpy(chain, h, (size_t)N * sizeof(int), cudaMemcpyHostToDevice);
  cudaMalloc(&atom, 4096 * sizeof(int));
  cudaMemset(atom, 0, 4096 * sizeof(int));
  long long* out;
  cudaMalloc(&out, 4096 * sizeof(long long));
  const int smem = STAGES * STAGE_BYTES + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long ho[4096];
  for (int far = 0; far < 2; ++far)
  for (int streaming = 0; streaming < 2; ++streaming)
    for (int cg = 1; cg < 2; ++cg) {
      printf("%s chain: ", far ? "2MB-page-hopping" : "1MB-local");
      probe<<<148, 128, smem>>>(buf, 1ll << 30, 8, far ? chain_far : chain, atom, out, streaming, cg);
      cudaDeviceSynchronize();
      cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
      long long ld = 0, at = 0;
      for (int i = 0; i < 8; ++i) { ld += ho[i * 4]; at += ho[i * 4 + 1]; }
      printf("streaming=%d ld%s: L2 load latency %lld cycles, atomic %lld cycles (avg of 8 SMs)\n",
             streaming, cg ? ".cg" : ".volatile", ld / 8, at / 8);
    }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
