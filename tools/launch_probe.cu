// Launch-overhead / streaming-ramp probe for the decode-step GEMM shape (tuning tool, not
// product code). Measures, back to back in one stream (and in a CUDA graph):
//   * an empty 148 x 256 kernel with ~1 KB of params at 0 / 208 KB dynamic smem, PDL on/off,
//     with and without a TMEM alloc/dealloc;
//   * a pure bulk-copy streaming kernel (cp.async.bulk global->smem ring, 8 x 16 KB stages,
//     one elected producer, 148 CTAs) over B bytes per launch, cycling through buffers larger
//     than L2 -- the per-launch ramp/drain cost of weight streaming at a given size.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o launch_probe launch_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

struct Big {
  unsigned char blob[960];
};

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <bool TMEM>
__global__ void __launch_bounds__(256, 1) empty_kernel(const __grid_constant__ Big b, int* out) {
  extern __shared__ uint8_t sm[];
  __shared__ uint32_t slot;
  pdl_launch();
  if (TMEM && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  __syncthreads();
  pdl_wait();
  if (threadIdx.x == 0 && b.blob[blockIdx.x & 511] == 7) out[blockIdx.x] = sm[0];
  __syncthreads();
  if (TMEM && threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(slot));
}

constexpr int STAGES = 12;
constexpr int STAGE_BYTES = 16384;

template <bool WAIT, bool TMEM>
__global__ void __launch_bounds__(128, 1)
    stream_kernel(const uint8_t* __restrict__ src, long long bytes, int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  if (TMEM && threadIdx.x >= 64 && threadIdx.x < 96) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_launch();
  const long long units = bytes / STAGE_BYTES;
  const long long b = (long long)blockIdx.x * units / gridDim.x;
  const long long e = (long long)(blockIdx.x + 1) * units / gridDim.x;
  const int warp = threadIdx.x >> 5;
  if (warp == 0 && (threadIdx.x & 31) == 0) {
    int st = 0;
    uint32_t ph = 0;
    for (long long u = b; u < e; ++u) {
      if (WAIT && u - b == STAGES) pdl_wait();
      if (u - b >= STAGES) {
        asm volatile(
            "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                smem_u32(&empty[st])),
            "r"(ph ^ 1));
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&full[st])),
                   "r"(STAGE_BYTES));
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              smem_u32(sm + st * STAGE_BYTES)),
          "l"(src + u * STAGE_BYTES), "r"(STAGE_BYTES), "r"(smem_u32(&full[st]))
          : "memory");
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1 && (threadIdx.x & 31) == 0) {
    int st = 0;
    uint32_t ph = 0;
    int acc = 0;
    for (long long u = b; u < e; ++u) {
      asm volatile(
          "{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(
              smem_u32(&full[st])),
          "r"(ph));
      acc += sm[st * STAGE_BYTES + 5];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[st])));
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
    if (acc == 123456) out[0] = acc;
  }
  __syncthreads();
  if (TMEM && threadIdx.x >= 64 && threadIdx.x < 96)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(tslot));
}

template <typename F>
static float time_launches(F launch, int n, cudaStream_t s, bool graph) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) launch(i);
  cudaStreamSynchronize(s);
  float ms = 0;
  if (graph) {
    cudaGraph_t g;
    cudaGraphExec_t ex;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < n; ++i) launch(i);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ex, g, 0);
    cudaGraphLaunch(ex, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ex, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(g);
  } else {
    cudaEventRecord(a, s);
    for (int i = 0; i < n; ++i) launch(i);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
  }
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return ms * 1e3f / n;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int* out;
  cudaMalloc(&out, 4096 * 4);
  Big big{};
  const int G = 148;
  for (int tmem = 0; tmem < 0; ++tmem)
    for (int smem_kb : {0, 208})
      for (int pdl = 0; pdl < 2; ++pdl)
        for (int graph = 0; graph < 2; ++graph) {
          auto k = tmem ? empty_kernel<true> : empty_kernel<false>;
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
          auto launch = [&](int) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(G);
            cfg.blockDim = dim3(256);
            cfg.dynamicSmemBytes = smem_kb * 1024;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = pdl;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k, big, out);
          };
          printf("empty tmem=%d smem=%3dKB pdl=%d graph=%d: %6.2f us/launch\n", tmem, smem_kb, pdl,
                 graph, time_launches(launch, 200, s, graph));
        }
  // streaming ramp: bytes per launch, buffers cycled over 2 GB (>> L2)
  const size_t total = 2ull << 30;
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  const int smem = STAGES * STAGE_BYTES + 1024;
  void (*kern[4])(const uint8_t*, long long, int*) = {stream_kernel<false, false>, stream_kernel<true, false>,
                                                      stream_kernel<false, true>, stream_kernel<true, true>};
  for (auto k : kern) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (long long mb : {8LL, 32LL, 117LL, 235LL}) {
    const long long bytes = mb << 20;
    const int nbuf = (int)(total / bytes);
    for (int variant = 0; variant < 4; ++variant)
      for (int pdl = 1, graph = 1; graph < 2; ++graph) {
        auto kk = kern[variant];
        auto launch = [&](int i) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(G);
          cfg.blockDim = dim3(128);
          cfg.dynamicSmemBytes = smem;
          cfg.stream = s;
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          attr[0].val.programmaticStreamSerializationAllowed = pdl;
          cfg.attrs = attr;
          cfg.numAttrs = 1;
          cudaLaunchKernelEx(&cfg, kk, (const uint8_t*)(buf + (size_t)(i % nbuf) * bytes),
                             bytes, out);
        };
        const float us = time_launches(launch, 64, s, graph);
        printf("stream %4lld MB wait=%d tmem=%d (pdl, graph): %8.2f us/launch  %7.0f GB/s\n", mb,
               variant & 1, variant >> 1, us, bytes / (us * 1e-6) / 1e9);
      }
  }
  return 0;
}
