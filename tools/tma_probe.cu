// Weight-streaming rate of TMA tensor boxes vs bulk copies (tuning tool, not product code).
// 148 CTAs stream a tile-major [tiles][128][64] bf16 matrix (16 KB per tile) through a
// 6-stage ring, like the decode GEMM's producer; variants: bulk copy, 3-D tensor box
// (128-byte swizzle), tensor box + a 2 KB activation box per stage, L2 evict-first hint.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_probe tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                   smem_u32(b)), "r"(ph));
}

constexpr int STAGES = 6, TILE = 16384, XB = 2048;

template <int MODE>  // 0 bulk, 1 tensor, 2 tensor + x, 3 bulk + evict_first, 4 tensor + evict_first
__global__ void __launch_bounds__(128, 1) stream(const __grid_constant__ CUtensorMap tw,
                                                 const __grid_constant__ CUtensorMap tx,
                                                 const uint8_t* __restrict__ w, long long tiles, long long toff, int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * (TILE + XB));
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const long long b = (long long)blockIdx.x * tiles / gridDim.x, e = (long long)(blockIdx.x + 1) * tiles / gridDim.x;
  const int warp = threadIdx.x >> 5;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  if (warp == 0 && (threadIdx.x & 31) == 0) {
    int st = 0;
    uint32_t ph = 0;
    for (long long u = b; u < e; ++u) {
      if (u - b >= STAGES) wait_bar(&empty[st], ph ^ 1);
      uint8_t* dst = sm + st * (TILE + XB);
      const uint32_t bytes = TILE + (MODE == 2 ? XB : 0);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&full[st])), "r"(bytes));
      if (MODE == 0)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         smem_u32(dst)), "l"(w + (u + toff) * TILE), "r"(TILE), "r"(smem_u32(&full[st]))
                     : "memory");
      else if (MODE == 3)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
                smem_u32(dst)), "l"(w + (u + toff) * TILE), "r"(TILE), "r"(smem_u32(&full[st])), "l"(pol)
            : "memory");
      else if (MODE == 4)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;\n" ::"r"(
                smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(&tw)), "r"(smem_u32(&full[st])), "r"(0), "r"(0), "r"((int)(u + toff)), "l"(pol)
            : "memory");
      else {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
                smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(&tw)), "r"(smem_u32(&full[st])), "r"(0), "r"(0), "r"((int)(u + toff))
            : "memory");
        if (MODE == 2)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
                  smem_u32(dst + TILE)), "l"(reinterpret_cast<uint64_t>(&tx)), "r"(smem_u32(&full[st])), "r"((int)(u % 64) * 64), "r"(0)
              : "memory");
      }
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1 && (threadIdx.x & 31) == 0) {
    int st = 0;
    uint32_t ph = 0, acc = 0;
    for (long long u = b; u < e; ++u) {
      wait_bar(&full[st], ph);
      acc += sm[st * (TILE + XB) + 7];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[st])));
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
    if (acc == 12345) out[0] = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  EncodeFn enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const long long tiles_per = 235ll * 1024 * 1024 / TILE;  // ~235 MB per launch (gate|up)
  const int nbuf = 8;
  const long long total_tiles = tiles_per * nbuf;
  uint8_t* w;
  cudaMalloc(&w, total_tiles * TILE);
  cudaMemset(w, 1, total_tiles * TILE);
  uint8_t* x;
  cudaMalloc(&x, 16 * 4096 * 2);
  cudaMemset(x, 1, 16 * 4096 * 2);
  int* out;
  cudaMalloc(&out, 64);
  CUtensorMap tw, tx;
  {
    cuuint64_t dims[3] = {64, 128, (cuuint64_t)total_tiles};
    cuuint64_t str[2] = {128, TILE};
    cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
    if (enc(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
      printf("encode w failed\n");
    cuuint64_t dx[2] = {4096, 16};
    cuuint64_t sx[1] = {4096 * 2};
    cuuint32_t bx[2] = {64, 16}, ex[2] = {1, 1};
    if (enc(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dx, sx, bx, ex, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
      printf("encode x failed\n");
  }
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int smem = STAGES * (TILE + XB) + 1024;
  void (*k[5])(CUtensorMap, CUtensorMap, const uint8_t*, long long, long long, int*) = {stream<0>, stream<1>, stream<2>, stream<3>, stream<4>};
  const char* names[5] = {"bulk 16KB", "tensor 3D box 16KB SW128", "tensor box + 2KB x box", "bulk + evict_first", "tensor + evict_first"};
  for (int m = 0; m < 5; ++m) {
    cudaFuncSetAttribute(k[m], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaGraph_t g;
    cudaGraphExec_t ex;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 32; ++i) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      // each launch streams a different 235 MB window (no L2 reuse); tensor variants index
      // tiles from the window start through a base offset folded into the tile coordinate
      const long long off = (i % nbuf) * tiles_per;
      cudaLaunchKernelEx(&cfg, k[m], tw, tx, (const uint8_t*)w, tiles_per, off, out);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ex, g, 0);
    cudaGraphLaunch(ex, s);
    cudaStreamSynchronize(s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ex, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / 32;
    printf("%-28s %8.2f us/launch  %7.0f GB/s\n", names[m], us, tiles_per * (double)TILE / (us * 1e-6) / 1e9);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("  error %s\n", cudaGetErrorString(e));
  }
  return 0;
}
