// tcgen05 stream-K weight-streaming GEMM with fused decode-step epilogues.
// See gemm.cuh for the design notes and the reference ops this replaces.
#include "gemm.cuh"
#include "kernels.h"

namespace icr {

constexpr int BM = 128;  // MMA M (weight rows per tile)
constexpr int BK = 64;   // K elements per stage (one 128-byte swizzle row)
constexpr uint32_t W_BYTES = BM * BK * 2;

template <int NT>
struct Cfg {
  static constexpr uint32_t X_BYTES = NT * BK * 2;
  static constexpr uint32_t STAGE = W_BYTES + X_BYTES;
  static constexpr int STAGES_RAW = (200 * 1024) / STAGE;
  static constexpr int STAGES = STAGES_RAW > 16 ? 16 : STAGES_RAW;
  static constexpr uint32_t TMEM_COLS = NT < 32 ? 32 : NT;
  static constexpr uint32_t IDESC = idesc_bf16_f32(BM, NT);
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE + 512;
};

struct Split {
  long long U;
  int Ut, G;
  __device__ __host__ long long ubegin(int c) const { return (long long)c * U / G; }
  // largest CTA whose range contains unit x
  __device__ __host__ int owner(long long x) const { return (int)(((x + 1) * G - 1) / U); }
};

__device__ __forceinline__ float silu_ref(float g) {
  // Sign-split logistic as in src/tensor.py:199-214 (_sigmoid, silu).
  float z = expf(-fabsf(g));
  float sig = g >= 0.f ? __fdiv_rn(1.f, 1.f + z) : __fdiv_rn(z, 1.f + z);
  return __fmul_rn(g, sig);
}

template <int NT>
__device__ __forceinline__ void finalize16(const GemmParams& p, int tile, int n0, float (&v)[16],
                                           int ep_t, float* red_val, int* red_idx) {
  const int m = tile * BM + ep_t;
  // ---- LoRA expand on decoder rows (segmented by adapter slot) ----
  if (p.lora_b != nullptr && m < p.lora_m) {
    const int uidx = (p.mode == EPI_SILU) ? (m & 1) : 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int n = n0 + j;
      if (n >= p.n_rows || p.row_kind[n] != 1) continue;
      const int a = p.row_adapter[n];
      if (a < 0) continue;  // base decoder row (read-only replay): no adapter
      const __nv_bfloat16* b = p.lora_b + ((size_t)a * p.lora_m + m) * p.rank;
      const float* u = p.lora_u + ((size_t)n * p.n_u + uidx) * p.rank;
      float acc = 0.f;
      for (int r = 0; r < p.rank; r += 8) {
        uint4 raw = *reinterpret_cast<const uint4*>(b + r);
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 f = __bfloat1622float2(h2[q]);
          acc = fmaf(u[r + 2 * q], f.x, acc);
          acc = fmaf(u[r + 2 * q + 1], f.y, acc);
        }
      }
      v[j] += acc;
    }
  }

  switch (p.mode) {
    case EPI_F32: {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + j;
        if (n < p.n_rows) p.out_f32[(size_t)n * p.ld_out + m] = v[j];
      }
    } break;
    case EPI_RESID: {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + j;
        if (n < p.n_rows && p.row_kind[n] >= 0) {
          float* r = p.resid + (size_t)n * p.M + m;
          *r = __fadd_rn(*r, v[j]);
        }
      }
    } break;
    case EPI_SILU: {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float partner = __shfl_xor_sync(0xffffffffu, v[j], 1);
        const int n = n0 + j;
        if ((m & 1) == 0 && n < p.n_rows && p.row_kind[n] >= 0) {
          const float f = __fmul_rn(silu_ref(v[j]), partner);
          p.out_bf16[(size_t)n * (p.M >> 1) + (m >> 1)] = __float2bfloat16_rn(f);
        }
      }
    } break;
    case EPI_QKV: {
      const int hd = p.head_dim;
      const int region = m < p.q_dim ? 0 : (m < p.q_dim + p.kv_dim ? 1 : 2);
      const int base = region == 0 ? 0 : (region == 1 ? p.q_dim : p.q_dim + p.kv_dim);
      const int i = (m - base) % hd;
      const int head = (m - base) / hd;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float partner = __shfl_xor_sync(0xffffffffu, v[j], 1);
        const int n = n0 + j;
        if (n >= p.n_rows) continue;
        const int kind = p.row_kind[n];
        if (kind < 0) continue;
        const int pos = p.row_pos[n];
        float out = v[j];
        if (region < 2) {
          // Interleaved-pair RoPE, src/tensor.py:309-315.
          const float2 cs = p.rope[(size_t)pos * (hd >> 1) + (i >> 1)];
          if ((i & 1) == 0)
            out = __fsub_rn(__fmul_rn(v[j], cs.x), __fmul_rn(partner, cs.y));
          else
            out = __fadd_rn(__fmul_rn(partner, cs.y), __fmul_rn(v[j], cs.x));
        }
        if (region == 0) {
          p.out_bf16[(size_t)n * p.q_dim + m] = __float2bfloat16_rn(out);
        } else if (kind == 0) {
          // Encoder rows only: K/V for position pos into its page (src/model.py:486-494).
          const int seq = p.row_seq[n];
          const int page = p.block_table[(size_t)seq * p.bt_stride + (pos >> 4)];
          __nv_bfloat16* dst = (region == 1 ? p.k_pages : p.v_pages) +
                               (((size_t)page * p.num_kv_heads + head) * 16 + (pos & 15)) * hd + i;
          *dst = __float2bfloat16_rn(out);
        }
      }
    } break;
    case EPI_ARGMAX: {
      const int wq = ep_t >> 5, ln = ep_t & 31;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + j;
        float val = (m < p.m_valid && n < p.n_rows) ? v[j] : -INFINITY;
        int idx = m;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, val, o);
          const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
          if (ov > val || (ov == val && oi < idx)) { val = ov; idx = oi; }
        }
        if (ln == 0) { red_val[wq * 16 + j] = val; red_idx[wq * 16 + j] = idx; }
      }
      named_bar_sync(1, 128);
      if (ep_t < 16) {
        float val = red_val[ep_t];
        int idx = red_idx[ep_t];
        for (int w = 1; w < 4; ++w) {
          const float ov = red_val[w * 16 + ep_t];
          const int oi = red_idx[w * 16 + ep_t];
          if (ov > val || (ov == val && oi < idx)) { val = ov; idx = oi; }
        }
        const int n = n0 + ep_t;
        if (n < p.n_rows)
          p.tile_best[(size_t)tile * p.best_stride + n] = make_float2(val, __int_as_float(idx));
      }
      named_bar_sync(1, 128);
    } break;
    default:
      break;
  }
}

template <int NT>
__global__ void __launch_bounds__(256, 1)
    gemm_streamk_kernel(const __grid_constant__ CUtensorMap tm_w,
                        const __grid_constant__ CUtensorMap tm_x, const GemmParams p,
                        int x_row0) {
  using C = Cfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tmem_full = empty + C::STAGES;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);
  float* red_val = reinterpret_cast<float*>(flag + 4);
  int* red_idx = reinterpret_cast<int*>(red_val + 64);

  const int warp = warp_id();
  Split sp;
  sp.Ut = p.K / BK;
  sp.U = (long long)(p.M / BM) * sp.Ut;
  sp.G = gridDim.x;
  const int c = blockIdx.x;
  const long long u_begin = sp.ubegin(c), u_end = sp.ubegin(c + 1);
  const int t_first = (int)(u_begin / sp.Ut), t_last = (int)((u_end - 1) / sp.Ut);

  if (warp == 0 && elect_one()) {
    for (int i = 0; i < C::STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 128);
    fence_barrier_init();
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_x);
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = t_first; t <= t_last; ++t) {
        const long long t0 = (long long)t * sp.Ut;
        const int kb = (int)((u_begin > t0 ? u_begin : t0) - t0);
        const int ke = (int)((u_end < t0 + sp.Ut ? u_end : t0 + sp.Ut) - t0);
        for (int k = kb; k < ke; ++k) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + (size_t)stage * C::STAGE;
          mbar_expect_tx(&full[stage], C::STAGE);
          tma_load_2d_hint(st, &tm_w, &full[stage], k * BK, t * BM, pol);
          tma_load_2d(st + W_BYTES, &tm_x, &full[stage], k * BK, x_row0);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- tcgen05.mma issuer ----------------
    int stage = 0;
    uint32_t phase = 0, tphase = 0;
    for (int t = t_first; t <= t_last; ++t) {
      const long long t0 = (long long)t * sp.Ut;
      const int kb = (int)((u_begin > t0 ? u_begin : t0) - t0);
      const int ke = (int)((u_end < t0 + sp.Ut ? u_end : t0 + sp.Ut) - t0);
      mbar_wait(tmem_empty, tphase ^ 1);
      tc_fence_after();
      for (int k = kb; k < ke; ++k) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a = smem_u32(smem + (size_t)stage * C::STAGE);
          const uint32_t b = a + W_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            tc_mma_bf16(tmem_base, sdesc_kmajor_sw128(a + kk * 32), sdesc_kmajor_sw128(b + kk * 32),
                        C::IDESC, (k > kb || kk > 0) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          if (k == ke - 1) tc_commit(tmem_full);
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      tphase ^= 1;
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (TMEM -> registers -> global) ----------------
    const int ep_t = threadIdx.x - 128;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    uint32_t tphase = 0;
    for (int t = t_first; t <= t_last; ++t) {
      const long long t0 = (long long)t * sp.Ut;
      const int c_first = sp.owner(t0), c_last = sp.owner(t0 + sp.Ut - 1);
      const int nseg = c_last - c_first + 1;
      mbar_wait(tmem_full, tphase);
      tc_fence_after();
      if (nseg == 1) {
        for (int cc = 0; cc < NT / 16; ++cc) {
          float v[16];
          tmem_ld16(tmem_base + lane_base + cc * 16, v);
          finalize16<NT>(p, t, cc * 16, v, ep_t, red_val, red_idx);
        }
        tc_fence_before();
        mbar_arrive(tmem_empty);
      } else {
        const int slot = (t == t_first) ? 0 : 1;
        float* wsp = p.ws + (((size_t)c * 2 + slot) * NT) * BM;
        for (int cc = 0; cc < NT / 16; ++cc) {
          float v[16];
          tmem_ld16(tmem_base + lane_base + cc * 16, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) __stcg(wsp + (size_t)(cc * 16 + j) * BM + ep_t, v[j]);
        }
        tc_fence_before();
        mbar_arrive(tmem_empty);
        __threadfence();
        named_bar_sync(1, 128);
        if (ep_t == 0) *flag = atomicAdd(&p.counters[t], 1);
        named_bar_sync(1, 128);
        const bool last = (*flag == nseg - 1);
        named_bar_sync(1, 128);
        if (last) {
          __threadfence();
          for (int cc = 0; cc < NT / 16; ++cc) {
            float v[16];
            for (int s = 0; s < nseg; ++s) {
              const int cs = c_first + s;
              const int ts = (int)(sp.ubegin(cs) / sp.Ut);
              const int sl = (t == ts) ? 0 : 1;
              const float* src = p.ws + (((size_t)cs * 2 + sl) * NT) * BM;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float x = __ldcg(src + (size_t)(cc * 16 + j) * BM + ep_t);
                v[j] = (s == 0) ? x : __fadd_rn(v[j], x);
              }
            }
            finalize16<NT>(p, t, cc * 16, v, ep_t, red_val, red_idx);
          }
          if (ep_t == 0) p.counters[t] = 0;
        }
      }
      tphase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<C::TMEM_COLS>(tmem_base);
}

// ------------------------------------------------------------------ host side
template <int NT>
static cudaError_t launch_nt(const CUtensorMap& tw, const CUtensorMap& tx, const GemmParams& p,
                             int x_row0, int num_sms, cudaStream_t s) {
  using C = Cfg<NT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_streamk_kernel<NT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long U = (long long)(p.M / BM) * (p.K / BK);
  const int G = (int)(U < num_sms ? U : num_sms);
  gemm_streamk_kernel<NT><<<G, 256, C::SMEM, s>>>(tw, tx, p, x_row0);
  return cudaGetLastError();
}

int gemm_pick_nt(int rows) {
  if (rows <= 16) return 16;
  if (rows <= 32) return 32;
  if (rows <= 64) return 64;
  if (rows <= 128) return 128;
  return 256;
}

cudaError_t gemm_launch(const CUtensorMap& tw, const CUtensorMap& tx, const GemmParams& p,
                        int x_row0, int nt, int num_sms, cudaStream_t s) {
  switch (nt) {
    case 16: return launch_nt<16>(tw, tx, p, x_row0, num_sms, s);
    case 32: return launch_nt<32>(tw, tx, p, x_row0, num_sms, s);
    case 64: return launch_nt<64>(tw, tx, p, x_row0, num_sms, s);
    case 128: return launch_nt<128>(tw, tx, p, x_row0, num_sms, s);
    case 256: return launch_nt<256>(tw, tx, p, x_row0, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

size_t gemm_ws_floats(int num_sms) { return (size_t)num_sms * 2 * 256 * BM; }

}  // namespace icr
