// tcgen05 stream-K weight-streaming GEMM with fused decode-step epilogues.
// See gemm.cuh for the design notes and the reference ops this replaces.
#include "gemm.cuh"
#include "kernels.h"

namespace icr {

constexpr int BM = 128;  // MMA M (weight rows per tile)
constexpr int BK = 64;   // K elements per stage (one 128-byte swizzle row)
constexpr uint32_t W_BYTES = BM * BK * 2;
constexpr int MAX_RANK = 32;
// stream-K scratch word that holds no published partial (an all-ones NaN: the tensor cores
// only ever produce the canonical 0x7fffffff NaN)
constexpr uint32_t WS_EMPTY = 0xFFFFFFFFu;
__device__ __forceinline__ bool ws_empty(const float4& x) {
  return (__float_as_uint(x.x) == WS_EMPTY) | (__float_as_uint(x.y) == WS_EMPTY) |
         (__float_as_uint(x.z) == WS_EMPTY) | (__float_as_uint(x.w) == WS_EMPTY);
}
// barriers, reduction scratch, staged row metadata and the LoRA U rows of the launch
template <int NT>
constexpr size_t aux_smem() {
  // + SGMV segment table: slots + 1 offsets and up to 256 row ids; + the residual epilogue's
  // per-warp sum-of-squares partials of every 16-column chunk (wide launches)
  return 2048 + (size_t)NT * 5 * 4 + (64 + 1 + 512) * 4 + (size_t)NT * 16;
}

template <int NT>
struct Cfg {
  static constexpr uint32_t X_BYTES = NT * BK * 2;
  static constexpr uint32_t STAGE = W_BYTES + X_BYTES;
  static constexpr int STAGES_RAW = (int)((220 * 1024 - aux_smem<NT>()) / STAGE);
  static constexpr int STAGES = STAGES_RAW > 16 ? 16 : STAGES_RAW;
  // two accumulator buffers of NT columns: a CTA's next (tile, row group) accumulates while
  // the epilogue drains the previous one
  static constexpr uint32_t TMEM_COLS = 2 * NT < 32 ? 32 : 2 * NT;
  static constexpr uint32_t IDESC = idesc_bf16_f32(BM, NT);
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE + aux_smem<NT>();
};

// Stream-K partition of U units over G CTAs. 32-bit arithmetic (the host guarantees
// U * (G + 1) < 2^32): 64-bit division is a ~100-instruction software sequence, and the
// epilogue's critical path evaluates these per tile and per reduced segment.
// Ring depth: 5 x (16 KB W + X) in flight per SM measured fastest for the decode step
// (3.594 ms vs 3.625 at 6 stages, 3.68 at 4 and 8; ICR_STAGES sweep); p.stages > 0 overrides.
constexpr int DEFAULT_STAGES = 5;
template <int NT>
__host__ __device__ constexpr int ring_stages(int requested) {
  const int want = requested > 0 ? requested : DEFAULT_STAGES;
  return want < Cfg<NT>::STAGES ? want : Cfg<NT>::STAGES;
}

struct Split {
  long long U;
  int Ut, G;
  __device__ __host__ long long ubegin(int c) const {
    return (long long)(((unsigned)c * (unsigned)U) / (unsigned)G);
  }
  // largest CTA whose range contains unit x
  __device__ __host__ int owner(long long x) const {
    return (int)(((unsigned)(x + 1) * (unsigned)G - 1u) / (unsigned)U);
  }
};

// Warp transpose-reduction of 16 per-lane values: 16 shuffles instead of 16 x 5. Returns in
// every lane the warp total of value index (lane >> 1) & 15. The tree for each index is fixed
// (independent of the other indices' values), so per-row sums stay batch-invariant.
__device__ __forceinline__ float warp_reduce16(const float (&v)[16], int lane) {
  float a8[8], a4[4], a2[2];
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float send = hi ? v[i] : v[8 + i];
      const float keep = hi ? v[8 + i] : v[i];
      a8[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 16));
    }
  }
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float send = hi ? a8[i] : a8[4 + i];
      const float keep = hi ? a8[4 + i] : a8[i];
      a4[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 8));
    }
  }
  {
    const bool hi = lane & 4;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float send = hi ? a4[i] : a4[2 + i];
      const float keep = hi ? a4[2 + i] : a4[i];
      a2[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 4));
    }
  }
  const bool hi = lane & 2;
  float a1 = __fadd_rn(hi ? a2[1] : a2[0], __shfl_xor_sync(0xffffffffu, hi ? a2[0] : a2[1], 2));
  return __fadd_rn(a1, __shfl_xor_sync(0xffffffffu, a1, 1));
}

// Same transpose pattern for (max value, lowest index) pairs; argmax with lowest-index ties is
// order independent, so the result equals a sequential scan (src/engine.py:75-76).
__device__ __forceinline__ void argmax_pick(float& v, int& i, float ov, int oi) {
  if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
}
__device__ __forceinline__ void warp_argmax16(const float (&v)[16], int idx, int lane, float& bv,
                                              int& bi) {
  float a8[8], a4[4], a2[2];
  int i8[8], i4[4], i2[2];
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float sv = hi ? v[i] : v[8 + i];
      a8[i] = hi ? v[8 + i] : v[i];
      i8[i] = idx;
      argmax_pick(a8[i], i8[i], __shfl_xor_sync(0xffffffffu, sv, 16), __shfl_xor_sync(0xffffffffu, idx, 16));
    }
  }
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float sv = hi ? a8[i] : a8[4 + i];
      const int si = hi ? i8[i] : i8[4 + i];
      a4[i] = hi ? a8[4 + i] : a8[i];
      i4[i] = hi ? i8[4 + i] : i8[i];
      argmax_pick(a4[i], i4[i], __shfl_xor_sync(0xffffffffu, sv, 8), __shfl_xor_sync(0xffffffffu, si, 8));
    }
  }
  {
    const bool hi = lane & 4;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float sv = hi ? a4[i] : a4[2 + i];
      const int si = hi ? i4[i] : i4[2 + i];
      a2[i] = hi ? a4[2 + i] : a4[i];
      i2[i] = hi ? i4[2 + i] : i4[i];
      argmax_pick(a2[i], i2[i], __shfl_xor_sync(0xffffffffu, sv, 4), __shfl_xor_sync(0xffffffffu, si, 4));
    }
  }
  const bool hi = lane & 2;
  bv = hi ? a2[1] : a2[0];
  bi = hi ? i2[1] : i2[0];
  argmax_pick(bv, bi, __shfl_xor_sync(0xffffffffu, hi ? a2[0] : a2[1], 2),
              __shfl_xor_sync(0xffffffffu, hi ? i2[0] : i2[1], 2));
  argmax_pick(bv, bi, __shfl_xor_sync(0xffffffffu, bv, 1), __shfl_xor_sync(0xffffffffu, bi, 1));
}

// Per-CTA shared state of the epilogue warps (16-byte aligned and sized: the row metadata
// that follows it is read as int4 vectors).
struct alignas(16) EpiShared {
  int flag;
  int shrink_ready;
  int fin_last;  // the epilogue's finalize decision for the CTA's last tile (helpers read it)
  float red_val[64];
  int red_idx[64];
};
// barriers (<= 16 stages) + TMEM slot, EpiShared, row metadata + SGMV table, helper EpiShared
static_assert((2 * 16 + 4) * 8 + 16 + 2 * sizeof(EpiShared) + (5 * 16 + 64 + 1 + 512 + 3) * 4 + 16 * 16 <=
                  aux_smem<16>(), "aux shared-memory layout overflows");


__device__ __forceinline__ float silu_ref(float g) {
  // Sign-split logistic as in src/tensor.py:199-214 (_sigmoid, silu): 1/(1+z) for g >= 0,
  // z/(1+z) otherwise, z = exp(-|g|) (never overflows). MUFU exp2 / reciprocal (a few f32
  // ulps, far below the bf16 rounding of the result): no division slow-path branch, so the
  // 16 rows of a finalize interleave instead of running one latency chain after another.
  const float z = __expf(-fabsf(g));
  const float sig = __fdividef(g >= 0.f ? 1.f : z, 1.f + z);
  return __fmul_rn(g, sig);
}

__device__ __forceinline__ void unpack8(const uint4& raw, float (&f)[8]) {
  const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 t = __bfloat1622float2(h2[q]);
    f[2 * q] = t.x;
    f[2 * q + 1] = t.y;
  }
}

// Row metadata staged in smem by the epilogue warps (after griddepcontrol.wait).
struct RowMeta {
  int* kind;
  int* ad;
  int* pos;
  int* kvoff;
  float* inv;
};

template <int NT, int MODE>
__device__ __forceinline__ void finalize16(const GemmParams& p, int row0, int n_rows, int tile, int n0,
                                           float (&v)[16], int ep_t, EpiShared& sh, const RowMeta& rm,
                                           int bar, const float* pre = nullptr,
                                           const float2* cs_pre = nullptr, float* ssq_part = nullptr) {
  const int m = tile * BM + ep_t;
  // row kinds of the 16 rows (-1: padding or beyond n_rows, staged that way)
  int kd[16];
#pragma unroll
  for (int j = 0; j < 16; j += 4) {
    const int4 k4 = *reinterpret_cast<const int4*>(rm.kind + n0 + j);
    kd[j] = k4.x; kd[j + 1] = k4.y; kd[j + 2] = k4.z; kd[j + 3] = k4.w;
  }
  // ---- RMSNorm of the input rows (X was the raw residual stream) ----
  if (p.in_ssq != nullptr) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __fmul_rn(v[j], rm.inv[n0 + j]);
  }
  if constexpr (MODE == EPI_F32) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + j;
        if (n < n_rows) p.out_f32[(size_t)(row0 + n) * p.ld_out + m] = v[j];
      }
  } else if constexpr (MODE == EPI_RESID) {
      // Every row's math first (16 independent chains the scheduler can interleave), then
      // the predicated stores: a per-row branch would serialise the rows' latencies.
      const int wq = ep_t >> 5, ln = ep_t & 31;
      float old[16], xn[16], sq[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + j;
        old[j] = pre != nullptr ? pre[j]
                 : kd[j] >= 0 ? __ldcg(p.resid + (size_t)(row0 + n) * p.M + m) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        xn[j] = __fadd_rn(old[j], v[j]);
        sq[j] = kd[j] >= 0 ? __fmul_rn(xn[j], xn[j]) : 0.f;
      }
      float* rp = p.resid + (size_t)(row0 + n0) * p.M + m;
      __nv_bfloat16* bp = p.resid_bf16 + (size_t)(row0 + n0) * p.M + m;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (kd[j] >= 0) {
          rp[(size_t)j * p.M] = xn[j];
          bp[(size_t)j * p.M] = __float2bfloat16_rn(xn[j]);
        }
      }
      const float wsum = warp_reduce16(sq, ln);
      if (ssq_part != nullptr) {
        // wide launches: the 4 warps' partials of every chunk are combined once, after the
        // last chunk (fin_chunks) -- no barrier pair per chunk
        if ((ln & 1) == 0) ssq_part[((n0 >> 4) * 4 + wq) * 16 + ((ln >> 1) & 15)] = wsum;
      } else {
        if ((ln & 1) == 0) sh.red_val[wq * 16 + ((ln >> 1) & 15)] = wsum;
        named_bar_sync(bar, 128);
        if (ep_t < 16) {
          const int n = n0 + ep_t;
          if (n < n_rows) {
            const float s = ((sh.red_val[ep_t] + sh.red_val[16 + ep_t]) + sh.red_val[32 + ep_t]) +
                            sh.red_val[48 + ep_t];
            p.out_ssq[(size_t)tile * p.ss_stride + row0 + n] = s;
          }
        }
        named_bar_sync(bar, 128);
      }
  } else if constexpr (MODE == EPI_SILU) {
      float f[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float partner = __shfl_xor_sync(0xffffffffu, v[j], 1);
        f[j] = __fmul_rn(silu_ref(v[j]), partner);
      }
      if ((m & 1) == 0) {
        __nv_bfloat16* op = p.out_bf16 + (size_t)(row0 + n0) * (p.M >> 1) + (m >> 1);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (kd[j] >= 0) op[(size_t)j * (p.M >> 1)] = __float2bfloat16_rn(f[j]);
      }
  } else if constexpr (MODE == EPI_QKV) {
      const int hd = p.head_dim;
      const int region = m < p.q_dim ? 0 : (m < p.q_dim + p.kv_dim ? 1 : 2);
      const int base = region == 0 ? 0 : (region == 1 ? p.q_dim : p.q_dim + p.kv_dim);
      const int i = (m - base) % hd;
      const int head = (m - base) / hd;
      // RoPE factors of all 16 rows loaded up front (one round trip, not one per row), or
      // already prefetched by the caller while the tile was streaming
      float2 csv[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + j;
        csv[j] = cs_pre != nullptr ? cs_pre[j]
                 : (region < 2 && kd[j] >= 0)
                     ? __ldg(p.rope + (size_t)rm.pos[n] * (hd >> 1) + (i >> 1))
                     : make_float2(1.f, 0.f);
      }
      float out[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float partner = __shfl_xor_sync(0xffffffffu, v[j], 1);
        // Interleaved-pair RoPE, src/tensor.py:309-315 (q and k only; v passes through).
        const float2 cs = csv[j];
        const float even = __fsub_rn(__fmul_rn(v[j], cs.x), __fmul_rn(partner, cs.y));
        const float odd = __fadd_rn(__fmul_rn(partner, cs.y), __fmul_rn(v[j], cs.x));
        out[j] = region == 2 ? v[j] : ((i & 1) == 0 ? even : odd);
      }
      if (region == 0) {
        __nv_bfloat16* qp = p.out_bf16 + (size_t)(row0 + n0) * p.q_dim + m;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (kd[j] >= 0) qp[(size_t)j * p.q_dim] = __float2bfloat16_rn(out[j]);
      } else {
        // Encoder rows only: K/V for position pos into its page (src/model.py:486-494).
        __nv_bfloat16* pages = (region == 1 ? p.k_pages : p.v_pages) + (size_t)head * 16 * hd + i;
        int ko[16];
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const int4 k4 = *reinterpret_cast<const int4*>(rm.kvoff + n0 + j);
          ko[j] = k4.x; ko[j + 1] = k4.y; ko[j + 2] = k4.z; ko[j + 3] = k4.w;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (kd[j] == 0) pages[ko[j]] = __float2bfloat16_rn(out[j]);
      }
  } else if constexpr (MODE == EPI_ARGMAX) {
      const int wq = ep_t >> 5, ln = ep_t & 31;
      float vals[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) vals[j] = (m < p.m_valid && n0 + j < n_rows) ? v[j] : -INFINITY;
      float bv;
      int bi;
      warp_argmax16(vals, m, ln, bv, bi);
      if ((ln & 1) == 0) { sh.red_val[wq * 16 + ((ln >> 1) & 15)] = bv; sh.red_idx[wq * 16 + ((ln >> 1) & 15)] = bi; }
      named_bar_sync(bar, 128);
      if (ep_t < 16) {
        float val = sh.red_val[ep_t];
        int idx = sh.red_idx[ep_t];
        for (int w = 1; w < 4; ++w) {
          const float ov = sh.red_val[w * 16 + ep_t];
          const int oi = sh.red_idx[w * 16 + ep_t];
          if (ov > val || (ov == val && oi < idx)) { val = ov; idx = oi; }
        }
        const int n = n0 + ep_t;
        if (n < n_rows)
          p.tile_best[(size_t)tile * p.best_stride + row0 + n] =
              make_float2(val, __int_as_float(idx));
      }
      named_bar_sync(bar, 128);
  }
}

// In-kernel LoRA shrink by the epilogue warps of all CTAs. A task is one adapter row
// (target t, slot a, rank index j) over one K slice of <= SHRINK_SLICE elements; all of
// a lane's loads for the slice are issued before use (one memory round trip). The warp
// that delivers a row's last slice folds the partials in slice order (deterministic).
// A task = one adapter row (target t, slot a, rank index j) over one K slice of SL elements
// (SL = 4096 when K fits: no cross-warp combine at all). The A slice of a warp's first task is
// loaded before griddepcontrol.wait (adapters do not depend on the previous kernel), so only
// the activation round trip remains on the critical path.
template <int SL>
struct ShrinkTask {
  static constexpr int NI = SL / 256;  // uint4 per lane
  uint4 a[NI];
};

// When the (target, slot, rank index) tasks are fewer than half the shrink warps (q, o:
// 128 tasks for 296 warps), each slot's decoder rows are split into rsplit contiguous parts
// handled by different warps -- every (row, j) dot is still computed whole by one warp
// (single-slice K only), so U's bits do not change.
template <int SL>
__device__ __forceinline__ int shrink_rsplit(const GemmParams& p, int nwarps, int n_dec) {
  const int splits = (p.sh_K + SL - 1) / SL;
  const int base = p.sh_targets * p.slots * p.rank * splits;
  const int rows_per_slot = n_dec / max(p.slots, 1);
  return splits > 1 ? 1 : max(1, min(min(8, rows_per_slot), nwarps / base));
}

template <int SL>
__device__ __forceinline__ int shrink_tasks_total(const GemmParams& p, int nwarps, int n_dec) {
  return p.sh_targets * p.slots * p.rank * ((p.sh_K + SL - 1) / SL) * shrink_rsplit<SL>(p, nwarps, n_dec);
}

template <int SL>
__device__ __forceinline__ void shrink_load_a(const GemmParams& p, int task, int lane, ShrinkTask<SL>& st) {
  // task: the (target, slot, j, slice) index, without the row split
  const int splits = (p.sh_K + SL - 1) / SL;
  const int per_t = p.slots * p.rank;
  const int ks = task % splits, combo = task / splits;
  const int t = combo / per_t, rem = combo % per_t;
  const int a = rem / p.rank, j = rem % p.rank;
  const __nv_bfloat16* A = (t == 0 ? p.sh_a0 : p.sh_a1) + ((size_t)a * p.rank + j) * p.sh_K;
#pragma unroll
  for (int i = 0; i < ShrinkTask<SL>::NI; ++i) {
    const int k = ks * SL + i * 256 + lane * 8;
    st.a[i] = k < p.sh_K ? __ldg(reinterpret_cast<const uint4*>(A + k)) : make_uint4(0, 0, 0, 0);
  }
}

template <int SL, bool SPLIT_ROWS>
__device__ __forceinline__ void lora_shrink_tasks(const GemmParams& p, int gwarp, int nwarps, int lane,
                                                  const int* s_off, const int* s_rows, ShrinkTask<SL>& st) {
  constexpr int NI = ShrinkTask<SL>::NI;
  const int per_t = p.slots * p.rank;
  const int splits = (p.sh_K + SL - 1) / SL;
  const int rsplit = SPLIT_ROWS ? shrink_rsplit<SL>(p, nwarps, s_off[p.slots]) : 1;
  const int tasks = p.sh_targets * per_t * splits * rsplit;
  for (int task = gwarp; task < tasks; task += nwarps) {
    const int rs = task % rsplit, btask = task / rsplit;
    const int ks = btask % splits, combo = btask / splits;
    const int t = combo / per_t, rem = combo % per_t;
    const int a = rem / p.rank, j = rem % p.rank;
    const int n_a = s_off[a + 1] - s_off[a];
    const int r0 = s_off[a] + (n_a * rs) / rsplit, r1 = s_off[a] + (n_a * (rs + 1)) / rsplit;
    if (task != gwarp) shrink_load_a<SL>(p, btask, lane, st);  // the first was preloaded
    if (r0 == r1) continue;
    const int k0 = ks * SL;
#pragma unroll 1
    for (int rr = r0; rr < r1; ++rr) {
      const int gr = s_rows[rr];
      if (gr < p.row0 || gr >= p.row0 + p.n_rows) continue;
      uint4 xraw[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int k = k0 + i * 256 + lane * 8;
        xraw[i] = k < p.sh_K ? __ldcg(reinterpret_cast<const uint4*>(p.sh_x + (size_t)gr * p.sh_ld + k))
                             : make_uint4(0, 0, 0, 0);
      }
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        float af[8], xf[8];
        unpack8(st.a[i], af);
        unpack8(xraw[i], xf);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = fmaf(xf[e], af[e], acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        const size_t slot = ((size_t)gr * 2 + t) * p.rank + j;
        if (splits == 1)
          p.ubd[(size_t)gr * p.ubd_ld + (size_t)t * p.slots * p.rank + a * p.rank + j] =
              __float2bfloat16_rn(acc);
        else
          p.sh_part[(size_t)ks * p.rows_total * 2 * p.rank + slot] = acc;
      }
    }
    if (splits > 1) {
      // the last split to arrive folds every split of every row of the segment: lanes cover
      // (row, split) pairs -- all loads in flight at once -- and the split sums are gathered
      // to the row's first lane and added in split order
      int last = 0;
      if (lane == 0) last = atom_add_acq_rel(p.sh_cnt + combo, 1) == splits - 1;
      if (__shfl_sync(0xffffffffu, last, 0)) {
        fence_acq_rel_gpu();  // every lane reads the other splits' partials
        const int per = 32 / splits;  // rows per pass (splits <= 32)
        const int q = lane % splits, g0 = (lane / splits) * splits;
#pragma unroll 1
        for (int rb = r0; rb < r1; rb += per) {
          const int rr = rb + lane / splits;
          const int gr = (lane < per * splits && rr < r1) ? s_rows[rr] : -1;
          const bool act = gr >= p.row0 && gr < p.row0 + p.n_rows;
          const size_t slot = act ? ((size_t)gr * 2 + t) * p.rank + j : 0;
          const float v = act ? __ldcg(p.sh_part + (size_t)q * p.rows_total * 2 * p.rank + slot) : 0.f;
          float sum = 0.f;
#pragma unroll 1
          for (int qq = 0; qq < splits; ++qq) {
            const float x = __shfl_sync(0xffffffffu, v, min(g0 + qq, 31));
            sum = qq == 0 ? x : __fadd_rn(sum, x);
          }
          if (act && q == 0)
            p.ubd[(size_t)gr * p.ubd_ld + (size_t)t * p.slots * p.rank + a * p.rank + j] =
                __float2bfloat16_rn(sum);
        }
        if (lane == 0) p.sh_cnt[combo] = 0;
      }
    }
  }
}

// The shrink of one warp: A of its first task preloaded before the PDL wait, then the tasks.
// One 4096-element slice per task: q, o, gate|up need no combine; down (K = 14336) combines 4.
constexpr int SHRINK_SL = 4096;
template <int SL, bool SPLIT_ROWS>
__device__ __forceinline__ void shrink_warp(const GemmParams& p, int gwarp, int nwarps, int lane,
                                            const int* s_off, const int* s_rows, bool wait_first) {
  ShrinkTask<SL> st;
  if constexpr (SPLIT_ROWS) {
    const int n_dec = s_off[p.slots];
    if (n_dec == 0) {  // no decoder rows (prefill): nothing to shrink
      if (wait_first) pdl_wait();
      return;
    }
    const int rsplit = shrink_rsplit<SL>(p, nwarps, n_dec);
    if (gwarp < shrink_tasks_total<SL>(p, nwarps, n_dec)) shrink_load_a<SL>(p, gwarp / rsplit, lane, st);
  } else {
    if (gwarp < p.sh_targets * p.slots * p.rank * ((p.sh_K + SL - 1) / SL)) shrink_load_a<SL>(p, gwarp, lane, st);
  }
  if (wait_first) pdl_wait();
  lora_shrink_tasks<SL, SPLIT_ROWS>(p, gwarp, nwarps, lane, s_off, s_rows, st);
}

template <int NT, int MODE>
__global__ void __launch_bounds__(256, 1)
    gemm_streamk_kernel(const __grid_constant__ CUtensorMap tm_w,
                        const __grid_constant__ CUtensorMap tm_x,
                        const __grid_constant__ CUtensorMap tm_lb,
                        const __grid_constant__ CUtensorMap tm_lu, const GemmParams p,
                        int x_row0) {
  using C = Cfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int NS = ring_stages<NT>(p.stages);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * C::STAGE);
  uint64_t* empty = full + NS;
  uint64_t* tmem_full = empty + NS;   // [2] per accumulator buffer
  uint64_t* tmem_empty = tmem_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  EpiShared& sh = *reinterpret_cast<EpiShared*>(tmem_slot + 4);
  RowMeta rm;
  rm.kind = reinterpret_cast<int*>(&sh + 1);
  rm.ad = rm.kind + NT;
  rm.pos = rm.ad + NT;
  rm.kvoff = rm.pos + NT;
  rm.inv = reinterpret_cast<float*>(rm.kvoff + NT);
  // [NT/16 chunks][4 warps][16 rows] sum-of-squares partials (after the helpers' EpiShared)
  float* ssq_part = reinterpret_cast<float*>(
      reinterpret_cast<EpiShared*>(rm.kind + ((5 * NT + 64 + 1 + 512 + 3) & ~3)) + 1);

  auto stamp = [&](int slot) {
    if (p.trace != nullptr) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      p.trace[(size_t)blockIdx.x * 16 + slot] = t;
    }
  };
  if (threadIdx.x == 0) {
    stamp(6);  // kernel entry (before any setup)
    if (p.trace != nullptr) {
      unsigned int smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      p.trace[(size_t)blockIdx.x * 16 + 8] = smid + 1;
    }
  }
  const int warp = warp_id();
  const int Kb = p.K / BK;  // base K chunks per tile
  const int Lc = p.lora_chunks;
  Split sp;
  sp.Ut = Kb + Lc;
  sp.U = (long long)(p.M / BM) * sp.Ut;
  sp.G = gridDim.x;
  const int c = blockIdx.x;
  const long long u_begin = sp.ubegin(c), u_end = sp.ubegin(c + 1);
  const int t_first = (int)((unsigned)u_begin / (unsigned)sp.Ut);
  const int t_last = (int)((unsigned)(u_end - 1) / (unsigned)sp.Ut);
  const int ntiles = t_last - t_first + 1;
  // shrink warps per CTA: 2-3, and in wide launches also the epilogue warps 4-7, which
  // otherwise only wait for the first accumulator during the main loop
  constexpr int SHRINK_WARPS = NT > 32 ? 6 : 2;

  if (warp == 0 && elect_one()) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tmem_full[b], 1); mbar_init(&tmem_empty[b], 128); }
    fence_barrier_init();
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_x);
    if (Lc > 0) { tma_prefetch_desc(&tm_lb); tma_prefetch_desc(&tm_lu); }
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  if (threadIdx.x == 128) { sh.shrink_ready = 0; sh.flag = 0; }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_launch();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) stamp(0);
  // stream-K partial of CTA cs (its first tile), 16-column chunk cc, for this thread's
  // feature: layout [cta][chunk][4 float4][128 features], a warp's float4 access is 512
  // contiguous bytes
  auto ws_slot = [&](int cs, int cc) {
    return reinterpret_cast<float4*>(p.ws) + (((size_t)cs * (NT / 16) + cc) * 4) * BM + (threadIdx.x & 127);
  };
  // Finalization of 16-column chunks [cc0, cc1) of tile t by one 128-thread group (thread
  // ep_t owns output feature t * 128 + ep_t; TMEM lane quarter = warp % 4). A tile split over
  // several CTAs is finalized by the CTA holding its FIRST K segment (segment 0: the tile
  // starts inside that CTA's range, so it is the CTA's last tile and its accumulator is the
  // last to complete). The other segments are the first tiles of the following CTAs; each
  // publishes its fp32 partial into its own ws slot, which holds the WS_EMPTY pattern
  // whenever it is unpublished. The finalizer folds seg 0 (TMEM) + seg 1 + ... in segment
  // order -- fixed by (M, K, grid) only -- polling each 4-byte word until it is not
  // WS_EMPTY (no atomics, no fences: one L2 round trip when the partials are there), and
  // re-arms the slots it consumed. Wide launches software-pipeline the residual rows.
  // Waiting on other CTAs is safe because a launch's CTAs are all resident together (grid =
  // min(units, #SMs), one CTA per SM; a PDL successor is only scheduled once every CTA of this
  // grid has started) -- the same assumption as the grid-wide LoRA-shrink count.
  auto fin_chunks = [&](int t, int b, int cc0, int cc1, int ep_t, EpiShared& shx, int bar,
                        const float* pre0, const float2* cs0) {
    const int grow0 = p.row0, gnr = p.n_rows;
    const long long t0 = (long long)t * sp.Ut;
    const int c_first = sp.owner(t0), c_last = sp.owner(t0 + sp.Ut - 1);
    const int nseg = c_last - c_first + 1;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    const bool stamps = ep_t == 0 && bar == 1;
    constexpr bool PIPE = NT > 16;
    float npre[16];
    auto fetch_resid = [&](int cc) {
      if (MODE == EPI_RESID) {
        const int m = t * BM + ep_t;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int n = cc * 16 + j;
          npre[j] = (n < gnr) ? __ldcg(p.resid + (size_t)(grow0 + n) * p.M + m) : 0.f;
        }
      }
    };
    if (PIPE) fetch_resid(cc0);
#pragma unroll 1
    for (int cc = cc0; cc < cc1; ++cc) {
      float cpre[16];
      if (PIPE) {
#pragma unroll
        for (int j = 0; j < 16; ++j) cpre[j] = npre[j];
        if (cc + 1 < cc1) fetch_resid(cc + 1);
      }
      float v[16];
      tmem_ld16(tmem_base + b * NT + lane_base + cc * 16, v);
      // segments 1.. in batches: every load of a batch issued before its first add
      constexpr int SEG_BATCH = 6;
#pragma unroll 1
      for (int s0 = 1; s0 < nseg; s0 += SEG_BATCH) {
        float4 buf[SEG_BATCH][4];
#pragma unroll
        for (int s = 0; s < SEG_BATCH; ++s)
          if (s0 + s < nseg) {
            const float4* src = ws_slot(c_first + s0 + s, cc);
#pragma unroll
            for (int q = 0; q < 4; ++q) buf[s][q] = ld_relaxed_f4(src + q * BM);
          }
#pragma unroll
        for (int s = 0; s < SEG_BATCH; ++s)
          if (s0 + s < nseg) {
            const float4* src = ws_slot(c_first + s0 + s, cc);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              while (ws_empty(buf[s][q])) buf[s][q] = ld_relaxed_f4(src + q * BM);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              v[4 * q + 0] = __fadd_rn(v[4 * q + 0], buf[s][q].x);
              v[4 * q + 1] = __fadd_rn(v[4 * q + 1], buf[s][q].y);
              v[4 * q + 2] = __fadd_rn(v[4 * q + 2], buf[s][q].z);
              v[4 * q + 3] = __fadd_rn(v[4 * q + 3], buf[s][q].w);
            }
          }
      }
      if (stamps && cc == 0) stamp(10);
      // re-arm the consumed slots for the next launch that uses this scratch
      const float4 empty4 = make_float4(__uint_as_float(WS_EMPTY), __uint_as_float(WS_EMPTY),
                                        __uint_as_float(WS_EMPTY), __uint_as_float(WS_EMPTY));
#pragma unroll 1
      for (int s = 1; s < nseg; ++s) {
        float4* dst = ws_slot(c_first + s, cc);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q * BM] = empty4;  // weak: never ahead of later loads
      }
      if (stamps && cc == 0) stamp(5);
      const float* prow = PIPE ? (MODE == EPI_RESID ? cpre : nullptr) : (cc == 0 ? pre0 : nullptr);
      finalize16<NT, MODE>(p, grow0, gnr, t, cc * 16, v, ep_t, shx, rm, bar, prow,
                           (MODE == EPI_QKV && cc == 0) ? cs0 : nullptr,
                           (MODE == EPI_RESID && PIPE) ? ssq_part : nullptr);
      if (stamps && cc == 0) stamp(11);
    }
    if constexpr (MODE == EPI_RESID && PIPE) {
      named_bar_sync(bar, 128);  // every warp of this group wrote its chunks' partials
      for (int idx = ep_t; idx < (cc1 - cc0) * 16; idx += 128) {
        const int cc = cc0 + (idx >> 4), r = idx & 15, n = cc * 16 + r;
        if (n < gnr) {
          const float* q = ssq_part + (cc * 4) * 16 + r;
          p.out_ssq[(size_t)t * p.ss_stride + grow0 + n] = ((q[0] + q[16]) + q[32]) + q[48];
        }
      }
      named_bar_sync(bar, 128);  // read before the next tile's chunks overwrite the partials
    }
  };
  constexpr bool HELPERS = NT >= 32;

  // pull the NEXT projection's adapter A matrices into L2 so its shrink loads hit L2

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      // Walk this CTA's units with running (tile, chunk) counters: no integer division on
      // the per-16KB path (a single thread must issue a tile every ~0.3 us).
      // LoRA chunk placement inside a tile (one rule for every CTA sharing the tile): the
      // last Lc units of the portion owned by the CTA whose range contains the tile start,
      // i.e. as late as possible in that CTA's range -- the shrink has finished by then.
      struct Cursor {
        int t, k;  // tile, position within the tile's Ut units
        int ls;    // first LoRA unit within the tile
      };
      auto tile_ls = [&](int t) {
        if (Lc == 0) return 0;
        const long long t0 = (long long)t * sp.Ut, t1 = t0 + sp.Ut;
        // first CTA portion of the tile long enough to hold the LoRA chunks; a portion
        // that ends before the tile does ends at that CTA's range end (late in its range)
        for (int cc = sp.owner(t0); cc < sp.G; ++cc) {
          const long long b = sp.ubegin(cc) > t0 ? sp.ubegin(cc) : t0;
          const long long e = sp.ubegin(cc + 1) < t1 ? sp.ubegin(cc + 1) : t1;
          if (e - b >= Lc) return (int)(e - Lc - t0);
          if (e >= t1) break;
        }
        return sp.Ut - Lc;
      };
      auto chunk_of = [&](const Cursor& cu, int& ch) {
        if (cu.k < cu.ls || Lc == 0) { ch = cu.k; return false; }
        if (cu.k < cu.ls + Lc) { ch = cu.k - cu.ls; return true; }
        ch = cu.k - Lc;
        return false;
      };
      auto advance = [&](Cursor& cu) {
        if (++cu.k == sp.Ut) { cu.k = 0; ++cu.t; cu.ls = tile_ls(cu.t); }
      };
      bool lora_ready = false;
      auto load_w = [&](const Cursor& cu, int stage) {
        int ch;
        const bool lo = chunk_of(cu, ch);
        uint8_t* st = smem + (size_t)stage * C::STAGE;
        mbar_expect_tx(&full[stage], C::STAGE);
        if (lo)
          tma_load_3d_hint(st, &tm_lb, &full[stage], 0, 0, cu.t * Lc + ch, pol);
        else if (p.w_blocked)
          tma_load_3d_hint(st, &tm_w, &full[stage], 0, 0, cu.t * Kb + ch, pol);
        else
          tma_load_2d_hint(st, &tm_w, &full[stage], ch * BK, cu.t * BM, pol);
      };
      auto load_x = [&](const Cursor& cu, int stage) {
        const int xr = x_row0;
        int ch;
        const bool lo = chunk_of(cu, ch);
        uint8_t* dst = smem + (size_t)stage * C::STAGE + W_BYTES;
        if (lo) {
          if (!lora_ready) {  // U is produced by this grid's shrink warps (2 per CTA)
            // every shrink warp (2 per CTA) of this launch published; earlier row-group
            // launches of the same projection already added their own 2 x grid arrivals
            const int target = gridDim.x * 2 * (p.sync_round > 0 ? p.sync_round : 1);
            stamp(2);
            while (ld_acquire(p.sync) < target) __nanosleep(32);
            stamp(3);
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
            lora_ready = true;
          }
          tma_load_2d(dst, &tm_lu, &full[stage], ch * BK, xr);
        } else {
          tma_load_2d(dst, &tm_x, &full[stage], ch * BK, xr);
        }
      };
      Cursor start;
      start.t = t_first;
      start.k = (int)(u_begin - (long long)t_first * sp.Ut);
      start.ls = tile_ls(t_first);
      // Weights do not depend on the previous kernel: fill the ring before waiting on it.
      const long long total = u_end - u_begin;
      const int pre = (int)(total < NS ? total : NS);
      const int pw = p.preissue_cap == 0 ? pre : (p.preissue_cap < 0 ? 0 : min(pre, p.preissue_cap));
      Cursor cu = start;
      for (int i = 0; i < pw; ++i) { load_w(cu, i); advance(cu); }
      pdl_wait();
      stamp(7);  // previous kernel complete
      cu = start;
      for (int i = 0; i < pre; ++i) {
        if (i >= pw) load_w(cu, i);
        load_x(cu, i);
        advance(cu);
      }
      int stage = pre % NS;
      uint32_t phase = (pre == NS) ? 1u : 0u;
      for (long long u = u_begin + pre; u < u_end; ++u) {
        mbar_wait(&empty[stage], phase ^ 1);
        load_w(cu, stage);
        load_x(cu, stage);
        advance(cu);
        if (++stage == NS) { stage = 0; phase ^= 1; }
      }
      stamp(4);
    }
  } else if (warp == 1) {
    // ---------------- tcgen05.mma issuer ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int job = 0; job < ntiles; ++job) {
      // the CTA's tiles alternate between the two accumulator buffers: a tile's MMAs never
      // wait for the previous tile's epilogue (publish) to drain TMEM
      const int t = t_first + job, bf = job & 1;
      const long long t0 = (long long)t * sp.Ut;
      const int kb = (int)((u_begin > t0 ? u_begin : t0) - t0);
      const int ke = (int)((u_end < t0 + sp.Ut ? u_end : t0 + sp.Ut) - t0);
      mbar_wait(&tmem_empty[bf], ((job >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int k = kb; k < ke; ++k) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (p.skip_mma) {
          if (elect_one()) {
            mbar_arrive(&empty[stage]);
            if (k == ke - 1) mbar_arrive(&tmem_full[bf]);
          }
        } else if (elect_one()) {
          const uint32_t a = smem_u32(smem + (size_t)stage * C::STAGE);
          const uint32_t b = a + W_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            tc_mma_bf16(tmem_base + bf * NT, sdesc_kmajor_sw128(a + kk * 32),
                        sdesc_kmajor_sw128(b + kk * 32), C::IDESC, (k > kb || kk > 0) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          if (k == ke - 1) { tc_commit(&tmem_full[bf]); stamp(12); }
        }
        __syncwarp();
        if (++stage == NS) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ---------------- LoRA shrink (SGMV) on the two otherwise idle warps ----------------
    if (p.sh_x != nullptr) {
      const int lane = lane_id();
      // stage the SGMV segment table (adapter slot -> decoder rows) in smem once; it is part
      // of the metadata uploaded before the forward, so it is read before the PDL wait
      int* s_off = rm.kind + 5 * NT;           // after the epilogue's row metadata
      int* s_rows = s_off + (p.slots + 1);
      const int t64 = threadIdx.x - 64;        // 0..63 across warps 2-3
      for (int i = t64; i <= p.slots; i += 64) s_off[i] = p.seg_off[i];
      named_bar_sync(3, 64);
      const int nseg = s_off[p.slots];
      for (int i = t64; i < nseg; i += 64) s_rows[i] = p.seg_rows[i];
      if constexpr (SHRINK_WARPS > 2) named_bar_arrive(6, 64 + 128);  // the table is staged
      named_bar_sync(3, 64);
      // wide launches (many decoder rows per adapter slot) split each slot's rows over warps
      shrink_warp<SHRINK_SL, (NT > 32)>(p, blockIdx.x * SHRINK_WARPS + (warp - 2), gridDim.x * SHRINK_WARPS,
                                        lane, s_off, s_rows, true);
      asm volatile("fence.proxy.async.global;\n" ::: "memory");  // U is read by TMA
      // the epilogue warps' shrink tasks of this CTA are done too: the CTA still counts 2
      // arrivals per launch, whatever its width (row-group launches share the counter)
      if constexpr (SHRINK_WARPS > 2) named_bar_sync(7, 64 + 128);
      __syncwarp();
      if (lane == 0) red_add_release(p.sync, 1);
      if (lane == 0 && warp == 2) stamp(1);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (TMEM -> registers -> global) ----------------
    const int ep_t = threadIdx.x - 128;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    if constexpr (SHRINK_WARPS > 2) {
      if (p.sh_x != nullptr) {
        // wide launches: shrink tasks first (the first accumulator is far away)
        const int* s_off = rm.kind + 5 * NT;
        const int* s_rows = s_off + (p.slots + 1);
        named_bar_sync(6, 64 + 128);  // warps 2-3 staged the SGMV table
        shrink_warp<SHRINK_SL, true>(p, blockIdx.x * SHRINK_WARPS + 2 + (warp - 4), gridDim.x * SHRINK_WARPS,
                                     lane_id(), s_off, s_rows, true);
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        __syncwarp();
        named_bar_arrive(7, 64 + 128);  // counted by warps 2-3
      }
    }
    pdl_wait();
    // the launch that used reset_sync has completed (PDL): re-arm its shrink counter for
    // its next use (two launches later at the earliest)
    if (p.reset_sync != nullptr && blockIdx.x == 0 && ep_t == 0) *p.reset_sync = 0;
    const int grow0 = p.row0, gnr = p.n_rows;
    // stage this launch's row metadata (+ RMSNorm inverse) in smem
    for (int n = ep_t; n < NT; n += 128) {
      int kind = -1, ad = -1, pos = 0, kvoff = 0;
      float inv = 1.f;
      if (n < gnr) {
        const int gn = grow0 + n;
        kind = p.row_kind ? p.row_kind[gn] : 0;
        ad = p.row_adapter ? p.row_adapter[gn] : -1;
        pos = p.row_pos ? p.row_pos[gn] : 0;
        if (MODE == EPI_QKV && kind == 0) {
          const int page = p.block_table[(size_t)p.row_seq[gn] * p.bt_stride + (pos >> 4)];
          kvoff = (page * p.num_kv_heads * 16 + (pos & 15)) * p.head_dim;
        }
        if (p.in_ssq != nullptr) {
          // the row's per-tile partial sums in tile order; wide launches keep 16 loads in
          // flight per batch (decode launches measured faster with the compact loop)
          float ss = 0.f;
          if constexpr (NT == 16) {
#pragma unroll 4
            for (int t = 0; t < p.ss_tiles; ++t) ss = __fadd_rn(ss, p.in_ssq[(size_t)t * p.ss_stride + gn]);
          } else {
#pragma unroll 1
          for (int t0 = 0; t0 < p.ss_tiles; t0 += 16) {
            float part[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
              part[q] = t0 + q < p.ss_tiles ? __ldcg(p.in_ssq + (size_t)(t0 + q) * p.ss_stride + gn) : 0.f;
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (t0 + q < p.ss_tiles) ss = __fadd_rn(ss, part[q]);
          }
          }
          inv = __fdiv_rn(1.f, sqrtf(__fadd_rn(__fdiv_rn(ss, p.ss_d), p.eps)));
        }
      }
      rm.kind[n] = kind;
      rm.ad[n] = ad;
      rm.pos[n] = pos;
      rm.kvoff[n] = kvoff;
      rm.inv[n] = inv;
    }
    named_bar_sync(1, 128);
    for (int t = t_first; t <= t_last; ++t) {
      const int job = t - t_first, bf = job & 1;
      const long long t0 = (long long)t * sp.Ut;
      const int c_first = sp.owner(t0), c_last = sp.owner(t0 + sp.Ut - 1);
      const int nseg = c_last - c_first + 1;
      // residual rows of this tile's first 16 columns: loaded before the accumulator is
      // ready so the epilogue's critical path has no dependent global load
      float pre[16];
      const bool have_pre = MODE == EPI_RESID;
      if (have_pre) {
        const int m = t * BM + ep_t;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          pre[j] = (j < gnr && rm.kind[j] >= 0) ? __ldcg(p.resid + (size_t)(grow0 + j) * p.M + m) : 0.f;
      }
      // likewise the RoPE factors of the first 16 rows (the table lines are evicted by the
      // weight stream between layers: an HBM round trip under load)
      float2 cs_pre[MODE == EPI_QKV ? 16 : 1];
      if constexpr (MODE == EPI_QKV) {
        const int m = t * BM + ep_t;
        const int region = m < p.q_dim ? 0 : (m < p.q_dim + p.kv_dim ? 1 : 2);
        const int base = region == 0 ? 0 : (region == 1 ? p.q_dim : p.q_dim + p.kv_dim);
        const int i = (m - base) % p.head_dim;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          cs_pre[j] = (region < 2 && j < gnr && rm.kind[j] >= 0)
                          ? __ldg(p.rope + (size_t)rm.pos[j] * (p.head_dim >> 1) + (i >> 1))
                          : make_float2(1.f, 0.f);
      }
      mbar_wait(&tmem_full[bf], (job >> 1) & 1);
      tc_fence_after();
      if (ep_t == 0) stamp(13);
      // A tile split over several CTAs: segment 0's CTA finalizes it (see fin_chunks); any
      // other segment publishes its partial and hands the accumulator back at once.
      const bool fin = nseg == 1 || c == c_first;
      if (!fin) {
#pragma unroll 1
        for (int cc = 0; cc < NT / 16; ++cc) {
          float v[16];
          tmem_ld16(tmem_base + bf * NT + lane_base + cc * 16, v);
          float4* wsp = ws_slot(c, cc);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            __stcg(wsp + q * BM, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
        }
        tc_fence_before();
        mbar_arrive(&tmem_empty[bf]);
        if (ep_t == 0) stamp(15);
      }
      // wide launches: warps 0-3 (their roles are over once the last tile's MMAs are issued)
      // finalize the upper half of the last tile's 16-column chunks
      const bool helped = HELPERS && t == t_last;
      if (helped) {
        if (ep_t == 0) sh.fin_last = fin ? 1 : 0;
        named_bar_sync(4, 256);
      }
      if (fin) {
        fin_chunks(t, bf, 0, helped ? NT / 32 : NT / 16, ep_t, sh, 1, have_pre ? pre : nullptr, cs_pre);
        if (helped) named_bar_sync(5, 256);
        tc_fence_before();
        mbar_arrive(&tmem_empty[bf]);
      }
      if (ep_t == 0) stamp(14);
    }
  }

  if (HELPERS && warp < 4) {
    __syncwarp();
    named_bar_sync(4, 256);  // the epilogue has decided whether this CTA finalizes t_last
    if (sh.fin_last) {
      tc_fence_after();
      EpiShared& sh2 = *reinterpret_cast<EpiShared*>(rm.kind + ((5 * NT + 64 + 1 + 512 + 3) & ~3));
      fin_chunks(t_last, (ntiles - 1) & 1, NT / 32, NT / 16, threadIdx.x, sh2, 2, nullptr, nullptr);
      tc_fence_before();
      named_bar_sync(5, 256);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<C::TMEM_COLS>(tmem_base);
  if (threadIdx.x == 0) stamp(9);  // exit
}

// ------------------------------------------------------------------ host side
// One kernel per (token-tile width, epilogue): each instantiation carries only its own
// epilogue, so the code a tile's tail executes stays small and hot in the instruction caches.
template <int NT, int MODE>
static cudaError_t launch_ntm(const CUtensorMap& tw, const CUtensorMap& tx, const CUtensorMap& tlb,
                              const CUtensorMap& tlu, const GemmParams& p, int x_row0, int num_sms,
                              cudaStream_t s) {
  using C = Cfg<NT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_streamk_kernel<NT, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long U = (long long)(p.M / BM) * (p.K / BK + p.lora_chunks);
  const int G = (int)(U < num_sms ? U : num_sms);
  if ((unsigned long long)U * (unsigned long long)(G + 1) >= (1ull << 32)) return cudaErrorInvalidValue;
  const int NS = ring_stages<NT>(p.stages);
  const size_t smem = 1024 + (size_t)NS * C::STAGE + aux_smem<NT>();
  return launch_pdl(gemm_streamk_kernel<NT, MODE>, dim3(G), dim3(256), smem, s, tw, tx, tlb, tlu, p,
                    x_row0);
}

template <int NT>
static cudaError_t launch_nt(const CUtensorMap& tw, const CUtensorMap& tx, const CUtensorMap& tlb,
                             const CUtensorMap& tlu, const GemmParams& p, int x_row0, int num_sms,
                             cudaStream_t s) {
  switch (p.mode) {
    case EPI_F32: return launch_ntm<NT, EPI_F32>(tw, tx, tlb, tlu, p, x_row0, num_sms, s);
    case EPI_RESID: return launch_ntm<NT, EPI_RESID>(tw, tx, tlb, tlu, p, x_row0, num_sms, s);
    case EPI_SILU: return launch_ntm<NT, EPI_SILU>(tw, tx, tlb, tlu, p, x_row0, num_sms, s);
    case EPI_QKV: return launch_ntm<NT, EPI_QKV>(tw, tx, tlb, tlu, p, x_row0, num_sms, s);
    case EPI_ARGMAX: return launch_ntm<NT, EPI_ARGMAX>(tw, tx, tlb, tlu, p, x_row0, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

int gemm_pick_nt(int rows) {
  if (rows <= 16) return 16;
  if (rows <= 32) return 32;
  if (rows <= 64) return 64;
  if (rows <= 128) return 128;
  return 256;
}

cudaError_t gemm_launch(const CUtensorMap& tw, const CUtensorMap& tx, const CUtensorMap* tlb,
                        const CUtensorMap* tlu, const GemmParams& p, int x_row0, int nt,
                        int num_sms, cudaStream_t s) {
  if (p.rank > MAX_RANK) return cudaErrorInvalidValue;
  if (p.lora_chunks > 0 && (tlb == nullptr || tlu == nullptr)) return cudaErrorInvalidValue;
  const CUtensorMap& lb = tlb ? *tlb : tw;
  const CUtensorMap& lu = tlu ? *tlu : tx;
  switch (nt) {
    case 16: return launch_nt<16>(tw, tx, lb, lu, p, x_row0, num_sms, s);
    case 32: return launch_nt<32>(tw, tx, lb, lu, p, x_row0, num_sms, s);
    case 64: return launch_nt<64>(tw, tx, lb, lu, p, x_row0, num_sms, s);
    case 128: return launch_nt<128>(tw, tx, lb, lu, p, x_row0, num_sms, s);
    case 256: return launch_nt<256>(tw, tx, lb, lu, p, x_row0, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

size_t gemm_ws_floats(int num_sms) { return (size_t)num_sms * 256 * BM; }

cudaError_t gemm_ws_clear(float* ws, int num_sms, cudaStream_t s) {
  return cudaMemsetAsync(ws, 0xFF, gemm_ws_floats(num_sms) * sizeof(float), s);
}

int gemm_stages(int nt) {
  switch (nt) {
    case 16: return Cfg<16>::STAGES;
    case 32: return Cfg<32>::STAGES;
    case 64: return Cfg<64>::STAGES;
    case 128: return Cfg<128>::STAGES;
    default: return Cfg<256>::STAGES;
  }
}

}  // namespace icr
