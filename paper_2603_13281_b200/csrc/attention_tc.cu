// Shared-KV paged decode attention on the 5th-generation tensor cores (head_dim 128).
// Reference semantics: `layer_attention` (src/model.py:384-425) over the fused 2H query
// heads of `block_forward` decode (src/model.py:495-501): scores = (q . k) * 1/sqrt(hd) with
// the causal mask, softmax, weights @ V -- per (row, head), batch-invariant.
//
// Persistent: one CTA per SM walks a host-scheduled (LPT) list of units = work item x KV
// head. A work item is a chunk of pages at fixed absolute positions shared by every sequence
// whose block table maps the same physical pages; its up to 128 query entries (row,
// head-in-group) -- the encoder and decoder heads of every model sharing the prefix -- are the
// M = 128 rows of the tcgen05 MMAs. The chunk is streamed in sub-chunks of SUBP = 8 pages
// (128 keys) through a 3-stage TMA ring:
//   S_j[128 x 128] = Q . K_j^T            (K-major Q and K; fp32, double-buffered in TMEM)
//   softmax        : 8 warps, two per TMEM lane quarter (each half of the key columns), exp2
//                    domain with the causal mask; running max m, sum l per entry; P_j bf16
//                    back into TMEM; O rescaled in TMEM when the max moves
//   O[128 x 128]  += P_j . V_j              (P from TMEM, V MN-major straight from the pages)
// so S_{j+1}, the loads of sub-chunk j+2 and the softmax of j overlap -- within a unit and
// across consecutive units of a CTA. The unnormalised partial (O, m, l) per (row, head, chunk)
// is written out and folded in chunk order by the merge kernel (attention.cu, attn_merge.cuh),
// launched behind this one with PDL: its small CTAs share SMs with the next projection GEMM,
// which streams its weights while the merge runs. Each K/V page is
// staged in shared memory once per KV head for all entries: HBM bytes scale with context, not
// with the number of models. Sub-chunk boundaries sit at fixed offsets from the chunk's
// absolute start, so a row's partial never depends on which other rows share the item or on
// which CTA runs it.
#include "kernels.h"
#include "ptx.cuh"
#include "attn_merge.cuh"

namespace icr {

constexpr int TC_THREADS = 384;  // w0 K TMA, w1 MMA + TMEM, w2 V TMA, w3-11 Q, w4-11 softmax
constexpr int TC_ROWS = 128;     // MMA M: query entries per item
constexpr int SUBP = 8;          // pages per sub-chunk (N = 128 keys per S MMA)

struct TcLayout {
  static constexpr uint32_t Q_OFF = 0;                     // 2 K-blocks x [128 rows x 128 B]
  static constexpr uint32_t HALF = SUBP * 16 * 128;        // 16 KB: one 64-dim half, 128 keys
  static constexpr uint32_t STAGE0 = 32768;                // stage s: K halves, then V halves
  static constexpr uint32_t STAGE_BYTES = 4 * HALF;        // 64 KB
  static constexpr int NSTAGE = 3;                         // K/V sub-chunks in flight
  static constexpr uint32_t BAR_OFF = STAGE0 + NSTAGE * STAGE_BYTES;
  static constexpr uint32_t RED_OFF = BAR_OFF + 256;       // float [2 halves][128]
  static constexpr uint32_t MROW_OFF = RED_OFF + 256 * 4;  // float [128]: row max of the unit
  // 231,168 B: within the opt-in maximum of 232,448 less the 1 KB the driver reserves
  static constexpr size_t SMEM = MROW_OFF + 128 * 4;
  // TMEM columns: S0 [0,128) S1 [128,256) O [256,384) P0 [384,448) P1 [448,512) -- P (bf16
  // pairs packed in 32-bit columns) is the A operand of P.V straight from TMEM, so shared
  // memory holds Q and three K/V stages
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t P_COL = 384;
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// MN-major, 128-byte-swizzle shared-memory descriptor (B operand of P.V): 64 consecutive
// N elements (one 128-byte row) per K index, 8 K rows per 1024-byte atom; SBO = bytes
// between 8-row K groups, LBO = bytes between 64-element N blocks.
__device__ __forceinline__ uint64_t sdesc_mnmajor_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

static_assert(TcLayout::SMEM <= 232448 - 1024, "exceeds the per-block shared memory limit");

__device__ __forceinline__ void cp_async16_s(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}

// The in-kernel merge as a call: its 24-chunk register batch gets its own allocation instead
// of raising the pressure of the whole kernel (inlined, the long-chunk variant spills).
__device__ __noinline__ void merge_unit_call(const float* __restrict__ part_o,
                                             const float2* __restrict__ part_ml, int kind, int nch,
                                             int r, int g, int num_heads, int group, int max_chunks,
                                             __nv_bfloat16* __restrict__ out, int out_ld, int lt) {
  merge_unit<128>(part_o, part_ml, kind, nch, r, g, num_heads, group, max_chunks, out, out_ld, lt, 128);
}

// Persistent: CTA c runs the (item, KV head) units sched_units[sched_off[c] .. sched_off[c+1])
// (a host LPT schedule over min(#SMs, units) CTAs, one per SM). Every role walks the same unit
// list, so each knows the item sequence without communication; mbarrier phases follow a
// global sub-chunk counter J (stages, S buffers, P buffers) or the CTA's item count (Q, O).
// Across units the K/V producers run ahead into the next unit's pages, the Q warp stages the
// next unit's queries as soon as the last S MMA of the current one has read Q, and the next
// unit's first S MMA overlaps the current unit's softmax tail and epilogue.
template <bool kNarrow>
__global__ void __launch_bounds__(TC_THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                   const __grid_constant__ CUtensorMap tm_k8, const __grid_constant__ CUtensorMap tm_v8,
                   const __nv_bfloat16* __restrict__ q, int q_ld, int num_kv_heads, int group,
                   const AttnItem* __restrict__ items, const int* __restrict__ item_pages,
                   const int2* __restrict__ item_rows, const int* __restrict__ row_pos,
                   int num_heads, int max_chunks, float scale, float* __restrict__ part_o,
                   float2* __restrict__ part_ml, const int* __restrict__ sched_off,
                   const int* __restrict__ sched_units, unsigned long long* __restrict__ trace,
                   int chunk_tokens, unsigned long long* __restrict__ span,
                   const int* __restrict__ row_kind, int n_rows, __nv_bfloat16* __restrict__ out,
                   int out_ld, int* __restrict__ merge_sync) {
  using L = TcLayout;
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  uint8_t* smem = tc_smem;  // no static shared memory: the dynamic window starts 1024-aligned
  uint8_t* sQ = smem + L::Q_OFF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_full = bars + 0;    // Q of the CTA's n-th unit staged (phase n)
  uint64_t* kv_full = bars + 20;  // [3] K landed
  uint64_t* kv_empty = bars + 23; // [3] K consumed by S
  uint64_t* s_full = bars + 5;    // [2]
  // P(J) written (+ O rescaled): bars[7] for P buffer 0, bars[17] for buffer 1
  uint64_t* o_done = bars + 8;    // one phase per P.V (the lazy rescale waits on it)
  uint64_t* p_free = bars + 9;    // [2]: TMEM P buffer b consumed by its P.V
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);
  uint64_t* v_full = bars + 26;   // [3] V landed
  uint64_t* v_empty = bars + 29;  // [3] V consumed by P.V
  uint64_t* o_final = bars + 16;  // the unit's last P.V landed (phase n)
  uint64_t* q_free = bars + 18;   // the unit's last S MMA has read Q (phase n)
  float* red = reinterpret_cast<float*>(smem + L::RED_OFF);
  float* mrow = reinterpret_cast<float*>(smem + L::MROW_OFF);

  const int cta = blockIdx.x;
  unsigned long long merge_target = 0;  // thread 0: the in-kernel merge's counter target
  auto stamp = [&](int k) {
    if (trace != nullptr && cta < 4096) trace[(size_t)cta * 16 + k] = globaltimer();
  };
  // per-sub-chunk timeline of CTA 0 (diagnostic): [J][0 K issued, 1 S done, 2 P written, 3 PV issued]
  auto sstamp = [&](int j, int k) {
    if (trace != nullptr && cta == 0 && j < 256) trace[(size_t)2 * 4096 * 16 + j * 8 + k] = globaltimer();
  };
  if (threadIdx.x == 0) {
    stamp(6);
    if (span != nullptr) atomicMin(span, globaltimer());
  }
  if ((smem_u32(tc_smem) & 1023) != 0) __trap();  // SW128 tiles need a 1024-byte base
  pdl_launch();
  const int warp = warp_id(), lane = lane_id();
  if ((warp == 0 || warp == 2) && lane == 0) {  // descriptor fetches off the critical path
    tma_prefetch_desc(warp == 0 ? &tm_k8 : &tm_v8);
    tma_prefetch_desc(warp == 0 ? &tm_k : &tm_v);
  }
  const int cp = chunk_tokens >> 4;
  // CTA c's first unit is unit c (schedule_units assigns the G longest units to CTAs 0..G-1):
  // its item, page ids and (Q warp) row table are requested right away, together with the
  // schedule, all uploaded before the forward -- one round trip, overlapping the set-up
  const int k_begin = sched_off[cta], k_end = sched_off[cta + 1];
  const AttnItem it0 = items[cta / num_kv_heads];
  int pid0 = 0;
  if ((warp == 0 || warp == 2) && lane < cp) pid0 = __ldg(item_pages + (cta / num_kv_heads) * cp + lane);

  if (threadIdx.x == 0) {
    mbar_init(q_full, 32);
    for (int b = 0; b < L::NSTAGE; ++b) {
      mbar_init(&kv_full[b], 1);
      mbar_init(&kv_empty[b], 1);
      mbar_init(&v_full[b], 1);
      mbar_init(&v_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) mbar_init(&s_full[b], 1);
    mbar_init(bars + 7, 256);
    mbar_init(bars + 17, 256);
    mbar_init(o_done, 1);
    mbar_init(o_final, 1);
    mbar_init(q_free, 1);
    mbar_init(&p_free[0], 1);
    mbar_init(&p_free[1], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<L::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tmem_o = tmem_base + 256;

  if (warp == 0 || warp == 2) {
    // ---------------- producers: K (warp 0) and V (warp 2) rings, decoupled: a K stage is
    // free once S has read it, a V stage only after P.V -- K runs ahead of the softmax. The
    // whole warp walks the pages: lane i holds the page id of position i of the current
    // 32-page window; lane 0 issues the TMAs ------------------------------------------------
    const bool is_k = warp == 0;
    const CUtensorMap* tm = is_k ? &tm_k : &tm_v;
    const CUtensorMap* tm8 = is_k ? &tm_k8 : &tm_v8;
    uint64_t* full = is_k ? kv_full : v_full;
    uint64_t* empty = is_k ? kv_empty : v_empty;
    bool waited = false;
    int J = 0;
    AttnItem it = it0;
    // K/V stream through L2 once per launch: evict first, so the partials written by the
    // units that finish early (read back by the merge) are not pushed out by the stream
    const uint64_t pol = policy_evict_first();
    int pid_cur = pid0;
    for (int k = k_begin; k < k_end; ++k) {
      const int unit = k == k_begin ? cta : sched_units[k];
      const int item = unit / num_kv_heads, g = unit % num_kv_heads;
      const int np = it.n_pages, nsub = (np + SUBP - 1) / SUBP;
      AttnItem it_n = it;
      int pid_n0 = 0, pid_nxt = 0, nunit = 0;
      for (int j = 0; j < nsub; ++j, ++J) {
        const int b = J % L::NSTAGE, ph = (J / L::NSTAGE) & 1;
        if (J >= L::NSTAGE) mbar_wait(&empty[b], ph ^ 1);
        const int p0 = j * SUBP, pn = min(SUBP, np - p0);
        if (p0 > 0 && (p0 & 31) == 0) {
          pid_cur = pid_nxt;
          pid_nxt = (p0 + 32 + lane < np) ? __ldg(item_pages + item * cp + p0 + 32 + lane) : 0;
        }
        uint8_t* st = smem + L::STAGE0 + b * L::STAGE_BYTES + (is_k ? 0 : 2 * L::HALF);
        if (lane == 0) mbar_expect_tx(&full[b], (uint32_t)pn * 2 * 2048);
        // a full sub-chunk of consecutive page ids (sequentially allocated prompts) is ONE
        // 32 KB TMA; otherwise one TMA per 64-dim half page
        const int w0 = p0 & 31;
        const int first = __shfl_sync(0xffffffffu, pid_cur, w0);
        const bool run = pn == SUBP &&
            __ballot_sync(0xffffffffu, lane >= w0 && lane < w0 + SUBP && pid_cur == first + (lane - w0)) ==
                (0xffu << w0);
        if (run) {
          if (!waited && p0 + SUBP > it.n_pre) {
            pdl_wait();
            if (is_k && lane == 0) stamp(7);
            waited = true;
          }
          if (lane == 0) tma_load_5d_hint(st, tm8, &full[b], 0, 0, first, 0, g, pol);
        } else {
          for (int pi = 0; pi < pn; ++pi) {
            if (!waited && p0 + pi >= it.n_pre) {
              pdl_wait();
              if (is_k && lane == 0) stamp(7);
              waited = true;
            }
            const int plane = __shfl_sync(0xffffffffu, pid_cur, (p0 + pi) & 31) * num_kv_heads + g;
            if (lane == 0) {
#pragma unroll
              for (int h = 0; h < 2; ++h)
                tma_load_4d_hint(st + h * L::HALF + pi * 2048, tm, &full[b], 0, 0, h, plane, pol);
            }
          }
        }
        if (is_k && lane == 0) sstamp(J, 0);
        // prefetches, each issued right after a sub-chunk's loads so that an in-order stall on
        // a dependent address never delays a TMA: this unit's second page window, the next
        // unit's id, then (last sub-chunk, the ring full) its record and first page window
        if (j == 0) {
          pid_nxt = (32 + lane < np) ? __ldg(item_pages + item * cp + 32 + lane) : 0;
          if (k + 1 < k_end) nunit = sched_units[k + 1];
        }
        if (j == nsub - 1 && k + 1 < k_end) {
          const int nitem = nunit / num_kv_heads;
          it_n = items[nitem];
          pid_n0 = lane < cp ? __ldg(item_pages + nitem * cp + lane) : 0;
        }
      }
      it = it_n;
      pid_cur = pid_n0;
    }
    if (!waited) pdl_wait();
    if constexpr (kNarrow) {
      // the merge's completion target, read while the units still stream (off the tail): this
      // launch's adds total < 2^20, so the value's generation is the previous launch's
      if (threadIdx.x == 0)
        merge_target = ((ld_acquire_u64(reinterpret_cast<const unsigned long long*>(merge_sync)) >> 20) + 1) << 20;
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int J = 0, n = 0;
    for (int k = k_begin; k < k_end; ++k, ++n) {
      const int np = k == k_begin ? it0.n_pages : items[sched_units[k] / num_kv_heads].n_pages;
      const int nsub = (np + SUBP - 1) / SUBP;
      auto issue_s = [&](int Jx, int jx) {
        const int st = Jx % L::NSTAGE, b = Jx & 1;
        mbar_wait(&kv_full[st], (Jx / L::NSTAGE) & 1);
        tc_fence_after();
        if (elect_one()) {
          const int keys = min(SUBP, np - jx * SUBP) * 16;
          const uint32_t idesc_s = idesc_bf16_f32(TC_ROWS, (uint32_t)keys);
          const uint32_t kb = smem_u32(smem + L::STAGE0 + st * L::STAGE_BYTES);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t a = smem_u32(sQ) + (kk >> 2) * (TC_ROWS * 128) + (kk & 3) * 32;
            const uint32_t bb = kb + (kk >> 2) * L::HALF + (kk & 3) * 32;
            tc_mma_bf16(tmem_base + b * 128, sdesc_kmajor_sw128(a), sdesc_kmajor_sw128(bb), idesc_s,
                        kk > 0 ? 1u : 0u);
          }
          tc_commit(&s_full[b]);
          tc_commit(&kv_empty[st]);
          if (jx == nsub - 1) tc_commit(q_free);  // Q may be restaged for the next unit
        }
        __syncwarp();
      };
      mbar_wait(q_full, n & 1);
      tc_fence_after();
      issue_s(J, 0);
      for (int j = 0; j < nsub; ++j, ++J) {
        if (j + 1 < nsub) issue_s(J + 1, j + 1);
        const int st = J % L::NSTAGE;
        mbar_wait((bars + ((J & 1) ? 17 : 7)), (J >> 1) & 1);  // softmax J wrote P and rescaled O
        mbar_wait(&v_full[st], (J / L::NSTAGE) & 1);
        tc_fence_after();
        if (elect_one()) {
          const int pn = min(SUBP, np - j * SUBP);
          const uint32_t idesc_o = idesc_bf16_f32(TC_ROWS, 128) | (1u << 16);  // B (V) MN-major
          const uint32_t vb = smem_u32(smem + L::STAGE0 + st * L::STAGE_BYTES) + 2 * L::HALF;
          const uint32_t pt = tmem_base + L::P_COL + (J & 1) * 64;
          for (int kk = 0; kk < pn; ++kk)  // 16 keys (one page, 8 P columns) per instruction
            tc_mma_bf16_ts(tmem_o, pt + kk * 8, sdesc_mnmajor_sw128(vb + kk * 2048, L::HALF, 1024),
                           idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          sstamp(J, 3);
          tc_commit(o_done);
          if (j == nsub - 1) tc_commit(o_final);
          tc_commit(&p_free[J & 1]);
          tc_commit(&v_empty[st]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 3) {
    // ---------------- Q staging: one warp, cp.async straight into the swizzled tile ----------
    int n = 0;
    for (int k = k_begin; k < k_end; ++k, ++n) {
      const int unit = k == k_begin ? cta : sched_units[k];
      const AttnItem it = k == k_begin ? it0 : items[unit / num_kv_heads];
      const int g = unit % num_kv_heads;
      // the row table (uploaded before the forward) before the wait: one round trip
      int2 rws[4];
#pragma unroll
      for (int m = 0; m < 4; ++m)
        rws[m] = (lane + 32 * m < it.n_rows) ? item_rows[it.row_off + lane + 32 * m] : make_int2(0, 0);
      if (n == 0) {
        pdl_wait();  // q comes from the q/k/v GEMM
        if (lane == 0) stamp(3);
      } else {
        mbar_wait(q_free, (n - 1) & 1);  // the previous unit's S MMAs have read Q
      }
      // entry e sits in M row / TMEM lane r(e) = (e % 4) * 32 + e / 4: the entries of a partly
      // filled item spread over all four lane quarters. Lane l stages entries l + 32 m (all 16
      // chunks each); the row table is read before the copies are issued (one round trip)
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int e = lane + 32 * m;
        if (e < it.n_rows) {
          const int r = (e & 3) * 32 + (e >> 2);
          const __nv_bfloat16* src = q + (size_t)rws[m].x * q_ld + (g * group + rws[m].y) * 128;
#pragma unroll
          for (int c = 0; c < 16; ++c)
            cp_async16_s(smem_u32(sQ + (c >> 3) * (TC_ROWS * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4)),
                         src + c * 8);
        }
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_arrive(q_full);
    }
  } else {
    // ---------------- softmax: warps w and w + 4 (same SM sub-partition, same TMEM lane
    // quarter w % 4) split each row's 128 key columns; the row max and sum are exchanged
    // through shared memory under a 64-thread barrier per quarter ------------------------
    const int sw = warp - 4;                       // 0..7
    const int quarter = sw & 3, half = sw >> 2;    // key columns [64 half, 64 half + 64)
    const int r = quarter * 32 + lane;             // TMEM lane = M row
    const int e = (r & 31) * 4 + (r >> 5);         // the query entry held in that row
    const uint32_t lane_base = (uint32_t)(32 * quarter) << 16;
    const float sl2 = scale * 1.4426950408889634f;
    int J = 0, n = 0;
    for (int k = k_begin; k < k_end; ++k, ++n) {
      const int unit = k == k_begin ? cta : sched_units[k];
      const AttnItem it = k == k_begin ? it0 : items[unit / num_kv_heads];
      const int g = unit % num_kv_heads;
      const int np = it.n_pages, nsub = (np + SUBP - 1) / SUBP;
      const bool valid = e < it.n_rows;
      int pos = -1;
      size_t slot = 0;
      if (valid) {
        const int2 rr = item_rows[it.row_off + e];
        pos = row_pos[rr.x];
        slot = ((size_t)rr.x * num_heads + g * group + rr.y) * max_chunks + it.chunk_idx;
      }
      float m_run = -INFINITY, l_part = 0.f;
      // Narrow units (<= 64 entries: every entry sits in lanes 0-15 of its lane quarter) read
      // and write only those 16 lanes (16x256b / 16x128b shapes): each thread holds two rows x
      // 16 keys, half the exponentials of the 32-lane form. The arithmetic per row is the same
      // as the wide form's -- thread t%4 of a row's group carries exactly the wide form's row-sum
      // chain t%4, combined in the same order -- so a row's partial does not depend on how many
      // entries share its item. Used for units of >= 4 sub-chunks, where the softmax sets the
      // pace (measured: C4 32k streaming 1.4 -> 1.1 us per sub-chunk).
      const bool narrow = kNarrow && it.n_rows <= 64 && nsub >= 4;
      if (narrow) {
        const int gq = lane & 3;
        const int rA = quarter * 32 + (lane >> 2), rB = rA + 8;
        const int eA = (lane >> 2) * 4 + quarter, eB = eA + 32;
        const bool vA = eA < it.n_rows, vB = eB < it.n_rows;
        const int posA = vA ? row_pos[item_rows[it.row_off + eA].x] : -1;
        const int posB = vB ? row_pos[item_rows[it.row_off + eB].x] : -1;
        float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;
        for (int j = 0; j < nsub; ++j, ++J) {
          const int b = J & 1;
          const int keys = min(SUBP, np - j * SUBP) * 16;
          const int kbase = it.chunk_start + j * SUBP * 16 + half * 64;
          const int hkeys = min(64, keys - half * 64);
          mbar_wait(&s_full[b], (J >> 1) & 1);
          tc_fence_after();
          if (r == 0 && half == 0) sstamp(J, 1);
          if (r == 0 && half == 0 && J == 0) stamp(2);
          uint32_t v[32];  // v[4i + c]: row A key 8i + 2gq + c; v[4i + 2 + c]: row B
          if (hkeys > 0) {
            tmem_ld_16x256b_x8(tmem_base + b * 128 + lane_base + half * 64, v);
            tmem_wait_ld();
            tmem_reg_fence32(v);
          }
          const int nvA = vA ? max(0, min(hkeys, posA + 1 - kbase)) : 0;
          const int nvB = vB ? max(0, min(hkeys, posB + 1 - kbase)) : 0;
          if ((nvA > 0 && nvA < 64) || (nvB > 0 && nvB < 64)) {
            asm volatile("" ::: "memory");
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                const int key = 8 * i + 2 * gq + c;
                if (key >= nvA) v[4 * i + c] = 0xff800000u;
                if (key >= nvB) v[4 * i + 2 + c] = 0xff800000u;
              }
          }
          float mxA = -INFINITY, mxB = -INFINITY;
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              mxA = fmaxf(mxA, __uint_as_float(v[4 * i + c]));
              mxB = fmaxf(mxB, __uint_as_float(v[4 * i + 2 + c]));
            }
          if (nvA == 0) mxA = -INFINITY;
          if (nvB == 0) mxB = -INFINITY;
          mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 1));
          mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 1));
          mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 2));
          mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 2));
          if (gq == 0) {
            red[half * 128 + rA] = mxA;
            red[half * 128 + rB] = mxB;
          }
          named_bar_sync(1 + quarter, 64);
          const float mcA = fmaxf(mA, __fmul_rn(fmaxf(red[rA], red[128 + rA]), sl2));
          const float mcB = fmaxf(mB, __fmul_rn(fmaxf(red[rB], red[128 + rB]), sl2));
          named_bar_sync(1 + quarter, 64);
          const float mnA = (mcA > mA + 8.f) ? mcA : mA;
          const float mnB = (mcB > mB + 8.f) ? mcB : mB;
          const float corrA = (mA == -INFINITY) ? 1.f : ex2_approx(mA - mnA);
          const float corrB = (mB == -INFINITY) ? 1.f : ex2_approx(mB - mnB);
          if (J >= 2) mbar_wait(&p_free[b], ((J >> 1) - 1) & 1);
          tc_fence_after();
          uint32_t pk[16];  // pk[2i]: row A P column 4i + gq (keys 8i + 2gq, +1); pk[2i + 1]: row B
          float lsA = 0.f, lsB = 0.f;
          const float nmA = -mnA, nmB = -mnB;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float a0 = nvA > 0 ? ex2_approx(fmaf(__uint_as_float(v[4 * i]), sl2, nmA)) : 0.f;
            const float a1 = nvA > 0 ? ex2_approx(fmaf(__uint_as_float(v[4 * i + 1]), sl2, nmA)) : 0.f;
            const float b0 = nvB > 0 ? ex2_approx(fmaf(__uint_as_float(v[4 * i + 2]), sl2, nmB)) : 0.f;
            const float b1 = nvB > 0 ? ex2_approx(fmaf(__uint_as_float(v[4 * i + 3]), sl2, nmB)) : 0.f;
            lsA += a0 + a1;
            lsB += b0 + b1;
            __nv_bfloat162 ha = __floats2bfloat162_rn(a0, a1), hb2 = __floats2bfloat162_rn(b0, b1);
            pk[2 * i] = *reinterpret_cast<uint32_t*>(&ha);
            pk[2 * i + 1] = *reinterpret_cast<uint32_t*>(&hb2);
          }
          if (hkeys > 0) tmem_st_16x128b_x8(tmem_base + lane_base + L::P_COL + b * 64 + half * 32, pk);
          float sA = lsA + __shfl_xor_sync(0xffffffffu, lsA, 1);
          float sB = lsB + __shfl_xor_sync(0xffffffffu, lsB, 1);
          sA = sA + __shfl_xor_sync(0xffffffffu, sA, 2);
          sB = sB + __shfl_xor_sync(0xffffffffu, sB, 2);
          lA = fmaf(lA, corrA, sA);
          lB = fmaf(lB, corrB, sB);
          mA = mnA;
          mB = mnB;
          if (j > 0 && __any_sync(0xffffffffu, (vA && corrA != 1.f) || (vB && corrB != 1.f))) {
            mbar_wait(o_done, (J - 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int hc = 0; hc < 2; ++hc) {  // 32 columns at a time (register budget)
              uint32_t o[16];
              tmem_ld_16x256b_x4(tmem_o + lane_base + half * 64 + hc * 32, o);
              tmem_wait_ld();
              tmem_reg_fence(o);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                o[4 * i] = __float_as_uint(__uint_as_float(o[4 * i]) * corrA);
                o[4 * i + 1] = __float_as_uint(__uint_as_float(o[4 * i + 1]) * corrA);
                o[4 * i + 2] = __float_as_uint(__uint_as_float(o[4 * i + 2]) * corrB);
                o[4 * i + 3] = __float_as_uint(__uint_as_float(o[4 * i + 3]) * corrB);
              }
              tmem_st_16x256b_x4(tmem_o + lane_base + half * 64 + hc * 32, o);
            }
          }
          asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
          tc_fence_before();
          mbar_arrive((bars + (b ? 17 : 7)));
          if (r == 0 && half == 0) sstamp(J, 2);
        }
        if (gq == 0) {
          red[half * 128 + rA] = lA;
          red[half * 128 + rB] = lB;
          if (half == 0) {
            mrow[rA] = mA;
            mrow[rB] = mB;
          }
        }
      } else {
        for (int j = 0; j < nsub; ++j, ++J) {
          const int b = J & 1;
          const int keys = min(SUBP, np - j * SUBP) * 16;
          const int kbase = it.chunk_start + j * SUBP * 16 + half * 64;
          const int hkeys = min(64, keys - half * 64);  // this half's columns (may be <= 0)
          mbar_wait(&s_full[b], (J >> 1) & 1);
          tc_fence_after();
          if (r == 0 && half == 0) sstamp(J, 1);
          if (r == 0 && half == 0 && J == 0) stamp(2);
          uint32_t v[4][16];  // raw q.k of this half's (<= 64) keys
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            if (q4 * 16 < hkeys) tmem_ld16_nowait(tmem_base + b * 128 + lane_base + half * 64 + q4 * 16, v[q4]);
          tmem_wait_ld();
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) tmem_reg_fence(v[q4]);
          // visible keys of this half: [kbase, kbase + nvis); max of raw scores x sl2 (> 0)
          // equals the max of the scaled scores (rounding is monotonic)
          const int nvis = valid ? max(0, min(hkeys, pos + 1 - kbase)) : 0;
          if (nvis > 0 && nvis < 64) {
            // rare (the row's causal edge or a short last sub-chunk): invisible keys become
            // -inf once, so the max and exp loops below carry no per-key predicates
            asm volatile("" ::: "memory");
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
              for (int jj = 0; jj < 16; ++jj)
                if (q4 * 16 + jj >= nvis) v[q4][jj] = 0xff800000u;  // -inf
          }
          float mx = -INFINITY;
          if (nvis > 0) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
              for (int jj = 0; jj < 16; ++jj) mx = fmaxf(mx, __uint_as_float(v[q4][jj]));
          }
          // exchange with the partner thread (same row, other half); the second barrier lets
          // the buffer be rewritten next iteration
          red[half * 128 + r] = mx;
          named_bar_sync(1 + quarter, 64);
          const float m_cand = fmaxf(m_run, __fmul_rn(fmaxf(red[r], red[128 + r]), sl2));
          named_bar_sync(1 + quarter, 64);
          // lazy max: keep the reference while the new scores stay within 2^8 of it (P <= 256
          // is exact enough in bf16 / fp32), so O is rescaled only when the max jumps
          const float m_new = (m_cand > m_run + 8.f) ? m_cand : m_run;
          const float corr = (m_run == -INFINITY) ? 1.f : ex2_approx(m_run - m_new);
          // P buffer b was last read by P.V(J - 2)
          if (J >= 2) mbar_wait(&p_free[b], ((J >> 1) - 1) & 1);
          tc_fence_after();
          // this half's 64 keys -> 32 packed bf16x2 columns of TMEM P buffer b
          const uint32_t pcol = tmem_base + lane_base + L::P_COL + b * 64 + half * 32;
          float ls[4] = {0.f, 0.f, 0.f, 0.f};  // four short row-sum chains instead of two long ones
          const float nm = -m_new;
#pragma unroll
          for (int hb = 0; hb < 2; ++hb) {  // 32 keys -> 16 packed columns, stored at once
            uint32_t pk[16];
            if (nvis > 0) {  // padding rows, rows past their position: P is zero
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                const int q4 = hb * 2 + q;
#pragma unroll
                for (int jj = 0; jj < 16; jj += 2) {
                  // every exponential on the SFU (measured faster than an FMA-pipe share); masked
                  // keys and columns past a short sub-chunk hold -inf: exp2(-inf) = +0
                  const float p0 = ex2_approx(fmaf(__uint_as_float(v[q4][jj]), sl2, nm));
                  const float p1 = ex2_approx(fmaf(__uint_as_float(v[q4][jj + 1]), sl2, nm));
                  ls[(jj >> 1) & 3] += p0 + p1;
                  __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                  pk[q * 8 + (jj >> 1)] = *reinterpret_cast<uint32_t*>(&h2);
                }
              }
            } else {
#pragma unroll
              for (int c = 0; c < 16; ++c) pk[c] = 0u;
            }
            // (columns past the sub-chunk's pages are never read by P.V)
            if (hkeys > 0) tmem_st16(pcol + hb * 16, pk);
          }
          l_part = fmaf(l_part, corr, (ls[0] + ls[1]) + (ls[2] + ls[3]));
          m_run = m_new;
          if (j > 0 && __any_sync(0xffffffffu, valid && corr != 1.f)) {
            // the max moved: rescale this half's 64 O columns once P.V(J - 1) has landed
            mbar_wait(o_done, (J - 1) & 1);
            tc_fence_after();
            uint32_t o[4][16];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) tmem_ld16_nowait(tmem_o + lane_base + half * 64 + q4 * 16, o[q4]);
            tmem_wait_ld();
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              tmem_reg_fence(o[q4]);
#pragma unroll
              for (int jj = 0; jj < 16; ++jj) o[q4][jj] = __float_as_uint(__uint_as_float(o[q4][jj]) * corr);
              tmem_st16(tmem_o + lane_base + half * 64 + q4 * 16, o[q4]);
            }
          }
          asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");  // P (and rescaled O) in TMEM
          tc_fence_before();
          mbar_arrive((bars + (b ? 17 : 7)));
          if (r == 0 && half == 0) sstamp(J, 2);
        }
        red[half * 128 + r] = l_part;
        if (half == 0) mrow[r] = m_run;
      }
      if (r == 0 && half == 0) stamp(4);
      // ---------------- epilogue: unnormalised partial O and (m, l), straight from TMEM
      // (each thread 256 contiguous bytes of its entry's row) ----------------
      mbar_wait(o_final, n & 1);  // the unit's last P.V landed (single phase per unit)
      tc_fence_after();
      // the partial buffers (and the merge counters) belong to this launch only once the
      // previous kernel has completed
      if (k == k_begin) pdl_wait();
      if (r == 0 && half == 0) stamp(0);
      named_bar_sync(1 + quarter, 64);
      const float l = red[r] + red[128 + r];
      m_run = mrow[r];
      named_bar_sync(1 + quarter, 64);  // red is rewritten by the next unit's first exchange
      uint32_t o[4][16];
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) tmem_ld16_nowait(tmem_o + lane_base + half * 64 + q4 * 16, o[q4]);
      tmem_wait_ld();
      if (k + 1 == k_end) {
        // the CTA's last unit (the one on the critical path): no K/V load is pending any more
        // and the last P.V has read its stage, so the partial goes through the free stage
        // memory -- rows of 512 B at a 528-byte pitch (bank-conflict-free float4 writes) -- and
        // leaves as one 512-byte TMA bulk copy per row instead of sixteen strided 16-byte
        // stores per thread (measured: ~1.5 us of store issue at the C4 tail)
        float4* srow = reinterpret_cast<float4*>(smem + L::STAGE0 + r * 528 + half * 256);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          tmem_reg_fence(o[q4]);
#pragma unroll
          for (int jj = 0; jj < 16; jj += 4)
            srow[q4 * 4 + jj / 4] = make_float4(__uint_as_float(o[q4][jj]), __uint_as_float(o[q4][jj + 1]),
                                                __uint_as_float(o[q4][jj + 2]), __uint_as_float(o[q4][jj + 3]));
        }
        fence_proxy_async();  // generic-proxy smem writes -> visible to the bulk copy
        named_bar_sync(1 + quarter, 64);
        if (valid && half == 0) {
          bulk_store(part_o + slot * 128, smem + L::STAGE0 + r * 528, 512);
          bulk_commit();
          part_ml[slot] = make_float2(m_run, l);
          bulk_wait_all();
        }
      } else if (valid) {
        float4* dst = reinterpret_cast<float4*>(part_o + slot * 128 + half * 64);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          tmem_reg_fence(o[q4]);
#pragma unroll
          for (int jj = 0; jj < 16; jj += 4)
            dst[q4 * 4 + jj / 4] = make_float4(__uint_as_float(o[q4][jj]), __uint_as_float(o[q4][jj + 1]),
                                               __uint_as_float(o[q4][jj + 2]), __uint_as_float(o[q4][jj + 3]));
        }
        if (half == 0) part_ml[slot] = make_float2(m_run, l);
        if (r == 0 && half == 0) stamp(1);
      }
      // O may now be overwritten: the next unit's first P.V waits for this group's P arrive
      tc_fence_before();
      if (r == 0 && half == 0) stamp(5);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<L::TMEM_COLS>(tmem_base);
  if constexpr (kNarrow) {
    // ---------------- merge, in-kernel (long-chunk configurations): every CTA publishes its
    // units' partials (the barrier orders all of the CTA's partial stores before thread 0's
    // release), then merges (row, KV head) tasks cta + i * G, one per 128-thread group at a
    // time, once every unit of the launch is in -- no second launch and no PDL hand-off on
    // the critical path. The fold is merge_unit (attn_merge.cuh), the same fixed-order
    // function as the separate merge kernel of short-chunk configurations.
    // One 64-bit counter that never needs re-arming: every launch adds exactly 2^20 to it
    // (CTA 0 adds 2^20 - (G - 1), the others 1, each after publishing its units), so the
    // launch is complete when the counter reaches the next multiple of 2^20 above the value
    // a CTA saw. (Launches are ordered: a CTA adds only after griddepcontrol.wait, i.e. after
    // the previous launch, whose adds all precede it.)
    unsigned long long* done = reinterpret_cast<unsigned long long*>(merge_sync);
    unsigned long long* s_target = reinterpret_cast<unsigned long long*>(red);
    if (threadIdx.x == 0) {
      stamp(8);
      const unsigned long long mine = cta == 0 ? (1ull << 20) - (gridDim.x - 1) : 1ull;
      red_add_release_u64(done, mine);
      *s_target = merge_target;
    }
    __syncthreads();
    const unsigned long long target = *s_target;
    const int grp = threadIdx.x >> 7, lt = threadIdx.x & 127;
    const int ngrp = TC_THREADS / 128;
    bool waited = false;
    for (int task = cta + grp * (int)gridDim.x; task < n_rows * num_kv_heads;
         task += ngrp * (int)gridDim.x) {
      const int r = task / num_kv_heads, g = task % num_kv_heads;
      const int kind = row_kind[r], nch = row_pos[r] / chunk_tokens + 1;  // before the wait
      if (!waited) {
        if (lt == 0)
          while (ld_acquire_u64(done) < target) __nanosleep(32);
        named_bar_sync(1 + grp, 128);
        if (grp == 0 && lt == 0) stamp(10);
        waited = true;
      }
      merge_unit_call(part_o, part_ml, kind, nch, r, g, num_heads, group, max_chunks, out, out_ld, lt);
    }
  }
  if (threadIdx.x == 0) {
    stamp(9);
    if (span != nullptr) atomicMax(span + 1, globaltimer());
  }
}

// The 16-lane softmax form only pays on units of >= 4 sub-chunks, i.e. chunks of >= 32 pages
// (a deployment constant, so a captured graph's kernel choice stays valid); compiled in, it
// costs the 32-lane form register spills (measured: C2 decode attention 331 -> 370 us per
// step), so short-chunk configurations run the kernel without it. Both forms produce the same
// bits for a row.
cudaError_t attn_tc_partial_launch(const AttnLaunch& a, int chunk_pages, cudaStream_t s) {
  using L = TcLayout;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int units = a.n_items_cap * a.num_kv_heads;
  const int grid = units < a.num_sms ? units : a.num_sms;
  auto kern = chunk_pages >= 4 * SUBP ? attn_tc_kernel<true> : attn_tc_kernel<false>;
  return launch_pdl(kern, dim3(grid), dim3(TC_THREADS), L::SMEM, s,
                    a.tm_k, a.tm_v, a.tm_k8, a.tm_v8, a.q, a.q_ld, a.num_kv_heads, a.group, a.items, a.item_pages,
                    a.item_rows, a.row_pos, a.num_heads, a.max_chunks, a.scale, a.part_o, a.part_ml,
                    a.sched_off, a.sched_units, a.trace, a.chunk_tokens, a.span,
                    a.row_kind, a.n_rows, a.out, a.out_ld, a.merge_cnt);
}

}  // namespace icr
