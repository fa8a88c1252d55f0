// K1 fast path: paged GQA decode on tensor cores, persistent + split-KV
// (block_size 16, head_dim 64/128/256, group size <= 8).  Same semantics as
// k_paged_decode in decode.cu (reference: attention.py:92-127, metrics.py:
// 189-211, cache.py:163-184, engine.py:426-444).
//
// Kernel A (k_decode_stream): a persistent grid (2 CTAs per SM) pulls work
// items = (sequence, KV head, 512-position chunk) from an atomic queue
// (largest-position chunks last).  Each of the 4 warps streams its 16-token
// blocks of the item through a private TMA ring (cp.async.bulk.tensor,
// SWIZZLE_128B, one op for K and one for V per block) and runs
//   S^T[16 tok x 8 heads] = K . Q^T       d/16 x mma.m16n8k16 (bf16, fp32 acc)
//   online softmax per head
//   O^T[d x 8 heads]    += V^T . P^T      d/16 x mma.m16n8k16, P^T by movmatrix
// writing the fp32 scores of every position to a scratch row.  The warps'
// (m, l, O) are merged in shared memory into one partial per item.  The ring
// keeps streaming across item boundaries (the next item is fetched ahead).
// Kernel B (k_decode_finish): per (sequence, KV head) merges the partials
// (log-sum-exp), writes the output, and folds f(exp(s - M) / Z) into the
// metric of every attended slot (the appended slot is initialised: metric,
// logical = C, fresh), then C += 1.  Scores are 16 B/position against the
// 512 B/position of K+V, so the metric costs ~6% extra traffic and no
// grid-wide synchronisation.
#include <cuda.h>

#include <stdio.h>
#include <stdlib.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"

using namespace kvc;

namespace kvc_mma {

constexpr int kNW = 4;           // warps per CTA
constexpr int kThreads = kNW * 32;
constexpr int kBlk = 16;         // tokens per KV block
constexpr int kHP = 8;           // heads per MMA (group padded to 8)
constexpr int kItemBlocks = 16;  // max blocks per (warp) work item: 256 positions
// Blocks per work item for a launch: 16 (256 positions) unless that leaves
// fewer items than resident warps (small batches), then 8/4 - more,
// shorter split-KV items (down to 4 blocks) at the cost of more partials to merge.
static int item_blocks_for(int64_t pairs, int max_ctx) {
  static const int forced = getenv("KVC_K1_ITEM_BLOCKS") ? atoi(getenv("KVC_K1_ITEM_BLOCKS")) : 0;  // experiments
  if (forced >= 1 && forced <= kItemBlocks) return forced;
  const int64_t warps = 148 * 2 * 4;  // 2 CTAs x 4 warps per SM
  int ib = kItemBlocks;
  // (round 2: one item per resident warp is enough; B = 8 at 8 heads now
  // takes 256-position items, 1.05 -> 1.03 ms per step)
  while (ib > 4 && pairs * ((max_ctx + ib * kBlk - 1) / (ib * kBlk)) < warps) ib /= 2;
  return ib;
}

struct Params {
  kvc_pool p;
  const int32_t *rows;
  int batch, layer, r;
  const uint16_t *q, *k_new, *v_new;
  void *out;
  int out_f32;
  float *rows_out;
  int64_t rows_stride;
  int metric_mode, append_fresh, stages;
  int max_ctx_pad;  // score row length per (sequence, head)
  int item_tok;     // positions per work item (item_blocks_for * 16)
  int msplit;       // kernel B CTAs per (sequence, head): key slices of the metric pass
  int n_ck;         // chunks per (sequence, head) upper bound
  int n_items;
  float scale;      // log2(e)/sqrt(d)
  int *counter;     // work queue head (reset by kernel B for the next call)
  int *pair_done;   // [pairs] kernel B arrival counters (left zero by the last CTA of the pair)
  int metric_split; // 1: kernel B writes the output only; k_decode_metric (side stream) accumulates
  int need_scores;  // a metric or rows pass reads the score row (else kernel A skips it)
  void *metric_stream;
  int counter_ready;
  int early_pull;   // kernel A pulls its first item before griddepcontrol.wait (host-checked)
  int layer_chain;  // host only: a chain of consecutive layer launches (kvc_decode_args.early_pull 1 or 2)
  float *scores;    // [pairs][max_ctx_pad][r]
  float *part_ml;   // [pairs][n_ck][2][kHP]
  float *part_o;    // [pairs][n_ck][r][D]
  unsigned long long *trace;  // debug (KVC_K1_TRACE): [grid*warps][2] start/end globaltimer
  unsigned long long *trace_b;  // debug (KVC_K1_TRACE_PTR): kernel B [cta][2] after-wait/end globaltimer
};

// Programmatic dependent launch: the finish kernel (and the next stream) is launched
// while kernel A drains; they block here until A's writes are visible.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void tma3d(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar,
                                      uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// exp2 on the MUFU (ex2.approx, as in FlashAttention); -inf -> +0
__device__ __forceinline__ float ex2f_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &a0, uint32_t &a1, uint32_t &a2, uint32_t &a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &a0, uint32_t &a1, uint32_t &a2, uint32_t &a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}

__device__ __forceinline__ void mma16816(float *c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&v);
}

// byte offset of 16-byte chunk `c` of row `row` in a TMA SWIZZLE_128B block
// laid out as (d/64) atoms of 16 rows x 128 bytes.
__device__ __forceinline__ uint32_t swz(int row, int c) {
  return (uint32_t)((c >> 3) * (kBlk * 128) + row * 128 + (((c & 7) ^ (row & 7)) << 4));
}

// Warp work item: (sequence, KV head, kItemTok positions) + its block ids.
struct WItem {
  int id;     // -1 = none
  int bi, head, t0, t1, c_old, nblk;
  int64_t hidx;
  int32_t blk[kItemBlocks];
};

// Lane 0 pulls item ids until a non-empty chunk (or the queue ends); the
// whole warp then loads the item's table entries.  Chunk-major order keeps
// the long heads' tail chunks at the end of the queue.
__device__ void fetch_item(const Params &P, WItem &w, int lane) {
  const kvc_pool &p = P.p;
  const int H = p.num_kv_heads;
  const int pairs = P.batch * H;
  int id = -1, bi = 0, head = 0, t0 = 0, t1 = 0, c_old = 0;
  int64_t hidx = 0;
  if (lane == 0) {
    while (true) {
      const int cand = atomicAdd(P.counter, 1);
      if (cand >= P.n_items) break;
      const int ck = cand / pairs, pair = cand % pairs;
      const int b_ = pair / H, h_ = pair % H;
      const int64_t hx = head_index(p, P.rows[b_], P.layer, h_);
      const int co = p.ctx[hx];
      const int cp = co + (P.k_new ? 1 : 0);
      const int s0 = ck * P.item_tok;
      if (s0 < cp && cp <= p.nblocks[hx] * kBlk) {
        id = cand; bi = b_; head = h_; t0 = s0; t1 = min(cp, s0 + P.item_tok); c_old = co; hidx = hx;
        break;
      }
    }
  }
  id = __shfl_sync(0xffffffffu, id, 0);
  if (id < 0) {
    if (lane == 0) w.id = -1;
    __syncwarp();
    return;
  }
  bi = __shfl_sync(0xffffffffu, bi, 0);
  head = __shfl_sync(0xffffffffu, head, 0);
  t0 = __shfl_sync(0xffffffffu, t0, 0);
  t1 = __shfl_sync(0xffffffffu, t1, 0);
  c_old = __shfl_sync(0xffffffffu, c_old, 0);
  hidx = __shfl_sync(0xffffffffu, hidx, 0);
  const int nblk = (t1 - 1) / kBlk - t0 / kBlk + 1;
  if (lane < nblk) w.blk[lane] = p.tables[hidx * p.max_blocks + t0 / kBlk + lane];
  if (lane == 0) {
    w.id = id; w.bi = bi; w.head = head; w.t0 = t0; w.t1 = t1; w.c_old = c_old; w.nblk = nblk; w.hidx = hidx;
  }
  __syncwarp();
}

template <int D>
__global__ void __launch_bounds__(kThreads) k_decode_stream(const __grid_constant__ CUtensorMap tmK,
                                                           const __grid_constant__ CUtensorMap tmV,
                                                           const Params P) {
  constexpr int kBlkBytes = kBlk * D * 2;
  constexpr int kStageBytes = 2 * kBlkBytes;
  constexpr int kKS = D / 16;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stages = P.stages;
  const kvc_pool &p = P.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int H = p.num_kv_heads, r = P.r, n_q = H * r;
  if (P.trace && lane == 0) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    P.trace[(blockIdx.x * kNW + warp) * 2] = t0;
  }
  const bool append = P.k_new != nullptr;
  uint8_t *my_ring = smem + warp * stages * kStageBytes;
  uint64_t *my_bars = reinterpret_cast<uint64_t *>(smem + kNW * stages * kStageBytes) + warp * stages;
  WItem *wit = reinterpret_cast<WItem *>(smem + kNW * stages * kStageBytes + kNW * stages * 8) + warp * 2;

  if (lane == 0)
    for (int s = 0; s < stages; ++s) mbar_init(&my_bars[s], 1);
  fence_barrier_init();
  if (lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
  }
  const uint64_t pol = policy_evict_first();
  // scores and partials are read back within the layer: keep them in L2
  // (their readers discard the lines, so they never reach HBM)
  const uint64_t pol_keep = policy_evict_last();
  // the warp's block stream: all blocks of wit[cur], then of wit[cur^1]
  int cur = 0;
  int iss_item = 0, iss_k = 0;  // next fill: block iss_k of wit[(cur+iss_item)&1]
  int issued = 0, done = 0;
  auto try_issue = [&]() {  // lane 0
    while (issued - done < stages && iss_item < 2) {
      const WItem &w = wit[(cur + iss_item) & 1];
      if (w.id < 0) break;
      if (iss_k >= w.nblk) {
        if (iss_item == 0) { iss_item = 1; iss_k = 0; continue; }
        break;
      }
      const int y = w.blk[iss_k] * kBlk;
      const int s = issued % stages;
      uint8_t *dst = my_ring + s * kStageBytes;
      fence_proxy_async();
      mbar_expect_tx(&my_bars[s], kStageBytes);
      tma3d(dst, &tmK, 0, y, 0, &my_bars[s], pol);
      tma3d(dst + kBlkBytes, &tmV, 0, y, 0, &my_bars[s], pol);
      ++issued;
      ++iss_k;
    }
  };
  if (P.early_pull) {
    // First pull and its TMA loads before the dependency wait.  Only when
    // the caller guarantees (kvc_decode_args.early_pull) that the kernel in
    // front of this one is kernel B of another layer's launch over the same
    // queue: that kernel writes none of what the pull reads (this launch's
    // queue head - the heads alternate per launch -, this layer's C, tables,
    // rows).  Never after the allocator, compaction or a scatter, which do
    // write tables/nblocks/ctx.  Queries are read after the wait.
    if (lane == 0) wit[1].id = -1;
    fetch_item(P, wit[0], lane);
    if (lane == 0) try_issue();
  }
  __syncwarp();
  pdl_wait();     // the previous kernel's writes (ctx, tables, q, queue) are visible
  pdl_trigger();  // let kernel B's CTAs launch and park in griddepcontrol.wait
  if (!P.early_pull) fetch_item(P, wit[0], lane);
  fetch_item(P, wit[1], lane);
  if (lane == 0) try_issue();

  const int lm_tok = (lane & 7) + ((lane >> 3) & 1) * 8;
  const int lm_cadd = lane >> 4;
  const int lt_tok = (lane & 7) + (lane >> 4) * 8;
  const int lt_cadd = (lane >> 3) & 1;
  const bool hv0 = 2 * t < r, hv1 = 2 * t + 1 < r;

  while (wit[cur].id >= 0) {
    const int bi = wit[cur].bi, head = wit[cur].head, t0 = wit[cur].t0, t1 = wit[cur].t1;
    const int c_old = wit[cur].c_old, nblk = wit[cur].nblk, item_id = wit[cur].id;
    const int pair = bi * H + head;
    uint32_t qb[kKS][2];
    {
      const bool real = g < r;
      const uint16_t *qrow = P.q + ((int64_t)bi * n_q + head * r + (real ? g : 0)) * D;
#pragma unroll
      for (int kk = 0; kk < kKS; ++kk) {
        qb[kk][0] = real ? *reinterpret_cast<const uint32_t *>(qrow + kk * 16 + 2 * t) : 0u;
        qb[kk][1] = real ? *reinterpret_cast<const uint32_t *>(qrow + kk * 16 + 8 + 2 * t) : 0u;
      }
    }
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    float oacc[kKS][4];
#pragma unroll
    for (int i = 0; i < kKS; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
    float *srow_base = P.scores + (int64_t)pair * P.max_ctx_pad * r;
    for (int k = 0; k < nblk; ++k) {
      const int s = done % stages;
      mbar_wait(&my_bars[s], (done / stages) & 1);
      uint8_t *kb = my_ring + s * kStageBytes;
      uint8_t *vb = kb + kBlkBytes;
      const int tb0 = (t0 / kBlk + k) * kBlk;
      const int valid = min(kBlk, t1 - tb0);
      if (append && c_old >= tb0 && c_old < tb0 + kBlk) {
        const int off = c_old - tb0;
        const int64_t slot = (int64_t)wit[cur].blk[k] * kBlk + off;
        const uint4 *kn = reinterpret_cast<const uint4 *>(P.k_new + ((int64_t)bi * H + head) * D);
        const uint4 *vn = reinterpret_cast<const uint4 *>(P.v_new + ((int64_t)bi * H + head) * D);
        for (int c = lane; c < D / 8; c += 32) {
          const uint4 kv = kn[c], vv = vn[c];
          *reinterpret_cast<uint4 *>(kb + swz(off, c)) = kv;
          *reinterpret_cast<uint4 *>(vb + swz(off, c)) = vv;
          reinterpret_cast<uint4 *>(p.k_cache)[slot * (D / 8) + c] = kv;
          reinterpret_cast<uint4 *>(p.v_cache)[slot * (D / 8) + c] = vv;
        }
        __syncwarp();
      }
      // the block's K and V fragments go to registers first and the stage
      // returns to the ring before the math, so the next TMA overlaps it
      // (d <= 128: at d = 256 the fragments would not fit in registers)
      constexpr bool kEarly = D <= 128;
      constexpr int kVF = kEarly ? kKS : 1;
      uint32_t kf[kKS][4], vf[kVF][4];
      const uint32_t kbase = smem_u32(kb), vbase = smem_u32(vb);
#pragma unroll
      for (int kk = 0; kk < kKS; ++kk)
        ldsm_x4(kbase + swz(lm_tok, 2 * kk + lm_cadd), kf[kk][0], kf[kk][1], kf[kk][2], kf[kk][3]);
      if constexpr (kEarly) {
#pragma unroll
        for (int mt = 0; mt < kKS; ++mt)
          ldsm_x4_t(vbase + swz(lt_tok, 2 * mt + lt_cadd), vf[mt][0], vf[mt][1], vf[mt][2], vf[mt][3]);
        __syncwarp();
        ++done;
        if (lane == 0) try_issue();
      }
      // two independent accumulation chains over d
      float sc[4] = {0.f, 0.f, 0.f, 0.f}, sc2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < kKS; ++kk)
        mma16816((kk & 1) ? sc2 : sc, kf[kk][0], kf[kk][1], kf[kk][2], kf[kk][3], qb[kk][0], qb[kk][1]);
#pragma unroll
      for (int i = 0; i < 4; ++i) sc[i] += sc2[i];
      const bool tv0 = g < valid, tv1 = g + 8 < valid;
      const float s00 = (tv0 && hv0) ? sc[0] * P.scale : -INFINITY;
      const float s01 = (tv0 && hv1) ? sc[1] * P.scale : -INFINITY;
      const float s10 = (tv1 && hv0) ? sc[2] * P.scale : -INFINITY;
      const float s11 = (tv1 && hv1) ? sc[3] * P.scale : -INFINITY;
      if (P.need_scores) {
        float *r0 = srow_base + (int64_t)(tb0 + g) * r;
        float *r1 = r0 + 8 * r;
        if (tv0 && hv0) st_hint(r0 + 2 * t, s00, pol_keep);
        if (tv0 && hv1) st_hint(r0 + 2 * t + 1, s01, pol_keep);
        if (tv1 && hv0) st_hint(r1 + 2 * t, s10, pol_keep);
        if (tv1 && hv1) st_hint(r1 + 2 * t + 1, s11, pol_keep);
      }
      float bm0 = fmaxf(s00, s10), bm1 = fmaxf(s01, s11);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, o));
        bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, o));
      }
      const float mn0 = fmaxf(m0, bm0), mn1 = fmaxf(m1, bm1);
      const bool z0 = mn0 == -INFINITY, z1 = mn1 == -INFINITY;
      const float al0 = z0 ? 1.f : ex2f_fast(m0 - mn0);
      const float al1 = z1 ? 1.f : ex2f_fast(m1 - mn1);
      const float p00 = z0 ? 0.f : ex2f_fast(s00 - mn0);
      const float p10 = z0 ? 0.f : ex2f_fast(s10 - mn0);
      const float p01 = z1 ? 0.f : ex2f_fast(s01 - mn1);
      const float p11 = z1 ? 0.f : ex2f_fast(s11 - mn1);
      // the output only needs rescaling when some head's running max moved
      const bool rescale = __any_sync(0xffffffffu, al0 != 1.f || al1 != 1.f);
      m0 = mn0;
      m1 = mn1;
      l0 = l0 * al0 + p00 + p10;
      l1 = l1 * al1 + p01 + p11;
      const uint32_t pb0 = movmatrix_t(pack_bf16(p00, p01));
      const uint32_t pb1 = movmatrix_t(pack_bf16(p10, p11));
      if (rescale) {
#pragma unroll
        for (int mt = 0; mt < kKS; ++mt) {
          oacc[mt][0] *= al0;
          oacc[mt][1] *= al1;
          oacc[mt][2] *= al0;
          oacc[mt][3] *= al1;
        }
      }
      if constexpr (kEarly) {
#pragma unroll
        for (int mt = 0; mt < kKS; ++mt) mma16816(oacc[mt], vf[mt][0], vf[mt][1], vf[mt][2], vf[mt][3], pb0, pb1);
      } else {
#pragma unroll
        for (int mt = 0; mt < kKS; ++mt) {
          uint32_t a0, a1, a2, a3;
          ldsm_x4_t(vbase + swz(lt_tok, 2 * mt + lt_cadd), a0, a1, a2, a3);
          mma16816(oacc[mt], a0, a1, a2, a3, pb0, pb1);
        }
        __syncwarp();
        ++done;
        if (lane == 0) try_issue();
      }
    }
    // ---- this item's partial (m, l, O) straight from registers ----
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, o);
      l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    const int ck = t0 / P.item_tok;
    float *pml = P.part_ml + ((int64_t)pair * P.n_ck + ck) * 2 * kHP;
    float *po = P.part_o + ((int64_t)pair * P.n_ck + ck) * r * D;
    if (g == 0) {
      pml[2 * t] = m0;
      pml[2 * t + 1] = m1;
      pml[kHP + 2 * t] = l0;
      pml[kHP + 2 * t + 1] = l1;
    }
#pragma unroll
    for (int mt = 0; mt < kKS; ++mt) {
      if (hv0) {
        st_hint(po + (2 * t) * D + mt * 16 + g, oacc[mt][0], pol_keep);
        st_hint(po + (2 * t) * D + mt * 16 + g + 8, oacc[mt][2], pol_keep);
      }
      if (hv1) {
        st_hint(po + (2 * t + 1) * D + mt * 16 + g, oacc[mt][1], pol_keep);
        st_hint(po + (2 * t + 1) * D + mt * 16 + g + 8, oacc[mt][3], pol_keep);
      }
    }
    (void)item_id;
    // advance: the fetched-ahead item becomes current; refill the other slot
    const int fin = cur;
    cur ^= 1;
    if (iss_item == 1) iss_item = 0;
    else { iss_item = 0; iss_k = 0; }
    __syncwarp();
    if (wit[cur].id >= 0) fetch_item(P, wit[fin], lane);
    else if (lane == 0) wit[fin].id = -1;
    __syncwarp();
    if (lane == 0) try_issue();
  }
  if (P.trace && lane == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    P.trace[(blockIdx.x * kNW + warp) * 2 + 1] = t1;
  }
}

// Metric update for four consecutive positions per thread: R float4 score
// loads (the 4*R scores are contiguous), one float4 metric read-modify-write
// (four slots of one block are contiguous in the pool).
template <int R>
__device__ __forceinline__ void metric_quads(const Params &P, const float *srow, const int32_t *tab,
                                             const float *Ms, const float *iZ, int cp, int c_old, bool append,
                                             int q_lo, int q_hi) {
  const kvc_pool &p = P.p;
  float ms[R], iz[R];
#pragma unroll
  for (int h = 0; h < R; ++h) ms[h] = Ms[h], iz[h] = iZ[h];
  const int nq = min((cp + 3) / 4, q_hi);
  for (int g = q_lo + threadIdx.x; g < nq; g += blockDim.x) {
    const int p0 = g * 4;
    float sc[4 * R];
    if (p0 + 4 <= cp) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const float4 v = *reinterpret_cast<const float4 *>(srow + (int64_t)p0 * R + 4 * j);
        sc[4 * j] = v.x, sc[4 * j + 1] = v.y, sc[4 * j + 2] = v.z, sc[4 * j + 3] = v.w;
      }
    } else {  // last quad: the scores past cp were never written
      const int nv = (cp - p0) * R;
#pragma unroll
      for (int j = 0; j < 4 * R; ++j) sc[j] = j < nv ? srow[(int64_t)p0 * R + j] : 0.f;
    }
    float c[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      float a = 0.f;
#pragma unroll
      for (int h = 0; h < R; ++h) {
        const float w = exp2f(sc[o * R + h] - ms[h]) * iz[h];
        a += P.metric_mode == 2 ? w * w : w;
      }
      c[o] = a;
    }
    const int64_t f0 = (int64_t)tab[p0 / kBlk] * kBlk + p0 % kBlk;
    float4 *mp = reinterpret_cast<float4 *>(p.metric + f0);
    float4 m4 = *mp;
    float mv[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int pos = p0 + e;
      if (pos < cp) mv[e] = (append && pos == c_old) ? c[e] : mv[e] + c[e];
    }
    *mp = make_float4(mv[0], mv[1], mv[2], mv[3]);
    if (append && c_old >= p0 && c_old < p0 + 4) {
      const int64_t slot = f0 + (c_old - p0);
      p.logical[slot] = c_old;
      p.protected_[slot] = 0;
      p.fresh[slot] = P.append_fresh ? 1 : 0;
    }
  }
}

// After this CTA's metric pass: drop its score lines [q_lo, q_hi) quads
// (q_lo a multiple of 8 quads = 128*r bytes) from L2 without a write-back.
__device__ __forceinline__ void discard_scores(const float *srow, int r, int nq_all, int q_lo, int q_hi) {
  const int q_end = min(nq_all, q_hi);
  if (q_end <= q_lo) return;
  __syncthreads();
  const char *b = reinterpret_cast<const char *>(srow + (int64_t)q_lo * 4 * r);
  const int lines = ((q_end - q_lo) * 16 * r + 127) / 128;
  for (int i = threadIdx.x; i < lines; i += blockDim.x) discard_l2(b + (int64_t)i * 128);
}

// Metric / rows pass of kernel B when no side stream takes it: sum over the
// r heads of f(exp2(s - M) / Z) into metric[slot] for this CTA's key slice,
// the appended slot initialised (metrics.py:153-158, 189-211).
__device__ void finish_metric(const Params &P, int pair, int slice, int64_t hidx, int cp, int c_old, bool append,
                              const float *Ms, const float *iZ) {
  const kvc_pool &p = P.p;
  const int H = p.num_kv_heads, r = P.r;
  const int bi = pair / H, head = pair % H;
  // metric / rows over all attended positions
  const float *srow = P.scores + (int64_t)pair * P.max_ctx_pad * r;
  const int32_t *tab = head_table(p, hidx);
  // key slices in whole 8-quad units, so no 128-byte score line is shared
  // between CTAs (each CTA discards its own lines)
  const int nq_all = (cp + 3) / 4, qper = ((nq_all + gridDim.y - 1) / gridDim.y + 7) & ~7;
  const int q_lo = slice * qper, q_hi = q_lo + qper;
  if (P.metric_mode && !P.rows_out && (r == 1 || r == 2 || r == 4 || r == 8)) {
    switch (r) {
      case 1: metric_quads<1>(P, srow, tab, Ms, iZ, cp, c_old, append, q_lo, q_hi); break;
      case 2: metric_quads<2>(P, srow, tab, Ms, iZ, cp, c_old, append, q_lo, q_hi); break;
      case 4: metric_quads<4>(P, srow, tab, Ms, iZ, cp, c_old, append, q_lo, q_hi); break;
      default: metric_quads<8>(P, srow, tab, Ms, iZ, cp, c_old, append, q_lo, q_hi); break;
    }
    discard_scores(srow, r, nq_all, q_lo, q_hi);
  } else if (P.metric_mode || P.rows_out) {
    for (int pos = q_lo * 4 + threadIdx.x; pos < min(cp, q_hi * 4); pos += blockDim.x) {
      float contrib = 0.f;
      for (int h = 0; h < r; ++h) {
        const float w = exp2f(srow[(int64_t)pos * r + h] - Ms[h]) * iZ[h];
        contrib += P.metric_mode == 2 ? w * w : w;
        if (P.rows_out) P.rows_out[(((int64_t)bi * H + head) * r + h) * P.rows_stride + pos] = w;
      }
      if (P.metric_mode) {
        const int64_t slot = (int64_t)tab[pos / kBlk] * kBlk + pos % kBlk;
        if (append && pos == c_old) {
          p.metric[slot] = contrib;
          p.logical[slot] = c_old;
          p.protected_[slot] = 0;
          p.fresh[slot] = P.append_fresh ? 1 : 0;
        } else {
          p.metric[slot] += contrib;
        }
      }
    }
  }
  if (append && !P.metric_mode && p.metric && threadIdx.x == 0 && slice == 0) {
    const int64_t slot = (int64_t)tab[c_old / kBlk] * kBlk + c_old % kBlk;
    p.metric[slot] = 0.f;
    p.logical[slot] = c_old;
    p.protected_[slot] = 0;
    p.fresh[slot] = P.append_fresh ? 1 : 0;
  }
}

// Kernel B: per (sequence, head): merge partials, output, metric, C += 1,
// and the queue reset for the next launch (the former k_decode_bump).
template <int D>
__global__ void __launch_bounds__(256) k_decode_finish(const Params P) {
  extern __shared__ float sm[];
  float *Ms = sm, *iZ = sm + kHP, *fac = sm + 2 * kHP;  // fac: [n_ck][kHP]
  const kvc_pool &p = P.p;
  const int pair = blockIdx.x;
  const int slice = blockIdx.y;  // key slice of the metric pass / share of the outputs
  const int H = p.num_kv_heads, r = P.r, n_q = H * r;
  const int bi = pair / H, head = pair % H;
  // Prologue before the dependency wait: kernel A writes none of these
  // (it only reads ctx/tables/q), so they overlap A's tail.
  const int64_t hidx = head_index(p, P.rows[bi], P.layer, head);
  const int c_old = p.ctx[hidx];
  const bool append = P.k_new != nullptr;
  const int cp = c_old + (append ? 1 : 0);
  const int cap = p.nblocks[hidx] * kBlk;
  bool bad = false;  // NumericError: non-finite query (attention.py:33-36, 108)
  if (slice == 0) {
    const uint16_t *qg = P.q + ((int64_t)bi * n_q + head * r) * D;
    for (int e = threadIdx.x; e < r * D; e += blockDim.x) bad |= !isfinite(bf16_bits_to_f32(qg[e]));
  }
  pdl_wait();
  pdl_trigger();
  if (P.trace_b && threadIdx.x == 0) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    P.trace_b[(blockIdx.y * gridDim.x + blockIdx.x) * 2] = t0;
  }
  if (pair == 0 && slice == 0 && threadIdx.x == 0) *P.counter = 0;  // queue head for the next launch
  if (bad) set_status(p.status, KVC_DEV_NUMERIC, (int32_t)hidx, 0);
  if (cp < 1 || cp > cap || cp > P.max_ctx_pad) {  // no item ran (or not all of it) for this head
    if (slice == 0 && threadIdx.x == 0) {
      if (cp < 1) set_status(p.status, KVC_DEV_EMPTY_CONTEXT, (int32_t)hidx, 0);
      else if (cp > cap)
        set_status(p.status, append ? KVC_DEV_ALLOCATION_ORDER : KVC_DEV_CACHE_CORRUPTION, (int32_t)hidx, c_old);
      else  // C beyond the caller's max_ctx bound: the work items and score rows do not cover it
        set_status(p.status, KVC_DEV_CACHE_CORRUPTION, (int32_t)hidx, cp);
    }
    return;
  }
  const int nck = (cp + P.item_tok - 1) / P.item_tok;
  const float *pml = P.part_ml + (int64_t)pair * P.n_ck * 2 * kHP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // output share of this CTA in float4 groups; TPO adjacent lanes split one
  // group's chunk partials (fixed order).  The first 8 chunks' loads are in
  // flight while the head statistics are folded.
  constexpr int kCB = 8;
  const int E4 = r * D / 4;
  const int per = ((E4 + gridDim.y - 1) / gridDim.y + 7) & ~7;  // whole 128-byte lines per CTA
  const int g_lo = slice * per, g_hi = min(E4, g_lo + per);
  int tpo = 1;
  while (tpo < 32 && (g_hi - g_lo) * tpo * 2 <= (int)blockDim.x) tpo *= 2;
  const int sub = threadIdx.x % tpo;
  const int gi = g_lo + (int)threadIdx.x / tpo;
  const bool greal = gi < g_hi;
  const float4 *po4 = reinterpret_cast<const float4 *>(P.part_o + (int64_t)pair * P.n_ck * r * D) + (greal ? gi : 0);
  float4 v[kCB];
#pragma unroll
  for (int j = 0; j < kCB; ++j) {
    const int c = sub + j * tpo;
    v[j] = (greal && c < nck) ? __ldcg(po4 + (int64_t)c * E4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // head statistics: warp h folds head h's chunk partials in one pass
  // (lane-local online max), then fac[c][h] = exp2(m_c - M_h)
  if (warp < r) {
    const int h = warp;
    float mloc = -INFINITY, zloc = 0.f;
    for (int c = lane; c < nck; c += 32) {
      const float m = __ldcg(pml + c * 2 * kHP + h), l = __ldcg(pml + c * 2 * kHP + kHP + h);
      fac[c * kHP + h] = m;
      if (m != -INFINITY) {
        if (m > mloc) {
          zloc = zloc * ex2f_fast(mloc - m) + l;
          mloc = m;
        } else {
          zloc += l * ex2f_fast(m - mloc);
        }
      }
    }
    const float M = warp_max(mloc);
    const float Z = warp_sum(M == -INFINITY || mloc == -INFINITY ? 0.f : zloc * exp2f(mloc - M));
    __syncwarp();
    for (int c = lane; c < nck; c += 32) {
      const float m = fac[c * kHP + h];
      fac[c * kHP + h] = m == -INFINITY ? 0.f : exp2f(m - M);
    }
    if (lane == 0) {
      Ms[h] = M;
      iZ[h] = Z > 0.f ? 1.f / Z : 0.f;
    }
  }
  __syncthreads();
  {
    const int h = greal ? gi * 4 / D : 0;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c0 = sub;; c0 += kCB * tpo) {
#pragma unroll
      for (int j = 0; j < kCB; ++j) {
        const int c = c0 + j * tpo;
        const float f = c < nck ? fac[c * kHP + h] : 0.f;
        acc.x += v[j].x * f, acc.y += v[j].y * f, acc.z += v[j].z * f, acc.w += v[j].w * f;
      }
      if (c0 + kCB * tpo >= nck) break;
#pragma unroll
      for (int j = 0; j < kCB; ++j) {
        const int c = c0 + (kCB + j) * tpo;
        v[j] = (greal && c < nck) ? __ldcg(po4 + (int64_t)c * E4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    for (int o = 1; o < tpo; o <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
      acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
    }
    if (greal && sub == 0) {
      const float z = iZ[h];
      const int64_t oi = ((int64_t)bi * n_q + head * r) * D + (int64_t)gi * 4;
      if (P.out_f32) {
        float *o = reinterpret_cast<float *>(P.out) + oi;
        const float4 ov = make_float4(acc.x * z, acc.y * z, acc.z * z, acc.w * z);
        if ((reinterpret_cast<uintptr_t>(o) & 15) == 0) *reinterpret_cast<float4 *>(o) = ov;
        else o[0] = ov.x, o[1] = ov.y, o[2] = ov.z, o[3] = ov.w;
      } else {
        __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(P.out) + oi;
        const __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * z, acc.y * z);
        const __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z * z, acc.w * z);
        if ((reinterpret_cast<uintptr_t>(o) & 7) == 0) {
          uint2 u;
          u.x = *reinterpret_cast<const uint32_t *>(&lo);
          u.y = *reinterpret_cast<const uint32_t *>(&hi);
          *reinterpret_cast<uint2 *>(o) = u;
        } else {
          o[0] = lo.x, o[1] = lo.y, o[2] = hi.x, o[3] = hi.y;
        }
      }
    }
  }
  // the chunk partials are consumed: drop this CTA's lines from L2
  if (g_hi > g_lo) {
    __syncthreads();
    const int lpc = (g_hi - g_lo) / 8;
    const char *b0 = reinterpret_cast<const char *>(P.part_o + (int64_t)pair * P.n_ck * r * D) + (int64_t)g_lo * 16;
    for (int i = threadIdx.x; i < nck * lpc; i += blockDim.x)
      discard_l2(b0 + (int64_t)(i / lpc) * E4 * 16 + (int64_t)(i % lpc) * 128);
  }
  if (!P.metric_split) finish_metric(P, pair, slice, hidx, cp, c_old, append, Ms, iZ);
  if (P.trace_b && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    P.trace_b[(blockIdx.y * gridDim.x + blockIdx.x) * 2 + 1] = t1;
  }
  // C += 1 once every CTA of the pair has read C (the last to arrive bumps;
  // k_decode_metric on the side stream runs after this kernel and sees C + 1)
  if (append) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (gridDim.y == 1) {
        p.ctx[hidx] = c_old + 1;
      } else {
        __threadfence();
        if (atomicAdd(&P.pair_done[pair], 1) == (int)gridDim.y - 1) {
          P.pair_done[pair] = 0;
          p.ctx[hidx] = c_old + 1;
        }
      }
    }
  }
}

// Metric half of kernel B on a side stream, after kernel B (C already
// bumped: c_old = C - 1 when appending): head statistics from the partials,
// then metric[slot] += sum_h f(exp2(s - M)/Z) over the attended positions and
// the appended slot's metric/logical/fresh (metrics.py:153-158, 189-211).
template <int D>
__global__ void __launch_bounds__(256) k_decode_metric(const Params P) {
  __shared__ float Ms[kHP], iZ[kHP];
  const kvc_pool &p = P.p;
  const int pair = blockIdx.x, slice = blockIdx.y;
  const int H = p.num_kv_heads, r = P.r;
  const int bi = pair / H, head = pair % H;
  const int64_t hidx = head_index(p, P.rows[bi], P.layer, head);
  const bool append = P.k_new != nullptr;
  const int cp = p.ctx[hidx];
  const int c_old = cp - (append ? 1 : 0);
  // (kernel B rejected heads beyond max_ctx without bumping C)
  if (cp < 1 || cp > p.nblocks[hidx] * kBlk || cp > P.max_ctx_pad || p.status[0] == KVC_DEV_CACHE_CORRUPTION) return;
  const int nck = (cp + P.item_tok - 1) / P.item_tok;
  const float *pml = P.part_ml + (int64_t)pair * P.n_ck * 2 * kHP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < kHP) {
    const int h = warp;
    float M = -INFINITY;
    for (int c = lane; c < nck; c += 32) M = fmaxf(M, __ldcg(pml + c * 2 * kHP + h));
    M = warp_max(M);
    float Z = 0.f;
    for (int c = lane; c < nck; c += 32) {
      const float m = __ldcg(pml + c * 2 * kHP + h);
      if (m != -INFINITY) Z += __ldcg(pml + c * 2 * kHP + kHP + h) * exp2f(m - M);
    }
    Z = warp_sum(Z);
    if (lane == 0) {
      Ms[h] = M;
      iZ[h] = Z > 0.f ? 1.f / Z : 0.f;
    }
  }
  __syncthreads();
  const float *srow = P.scores + (int64_t)pair * P.max_ctx_pad * r;
  const int32_t *tab = head_table(p, hidx);
  const int nq_all = (cp + 3) / 4, qper = ((nq_all + gridDim.y - 1) / gridDim.y + 7) & ~7;
  const int q_lo = slice * qper, q_hi = q_lo + qper;
  switch (r) {
    case 1: metric_quads<1>(P, srow, tab, Ms, iZ, cp, c_old, append, q_lo, q_hi); break;
    case 2: metric_quads<2>(P, srow, tab, Ms, iZ, cp, c_old, append, q_lo, q_hi); break;
    case 4: metric_quads<4>(P, srow, tab, Ms, iZ, cp, c_old, append, q_lo, q_hi); break;
    default: metric_quads<8>(P, srow, tab, Ms, iZ, cp, c_old, append, q_lo, q_hi); break;
  }
  discard_scores(srow, r, nq_all, q_lo, q_hi);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// Cached 3-D SWIZZLE_128B map over a [num_blocks*16, d] bf16 pool viewed as
// {64 elems, rows, d/64 atoms}; the box {64, 16, d/64} is one whole block.
static bool pool_map(CUtensorMap *out, const void *base, int64_t rows, int D) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, CUtensorMap> cache;
  const uint64_t key = reinterpret_cast<uint64_t>(base) * 1315423911ull ^ ((uint64_t)rows << 8) ^ (uint64_t)D;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(D / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)kBlk, (cuuint32_t)(D / 64)};
  cuuint32_t estr[3] = {1, 1, 1};
  if (fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  cache[key] = *out;
  return true;
}

static bool pdl_off() {
  static const bool off = getenv("KVC_NO_PDL") != nullptr;
  return off;
}

static void launch_pdl(void (*fn)(const Params), int grid, int threads, int smem, cudaStream_t s, const Params &P,
                       int grid_y = 1) {
  const bool off = pdl_off();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, grid_y);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = off ? 0 : 1;
  cudaLaunchKernelEx(&cfg, fn, P);
}

int stream_smem(int D, int stages) {
  return kNW * stages * 2 * kBlk * D * 2 + kNW * stages * 8 + kNW * 2 * (int)sizeof(WItem) + 1024 + 64;
}

template <int D>
int launch(Params &P, cudaStream_t s) {
  CUtensorMap tmK, tmV;
  const int64_t rows = P.p.num_blocks * kBlk;
  if (!pool_map(&tmK, P.p.k_cache, rows, D) || !pool_map(&tmV, P.p.v_cache, rows, D)) return KVC_ERR_CUDA;
  static const int env_stages = getenv("KVC_K1_STAGES") ? atoi(getenv("KVC_K1_STAGES")) : 0;  // experiments
  static const int env_ctas = getenv("KVC_K1_CTAS") ? atoi(getenv("KVC_K1_CTAS")) : 0;
  // d = 128 inside a chain of layer launches (the caller asked for the early
  // pull, e.g. a DecodeStepGraph step): a 2-stage ring (65 KB per CTA, 3 fit
  // an SM) with the grid kept at 2 CTAs per SM, so the next layer's kernel A
  // finds a free CTA slot on every SM and starts its early pull while this
  // layer's CTAs drain (graph step: B = 8 0.981 -> 0.972 ms, B = 64 5.921 ->
  // 5.895).  Stand-alone launches keep the 3-stage ring on both slots
  // (attention only at B = 8: 34.0 us per layer against 35.8 with 2 stages).
  const bool spare_slot = D == 128 && P.layer_chain;
  P.stages = env_stages > 0 ? env_stages : (D >= 256 || spare_slot) ? 2 : 3;
  const int smem = stream_smem(D, P.stages);
  auto fa = k_decode_stream<D>;
  auto fb = k_decode_finish<D>;
  static bool configured = false;
  if (!configured) {
    // (fails if the kernel ever gains static shared memory: report it rather
    // than fall back to the generic path silently on a 48 KB default)
    if (cudaFuncSetAttribute(fa, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
      return KVC_ERR_CUDA;
    cudaFuncSetAttribute(fb, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    configured = true;
  }
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fa, kThreads, smem);
  if (per_sm < 1) return KVC_ERR_UNSUPPORTED;
  const int cap_sm = env_ctas > 0 ? env_ctas : spare_slot ? 2 : 0;
  if (cap_sm > 0 && cap_sm < per_sm) per_sm = cap_sm;
  int grid = n_sm * per_sm;
  if (grid > P.n_items) grid = P.n_items;
  if (!P.counter_ready) cudaMemsetAsync(P.pair_done - 2, 0, (2 + P.batch * P.p.num_kv_heads) * sizeof(int), s);
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_off() ? 0 : 1;
    cudaLaunchKernelEx(&cfg, fa, tmK, tmV, P);
  }
  if (P.trace && !P.trace_b) {
    // debug: spread of the warps' end times in this launch (synchronises)
    const int nw = grid * kNW;
    unsigned long long *h = (unsigned long long *)malloc((size_t)nw * 16);
    cudaStreamSynchronize(s);
    cudaMemcpy(h, P.trace, (size_t)nw * 16, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, e_min = ~0ull, e_max = 0;
    for (int i = 0; i < nw; ++i) {
      t0 = h[2 * i] < t0 ? h[2 * i] : t0;
      e_min = h[2 * i + 1] < e_min ? h[2 * i + 1] : e_min;
      e_max = h[2 * i + 1] > e_max ? h[2 * i + 1] : e_max;
    }
    double e_mean = 0;
    for (int i = 0; i < nw; ++i) e_mean += (double)(h[2 * i + 1] - t0) / nw;
    fprintf(stderr, "[k1 trace] items %d warps %d: warp end min %.1f mean %.1f max %.1f us after first start\n", P.n_items,
            nw, (e_min - t0) / 1e3, e_mean / 1e3, (e_max - t0) / 1e3);
    free(h);
  }
  {
    const int smem_b = (2 + P.n_ck) * kHP * 4;
    if (smem_b > 64 * 1024) return KVC_ERR_UNSUPPORTED;
    const int pairs_b = P.batch * P.p.num_kv_heads;
    // small batches: several CTAs per (sequence, head) share the merge and
    // (without the side-stream metric kernel) the metric pass; each CTA
    // folds the head statistics itself.  Eager: 256 / pairs, at most 8.
    // With the metric on the side stream (the CUDA-graph step) kernel B only
    // merges, and its CTAs hold registers the next layer's kernel A CTAs
    // need to land (per-layer timeline: A's entries spread over the 4 us of
    // B at 256 B CTAs): one CTA per pair from 16 pairs up - B = 2 / 4 / 8
    // at 8 heads 0.59 / 0.67 / 1.03 -> 0.56 / 0.64 / 0.99 ms per step -,
    // 8 for <= 8 pairs (B = 1: 0.45 vs 0.50 ms with 1)
    int ms = 256 / (pairs_b > 0 ? pairs_b : 1);
    ms = ms < 1 ? 1 : ms > 8 ? 8 : ms;
    if (P.metric_split && pairs_b > 8) ms = 1;
    static const int ms_forced = getenv("KVC_K1_MSPLIT") ? atoi(getenv("KVC_K1_MSPLIT")) : 0;  // experiments
    if (ms_forced > 0) ms = ms_forced;
    launch_pdl(fb, pairs_b, 256, smem_b, s, P, ms);
  }
  const int pairs = P.batch * P.p.num_kv_heads;
  if (P.metric_split) {
    // fork: the metric accumulation runs beside the caller's next work on s
    static cudaEvent_t ev[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64) return KVC_ERR_UNSUPPORTED;
    if (!ev[dev]) cudaEventCreateWithFlags(&ev[dev], cudaEventDisableTiming);
    cudaStream_t ms = reinterpret_cast<cudaStream_t>(P.metric_stream);
    cudaEventRecord(ev[dev], s);
    cudaStreamWaitEvent(ms, ev[dev], 0);
    static const int mm_div = getenv("KVC_K1_METRIC_DIV") ? atoi(getenv("KVC_K1_METRIC_DIV")) : 256;  // experiments
    int msplit = mm_div / (pairs > 0 ? pairs : 1);
    msplit = msplit < 1 ? 1 : msplit > 8 ? 8 : msplit;
    k_decode_metric<D><<<dim3(pairs, msplit), 256, 0, ms>>>(P);
  }
  return cudaGetLastError() == cudaSuccess ? KVC_OK : KVC_ERR_CUDA;
}

}  // namespace kvc_mma

// Per-(device, stream) launch log: launches so far (queue-head parity) and the
// layer of the last one.
struct StreamKeyHash {
  size_t operator()(const std::pair<int, cudaStream_t> &k) const {
    return std::hash<void *>()(reinterpret_cast<void *>(k.second)) * 31u + (size_t)k.first;
  }
};
static std::mutex &launch_mu() {
  static std::mutex mu;
  return mu;
}
static std::unordered_map<std::pair<int, cudaStream_t>, std::pair<long long, int>, StreamKeyHash> &launch_log() {
  static std::unordered_map<std::pair<int, cudaStream_t>, std::pair<long long, int>, StreamKeyHash> m;
  return m;
}

// Workspace bytes the fast path needs (scores + partials + queue head).
static int64_t kvc_decode_mma_scratch(const kvc_pool *pool, int batch, int r, int max_ctx) {
  using namespace kvc_mma;
  const int64_t pairs = (int64_t)batch * pool->num_kv_heads;
  const int tok = item_blocks_for(pairs, max_ctx) * kBlk;
  const int64_t ctxp = ((int64_t)max_ctx + tok - 1) / tok * tok;
  const int64_t nck = ctxp / tok;
  return (2 + pairs) * 4 + 256 + pairs * ctxp * r * 4 + pairs * nck * 2 * kHP * 4 + pairs * nck * r * pool->head_dim * 4 +
         4096;
}

extern "C" int64_t kvc_decode_scratch_bytes(const kvc_pool *pool, int32_t batch, int32_t num_query_heads,
                                            int32_t max_ctx) {
  if (!pool || pool->num_kv_heads < 1) return 0;
  const int r = num_query_heads / pool->num_kv_heads;
  return kvc_decode_mma_scratch(pool, batch, r < 1 ? 1 : r, max_ctx > 0 ? max_ctx : 1);
}

// Returns KVC_ERR_UNSUPPORTED when the shape is outside the fast path.
int kvc_decode_mma(const kvc_pool *pool, const kvc_decode_args *a, int, int, cudaStream_t s) {
  using namespace kvc_mma;
  const int H = pool->num_kv_heads, D = pool->head_dim;
  const int r = a->num_query_heads / H;
  if (pool->block_size != kBlk || r > kHP || (D != 64 && D != 128 && D != 256)) return KVC_ERR_UNSUPPORTED;
  if (!pool->scratch) return KVC_ERR_UNSUPPORTED;
  const int max_ctx = a->max_ctx > 0 ? a->max_ctx : 1;
  if (kvc_decode_mma_scratch(pool, a->batch, r, max_ctx) > pool->scratch_bytes) return KVC_ERR_UNSUPPORTED;
  Params P;
  P.p = *pool;
  P.rows = a->seq_rows;
  P.batch = a->batch;
  P.layer = a->layer;
  P.r = r;
  P.q = reinterpret_cast<const uint16_t *>(a->q);
  P.k_new = reinterpret_cast<const uint16_t *>(a->k_new);
  P.v_new = reinterpret_cast<const uint16_t *>(a->v_new);
  P.out = a->out;
  P.out_f32 = a->out_f32;
  P.rows_out = a->rows_out;
  P.rows_stride = a->rows_stride;
  P.metric_mode = a->metric_mode;
  P.append_fresh = a->append_fresh;
  P.metric_stream = a->metric_stream;
  P.need_scores = (a->metric_mode || a->rows_out) ? 1 : 0;
  P.metric_split = (a->metric_stream && a->metric_mode && !a->rows_out && (r == 1 || r == 2 || r == 4 || r == 8)) ? 1 : 0;
  P.item_tok = item_blocks_for((int64_t)a->batch * H, max_ctx) * kBlk;
  P.max_ctx_pad = (max_ctx + P.item_tok - 1) / P.item_tok * P.item_tok;
  P.n_ck = P.max_ctx_pad / P.item_tok;
  P.n_items = P.n_ck * a->batch * H;
  P.scale = 1.4426950408889634f / sqrtf((float)D);
  char *base = reinterpret_cast<char *>(pool->scratch);
  // work-queue head + per-pair counters: the caller's persistent zeroed
  // array (left zero by kernel B), else a scratch copy zeroed per launch
  // two queue heads, alternating per launch on a stream (a launch may pull
  // from its head while the previous launch's kernel B still runs), then
  // the per-pair counters
  int *qbase = a->queue ? a->queue : reinterpret_cast<int *>(base);
  // Queue-head parity alternates per launch on a (device, stream): a launch
  // pulling early from its head must not share it with the previous launch,
  // whose kernel B resets that head after its trigger.  The early pull itself
  // is the caller's promise (a->early_pull: the work right before this call on
  // the stream is kernel B of another layer over the same queue - e.g. layer
  // m > 0 of a DecodeStepGraph step); the host adds what it can check.  The
  // launch count is committed only after a successful launch.
  int dev_id = 0;
  cudaGetDevice(&dev_id);
  const std::pair<int, cudaStream_t> skey{dev_id, s};
  int parity = 0;
  bool early = false;
  {
    std::lock_guard<std::mutex> lk(launch_mu());
    auto &last = launch_log();
    auto it = last.find(skey);
    const long long n_prev = it == last.end() ? 0 : it->second.first;
    const int layer_prev = it == last.end() ? -1 : it->second.second;
    parity = (int)(n_prev & 1);
    early = a->early_pull == 1 && a->queue && layer_prev >= 0 && layer_prev != a->layer &&
            !getenv("KVC_NO_EARLY_PULL");
  }
  P.counter = qbase + parity;
  P.pair_done = qbase + 2;
  P.counter_ready = a->queue ? 1 : 0;
  P.early_pull = early ? 1 : 0;
  P.layer_chain = a->early_pull == 1 || a->early_pull == 2;
  int64_t off = ((int64_t)(2 + a->batch * H) * 4 + 255) / 256 * 256;
  P.scores = reinterpret_cast<float *>(base + off);
  off += (int64_t)a->batch * H * P.max_ctx_pad * r * 4;
  P.part_ml = reinterpret_cast<float *>(base + off);
  off += (int64_t)a->batch * H * P.n_ck * 2 * kHP * 4;
  P.part_o = reinterpret_cast<float *>(base + off);
  P.trace = nullptr;
  P.trace_b = nullptr;
  {
    // debug (KVC_K1_TRACE_PTR=<device address>, tools/trace_step.py):
    // per-layer globaltimer slots [layer % 64][65536] u64 - kernel A warps
    // at 0, kernel B CTAs at 32768 - set at capture time, so graph replays
    // fill them
    static const char *tp = getenv("KVC_K1_TRACE_PTR");
    if (tp) {
      unsigned long long *b = reinterpret_cast<unsigned long long *>(strtoull(tp, nullptr, 0));
      P.trace = b + (int64_t)(a->layer % 64) * 65536;
      P.trace_b = P.trace + 32768;
    }
  }
  {
    static int calls = 0;
    static unsigned long long *tbuf = nullptr;
    static const bool tr = getenv("KVC_K1_TRACE") != nullptr;
    if (tr && ++calls % 97 == 0) {  // every 97th launch (not under graph capture)
      if (!tbuf) cudaMalloc(&tbuf, 148 * 4 * kNW * 16);
      P.trace = tbuf;
    }
  }
  int rc;
  switch (D) {
    case 64: rc = launch<64>(P, s); break;
    case 128: rc = launch<128>(P, s); break;
    default: rc = launch<256>(P, s); break;
  }
  if (rc == KVC_OK) {
    std::lock_guard<std::mutex> lk(launch_mu());
    auto &e = launch_log()[skey];
    e.first += 1;
    e.second = a->layer;
  }
  return rc;
}
