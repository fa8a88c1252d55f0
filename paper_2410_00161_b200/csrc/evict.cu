// K3 eviction scheduler + K4 compaction (MoveCache) for a batch of sequences.
//
// Reference (pkg/src/pagedkv/compression.py): per head, slots get an
// effective metric (0 if empty, +inf if protected|fresh, :131-133) and are
// sorted by (metric, occupied, logical, position) (:156-166); threshold
// th[e-1] is the (b*e)-th smallest effective metric (:169-177); candidate
// rows of a sequence are ranked by (threshold, head_idx, row) and the first
// E rows with row < cap_h are evicted (:180-231); MoveCache then fills the
// holes below each head's eviction range with the range's survivors
// (:234-280) and the trailing blocks are freed and logicals renumbered
// (:283-309).
//
// B200 formulation (no sort at all, exact):
//  * #rows of head h with th <= v  ==  min(cap_h, floor(cnt_h(<= v) / b)),
//    where cnt_h counts slots with key <= v.  So the E-th smallest eligible
//    threshold T* of a sequence is found by an MSB radix search (11+11+10
//    bits) over per-head histograms of 32-bit order keys, with per-head
//    contributions min(cap, floor(cnt/b)) summed per sequence.
//  * e_h = L_h + take_h with L_h/U_h = rows with th < / <= T*, ties taken
//    in head order (head_idx is the reference's tie-break).
//  * the evicted slot set of a head = keys < T_h plus the first `need` ties
//    at T_h = (b*e_h)-th smallest key, ties ordered by (occupied, logical,
//    position) - a per-head radix select, not a sort.
//  * MoveCache pairing: k-th hole (ascending) below the range <-> k-th
//    survivor (descending) inside it; all pairs are disjoint, so K/V/metric
//    copies run concurrently.  Logical renumbering = rank via a bitmap
//    prefix-popcount (logicals are distinct).
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <climits>
#include <utility>

#include "common.cuh"

using namespace kvc;

namespace {

// Launch with programmatic stream serialisation: the kernel's CTAs may start
// while the previous kernel of the stream drains; every kernel of the chain
// opens with grid_dep_wait() before touching what its predecessor wrote.
template <typename... P, typename... A>
void launch_pdl(void (*fn)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, fn, std::forward<A>(args)...);
}

#ifndef KVC_C16_REGS
#define KVC_C16_REGS 64  // two 512-thread CTAs per SM
#endif
constexpr int kBins = 2048;       // 11-bit digits
constexpr int kThreads = 512;
constexpr uint32_t kKeyInf = 0xFF800000u;  // f32_order_key(+inf)
constexpr int kCand = 256;
#ifndef KVC_SH_U
#define KVC_SH_U 2  // short-head k_hist: uint4 key loads in flight per thread
#endif                 // candidate list capacity per head (short-head path)

struct EvictState {
  // per head (T = n_seqs * hp)
  uint32_t *keys;     // [T][max_slots]
  int32_t *cap;       // [T]
  int32_t *lo;        // [T] L_h
  int32_t *hi;        // [T] U_h
  int32_t *ltc;       // [T] keys < T*
  int32_t *lec;       // [T] keys <= T*
  int32_t *lt1, *lt2; // [T] keys < T* sharing T*'s top 11 / top 22 bits (select shortcuts)
  // per sequence
  int32_t *R;         // [n_seqs][kBins] contribution deltas per digit
  int32_t *done;      // [n_seqs] heads finished in the current histogram kernel (last one finds the digit)
  int32_t *done_all;  // [1] sequences whose select finished (the last one makes the offsets global)
  int32_t *kv_ready;  // [T] K/V move list published by the head's compaction CTA: moves + 1 (0 = not yet)
  int32_t *c16_done;  // [1] k_compact16 CTAs finished (the last one sums the free tiles)
  // long heads: the last digit level also yields the bounds (no k_bounds pass)
  int32_t *cum1;      // [T][2048] inclusive level-1 histogram (top 11 bits) of all keys
  int32_t *cum2;      // [T][2048] inclusive level-2 histogram of the keys matching T*'s top 11 bits
  int32_t *cum3;      // [T][1024] inclusive level-3 histogram of the keys matching T*'s top 22 bits
  int32_t *below3;    // [T] keys whose top 22 bits are below T*'s
  int32_t *lt1p;      // [T] keys with T*'s top 11 bits but lower top 22 bits
  // K/V copy queue: each published head appends its 32-move chunks
  int32_t *pub_count;  // [1] heads published
  int32_t *chunk_tail; // [1] chunks appended
  int32_t *claim_next; // [1] next chunk a copier warp takes
  unsigned long long *chunks;  // [max_chunks] (head + 1) << 32 | chunk of the head; 0 = not yet written
  int64_t max_chunks;
  int64_t *totals;    // nullable [4]: zeroed by k_load's first CTA
  int32_t *zero;      // R .. c16_done: one memset per call
  int64_t zero_n;
  uint32_t *prefix;   // [n_seqs] T* digits found so far
  int64_t *E;         // [n_seqs] clamped budget (0 = inactive)
  int64_t *seq_moves; // [n_seqs] move slots of the sequence, then its base offset
  unsigned long long *cand;  // nullable [T][2][kCand]: (key << 32 | secondary) of keys < T* / == T*
  unsigned long long *trace; // debug (KVC_K4_TRACE): [T][8] phase stamps of k_compact16
  int64_t max_slots;
  int hp;
  int32_t *status;
};

__device__ __forceinline__ uint32_t slot_key(const kvc_pool &p, int64_t f, bool occ) {
  if (!occ) return f32_order_key(0.f);
  if (p.protected_[f] | p.fresh[f]) return kKeyInf;
  return f32_order_key(p.metric[f]);
}

__device__ __forceinline__ int ld_acquire(const int32_t *a) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// Shared-memory histogram increment (same-bin lanes serialise in hardware;
// warp aggregation with match.any measured slower for metric keys).
__device__ __forceinline__ void hist_add(int32_t *hist, uint32_t bin, bool active) {
  if (active) atomicAdd(&hist[bin], 1);
}

// Four consecutive positions of one thread: equal active bins in a row (the
// pooled metric repeats a window maximum) are added with one atomic.
__device__ __forceinline__ void hist_add4(int32_t *hist, const uint32_t bin[4], const bool act[4]) {
  uint32_t cur = 0;
  int run = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (!act[e]) continue;
    if (run && bin[e] != cur) {
      atomicAdd(&hist[cur], run);
      run = 0;
    }
    cur = bin[e];
    ++run;
  }
  if (run) atomicAdd(&hist[cur], run);
}

// Per-head inclusive scan of a kBins histogram in smem (NT threads,
// 4 bins each).  Writes the inclusive cumulative counts back into hist.
template <int NT>
__device__ void scan_hist(int32_t *hist) {
  using Scan = cub::BlockScan<int32_t, NT>;
  __shared__ typename Scan::TempStorage tmp;
  constexpr int per = kBins / NT;
  int32_t v[per];
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < per; ++i) {
    v[i] = hist[threadIdx.x * per + i];
    s += v[i];
  }
  int32_t excl;
  __syncthreads();
  Scan(tmp).ExclusiveSum(s, excl);
#pragma unroll
  for (int i = 0; i < per; ++i) {
    excl += v[i];
    hist[threadIdx.x * per + i] = excl;
  }
  __syncthreads();
}

// Add this head's contribution deltas min(cap, floor((base+cum[c])/b)) to R
// (counts are < 2^31: one head's slots).
template <int NT>
__device__ void add_contrib(const int32_t *cum, int32_t base, int cap, int b, int32_t *R, int nbins) {
  // each thread takes nbins / NT consecutive bins (the delta of bin c needs
  // the row count of bin c - 1: one division per bin, none for the bins
  // whose cumulative count does not move); b is a power of two in practice
  const int per = nbins / NT;
  const int sh = (b & (b - 1)) == 0 ? __ffs(b) - 1 : -1;
  auto rows = [&](int32_t x) {
    const int32_t z = sh >= 0 ? x >> sh : x / b;
    return z > cap ? cap : z;
  };
  const int c0 = threadIdx.x * per;
  int32_t prev_cum = c0 > 0 ? cum[c0 - 1] : -1;
  int32_t a = c0 > 0 ? rows(base + prev_cum) : 0;
  for (int i = 0; i < per; ++i) {
    const int c = c0 + i;
    const int32_t cc = cum[c];
    if (cc == prev_cum) continue;  // empty bin: the row count stays
    const int32_t z = rows(base + cc);
    if (z > a) atomicAdd(&R[c], z - a);
    a = z;
    prev_cum = cc;
  }
}

// (2/4/6) per sequence: clamp E, find the first digit whose cumulative row
// count reaches E, append it to the prefix, reset R.  Run by the last CTA of
// the sequence to finish the preceding histogram kernel (NT threads).
template <int NT>
__device__ void find_digit(const int64_t *req, EvictState &S, int si, int level, int bits, int64_t *clamped) {
  using Scan = cub::BlockScan<int32_t, NT>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int found;
  int32_t *R = S.R + (int64_t)si * kBins;
  const int nbins = 1 << bits;
  if (level == 1) {
    // level 1 also computes the clamp: R summed over all bins = sum cap
    if (req[si] <= 0) {
      if (threadIdx.x == 0) { S.E[si] = 0; clamped[si] = req[si]; }  // min(req, sum cap) = req
      for (int c = threadIdx.x; c < kBins; c += NT) R[c] = 0;
      return;
    }
  } else if (S.E[si] <= 0) {
    return;
  }
  constexpr int per = kBins / NT;
  int32_t v[per];
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < per; ++i) {
    const int c = threadIdx.x * per + i;
    v[i] = c < nbins ? __ldcg(R + c) : 0;  // accumulated by other CTAs' atomics
    s += v[i];
  }
  int32_t excl, total;
  Scan(tmp).ExclusiveSum(s, excl, total);
  if (threadIdx.x == 0) found = kBins;
  __syncthreads();
  const int64_t E = level == 1 ? (req[si] < total ? req[si] : total) : S.E[si];  // min(requested, sum cap)
  if (E > 0) {
    int32_t run = excl;
#pragma unroll
    for (int i = 0; i < per; ++i) {
      run += v[i];
      const int c = threadIdx.x * per + i;
      if (c < nbins && run >= E) { atomicMin(&found, c); break; }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < kBins; c += NT) R[c] = 0;
  if (threadIdx.x == 0 && E > 0 && found >= nbins) set_status(S.status, KVC_DEV_SCHEDULE_CORRUPTION, si, level);
  if (threadIdx.x == 0) {
    if (level == 1) {
      S.E[si] = E;
      clamped[si] = E;
      S.prefix[si] = (uint32_t)found;
    } else {
      S.prefix[si] = (S.prefix[si] << bits) | (uint32_t)found;
    }
  }
}

// True in every thread of the CTA that is the last of sequence si's heads to
// arrive (its contributions and everyone else's are then visible); that CTA
// also re-arms the counter for the next kernel.
__device__ __forceinline__ bool last_of_sequence(EvictState &S, int si) {
  __shared__ int last_s;
  __syncthreads();
  if (threadIdx.x == 0) {
    // acq_rel arrival: releases this CTA's contributions (ordered before it
    // by the CTA barrier), and the last arrival acquires everyone else's
    // (read through L2 by find_digit)
    int prev;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(&S.done[si]) : "memory");
    last_s = prev == S.hp - 1;
    if (last_s) S.done[si] = 0;
  }
  __syncthreads();
  return last_s != 0;
}

// (1) keys + cap + level-1 histogram contributions.
// Returns true in the CTA that was the sequence's last to arrive (it found
// the level-1 digit).
template <int NT>
__device__ bool load_body(const kvc_pool &p, const int32_t *rows, const int64_t *req, EvictState &S, int with_hist,
                          int64_t *clamped) {
  __shared__ int32_t hist[kBins];
  __shared__ int32_t shield_s;
  const int g = blockIdx.x;
  if (g == 0 && threadIdx.x < 4 && S.totals) S.totals[threadIdx.x] = 0;  // the compaction accumulates them
  const int si = g / S.hp, hi = g % S.hp;
  const int64_t hidx = (int64_t)rows[si] * S.hp + hi;
  const int b = p.block_size;
  const int nb = p.nblocks[hidx];
  const int C = p.ctx[hidx];
  const int64_t n = (int64_t)nb * b;
  const int32_t *tab = head_table(p, hidx);
  uint32_t *keys = S.keys + (int64_t)g * S.max_slots;
  if (n > S.max_slots) {
    if (threadIdx.x == 0) set_status(p.status, KVC_DEV_CAPACITY, (int32_t)hidx, (int32_t)n);
    if (with_hist && last_of_sequence(S, si)) {
      find_digit<NT>(req, S, si, 1, 11, clamped);
      return true;
    }
    return false;
  }
  for (int i = threadIdx.x; i < kBins; i += NT) hist[i] = 0;
  if (threadIdx.x == 0) shield_s = 0;
  __syncthreads();
  int shield = 0;
  if (b == 16 && NT >= 512) {
    // one thread per 16-slot block (64 B metric, 16 B flags in, 64 B keys
    // out); the table entry of the thread's next block is loaded a round
    // ahead, so each round waits for one load latency, not two
    constexpr int U = 1;
    int32_t nxt = threadIdx.x < nb ? tab[threadIdx.x] : -1;
    for (int64_t base = 0; base < nb; base += NT * U) {
      int32_t blk[U];
      blk[0] = nxt;
      nxt = base + NT + threadIdx.x < nb ? tab[base + NT + threadIdx.x] : -1;
      float4 mv[U][4];
      uint4 pr[U], fr[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (blk[u] < 0) continue;
        const int64_t f0 = (int64_t)blk[u] * 16;
        const float4 *mp = reinterpret_cast<const float4 *>(p.metric + f0);
#pragma unroll
        for (int q = 0; q < 4; ++q) mv[u][q] = mp[q];
        pr[u] = *reinterpret_cast<const uint4 *>(p.protected_ + f0);
        fr[u] = *reinterpret_cast<const uint4 *>(p.fresh + f0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (blk[u] < 0) continue;
        const int64_t f0 = (int64_t)blk[u] * 16;
        const float4 *mp = reinterpret_cast<const float4 *>(p.metric + f0);
#pragma unroll
        for (int q = 0; q < 4; ++q) mv[u][q] = mp[q];
        pr[u] = *reinterpret_cast<const uint4 *>(p.protected_ + f0);
        fr[u] = *reinterpret_cast<const uint4 *>(p.fresh + f0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (blk[u] < 0) continue;  // (the block loop's tail: no histogram votes to keep uniform)
        const int64_t bl = base + u * NT + threadIdx.x;
        const uint32_t pw[4] = {pr[u].x | fr[u].x, pr[u].y | fr[u].y, pr[u].z | fr[u].z, pr[u].w | fr[u].w};
        uint4 *kp = reinterpret_cast<uint4 *>(keys + bl * 16);
        // runs of equal top digits (the pooled metric repeats a window
        // maximum over neighbouring slots) add to the histogram once per run
        uint32_t cur = 0xffffffffu;
        int run = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float mf[4] = {mv[u][q].x, mv[u][q].y, mv[u][q].z, mv[u][q].w};
          uint32_t kq[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int64_t pos = bl * 16 + q * 4 + e;
            const bool occ = pos < C;
            const bool sh = occ && ((pw[q] >> (8 * e)) & 0xff);
            shield += sh ? 1 : 0;
            kq[e] = !occ ? f32_order_key(0.f) : sh ? kKeyInf : f32_order_key(mf[e]);
            if (with_hist) {
              const uint32_t bin = kq[e] >> 21;
              if (bin != cur) {
                if (run) atomicAdd(&hist[cur], run);
                cur = bin;
                run = 0;
              }
              ++run;
            }
          }
          kp[q] = make_uint4(kq[0], kq[1], kq[2], kq[3]);
        }
        if (with_hist && run) atomicAdd(&hist[cur], run);
      }
    }
  } else if (b == 16) {
    // short heads (many CTAs: registers matter more than latency hiding)
    for (int64_t base = 0; base < nb; base += NT) {
      const int64_t bl = base + threadIdx.x;
      const bool in = bl < nb;
      uint32_t kk[16];
      if (in) {
        const int64_t f0 = (int64_t)tab[bl] * 16;
        const float4 *mp = reinterpret_cast<const float4 *>(p.metric + f0);
        const uint4 pr = *reinterpret_cast<const uint4 *>(p.protected_ + f0);
        const uint4 fr = *reinterpret_cast<const uint4 *>(p.fresh + f0);
        const uint32_t pw[4] = {pr.x | fr.x, pr.y | fr.y, pr.z | fr.z, pr.w | fr.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 mv = mp[q];
          const float mf[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int o = q * 4 + e;
            const int64_t pos = bl * 16 + o;
            const bool occ = pos < C;
            const bool sh = occ && ((pw[q] >> (8 * e)) & 0xff);
            shield += sh ? 1 : 0;
            kk[o] = !occ ? f32_order_key(0.f) : sh ? kKeyInf : f32_order_key(mf[e]);
          }
        }
        uint4 *kp = reinterpret_cast<uint4 *>(keys + bl * 16);
#pragma unroll
        for (int q = 0; q < 4; ++q) kp[q] = make_uint4(kk[4 * q], kk[4 * q + 1], kk[4 * q + 2], kk[4 * q + 3]);
      }
      if (with_hist) {
#pragma unroll
        for (int o = 0; o < 16; ++o) hist_add(hist, in ? kk[o] >> 21 : 0, in);
      }
    }
  } else {
    for (int64_t base = 0; base < n; base += NT) {
      const int64_t pos = base + threadIdx.x;
      const bool in = pos < n;
      uint32_t key = 0;
      if (in) {
        const int64_t f = (int64_t)tab[pos / b] * b + pos % b;
        const bool occ = pos < C;
        key = slot_key(p, f, occ);
        shield += (occ && (p.protected_[f] | p.fresh[f])) ? 1 : 0;
        keys[pos] = key;
      }
      if (with_hist) hist_add(hist, key >> 21, in);
    }
  }
  shield = __reduce_add_sync(0xffffffffu, shield);
  if ((threadIdx.x & 31) == 0) atomicAdd(&shield_s, shield);
  __syncthreads();
  const int sh_blocks = (shield_s + b - 1) / b;
  int cap = nb - (sh_blocks > 1 ? sh_blocks : 1);
  if (cap < 0) cap = 0;
  if (threadIdx.x == 0) S.cap[g] = cap;
  if (!with_hist) return false;
  if (req[si] > 0) {
    scan_hist<NT>(hist);
    if (S.cum1) {  // long heads: kept for k_compact16's threshold select
      int32_t *row = S.cum1 + (int64_t)g * kBins;
      for (int i = threadIdx.x; i < kBins; i += NT) row[i] = hist[i];
    }
    add_contrib<NT>(hist, 0, cap, b, S.R + (int64_t)si * kBins, kBins);
  }
  if (!last_of_sequence(S, si)) return false;
  find_digit<NT>(req, S, si, 1, 11, clamped);
  return true;
}

template <int NT>
__global__ void __launch_bounds__(NT, NT <= 256 ? 8 : 2) k_load(kvc_pool p, const int32_t *rows, const int64_t *req,
                                                  EvictState S, int with_hist, int64_t *clamped) {
  grid_dep_wait();
  grid_dep_trigger();
  load_body<NT>(p, rows, req, S, with_hist, clamped);
}

// (3/5) per head: histogram of the next digit among keys matching the prefix.
template <int NT>
__device__ bool hist_body(const kvc_pool &p, const int32_t *rows, EvictState &S, int shift_hi, int shift, int bits,
                          const int64_t *req, int level, int64_t *clamped) {
  __shared__ int32_t hist[kBins];
  __shared__ int64_t below_s;
  const int g = blockIdx.x;
  const int si = g / S.hp, hi = g % S.hp;
  if (S.E[si] <= 0) return false;
  const int64_t hidx = (int64_t)rows[si] * S.hp + hi;
  const int b = p.block_size;
  const int64_t n = (int64_t)p.nblocks[hidx] * b;
  const uint32_t pre = S.prefix[si];
  const uint32_t *keys = S.keys + (int64_t)g * S.max_slots;
  const uint32_t dmask = (1u << bits) - 1;
  for (int i = threadIdx.x; i < kBins; i += NT) hist[i] = 0;
  if (threadIdx.x == 0) below_s = 0;
  __syncthreads();
  int32_t below = 0;
  // long heads (NT = 512: one wave of CTAs, occupancy irrelevant): U uint4
  // loads per thread in flight before the histogram updates; the decode
  // round's short heads (NT = 256) keep one, for occupancy
  constexpr int U = NT >= 512 ? 8 : 1;
  if constexpr (U == 1) {
    // short heads (n <= 8192: 32-bit positions): KVC_SH_U uint4 loads per
    // thread in flight (one kept the decode round's k_hist latency-bound:
    // 4 dependent round trips per head at 2.2 TB/s)
    constexpr int V = KVC_SH_U;
    const int n32 = (int)n;
    for (int base = 0; base < n32; base += 4 * NT * V) {
      uint4 k4[V];
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const int pos = base + 4 * (u * NT + (int)threadIdx.x);  // max_slots is a multiple of 4
        k4[u] = pos < n32 ? __ldcg(reinterpret_cast<const uint4 *>(keys + pos))
                          : make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
      }
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const int pos = base + 4 * (u * NT + (int)threadIdx.x);
        const uint32_t kv[4] = {k4[u].x, k4[u].y, k4[u].z, k4[u].w};
        uint32_t bin[4];
        bool act[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool in = pos + e < n32;
          const uint32_t top = kv[e] >> shift_hi;
          below += (in && top < pre) ? 1 : 0;
          bin[e] = (kv[e] >> shift) & dmask;
          act[e] = in && top == pre;
        }
        hist_add4(hist, bin, act);
      }
    }
  } else {
    for (int64_t base = 0; base < n; base += 4 * NT * U) {
      uint4 k4[U];
  #pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t pos = base + 4 * ((int64_t)u * NT + threadIdx.x);  // max_slots is a multiple of 4
        k4[u] = pos < n ? *reinterpret_cast<const uint4 *>(keys + pos)
                        : make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
      }
  #pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t pos = base + 4 * ((int64_t)u * NT + threadIdx.x);
        const uint32_t kv[4] = {k4[u].x, k4[u].y, k4[u].z, k4[u].w};
        uint32_t bin[4];
        bool act[4];
  #pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool in = pos + e < n;
          const uint32_t top = kv[e] >> shift_hi;
          below += (in && top < pre) ? 1 : 0;
          bin[e] = (kv[e] >> shift) & dmask;
          act[e] = in && top == pre;
        }
        hist_add4(hist, bin, act);
      }
    }
  }
  below = __reduce_add_sync(0xffffffffu, below);
  if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long *)&below_s, (unsigned long long)below);
  __syncthreads();
  scan_hist<NT>(hist);
  if (S.cum2 && level == 2) {  // long heads: kept for k_compact16's threshold select
    int32_t *row = S.cum2 + (int64_t)g * kBins;
    for (int i = threadIdx.x; i < kBins; i += NT) row[i] = hist[i];
  }
  add_contrib<NT>(hist, (int32_t)below_s, S.cap[g], b, S.R + (int64_t)si * kBins, 1 << bits);
  if (!last_of_sequence(S, si)) return false;
  find_digit<NT>(req, S, si, level, bits, clamped);
  return true;
}

template <int NT>
__global__ void __launch_bounds__(NT, NT <= 256 ? 8 : 2) k_hist(kvc_pool p, const int32_t *rows, EvictState S, int shift_hi,
                                                  int shift, int bits, const int64_t *req, int level,
                                                  int64_t *clamped) {
  grid_dep_wait();
  grid_dep_trigger();
  hist_body<NT>(p, rows, S, shift_hi, shift, bits, req, level, clamped);
}

// (7) per head: rows with threshold < T* and <= T*.  With S.cand, also the
// composites (key << 32 | secondary) of the keys < T* and of the ties at T*
// (first kCand of each, any order) for k_compact_warp.
template <int NT>
__device__ void bounds_counts(const kvc_pool &p, const int32_t *rows, EvictState &S, int g, int si, int hi);
template <int NT>
__device__ void select_seq(EvictState &S, int si, int bsz, int32_t *evict, int64_t *move_off, int32_t *status);
template <int NT>
__device__ void offsets_all(EvictState &S, int n_seqs, int64_t *move_off);

// (7-8) per head: rows with threshold < T* and <= T*; then the last CTA of
// each sequence takes the tie rows in head order (e_h) and the last sequence
// makes the move offsets global.
template <int NT>
__device__ void bounds_body(const kvc_pool &p, const int32_t *rows, EvictState &S, int n_seqs, int bsz,
                            int32_t *evict, int64_t *move_off) {
  const int g = blockIdx.x;
  const int si = g / S.hp, hi = g % S.hp;
  if (S.E[si] > 0) bounds_counts<NT>(p, rows, S, g, si, hi);
  else if (threadIdx.x == 0) { S.lo[g] = 0; S.hi[g] = 0; }
}

// (8) short heads (the decode-time batch of thousands of heads): the tie
// rows of each sequence and the global move offsets in two small grids, so
// the many-CTA k_bounds stays lean (registers, shared memory, occupancy).
__global__ void __launch_bounds__(1024) k_select(EvictState S, int bsz, int32_t *evict, int64_t *move_off,
                                                int32_t *status) {
  grid_dep_wait();
  grid_dep_trigger();
  select_seq<1024>(S, blockIdx.x, bsz, evict, move_off, status);
}

__global__ void __launch_bounds__(1024) k_offsets(EvictState S, int n_seqs, int64_t *move_off) {
  grid_dep_wait();
  grid_dep_trigger();
  offsets_all<1024>(S, n_seqs, move_off);
}

template <int NT>
__global__ void __launch_bounds__(NT) k_bounds(kvc_pool p, const int32_t *rows, EvictState S, int n_seqs, int bsz,
                                                    int32_t *evict, int64_t *move_off) {
  grid_dep_wait();
  grid_dep_trigger();
  bounds_body<NT>(p, rows, S, n_seqs, bsz, evict, move_off);
}

// (5-8) long heads: the last digit level (10 bits of the keys matching T*'s
// top 22) with the bounds folded in.  Each head CTA keeps its inclusive
// histogram and its counts below the prefix; once the sequence's last CTA
// has T*, the per-head counts follow from them (rows < / <= T*, and the keys
// below T* that share its top 11 / 22 bits), so no pass re-reads the keys.
// That CTA then takes the tie rows (select_seq); the last sequence makes the
// move offsets global.
template <int NT>
__global__ void __launch_bounds__(NT) k_hist_final(kvc_pool p, const int32_t *rows, EvictState S, const int64_t *req,
                                                        int64_t *clamped, int n_seqs, int bsz, int32_t *evict,
                                                        int64_t *move_off) {
  grid_dep_wait();
  grid_dep_trigger();
  __shared__ int32_t hist[kBins];
  __shared__ int32_t below_s, lt1_s;
  const int g = blockIdx.x;
  const int si = g / S.hp, hi = g % S.hp;
  const int b = p.block_size;
  const bool active = S.E[si] > 0;
  if (active) {
    const int64_t hidx = (int64_t)rows[si] * S.hp + hi;
    const int64_t n = (int64_t)p.nblocks[hidx] * b;
    const uint32_t pre = S.prefix[si];  // T*'s top 22 bits
    const uint32_t pre1 = pre >> 11;     // its top 11
    const uint32_t *keys = S.keys + (int64_t)g * S.max_slots;
    for (int i = threadIdx.x; i < kBins; i += NT) hist[i] = 0;  // (the upper half stays zero for the scan)
    if (threadIdx.x == 0) { below_s = 0; lt1_s = 0; }
    __syncthreads();
    int32_t below = 0, lt1 = 0;
    constexpr int U = 8;
    for (int64_t base = 0; base < n; base += 4 * NT * U) {
      uint4 k4[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t pos = base + 4 * ((int64_t)u * NT + threadIdx.x);  // max_slots is a multiple of 4
        k4[u] = pos < n ? *reinterpret_cast<const uint4 *>(keys + pos) : make_uint4(~0u, ~0u, ~0u, ~0u);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t pos = base + 4 * ((int64_t)u * NT + threadIdx.x);
        const uint32_t kv[4] = {k4[u].x, k4[u].y, k4[u].z, k4[u].w};
        uint32_t bin[4];
        bool act[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool in = pos + e < n;
          const uint32_t top = kv[e] >> 10;
          below += (in && top < pre) ? 1 : 0;
          lt1 += (in && top < pre && (kv[e] >> 21) == pre1) ? 1 : 0;
          bin[e] = kv[e] & 1023u;
          act[e] = in && top == pre;
        }
        hist_add4(hist, bin, act);
      }
    }
    below = __reduce_add_sync(0xffffffffu, below);
    lt1 = __reduce_add_sync(0xffffffffu, lt1);
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&below_s, below);
      atomicAdd(&lt1_s, lt1);
    }
    __syncthreads();
    scan_hist<NT>(hist);  // inclusive
    int32_t *row = S.cum3 + (int64_t)g * 1024;
    for (int i = threadIdx.x; i < 1024; i += NT) row[i] = hist[i];
    if (threadIdx.x == 0) {
      S.below3[g] = below_s;
      S.lt1p[g] = lt1_s;
    }
    add_contrib<NT>(hist, below_s, S.cap[g], b, S.R + (int64_t)si * kBins, 1024);
  }
  if (!last_of_sequence(S, si)) return;
  if (active) {
    find_digit<NT>(req, S, si, 3, 10, clamped);
    __syncthreads();
    const uint32_t Ts = S.prefix[si];
    const int d3 = (int)(Ts & 1023u);
    for (int h = threadIdx.x; h < S.hp; h += NT) {
      const int64_t gg = (int64_t)si * S.hp + h;
      const int32_t *row = S.cum3 + gg * 1024;
      const int32_t c_lt = d3 > 0 ? __ldcg(row + d3 - 1) : 0;
      const int32_t c_le = __ldcg(row + d3);
      const int32_t bl = __ldcg(S.below3 + gg);
      const int32_t lt = bl + c_lt, le = bl + c_le;
      const int cap = __ldcg(S.cap + gg);
      S.lo[gg] = lt / b < cap ? lt / b : cap;
      S.hi[gg] = le / b < cap ? le / b : cap;
      S.ltc[gg] = lt;
      S.lec[gg] = le;
      S.lt2[gg] = c_lt;
      S.lt1[gg] = __ldcg(S.lt1p + gg) + c_lt;
    }
    __syncthreads();
  } else {
    for (int h = threadIdx.x; h < S.hp; h += NT) {
      const int64_t gg = (int64_t)si * S.hp + h;
      S.lo[gg] = 0;
      S.hi[gg] = 0;
    }
    __syncthreads();
  }
  select_seq<NT>(S, si, bsz, evict, move_off, p.status);
  __shared__ int last_all;
  __syncthreads();
  if (threadIdx.x == 0) {
    int prev;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(S.done_all) : "memory");
    last_all = prev == n_seqs - 1;
    if (last_all) *S.done_all = 0;
  }
  __syncthreads();
  if (last_all) offsets_all<NT>(S, n_seqs, move_off);
}


template <int NT>
__device__ void bounds_counts(const kvc_pool &p, const int32_t *rows, EvictState &S, int g, int si, int hi) {
  using Red = cub::BlockReduce<int32_t, NT>;
  __shared__ typename Red::TempStorage tmp;
  __shared__ int32_t cnt_s[2];
  const int64_t hidx = (int64_t)rows[si] * S.hp + hi;
  const int b = p.block_size;
  const int64_t n = (int64_t)p.nblocks[hidx] * b;
  const int C = p.ctx[hidx];
  const int32_t *tab = head_table(p, hidx);
  const uint32_t T = S.prefix[si];
  const uint32_t *keys = S.keys + (int64_t)g * S.max_slots;
  unsigned long long *cand = S.cand ? S.cand + (int64_t)g * 2 * kCand : nullptr;
  if (threadIdx.x < 2) cnt_s[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int32_t lt = 0, le = 0, l1 = 0, l2 = 0;
  const uint32_t T1 = T >> 21, T2 = T >> 10;
  if (!cand) {
    // batches of 8 uint4 per thread in flight
    constexpr int U = 8;
    for (int64_t base = 0; base < n; base += 4 * NT * U) {
      uint4 k4[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t pos = base + 4 * ((int64_t)u * NT + threadIdx.x);  // max_slots is a multiple of 4
        k4[u] = pos < n ? *reinterpret_cast<const uint4 *>(keys + pos) : make_uint4(~0u, ~0u, ~0u, ~0u);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t pos = base + 4 * ((int64_t)u * NT + threadIdx.x);
        const uint32_t kv[4] = {k4[u].x, k4[u].y, k4[u].z, k4[u].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool in = pos + e < n;
          const bool below = in && kv[e] < T;
          lt += below ? 1 : 0;
          le += (in && kv[e] <= T) ? 1 : 0;
          l1 += (below && (kv[e] >> 21) == T1) ? 1 : 0;
          l2 += (below && (kv[e] >> 10) == T2) ? 1 : 0;
        }
      }
    }
  } else {
    // short heads (n <= 8192): all of the head's keys in flight at once, 4
    // per uint4; match masks per thread, then block scans place the
    // candidates (no per-element votes)
    constexpr int U = 8192 / (4 * NT);
    uint4 k4[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int pos0 = (u * NT + threadIdx.x) * 4;
      k4[u] = pos0 < n ? *reinterpret_cast<const uint4 *>(keys + pos0) : make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    uint32_t mlt = 0, meq = 0;  // bit u*4+i
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int pos0 = (u * NT + threadIdx.x) * 4;
      const uint32_t kv[4] = {k4[u].x, k4[u].y, k4[u].z, k4[u].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool in = pos0 + i < n;
        const bool below = in && kv[i] < T;
        mlt |= (below ? 1u : 0u) << (u * 4 + i);
        meq |= (in && kv[i] == T ? 1u : 0u) << (u * 4 + i);
      }
    }
    using Scan = cub::BlockScan<int32_t, NT>;
    __shared__ typename Scan::TempStorage stmp;
    __shared__ int32_t tot_s[2];
    const uint32_t masks[2] = {mlt, meq};
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      int32_t excl, tot;
      Scan(stmp).ExclusiveSum(__popc(masks[l]), excl, tot);
      if (threadIdx.x == 0) tot_s[l] = tot;
      __syncthreads();
      if (tot_s[l] <= kCand) {
        for (uint32_t mb = masks[l]; mb; mb &= mb - 1) {
          const int bit = __ffs(mb) - 1;
          const int u = bit >> 2, i = bit & 3;
          const int pos = (u * NT + threadIdx.x) * 4 + i;
          const uint32_t kk = keys[pos];  // (re-read: indexing k4 here would put it in local memory)
          const int32_t lg = p.logical[(int64_t)tab[pos >> 4] * 16 + (pos & 15)];
          const uint32_t sc = pos < C ? (0x80000000u | (uint32_t)(lg + 1)) : (uint32_t)pos;
          cand[l * kCand + excl++] = ((unsigned long long)kk << 32) | sc;
        }
      }
    }
    lt = __popc(mlt);
    le = lt + __popc(meq);
  }
  lt = Red(tmp).Sum(lt);
  __syncthreads();
  le = Red(tmp).Sum(le);
  if (!cand) {  // top-bin counts for k_compact16's select shortcut (long heads only)
    __syncthreads();
    l1 = Red(tmp).Sum(l1);
    __syncthreads();
    l2 = Red(tmp).Sum(l2);
  }
  if (threadIdx.x == 0) {
    S.lt1[g] = l1;
    S.lt2[g] = l2;
    const int cap = S.cap[g];
    S.lo[g] = lt / b < cap ? lt / b : cap;
    S.hi[g] = le / b < cap ? le / b : cap;
    S.ltc[g] = lt;
    S.lec[g] = le;
  }
}

// (8) last CTA of a sequence: e_h = L_h + ties taken in head order, and the
// sequence-local exclusive offsets of e_h*b (made global by offsets_all).
// Other CTAs' counts are read through L2 (acquired by the arrival).
template <int NT>
__device__ void select_seq(EvictState &S, int si, int bsz, int32_t *evict, int64_t *move_off, int32_t *status) {
  using Scan = cub::BlockScan<int64_t, NT>;
  using Red = cub::BlockReduce<int64_t, NT>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ typename Red::TempStorage rtmp;
  __shared__ int64_t less_s;
  const int hp = S.hp;
  const int64_t E = S.E[si];
  // total rows strictly below T*
  int64_t less = 0;
  for (int h = threadIdx.x; h < hp; h += NT) less += E > 0 ? __ldcg(S.lo + (int64_t)si * hp + h) : 0;
  less = Red(rtmp).Sum(less);
  if (threadIdx.x == 0) less_s = less;
  __syncthreads();
  const int64_t need = E - less_s;  // tie rows to take at T*, in head order
  int64_t tcarry = 0, ocarry = 0;
  for (int base = 0; base < hp; base += NT) {
    const int h = base + threadIdx.x;
    const int64_t g = (int64_t)si * hp + h;
    int64_t ties = 0, lo = 0;
    if (h < hp && E > 0) {
      lo = __ldcg(S.lo + g);
      ties = __ldcg(S.hi + g) - lo;
    }
    int64_t excl, tot;
    Scan(tmp).ExclusiveSum(ties, excl, tot);
    int32_t eh = 0;
    if (h < hp) {
      int64_t take = need - (tcarry + excl);
      if (take < 0) take = 0;
      if (take > ties) take = ties;
      eh = E > 0 ? (int32_t)(lo + take) : 0;
      evict[g] = eh;
    }
    __syncthreads();
    int64_t oex, otot;
    Scan(tmp).ExclusiveSum((int64_t)eh * bsz, oex, otot);
    if (h < hp) move_off[g] = ocarry + oex;
    __syncthreads();
    tcarry += tot;
    ocarry += otot;
  }
  if (threadIdx.x == 0) {
    S.seq_moves[si] = ocarry;
    if (E > 0 && (need < 0 || need > tcarry)) set_status(status, KVC_DEV_SCHEDULE_CORRUPTION, si, (int32_t)need);
  }
}

// (8b) last sequence: sequence bases -> global exclusive offsets over all heads.
template <int NT>
__device__ void offsets_all(EvictState &S, int n_seqs, int64_t *move_off) {
  using Scan = cub::BlockScan<int64_t, NT>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int64_t T = (int64_t)n_seqs * S.hp;
  if (n_seqs == 1) {  // offsets are already global
    if (threadIdx.x == 0) move_off[T] = __ldcg(S.seq_moves);
    return;
  }
  for (int base = 0; base < n_seqs; base += NT) {
    const int si = base + threadIdx.x;
    const int64_t v = si < n_seqs ? __ldcg(S.seq_moves + si) : 0;
    int64_t excl, tot;
    Scan(tmp).ExclusiveSum(v, excl, tot);
    if (si < n_seqs) S.seq_moves[si] = carry + excl;  // now the sequence base
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  // eight independent loads in flight per thread (a decode round has
  // thousands of heads)
  for (int64_t g0 = threadIdx.x; g0 < T; g0 += 8 * NT) {
    int64_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t g = g0 + (int64_t)u * NT;
      v[u] = g < T ? __ldcg(move_off + g) + S.seq_moves[g / S.hp] : 0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t g = g0 + (int64_t)u * NT;
      if (g < T) move_off[g] = v[u];
    }
  }
  if (threadIdx.x == 0) move_off[T] = carry;
}

// Radix select inside one CTA: value of the `rank`-th (0-based) smallest of
// the values v(pos) over pos in [0, n) with pred(pos); returns the value and
// leaves in *rank_out the rank of the target among values equal to it.
template <typename GetV>
__device__ uint32_t cta_select(int32_t *hist, int64_t n, int64_t rank, GetV getv, int64_t *rank_out) {
  __shared__ uint32_t pre_s;
  __shared__ int64_t rank_s;
  const int shifts[3] = {21, 10, 0};
  const int bitsv[3] = {11, 11, 10};
  uint32_t pre = 0;
  for (int lv = 0; lv < 3; ++lv) {
    const int shift = shifts[lv], bits = bitsv[lv];
    const int shift_hi = shift + bits;
    const uint32_t dmask = (1u << bits) - 1;
    for (int i = threadIdx.x; i < kBins; i += kThreads) hist[i] = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += kThreads) {
      const int64_t pos = base + threadIdx.x;
      bool ok = false;
      uint32_t v = 0;
      if (pos < n) ok = getv(pos, v);
      const bool match = ok && (shift_hi >= 32 || (v >> shift_hi) == pre);
      hist_add(hist, (v >> shift) & dmask, match);
    }
    __syncthreads();
    scan_hist<kThreads>(hist);  // inclusive
    for (int c = threadIdx.x; c < (1 << bits); c += kThreads) {
      const int64_t excl = c > 0 ? hist[c - 1] : 0;
      if (excl <= rank && rank < hist[c]) {
        pre_s = (pre << bits) | (uint32_t)c;
        rank_s = rank - excl;
      }
    }
    __syncthreads();
    pre = pre_s;
    rank = rank_s;
    __syncthreads();
  }
  *rank_out = rank;
  return pre;
}

struct MoveArgs {
  int32_t *evict;
  int32_t *evicted_kvs;
  int32_t *freed;       // nullable [T][max_blocks]
  int32_t *moves;       // [cap][2]
  int64_t *move_off;
  int32_t *move_counts;
  int64_t *totals;
  int32_t *src_pos;     // nullable [T][max_slots]: pre-renumbering logical of each kept position
  int64_t src_stride;
  int publish;          // k_compact16 publishes each head's move list for k_copy_published
  int64_t n_heads;      // T
};

// Named barrier over `count` threads (a warp-aligned group of the CTA).
// (ids 1 and 2 only, as immediates, so ptxas reserves three barriers)
__device__ __forceinline__ void group_sync(int id, int count) {
  if (id == 1) asm volatile("bar.sync 1, %0;" ::"r"(count) : "memory");
  else asm volatile("bar.sync 2, %0;" ::"r"(count) : "memory");
}

// Exclusive scan over a warp-aligned group of GT threads (gtid = rank in the
// group); wsum = 32 ints of shared memory owned by the group.
__device__ __forceinline__ int32_t group_excl_scan(int32_t v, int gtid, int GT, int bar, int32_t *wsum,
                                                   int32_t &total) {
  const int lane = gtid & 31, w = gtid >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  group_sync(bar, GT);
  int32_t pre = 0, tot = 0;
  for (int i = 0; i < GT / 32; ++i) {
    const int32_t t = wsum[i];
    pre += i < w ? t : 0;
    tot += t;
  }
  group_sync(bar, GT);
  total = tot;
  return pre + x - v;
}

// k_compact16 (whole CTA): head h's move list (nm moves) is complete; append
// its 32-move chunks to the copy queue (the list is released before the
// chunk entries, the entries before the head counts as published).
template <int NT>
__device__ void publish_moves(const EvictState &S, int64_t h, int nm) {
  __shared__ int base_s;
  const int nch = (nm + 31) / 32;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(S.kv_ready + h), "r"(nm + 1) : "memory");
    base_s = nch ? atomicAdd(S.chunk_tail, nch) : 0;
  }
  __syncthreads();
  __threadfence();
  for (int c = threadIdx.x; c < nch; c += NT) {
    const unsigned long long v = ((unsigned long long)(h + 1) << 32) | (unsigned)c;
    if (base_s + c < S.max_chunks)  // (sized from moves_capacity: a short buffer is a caller error)
      asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(S.chunks + base_s + c), "l"(v) : "memory");
    else
      set_status(S.status, KVC_DEV_CAPACITY, (int32_t)h, base_s + c);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(S.pub_count) : "memory");
  }
}

__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long *a) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}

// K/V rows of every move of the round, running beside k_compact16 (launched
// programmatically: its CTAs take the SMs compact16's CTAs leave).  A warp
// claims queue chunks one at a time (32 moves, one (src, dst) per lane).  All
// compact16 CTAs are resident by the time this grid launches (they trigger
// first) and every one of them publishes (0 moves when it evicts nothing), so
// waiting for a chunk entry cannot deadlock; a bounded wait still turns a
// missing publication into a status error instead of a hang.  The final
// griddepcontrol.wait makes this grid's completion imply compact16's.
// Lane 0: the queue entry `id` once it is written (0 when the queue is
// exhausted, or after a 2 s wait: a head never published).
__device__ __forceinline__ unsigned long long wait_chunk(const EvictState &S, const kvc_pool &p, int id, int T,
                                                         unsigned long long t0) {
  if (id >= S.max_chunks) return 0;  // beyond the queue (publish flagged any overflow)
  for (int spin = 0;; ++spin) {
    const unsigned long long d = ld_acquire64(S.chunks + id);
    if (d) return d;
    if (ld_acquire(S.pub_count) == T && id >= __ldcg(S.chunk_tail)) return 0;  // all published, no more work
    if ((spin & 63) == 63) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      if (t - t0 > 2000000000ull) {
        set_status(p.status, KVC_DEV_SCHEDULE_CORRUPTION, -1, id);
        return 0;
      }
    }
    __nanosleep(128);
  }
}

// A chunk's moves: lane j holds move j's (src, dst); returns the move count.
__device__ __forceinline__ int chunk_pairs(const EvictState &S, const MoveArgs &M, unsigned long long d, int lane,
                                           int2 &sd) {
  const int64_t h = (int64_t)(d >> 32) - 1;
  const int k0 = (int)(d & 0xffffffffu) * 32;
  const int nm = __ldcg(S.kv_ready + h) - 1;  // released before the chunk entry
  const int cnt = nm - k0 < 32 ? nm - k0 : 32;
  sd = make_int2(0, 0);
  if (lane < cnt) sd = __ldcg(reinterpret_cast<const int2 *>(M.moves) + __ldcg(M.move_off + h) + k0 + lane);
  return cnt;
}

// K/V rows of every move of the round, running beside k_compact16 (launched
// programmatically: its CTAs take the SMs compact16's CTAs leave).  A warp
// claims queue chunks (32 moves, one (src, dst) per lane); the next chunk is
// claimed when the current one starts and its pairs are fetched halfway
// through it, so queue latency hides under the copy.  All compact16 CTAs are
// resident by the time this grid launches (they trigger first) and every one
// of them publishes (0 moves when it evicts nothing), so waiting for a chunk
// entry cannot deadlock; a bounded wait still turns a missing publication
// into a status error instead of a hang.  The final griddepcontrol.wait makes
// this grid's completion imply compact16's.
template <int U>
__global__ void __launch_bounds__(256) k_copy_published(kvc_pool p, EvictState S, MoveArgs M) {
  const int lane = threadIdx.x & 31;
  const int T = (int)M.n_heads;
  const int vec = p.head_dim / 8, cm = 2 * vec;  // 16-byte units per move (K row, then V row)
  uint4 *kc = reinterpret_cast<uint4 *>(p.k_cache);
  uint4 *vc = reinterpret_cast<uint4 *>(p.v_cache);
  unsigned long long t0 = 0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  unsigned long long d = 0;
  if (lane == 0) d = wait_chunk(S, p, atomicAdd(S.claim_next, 1), T, t0);
  d = __shfl_sync(0xffffffffu, d, 0);
  int2 sd;
  int cnt = d ? chunk_pairs(S, M, d, lane, sd) : 0;
  while (d) {
    int id_next = 0;
    if (lane == 0) id_next = atomicAdd(S.claim_next, 1);
    unsigned long long d_next = 0;
    int2 sd_next = make_int2(0, 0);
    int cnt_next = 0;
    const int units = cnt * cm;
    const int half = (units / (32 * U) / 2) * 32 * U;  // the round after which the next chunk is fetched
    for (int b = 0; b < units; b += 32 * U) {
      uint4 val[U];
      uint4 *dst[U];
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const int u = b + i * 32 + lane;
        const int j = u / cm;
        const int src = __shfl_sync(0xffffffffu, sd.x, j & 31);
        const int dd = __shfl_sync(0xffffffffu, sd.y, j & 31);
        dst[i] = nullptr;
        if (u < units) {
          int c = u - j * cm;
          uint4 *base = c >= vec ? vc : kc;
          c -= c >= vec ? vec : 0;
          val[i] = __ldg(base + (int64_t)src * vec + c);  // read-only path: no K/V is written meanwhile
          dst[i] = base + (int64_t)dd * vec + c;
        }
      }
      if (b == half) {  // the next chunk's entry and pairs, while these loads are in flight
        if (lane == 0) d_next = wait_chunk(S, p, id_next, T, t0);
        d_next = __shfl_sync(0xffffffffu, d_next, 0);
        if (d_next) cnt_next = chunk_pairs(S, M, d_next, lane, sd_next);
      }
#pragma unroll
      for (int i = 0; i < U; ++i)
        if (dst[i]) *dst[i] = val[i];
    }
    d = d_next;
    sd = sd_next;
    cnt = cnt_next;
  }
  grid_dep_wait();
}

// (9) per head with e > 0: mask, MoveCache pairing, copies, free, renumber.
__global__ void __launch_bounds__(kThreads) k_compact(kvc_pool p, const int32_t *rows, EvictState S,
                                                     MoveArgs M) {
  grid_dep_wait();
  grid_dep_trigger();
  extern __shared__ uint32_t bitmap[];  // max_slots bits
  __shared__ int32_t hist[kBins];
  __shared__ int32_t cnt_s[4];
  using Scan = cub::BlockScan<int32_t, kThreads>;
  __shared__ typename Scan::TempStorage stmp;
  const int g = blockIdx.x;
  const int si = g / S.hp, hi = g % S.hp;
  const int e = M.evict[g];
  if (threadIdx.x == 0 && M.move_counts) M.move_counts[g] = 0;
  if (threadIdx.x == 0 && M.evicted_kvs) M.evicted_kvs[g] = 0;
  if (e <= 0) return;
  const int64_t hidx = (int64_t)rows[si] * S.hp + hi;
  const int b = p.block_size;
  const int D = p.head_dim;
  const int nb = p.nblocks[hidx];
  const int C = p.ctx[hidx];
  const int64_t n = (int64_t)nb * b;
  int32_t *tab = head_table(p, hidx);
  const uint32_t *keys = S.keys + (int64_t)g * S.max_slots;
  auto flat = [&](int64_t pos) { return (int64_t)tab[pos / b] * b + pos % b; };

  // threshold T_h = (b*e)-th smallest key, then the tie cut S_h
  int64_t tie_rank;
  const int64_t target = (int64_t)b * e - 1;
  const uint32_t T = cta_select(hist, n, target, [&](int64_t pos, uint32_t &v) { v = keys[pos]; return true; },
                                &tie_rank);
  auto sec = [&](int64_t pos) -> uint32_t {
    const bool occ = pos < C;
    return occ ? (0x80000000u | (uint32_t)(p.logical[flat(pos)] + 1)) : (uint32_t)pos;
  };
  int64_t dummy;
  const uint32_t Sx = cta_select(hist, n, tie_rank, [&](int64_t pos, uint32_t &v) {
    if (keys[pos] != T) return false;
    v = sec(pos);
    return true;
  }, &dummy);
  auto masked = [&](int64_t pos) {
    const uint32_t k = keys[pos];
    return k < T || (k == T && sec(pos) <= Sx);
  };

  // pairing: holes below R0 ascending -> dst; survivors in [R0, n) descending -> src
  const int64_t R0 = n - (int64_t)e * b;
  const int64_t off = M.move_off[g];
  int32_t *mv = M.moves + off * 2;
  if (threadIdx.x == 0) { cnt_s[0] = 0; cnt_s[1] = 0; cnt_s[2] = 0; }
  __syncthreads();
  int32_t evk = 0;
  {
    int32_t carry = 0;
    for (int64_t base = 0; base < R0; base += kThreads) {
      const int64_t pos = base + threadIdx.x;
      int32_t hole = 0;
      if (pos < R0) {
        const bool m = masked(pos);
        evk += (m && pos < C) ? 1 : 0;
        hole = (m || p.logical[flat(pos)] < 0) ? 1 : 0;
      }
      int32_t excl, tot;
      Scan(stmp).ExclusiveSum(hole, excl, tot);
      if (hole) {
        const int64_t k = carry + excl;
        if (k < (int64_t)e * b) mv[2 * k + 1] = (int32_t)flat(pos);
      }
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) cnt_s[0] = carry;  // holes available
  }
  {
    int32_t carry = 0;
    for (int64_t base = 0; base < n - R0; base += kThreads) {
      const int64_t pos = n - 1 - (base + threadIdx.x);  // descending
      int32_t surv = 0;
      if (pos >= R0) {
        const bool m = masked(pos);
        evk += (m && pos < C) ? 1 : 0;
        surv = (!m && p.logical[flat(pos)] >= 0) ? 1 : 0;
      }
      int32_t excl, tot;
      Scan(stmp).ExclusiveSum(surv, excl, tot);
      if (surv) mv[2 * (carry + excl)] = (int32_t)flat(pos);
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) cnt_s[1] = carry;  // survivors to move
  }
  atomicAdd(&cnt_s[2], evk);
  __syncthreads();
  const int32_t nmoves = cnt_s[1];
  if (nmoves > cnt_s[0]) {
    if (threadIdx.x == 0) set_status(p.status, KVC_DEV_SCHEDULE_CORRUPTION, (int32_t)hidx, nmoves);
    return;
  }
  // the metric/logical/flag moves happen here (renumbering below needs them);
  // the K/V rows move in k_copy_kv, a bandwidth kernel over all move lists
  for (int k = threadIdx.x; k < nmoves; k += kThreads) {
    const int64_t src = mv[2 * k], dst = mv[2 * k + 1];
    p.metric[dst] = p.metric[src];
    p.logical[dst] = p.logical[src];
    p.protected_[dst] = p.protected_[src];
    p.fresh[dst] = p.fresh[src];
  }
  (void)D;
  __syncthreads();
  // free the trailing e blocks, reset their slots
  for (int64_t i = threadIdx.x; i < (int64_t)e * b; i += kThreads) {
    const int j = nb - e + (int)(i / b);
    const int32_t blk = tab[j];
    const int64_t f = (int64_t)blk * b + i % b;
    p.metric[f] = 0.f;
    p.logical[f] = -1;
    p.protected_[f] = 0;
    p.fresh[f] = 0;
    if (i % b == 0) {
      p.free_flag[blk] = 1;
      atomicAdd(&p.free_tile[blk / KVC_FREE_TILE], 1);
      if (M.freed) M.freed[(int64_t)g * p.max_blocks + (j - (nb - e))] = blk;
    }
  }
  const int keep = nb - e;
  const int Cn = C < keep * b ? C : keep * b;
  // logical renumbering: rank among kept logicals (distinct, < n)
  const int words = (int)((n + 31) / 32);
  for (int w = threadIdx.x; w < words; w += kThreads) bitmap[w] = 0;
  __syncthreads();
  for (int64_t pos = threadIdx.x; pos < Cn; pos += kThreads) {
    const int32_t lg = p.logical[flat(pos)];
    if (lg < 0 || lg >= n) {
      set_status(p.status, KVC_DEV_CACHE_CORRUPTION, (int32_t)hidx, lg);
      continue;
    }
    const uint32_t bit = 1u << (lg & 31);
    if (atomicOr(&bitmap[lg >> 5], bit) & bit) set_status(p.status, KVC_DEV_CACHE_CORRUPTION, (int32_t)hidx, lg);
  }
  __syncthreads();
  // exclusive popcount prefix per word, stored in hist-sized chunks
  int32_t *wpre = reinterpret_cast<int32_t *>(bitmap) + words;  // second half of the smem window
  {
    int32_t carry = 0;
    for (int base = 0; base < words; base += kThreads) {
      const int w = base + threadIdx.x;
      const int32_t c = w < words ? __popc(bitmap[w]) : 0;
      int32_t excl, tot;
      Scan(stmp).ExclusiveSum(c, excl, tot);
      if (w < words) wpre[w] = carry + excl;
      carry += tot;
      __syncthreads();
    }
  }
  __syncthreads();
  for (int64_t pos = threadIdx.x; pos < Cn; pos += kThreads) {
    const int64_t f = flat(pos);
    const int32_t lg = p.logical[f];
    if (lg < 0 || lg >= n) continue;
    const uint32_t w = bitmap[lg >> 5] & ((1u << (lg & 31)) - 1u);
    p.logical[f] = wpre[lg >> 5] + __popc(w);
  }
  if (threadIdx.x == 0) {
    p.nblocks[hidx] = keep;
    p.ctx[hidx] = Cn;
    if (M.move_counts) M.move_counts[g] = nmoves;
    if (M.evicted_kvs) M.evicted_kvs[g] = cnt_s[2];
    if (M.totals) {
      atomicAdd((unsigned long long *)&M.totals[0], (unsigned long long)e);
      atomicAdd((unsigned long long *)&M.totals[1], (unsigned long long)cnt_s[2]);
      atomicAdd((unsigned long long *)&M.totals[2], (unsigned long long)nmoves);
    }
  }
}

// ---------------------------------------------------------------------------
// k_compact16: k_compact for block_size 16, 1024 threads, one thread per
// 16-slot block in every pass (uint4 key / int4 logical rows).
// ---------------------------------------------------------------------------


template <int NT>
__device__ void scan_hist16(int32_t *hist) {  // inclusive, NT threads
  using Scan = cub::BlockScan<int32_t, NT>;
  __shared__ typename Scan::TempStorage tmp;
  constexpr int per = kBins / NT;
  int32_t v[per];
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < per; ++i) {
    v[i] = hist[threadIdx.x * per + i];
    s += v[i];
  }
  int32_t excl;
  __syncthreads();
  Scan(tmp).ExclusiveSum(s, excl);
#pragma unroll
  for (int i = 0; i < per; ++i) {
    excl += v[i];
    hist[threadIdx.x * per + i] = excl;
  }
  __syncthreads();
}

// rank-th smallest value among the positions `get4` marks valid, 4 per call.
// Returns the value; *rank_out = its rank among equal values, *eq_out = how
// many valid positions hold it.
template <int NT, typename Get4>
__device__ uint32_t select16(int32_t *hist, int64_t n, int64_t rank, Get4 get4, int64_t *rank_out,
                             int64_t *eq_out, int lv0 = 0, uint32_t pre0 = 0) {
  __shared__ uint32_t pre_s;
  __shared__ int64_t rank_s, eq_s;
  const int shifts[3] = {21, 10, 0};
  const int bitsv[3] = {11, 11, 10};
  uint32_t pre = pre0;  // the digits above level lv0, when known
  int64_t eq = 0;
  for (int lv = lv0; lv < 3; ++lv) {
    const int shift = shifts[lv], bits = bitsv[lv];
    const int shift_hi = shift + bits;
    const uint32_t dmask = (1u << bits) - 1;
    for (int i = threadIdx.x; i < kBins; i += NT) hist[i] = 0;
    __syncthreads();
    for (int64_t qb = 0; qb * 4 < n; qb += NT) {  // warp-uniform trip count (hist_add votes)
      const int64_t q = qb + threadIdx.x;
      uint32_t v[4] = {0u, 0u, 0u, 0u};
      bool ok[4] = {false, false, false, false};
      if (q * 4 < n) get4(q * 4, v, ok);
      uint32_t bin[4];
      bool act[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        act[e] = ok[e] && (shift_hi >= 32 || (v[e] >> shift_hi) == pre);
        bin[e] = (v[e] >> shift) & dmask;
      }
      hist_add4(hist, bin, act);
    }
    __syncthreads();
    scan_hist16<NT>(hist);
    for (int c = threadIdx.x; c < (1 << bits); c += NT) {
      const int64_t excl = c > 0 ? hist[c - 1] : 0;
      if (excl <= rank && rank < hist[c]) {
        pre_s = (pre << bits) | (uint32_t)c;
        rank_s = rank - excl;
        eq_s = hist[c] - excl;
      }
    }
    __syncthreads();
    pre = pre_s;
    rank = rank_s;
    eq = eq_s;
    __syncthreads();
  }
  *rank_out = rank;
  *eq_out = eq;
  return pre;
}

template <int NT>
__device__ void compact16_head(kvc_pool &p, const int32_t *rows, EvictState &S, const MoveArgs &M, uint32_t *bitmap);

// Last CTA of the grid to arrive: free-block total over the tiles (after every
// CTA's free-tile atomics, acquired by the arrival).
template <int NT>
__device__ void free_total_last(const kvc_pool &p, int32_t *done, int64_t *totals) {
  __shared__ int last_s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int prev;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(done) : "memory");
    last_s = prev == (int)gridDim.x - 1;
    if (last_s) *done = 0;
  }
  __syncthreads();
  if (!last_s) return;
  using Red = cub::BlockReduce<int64_t, NT>;
  __shared__ typename Red::TempStorage tmp;
  int64_t s = 0;
  for (int t = threadIdx.x; t < num_tiles(&p); t += NT) s += __ldcg(p.free_tile + t);
  s = Red(tmp).Sum(s);
  if (threadIdx.x == 0) totals[3] = s;
}

template <int NT>
__global__ void __maxnreg__(KVC_C16_REGS) k_compact16(kvc_pool p, const int32_t *rows, EvictState S, MoveArgs M) {
  grid_dep_wait();
  grid_dep_trigger();
  extern __shared__ uint32_t bitmap[];  // [words] bitmap + [words] prefix
  compact16_head<NT>(p, rows, S, M, bitmap);
  if (M.totals) free_total_last<NT>(p, S.c16_done, M.totals);
}

template <int NT>
__device__ void compact16_head(kvc_pool &p, const int32_t *rows, EvictState &S, const MoveArgs &M, uint32_t *bitmap) {
  __shared__ int32_t hist[kBins];
  __shared__ int32_t cnt_s[4];
  using Scan = cub::BlockScan<int32_t, NT>;
  __shared__ typename Scan::TempStorage stmp;
  const int g = blockIdx.x;
  const int si = g / S.hp, hi = g % S.hp;
  const int e = M.evict[g];
  if (threadIdx.x == 0 && M.move_counts) M.move_counts[g] = 0;
  if (threadIdx.x == 0 && M.evicted_kvs) M.evicted_kvs[g] = 0;
  if (e <= 0) {
    if (M.publish) publish_moves<NT>(S, g, 0);
    return;
  }
  const int64_t hidx = (int64_t)rows[si] * S.hp + hi;
  const int nb = p.nblocks[hidx];
  const int C = p.ctx[hidx];
  const int64_t n = (int64_t)nb * 16;
  int32_t *tab = head_table(p, hidx);
  const uint32_t *keys = S.keys + (int64_t)g * S.max_slots;

  if (S.trace && threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); S.trace[g * 8 + 0] = t_; }
  // ---- threshold T_h = (16 e)-th smallest key; shortcut when it is T* ----
  const uint32_t Tstar = S.prefix[si];
  const int64_t lt = S.ltc[g], le = S.lec[g];
  const int64_t target = (int64_t)16 * e - 1;
  uint32_t T;
  int64_t tie_rank, tie_cnt;
  if (target >= lt) {
    T = Tstar;
    tie_rank = target - lt;
    tie_cnt = le - lt;
  } else {
    // The keys < T* that share T*'s top 22 (11) bits are exactly the largest
    // lt2 (lt1) keys below T*: when the target is among them the select
    // starts at level 3 (2) with that prefix (one or two passes fewer).
    const int64_t from_top = lt - 1 - target;
    int lv0 = 0;
    uint32_t pre0 = 0;
    int64_t rank0 = target;
    if (S.lt2[g] > from_top) {
      lv0 = 2; pre0 = Tstar >> 10; rank0 = S.lt2[g] - 1 - from_top;
    } else if (S.lt1[g] > from_top) {
      lv0 = 1; pre0 = Tstar >> 21; rank0 = S.lt1[g] - 1 - from_top;
    }
    if (S.cum3) {
      // Long heads: the histograms K3 kept give the threshold's digits down
      // to the first level that is not T*'s: level 1 from all keys' top-11
      // histogram, level 2 from that of T*'s 11-bit bucket, level 3 from that
      // of its 22-bit bucket (a bucket's keys below T* are its smallest, so
      // ranks inside it are ranks among the keys below T*).  One or two key
      // passes fewer, none when the threshold shares T*'s top 22 bits.
      const int32_t *rows3[3] = {S.cum1 + (int64_t)g * kBins, S.cum2 + (int64_t)g * kBins,
                                 S.cum3 + (int64_t)g * 1024};
      const int nbins[3] = {kBins, kBins, 1024};
      const int bitsv[3] = {11, 11, 10};
      __shared__ uint32_t d_s;
      __shared__ int64_t r_s, c_s;
      const int lv = lv0;
      const int32_t *row = rows3[lv];
      for (int d = threadIdx.x; d < nbins[lv]; d += NT) {
        const int32_t lo_c = d > 0 ? __ldcg(row + d - 1) : 0, hi_c = __ldcg(row + d);
        if (lo_c <= rank0 && rank0 < hi_c) {
          d_s = (uint32_t)d;
          r_s = rank0 - lo_c;
          c_s = hi_c - lo_c;
        }
      }
      __syncthreads();
      const uint32_t pre1 = (pre0 << bitsv[lv]) | d_s;
      const int64_t rank1 = r_s, cnt1 = c_s;
      __syncthreads();
      if (lv == 2) {
        T = pre1;
        tie_rank = rank1;
        tie_cnt = cnt1;
      } else {
        T = select16<NT>(hist, n, rank1, [&](int64_t pos, uint32_t *v, bool *ok) {
          const uint4 k4 = *reinterpret_cast<const uint4 *>(keys + pos);
          v[0] = k4.x; v[1] = k4.y; v[2] = k4.z; v[3] = k4.w;
#pragma unroll
          for (int i = 0; i < 4; ++i) ok[i] = pos + i < n && v[i] < Tstar;
        }, &tie_rank, &tie_cnt, lv + 1, pre1);
      }
    } else {
      T = select16<NT>(hist, n, rank0, [&](int64_t pos, uint32_t *v, bool *ok) {
        const uint4 k4 = *reinterpret_cast<const uint4 *>(keys + pos);
        v[0] = k4.x; v[1] = k4.y; v[2] = k4.z; v[3] = k4.w;
#pragma unroll
        for (int i = 0; i < 4; ++i) ok[i] = pos + i < n && v[i] < Tstar;
      }, &tie_rank, &tie_cnt, lv0, pre0);
    }
  }
  if (S.trace && threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); S.trace[g * 8 + 1] = t_; }
  // ---- tie cut: ties at T ordered by (occupied, logical, position) ----
  auto sec = [&](int64_t pos, int32_t lg) -> uint32_t {
    return pos < C ? (0x80000000u | (uint32_t)(lg + 1)) : (uint32_t)pos;
  };
  uint32_t Sx = 0xffffffffu;
  constexpr int kTieMax = 512;
  if (tie_rank + 1 < tie_cnt && tie_cnt <= kTieMax) {
    // few ties (the pooled metric repeats a local maximum over neighbouring
    // slots): one pass collects their secondary keys (distinct: logical
    // positions, or positions past C) into shared memory; the tie_rank-th
    // smallest is the value with exactly tie_rank smaller ones
    __shared__ uint32_t tie_s[kTieMax];
    __shared__ int tie_n;
    if (threadIdx.x == 0) tie_n = 0;
    __syncthreads();
    for (int64_t q = threadIdx.x; q * 4 < n; q += NT) {
      const int64_t pos = q * 4;  // rows padded to 4
      const uint4 k4 = *reinterpret_cast<const uint4 *>(keys + pos);
      const uint32_t kv[4] = {k4.x, k4.y, k4.z, k4.w};
      bool any = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) any |= pos + i < n && kv[i] == T;
      if (!any) continue;
      const int4 l4 = *reinterpret_cast<const int4 *>(p.logical + (int64_t)tab[pos / 16] * 16 + pos % 16);
      const int32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (pos + i < n && kv[i] == T) {
          const int k = atomicAdd(&tie_n, 1);
          if (k < kTieMax) tie_s[k] = sec(pos + i, lv[i]);
        }
      }
    }
    __syncthreads();
    const int nt = tie_n < kTieMax ? tie_n : kTieMax;
    __shared__ uint32_t sx_s;
    if (threadIdx.x == 0) sx_s = 0xffffffffu;
    __syncthreads();
    for (int i = threadIdx.x; i < nt; i += NT) {
      const uint32_t v = tie_s[i];
      int below = 0;
      for (int j = 0; j < nt; ++j) below += tie_s[j] < v ? 1 : 0;
      if (below == tie_rank) sx_s = v;
    }
    __syncthreads();
    Sx = sx_s;
    if (threadIdx.x == 0 && tie_n != tie_cnt) set_status(S.status, KVC_DEV_SCHEDULE_CORRUPTION, (int32_t)hidx, tie_n);
  } else if (tie_rank + 1 < tie_cnt) {
    int64_t dummy, dummy2;
    Sx = select16<NT>(hist, n, tie_rank, [&](int64_t pos, uint32_t *v, bool *ok) {
      const uint4 k4 = *reinterpret_cast<const uint4 *>(keys + pos);  // pos % 4 == 0, rows padded to 4
      const uint32_t kv[4] = {k4.x, k4.y, k4.z, k4.w};
      bool any = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ok[i] = pos + i < n && kv[i] == T;
        any |= ok[i];
      }
      int4 l4 = make_int4(0, 0, 0, 0);
      if (any) l4 = *reinterpret_cast<const int4 *>(p.logical + (int64_t)tab[pos / 16] * 16 + pos % 16);
      const int32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = ok[i] ? sec(pos + i, lv[i]) : 0u;
    }, &dummy, &dummy2);
  }

  if (S.trace && threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); S.trace[g * 8 + 2] = t_; }
  // ---- MoveCache pairing (holes ascending below R0, survivors descending) ----
  const int rb = nb - e;  // first block of the eviction range
  int32_t *mv = M.moves + M.move_off[g] * 2;
  const int64_t cap_mv = (int64_t)16 * e;
  if (threadIdx.x == 0) { cnt_s[0] = 0; cnt_s[1] = 0; cnt_s[2] = 0; }
  __syncthreads();
  int32_t evk = 0;
  auto block_flags_at = [&](int bl, int32_t blk, uint32_t &masked_bits, uint32_t &live_bits) {
    const int64_t f0 = (int64_t)blk * 16;
    const uint4 *kp = reinterpret_cast<const uint4 *>(keys + (int64_t)bl * 16);
    const int4 *lp = reinterpret_cast<const int4 *>(p.logical + f0);
    masked_bits = 0;
    live_bits = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 k4 = kp[q];
      const int4 l4 = lp[q];
      const uint32_t kv[4] = {k4.x, k4.y, k4.z, k4.w};
      const int32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int o = q * 4 + i;
        const int64_t pos = (int64_t)bl * 16 + o;
        const bool m = kv[i] < T || (kv[i] == T && (Sx == 0xffffffffu || sec(pos, lv[i]) <= Sx));
        masked_bits |= (m ? 1u : 0u) << o;
        live_bits |= (lv[i] >= 0 ? 1u : 0u) << o;
      }
    }
  };
  auto block_flags = [&](int bl, uint32_t &masked_bits, uint32_t &live_bits) {
    block_flags_at(bl, tab[bl], masked_bits, live_bits);
  };
  {
    int32_t carry = 0;
    for (int base = 0; base < rb; base += NT) {
      const int bl = base + threadIdx.x;
      uint32_t holes = 0;
      int64_t f0 = 0;
      if (bl < rb) {
        uint32_t mb, lb;
        block_flags(bl, mb, lb);
        holes = mb | ~lb;
        holes &= 0xffffu;
        const int occ_n = C - bl * 16;
        const uint32_t occ_bits = occ_n >= 16 ? 0xffffu : occ_n <= 0 ? 0u : ((1u << occ_n) - 1u);
        evk += __popc(mb & occ_bits);
        f0 = (int64_t)tab[bl] * 16;
      }
      int32_t excl, tot;
      Scan(stmp).ExclusiveSum(__popc(holes), excl, tot);
      int64_t k = carry + excl;
      for (uint32_t hb = holes; hb; hb &= hb - 1) {
        const int o = __ffs(hb) - 1;
        if (k < cap_mv) mv[2 * k + 1] = (int32_t)(f0 + o);
        ++k;
      }
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) cnt_s[0] = carry;
  }
  {
    // (the table entry of a thread's next block is loaded a round ahead)
    int32_t carry = 0;
    int32_t nxt = threadIdx.x < e ? tab[nb - 1 - threadIdx.x] : 0;
    for (int base = 0; base < e; base += NT) {
      const int t = base + threadIdx.x;
      const int bl = nb - 1 - t;  // descending blocks
      const int32_t blk = nxt;
      nxt = t + NT < e ? tab[nb - 1 - (t + NT)] : 0;
      uint32_t surv = 0;
      int64_t f0 = 0;
      if (t < e) {
        uint32_t mb, lb;
        block_flags_at(bl, blk, mb, lb);
        surv = ~mb & lb & 0xffffu;
        const int occ_n = C - bl * 16;
        const uint32_t occ_bits = occ_n >= 16 ? 0xffffu : occ_n <= 0 ? 0u : ((1u << occ_n) - 1u);
        evk += __popc(mb & occ_bits);
        f0 = (int64_t)blk * 16;
      }
      int32_t excl, tot;
      Scan(stmp).ExclusiveSum(__popc(surv), excl, tot);
      int64_t k = carry + excl;
      for (int o = 15; o >= 0; --o) {  // descending positions within the block
        if (surv >> o & 1u) {
          mv[2 * k] = (int32_t)(f0 + o);
          ++k;
        }
      }
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) cnt_s[1] = carry;
  }
  atomicAdd(&cnt_s[2], evk);
  __syncthreads();
  const int32_t nmoves = cnt_s[1];
  if (nmoves > cnt_s[0]) {
    if (threadIdx.x == 0) set_status(p.status, KVC_DEV_SCHEDULE_CORRUPTION, (int32_t)hidx, nmoves);
    if (M.publish) publish_moves<NT>(S, g, 0);
    return;
  }
  if (S.trace && threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); S.trace[g * 8 + 3] = t_; }
  // the move list is complete: the concurrent copy kernel can take it
  if (M.publish) publish_moves<NT>(S, g, nmoves);
  constexpr int GT = NT;
  const int gtid = threadIdx.x;
  constexpr int bar = 1;
  __shared__ int32_t wsum_s[32];
  const int keep = rb;
  const int Cn = C < keep * 16 ? C : keep * 16;
  {
    constexpr int MU = 8;  // moves' loads in flight per thread
    const int2 *mv2 = reinterpret_cast<const int2 *>(mv);
    for (int k0 = gtid; k0 < nmoves; k0 += MU * GT) {
      int2 sd[MU];
      float mt[MU];
      int32_t lg[MU];
      uint8_t pr[MU], fr[MU];
#pragma unroll
      for (int u = 0; u < MU; ++u) {
        const int k = k0 + u * GT;
        sd[u] = k < nmoves ? mv2[k] : make_int2(-1, -1);
      }
#pragma unroll
      for (int u = 0; u < MU; ++u)
        if (sd[u].x >= 0) {
          mt[u] = p.metric[sd[u].x];
          lg[u] = p.logical[sd[u].x];
          pr[u] = p.protected_[sd[u].x];
          fr[u] = p.fresh[sd[u].x];
        }
#pragma unroll
      for (int u = 0; u < MU; ++u)
        if (sd[u].x >= 0) {
          p.metric[sd[u].y] = mt[u];
          p.logical[sd[u].y] = lg[u];
          p.protected_[sd[u].y] = pr[u];
          p.fresh[sd[u].y] = fr[u];
        }
    }
    group_sync(bar, GT);
    if (S.trace && threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); S.trace[g * 8 + 4] = t_; }
    // ---- free the trailing e blocks and reset their slots ----
    // four table entries per thread in flight; free-tile counts with one
    // atomic per (warp, tile) (a head's blocks sit in a few tiles, so
    // per-block atomics would serialise)
    for (int base = 0; base < e; base += 4 * GT) {
      int32_t blk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = base + u * GT + gtid;
        blk[u] = t < e ? tab[rb + t] : -1;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = base + u * GT + gtid;
        const bool act = blk[u] >= 0;
        const unsigned am = __ballot_sync(0xffffffffu, act);
        if (!act) continue;
        const int64_t f0 = (int64_t)blk[u] * 16;
        float4 *mp = reinterpret_cast<float4 *>(p.metric + f0);
        int4 *lp = reinterpret_cast<int4 *>(p.logical + f0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          mp[q] = make_float4(0.f, 0.f, 0.f, 0.f);
          lp[q] = make_int4(-1, -1, -1, -1);
        }
        *reinterpret_cast<uint4 *>(p.protected_ + f0) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4 *>(p.fresh + f0) = make_uint4(0, 0, 0, 0);
        p.free_flag[blk[u]] = 1;
        if (M.freed) M.freed[(int64_t)g * p.max_blocks + t] = blk[u];
        const int tile = blk[u] / KVC_FREE_TILE;
        const unsigned peers = __match_any_sync(am, tile);
        if ((gtid & 31) == __ffs(peers) - 1) atomicAdd(&p.free_tile[tile], __popc(peers));
      }
    }
    if (S.trace && threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); S.trace[g * 8 + 5] = t_; }
    // ---- logical renumbering: rank among the kept logicals ----
    const int words = (int)((n + 31) / 32);
    uint32_t *wpre = bitmap + words;
    for (int w = gtid; w < words; w += GT) bitmap[w] = 0;
    group_sync(bar, GT);
    const int kb = (Cn + 15) / 16;
    for (int bl = gtid; bl < kb; bl += GT) {
      const int4 *lp = reinterpret_cast<const int4 *>(p.logical + (int64_t)tab[bl] * 16);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int4 l4 = lp[q];
        const int32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int pos = bl * 16 + q * 4 + i;
          if (pos >= Cn) continue;
          const int32_t lg = lv[i];
          if (lg < 0 || lg >= n) {
            set_status(p.status, KVC_DEV_CACHE_CORRUPTION, (int32_t)hidx, lg);
            continue;
          }
          const uint32_t bit = 1u << (lg & 31);
          if (atomicOr(&bitmap[lg >> 5], bit) & bit) set_status(p.status, KVC_DEV_CACHE_CORRUPTION, (int32_t)hidx, lg);
        }
      }
    }
    group_sync(bar, GT);
    {
      int32_t carry = 0;
      for (int base = 0; base < words; base += GT) {
        const int w = base + gtid;
        const int32_t c = w < words ? __popc(bitmap[w]) : 0;
        int32_t tot;
        const int32_t excl = group_excl_scan(c, gtid, GT, bar, wsum_s, tot);
        if (w < words) wpre[w] = carry + excl;
        carry += tot;
      }
    }
    group_sync(bar, GT);
    for (int bl = gtid; bl < kb; bl += GT) {
      int4 *lp = reinterpret_cast<int4 *>(p.logical + (int64_t)tab[bl] * 16);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int4 l4 = lp[q];
        int32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int pos = bl * 16 + q * 4 + i;
          const int32_t lg = lv[i];
          if (M.src_pos && pos < Cn) M.src_pos[g * M.src_stride + pos] = (lg < 0 || lg >= n) ? -1 : lg;
          if (pos >= Cn || lg < 0 || lg >= n) continue;
          lv[i] = (int32_t)wpre[lg >> 5] + __popc(bitmap[lg >> 5] & ((1u << (lg & 31)) - 1u));
        }
        lp[q] = make_int4(lv[0], lv[1], lv[2], lv[3]);
      }
    }
    if (S.trace && threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); S.trace[g * 8 + 6] = t_; }
  }
  __syncthreads();
  if (S.trace && threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); S.trace[g * 8 + 7] = t_; }
  if (threadIdx.x == 0) {
    p.nblocks[hidx] = keep;
    p.ctx[hidx] = Cn;
    if (M.move_counts) M.move_counts[g] = nmoves;
    if (M.evicted_kvs) M.evicted_kvs[g] = cnt_s[2];
    if (M.totals) {
      atomicAdd((unsigned long long *)&M.totals[0], (unsigned long long)e);
      atomicAdd((unsigned long long *)&M.totals[1], (unsigned long long)cnt_s[2]);
      atomicAdd((unsigned long long *)&M.totals[2], (unsigned long long)nmoves);
    }
  }
}

// ---------------------------------------------------------------------------
// k_compact_warp: one warp per head for heads of at most 8192 slots (the
// decode-time batch: thousands of short heads, a few evicted blocks each).
// No CTA barriers; one head per (one-warp) CTA, 4 KB of shared memory.
//  * T_h and the tie cut come from the candidates (keys < T*, or the ties at
//    T*) sorted by (key, secondary) in shared memory when there are at most
//    kCand of them, else from a warp radix select over the head's keys.
//  * holes / survivors / pairs / free / renumber as k_compact16, each pass
//    one 16-slot block per lane with warp scans.
// ---------------------------------------------------------------------------
#ifndef KVC_CW_WARPS
#define KVC_CW_WARPS 1
#endif
// warps (heads) per CTA.  One: a CTA retires with its head, so a short or
// non-evicting head frees its slot at once (8 heads per CTA held each CTA
// until its slowest head: 33% achieved occupancy; decode round -2%)
constexpr int kWC = KVC_CW_WARPS;

struct WarpArea {
  unsigned long long cand[kCand];  // composites (key << 32 | secondary); or a 256-bin histogram
  uint32_t bitmap[256];            // kept-logical bitmap (n <= 8192)
  int32_t wpre[256];               // its word prefix counts
};

__device__ __forceinline__ int warp_excl_scan(int v, int lane, int &total) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

// rank-th smallest (0-based) of getv over positions [0, n); 8-bit digits.
template <typename GetV>
__device__ uint32_t warp_select(int32_t *hist, int n, int64_t rank, GetV getv, int lane, int64_t *rank_out,
                                int64_t *eq_out) {
  uint32_t pre = 0;
  int64_t eq = 0;
  for (int lv = 0; lv < 4; ++lv) {
    const int shift = 24 - 8 * lv;
    for (int i = lane; i < 256; i += 32) hist[i] = 0;
    __syncwarp();
    for (int pos = lane; pos < n; pos += 32) {
      uint32_t v;
      if (getv(pos, v) && (lv == 0 || (v >> (shift + 8)) == pre)) atomicAdd(&hist[(v >> shift) & 255], 1);
    }
    __syncwarp();
    int h[8], sum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      h[i] = hist[lane * 8 + i];
      sum += h[i];
    }
    int tot;
    int64_t run = warp_excl_scan(sum, lane, tot);
    int found = -1;
    int64_t frank = 0, feq = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (found < 0 && run <= rank && rank < run + h[i]) {
        found = lane * 8 + i;
        frank = rank - run;
        feq = h[i];
      }
      run += h[i];
    }
    const unsigned fm = __ballot_sync(0xffffffffu, found >= 0);
    const int src = fm ? __ffs(fm) - 1 : 0;
    found = __shfl_sync(0xffffffffu, found, src);
    frank = __shfl_sync(0xffffffffu, frank, src);
    feq = __shfl_sync(0xffffffffu, feq, src);
    pre = (pre << 8) | (uint32_t)(found < 0 ? 0 : found);
    rank = frank;
    eq = feq;
    __syncwarp();
  }
  *rank_out = rank;
  *eq_out = eq;
  return pre;
}

// Bitonic sort of cnt (<= kCand) composites ascending, padded with ~0.
__device__ void warp_sort(unsigned long long *a, int cnt, int lane) {
  int m = 32;
  while (m < cnt) m <<= 1;
  for (int i = cnt + lane; i < m; i += 32) a[i] = ~0ull;
  __syncwarp();
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < m; i += 32) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long x = a[i], y = a[l];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            a[i] = y;
            a[l] = x;
          }
        }
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kWC * 32, 32 / kWC) k_compact_warp(kvc_pool p, const int32_t *rows, EvictState S,
                                                          MoveArgs M, int64_t T_heads) {
  grid_dep_wait();
  grid_dep_trigger();
  __shared__ WarpArea area[kWC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * kWC + warp;
  if (g >= T_heads) return;
  WarpArea &A = area[warp];
  const int si = (int)(g / S.hp), hi = (int)(g % S.hp);
  const int e = M.evict[g];
  if (lane == 0 && M.move_counts) M.move_counts[g] = 0;
  if (lane == 0 && M.evicted_kvs) M.evicted_kvs[g] = 0;
  if (e <= 0) return;
  const int64_t hidx = (int64_t)rows[si] * S.hp + hi;
  const int nb = p.nblocks[hidx];
  const int C = p.ctx[hidx];
  const int n = nb * 16;
  const int32_t *tab = head_table(p, hidx);
  const uint32_t *keys = S.keys + g * S.max_slots;
  auto sec = [&](int pos, int32_t lg) -> uint32_t {
    return pos < C ? (0x80000000u | (uint32_t)(lg + 1)) : (uint32_t)pos;
  };
  auto lg_at = [&](int pos) -> int32_t { return p.logical[(int64_t)tab[pos >> 4] * 16 + (pos & 15)]; };
  // candidate list l (0: keys < T*, 1: ties at T*) written by k_bounds -> smem
  auto load_cand = [&](int l, int cnt) {
    const unsigned long long *src = S.cand + g * 2 * kCand + l * kCand;
    for (int i = lane; i < cnt; i += 32) A.cand[i] = src[i];
    __syncwarp();
  };
  // ---- threshold T_h and tie cut Sx: masked iff (key, sec) <= (T, Sx) ----
  const uint32_t Tstar = S.prefix[si];
  const int64_t lt = S.ltc[g], le = S.lec[g];
  const int64_t target = (int64_t)16 * e - 1;
  uint32_t T, Sx = 0xffffffffu;
  int32_t *hist = reinterpret_cast<int32_t *>(A.cand);
  if (target >= lt) {
    T = Tstar;
    const int64_t tie_rank = target - lt, tie_cnt = le - lt;
    if (tie_rank + 1 < tie_cnt) {
      if (tie_cnt <= kCand) {
        const int cnt = (int)tie_cnt;
        load_cand(1, cnt);
        warp_sort(A.cand, cnt, lane);
        Sx = (uint32_t)(A.cand[tie_rank] & 0xffffffffu);
      } else {
        int64_t d0, d1;
        Sx = warp_select(hist, n, tie_rank, [&](int pos, uint32_t &v) {
          if (keys[pos] != Tstar) return false;
          v = sec(pos, lg_at(pos));
          return true;
        }, lane, &d0, &d1);
      }
    }
  } else if (lt <= kCand) {
    const int cnt = (int)lt;
    load_cand(0, cnt);
    warp_sort(A.cand, cnt, lane);
    const unsigned long long c = A.cand[target];
    T = (uint32_t)(c >> 32);
    Sx = (uint32_t)(c & 0xffffffffu);
  } else {
    int64_t tie_rank, tie_cnt;
    T = warp_select(hist, n, target, [&](int pos, uint32_t &v) { v = keys[pos]; return v < Tstar; }, lane,
                    &tie_rank, &tie_cnt);
    if (tie_rank + 1 < tie_cnt) {
      int64_t d0, d1;
      Sx = warp_select(hist, n, tie_rank, [&](int pos, uint32_t &v) {
        if (keys[pos] != T) return false;
        v = sec(pos, lg_at(pos));
        return true;
      }, lane, &d0, &d1);
    }
  }
  __syncwarp();
  // kept-logical bitmap built while the passes read the logicals: the kept
  // set is the logicals of unmasked live slots whenever every hole is filled
  // (the normal case); otherwise it is rebuilt after the moves below
  const int words = (n + 31) / 32;
  for (int w = lane; w < words; w += 32) A.bitmap[w] = 0;
  __syncwarp();
  bool bad = false;
  auto block_flags = [&](int bl, int64_t f0, uint32_t &mb, uint32_t &lb) {
    const uint4 *kp = reinterpret_cast<const uint4 *>(keys + bl * 16);
    const int4 *lp = reinterpret_cast<const int4 *>(p.logical + f0);
    mb = 0;
    lb = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 k4 = kp[q];
      const int4 l4 = lp[q];
      const uint32_t kv[4] = {k4.x, k4.y, k4.z, k4.w};
      const int32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int o = q * 4 + i;
        const bool m = kv[i] < T || (kv[i] == T && sec(bl * 16 + o, lv[i]) <= Sx);
        mb |= (m ? 1u : 0u) << o;
        lb |= (lv[i] >= 0 ? 1u : 0u) << o;
        if (!m && lv[i] >= 0) {
          if (lv[i] >= n) {
            bad = true;
          } else {
            const uint32_t bit = 1u << (lv[i] & 31);
            if (atomicOr(&A.bitmap[lv[i] >> 5], bit) & bit) bad = true;
          }
        }
      }
    }
  };
  auto occ_bits = [&](int bl) -> uint32_t {
    const int occ_n = C - bl * 16;
    return occ_n >= 16 ? 0xffffu : occ_n <= 0 ? 0u : ((1u << occ_n) - 1u);
  };
  const int rb = nb - e;
  int32_t *mv = M.moves + M.move_off[g] * 2;
  const int64_t cap_mv = (int64_t)16 * e;
  int evk = 0;
  // ---- holes ascending below the range ----
  int nholes = 0;
  for (int base = 0; base < rb; base += 64) {  // blocks base+lane and base+32+lane: loads of both in flight
    uint32_t holes[2] = {0u, 0u};
    int64_t f0[2] = {0, 0};
    uint32_t mb[2], lb[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int bl = base + u * 32 + lane;
      if (bl < rb) f0[u] = (int64_t)tab[bl] * 16;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int bl = base + u * 32 + lane;
      if (bl < rb) {
        block_flags(bl, f0[u], mb[u], lb[u]);
        holes[u] = (mb[u] | ~lb[u]) & 0xffffu;
        evk += __popc(mb[u] & occ_bits(bl));
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int tot;
      int k = nholes + warp_excl_scan(__popc(holes[u]), lane, tot);
      for (uint32_t hb = holes[u]; hb; hb &= hb - 1) {
        if (k < cap_mv) mv[2 * k + 1] = (int32_t)(f0[u] + __ffs(hb) - 1);
        ++k;
      }
      nholes += tot;
    }
  }
  // ---- survivors descending inside the range ----
  int nmoves = 0;
  for (int base = 0; base < e; base += 32) {
    const int t = base + lane;
    const int bl = nb - 1 - t;
    uint32_t surv = 0;
    int64_t f0 = 0;
    if (t < e) {
      f0 = (int64_t)tab[bl] * 16;
      uint32_t mb, lb;
      block_flags(bl, f0, mb, lb);
      surv = ~mb & lb & 0xffffu;
      evk += __popc(mb & occ_bits(bl));
    }
    int tot;
    int k = nmoves + warp_excl_scan(__popc(surv), lane, tot);
    for (int o = 15; o >= 0; --o) {
      if (surv >> o & 1u) {
        if (k < cap_mv) mv[2 * k] = (int32_t)(f0 + o);
        ++k;
      }
    }
    nmoves += tot;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) evk += __shfl_xor_sync(0xffffffffu, evk, o);
  __syncwarp();
  if (nmoves > nholes) {
    if (lane == 0) set_status(p.status, KVC_DEV_SCHEDULE_CORRUPTION, (int32_t)hidx, nmoves);
    return;
  }
  // ---- pair metadata (holes below the range, survivors inside: disjoint) ----
  for (int k = lane; k < nmoves; k += 32) {
    const int64_t src = mv[2 * k], dst = mv[2 * k + 1];
    p.metric[dst] = p.metric[src];
    p.logical[dst] = p.logical[src];
    p.protected_[dst] = p.protected_[src];
    p.fresh[dst] = p.fresh[src];
  }
  __syncwarp();
  // ---- free the trailing e blocks and reset their slots ----
  for (int t = lane; t < e; t += 32) {
    const int32_t blk = tab[rb + t];
    const int64_t f0 = (int64_t)blk * 16;
    float4 *mp = reinterpret_cast<float4 *>(p.metric + f0);
    int4 *lp = reinterpret_cast<int4 *>(p.logical + f0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      mp[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      lp[q] = make_int4(-1, -1, -1, -1);
    }
    *reinterpret_cast<uint4 *>(p.protected_ + f0) = make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4 *>(p.fresh + f0) = make_uint4(0, 0, 0, 0);
    p.free_flag[blk] = 1;
    atomicAdd(&p.free_tile[blk / KVC_FREE_TILE], 1);
    if (M.freed) M.freed[g * p.max_blocks + t] = blk;
  }
  // ---- logical renumbering: rank among the kept logicals ----
  const int Cn = C < rb * 16 ? C : rb * 16;
  const int kb = (Cn + 15) / 16;
  const bool fast = nholes == nmoves;
  if (fast) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) set_status(p.status, KVC_DEV_CACHE_CORRUPTION, (int32_t)hidx, -1);
  } else {
  for (int w = lane; w < words; w += 32) A.bitmap[w] = 0;
  __syncwarp();
  for (int bl0 = lane; bl0 < kb; bl0 += 64) {
    int4 l4s[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int bl = bl0 + 32 * u;
      if (bl < kb) {
        const int4 *lp = reinterpret_cast<const int4 *>(p.logical + (int64_t)tab[bl] * 16);
#pragma unroll
        for (int q = 0; q < 4; ++q) l4s[u][q] = lp[q];
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
    const int bl = bl0 + 32 * u;
    if (bl >= kb) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int4 l4 = l4s[u][q];
      const int32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int pos = bl * 16 + q * 4 + i;
        if (pos >= Cn) continue;
        const int32_t lg = lv[i];
        if (lg < 0 || lg >= n) {
          set_status(p.status, KVC_DEV_CACHE_CORRUPTION, (int32_t)hidx, lg);
          continue;
        }
        const uint32_t bit = 1u << (lg & 31);
        if (atomicOr(&A.bitmap[lg >> 5], bit) & bit) set_status(p.status, KVC_DEV_CACHE_CORRUPTION, (int32_t)hidx, lg);
      }
    }
    }
  }
  }
  __syncwarp();
  {
    int c[8], sum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int w = lane * 8 + i;
      c[i] = w < words ? __popc(A.bitmap[w]) : 0;
      sum += c[i];
    }
    int tot;
    int run = warp_excl_scan(sum, lane, tot);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int w = lane * 8 + i;
      if (w < words) A.wpre[w] = run;
      run += c[i];
    }
  }
  __syncwarp();
  for (int bl0 = lane; bl0 < kb; bl0 += 64) {
    int4 l4s[2][4];
    int4 *lps[2] = {nullptr, nullptr};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int bl = bl0 + 32 * u;
      if (bl < kb) {
        lps[u] = reinterpret_cast<int4 *>(p.logical + (int64_t)tab[bl] * 16);
#pragma unroll
        for (int q = 0; q < 4; ++q) l4s[u][q] = lps[u][q];
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
    const int bl = bl0 + 32 * u;
    if (bl >= kb) continue;
    int4 *lp = lps[u];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int4 l4 = l4s[u][q];
      int32_t lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int pos = bl * 16 + q * 4 + i;
        const int32_t lg = lv[i];
        if (pos >= Cn) continue;
        if (M.src_pos) M.src_pos[g * M.src_stride + pos] = (lg < 0 || lg >= n) ? -1 : lg;
        if (lg < 0 || lg >= n) {
          if (fast) set_status(p.status, KVC_DEV_CACHE_CORRUPTION, (int32_t)hidx, lg);
          continue;
        }
        lv[i] = A.wpre[lg >> 5] + __popc(A.bitmap[lg >> 5] & ((1u << (lg & 31)) - 1u));
      }
      lp[q] = make_int4(lv[0], lv[1], lv[2], lv[3]);
    }
    }
  }
  if (lane == 0) {
    p.nblocks[hidx] = rb;
    p.ctx[hidx] = Cn;
    if (M.move_counts) M.move_counts[g] = nmoves;
    if (M.evicted_kvs) M.evicted_kvs[g] = evk;
    if (M.totals) {
      atomicAdd((unsigned long long *)&M.totals[0], (unsigned long long)e);
      atomicAdd((unsigned long long *)&M.totals[1], (unsigned long long)evk);
      atomicAdd((unsigned long long *)&M.totals[2], (unsigned long long)nmoves);
    }
  }
}

// K/V rows of every move of the round, as one flat persistent grid: warp
// tasks of 32 consecutive move-list entries (the lists are laid out by the
// exclusive offsets of e_h * b); each lane finds its entry's head by binary
// search over the offsets and keeps it if it is below that head's move count.
// The valid moves' rows are then copied in 16-byte chunks (2-byte elements
// for head_dim % 8 != 0), several chunks in flight per lane.  Sources are in
// blocks freed by k_compact; nothing can reuse them before this kernel
// completes (stream order).
template <typename Chunk>
__device__ __forceinline__ void copy_rows(Chunk *kc, Chunk *vc, const int64_t *src, const int64_t *dst, int nvalid,
                                          int per_row, int lane) {
  const int nch = 2 * per_row;  // K chunks then V chunks
  const int total = nvalid * nch;
  for (int i0 = 0; i0 < total; i0 += 32 * 4) {
    Chunk val[4];
    int64_t to[4];
    bool isv[4], ok[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = i0 + u * 32 + lane;
      ok[u] = idx < total;
      if (ok[u]) {
        const int m = idx / nch, c0 = idx % nch;
        isv[u] = c0 >= per_row;
        const int c = isv[u] ? c0 - per_row : c0;
        const Chunk *base = isv[u] ? vc : kc;
        val[u] = base[src[m] * per_row + c];
        to[u] = dst[m] * per_row + c;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (ok[u]) (isv[u] ? vc : kc)[to[u]] = val[u];
  }
}

__global__ void __launch_bounds__(256) k_copy_kv(kvc_pool p, const int32_t *moves, const int64_t *move_off,
                                                const int32_t *move_counts, int64_t T) {
  grid_dep_wait();
  grid_dep_trigger();
  __shared__ int64_t s_src[8][32], s_dst[8][32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t cap = move_off[T];
  const int64_t tasks = (cap + 31) / 32;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  const int D = p.head_dim;
  for (int64_t task = (int64_t)blockIdx.x * 8 + warp; task < tasks; task += nwarps) {
    const int64_t k = task * 32 + lane;
    bool valid = false;
    if (k < cap) {
      int64_t lo = 0, hi = T - 1;  // last g with move_off[g] <= k
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (__ldg(move_off + mid) <= k) lo = mid;
        else hi = mid - 1;
      }
      valid = k - move_off[lo] < move_counts[lo];
    }
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    if (valid) {
      const int r = __popc(vm & ((1u << lane) - 1u));
      s_src[warp][r] = moves[2 * k];
      s_dst[warp][r] = moves[2 * k + 1];
    }
    __syncwarp();
    const int nvalid = __popc(vm);
    if (D % 8 == 0)
      copy_rows(reinterpret_cast<uint4 *>(p.k_cache), reinterpret_cast<uint4 *>(p.v_cache), s_src[warp], s_dst[warp],
                nvalid, D / 8, lane);
    else
      copy_rows(reinterpret_cast<uint16_t *>(p.k_cache), reinterpret_cast<uint16_t *>(p.v_cache), s_src[warp],
                s_dst[warp], nvalid, D, lane);
    __syncwarp();
  }
}

// K/V rows of every move of the round for long heads: grid (head, part); a warp moves one
// (K, V) row pair per step with 16-byte lanes, 4 pairs in flight per warp.
// Sources are inside blocks freed by k_compact; nothing can reuse them before
// this kernel completes (stream order).
__global__ void __launch_bounds__(256) k_copy_kv_heads(kvc_pool p, const int32_t *moves, const int64_t *move_off,
                                                const int32_t *move_counts) {
  grid_dep_wait();
  grid_dep_trigger();
  const int g = blockIdx.x;
  const int n = move_counts[g];
  if (n == 0) return;
  const int D = p.head_dim;
  const int32_t *mv = moves + move_off[g] * 2;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nwarps = blockDim.x / 32 * gridDim.y;
  const int wid = blockIdx.y * (blockDim.x / 32) + warp;
  if (D % 8 == 0 && D <= 256) {
    const int vec = D / 8;  // 16-byte chunks per row (16 for d=128)
    uint4 *kc = reinterpret_cast<uint4 *>(p.k_cache);
    uint4 *vc = reinterpret_cast<uint4 *>(p.v_cache);
    // each lane covers chunk (lane % vec) of K (lane < 16) or V rows
    const int per = 32 / (2 * vec) > 0 ? 32 / (2 * vec) : 1;  // moves per warp step
    for (int base = wid * per * 4; base < n; base += nwarps * per * 4) {
      uint4 val[4];
      int64_t dst[4];
      bool ok[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int slot_lane = lane / (2 * vec);
        const int k = base + u * per + slot_lane;
        const int sub = lane % (2 * vec);
        const bool isv = sub >= vec;
        const int c = isv ? sub - vec : sub;
        ok[u] = k < n && slot_lane < per;
        if (ok[u]) {
          const int64_t src = mv[2 * k];
          dst[u] = (int64_t)mv[2 * k + 1] * vec + c;
          val[u] = isv ? vc[src * vec + c] : kc[src * vec + c];
          if (isv) dst[u] = -1 - dst[u];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (!ok[u]) continue;
        if (dst[u] >= 0) kc[dst[u]] = val[u];
        else vc[-1 - dst[u]] = val[u];
      }
      if (2 * vec > 32) {  // d = 256: second half of the row
        for (int u = 0; u < 4; ++u) {
          const int k = base + u * per;
          if (k >= n) continue;
          const int64_t src = mv[2 * k], d0 = mv[2 * k + 1];
          for (int c = lane; c < 2 * vec; c += 32) {
            if (c < 32) continue;
            const bool isv = c >= vec;
            const int cc = isv ? c - vec : c;
            if (isv) vc[d0 * vec + cc] = vc[src * vec + cc];
            else kc[d0 * vec + cc] = kc[src * vec + cc];
          }
        }
      }
    }
  } else {  // small or odd head_dim: element copies
    uint16_t *kc = reinterpret_cast<uint16_t *>(p.k_cache);
    uint16_t *vc = reinterpret_cast<uint16_t *>(p.v_cache);
    const int64_t total = (int64_t)n * D;
    for (int64_t i = (int64_t)wid * 32 + lane; i < total; i += (int64_t)nwarps * 32) {
      const int64_t k = i / D, c = i % D;
      const int64_t src = mv[2 * k], dst = mv[2 * k + 1];
      kc[dst * D + c] = kc[src * D + c];
      vc[dst * D + c] = vc[src * D + c];
    }
  }
}

// Fused prefill + compress: write every kept position's prompt row straight
// to its final slot.  Position pos of head g (table order, after compaction)
// holds prompt row src_pos[g][pos] (heads that evicted nothing: row pos).
// A warp places one 16-slot block: 2 rows per instruction, 16 B per lane.
__global__ void __launch_bounds__(256) k_place_prompt_kv(kvc_pool p, const int32_t *rows, int hp,
                                                         const int32_t *evict, const int32_t *src_pos,
                                                         int64_t src_stride, const uint4 *k, const uint4 *v,
                                                         int L) {
  grid_dep_wait();
  grid_dep_trigger();
  const int g = blockIdx.x;
  const int si = g / hp, hi = g % hp;
  const int64_t hidx = (int64_t)rows[si] * hp + hi;
  const int b = p.block_size;
  const int vec = p.head_dim / 8;
  const int Cn = p.ctx[hidx];
  const int nbl = (Cn + b - 1) / b;
  const bool moved = evict[g] > 0;
  const int32_t *sp = src_pos + g * src_stride;
  const uint4 *ks = k + (int64_t)hi * L * vec;  // [layer][head] = head_idx (layer-major)
  const uint4 *vs = v + (int64_t)hi * L * vec;
  uint4 *kc = reinterpret_cast<uint4 *>(p.k_cache);
  uint4 *vc = reinterpret_cast<uint4 *>(p.v_cache);
  const int32_t *tab = head_table(p, hidx);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nw = gridDim.y * 8;
  for (int bl = blockIdx.y * 8 + warp; bl < nbl; bl += nw) {
    const int64_t f0 = (int64_t)tab[bl] * b;
    const int n = b * vec;  // chunks of the block
    for (int c0 = 0; c0 < n; c0 += 4 * 32) {
      uint4 tk[4], tv[4];
      int64_t dst[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + u * 32 + lane;
        const int o = c / vec, pos = bl * b + o;
        dst[u] = -1;
        if (c < n && pos < Cn) {
          const int src = moved ? __ldg(sp + pos) : pos;
          if (src >= 0 && src < L) {
            tk[u] = __ldcs(ks + (int64_t)src * vec + c % vec);
            tv[u] = __ldcs(vs + (int64_t)src * vec + c % vec);
            dst[u] = (f0 + o) * vec + c % vec;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (dst[u] >= 0) { kc[dst[u]] = tk[u]; vc[dst[u]] = tv[u]; }
    }
  }
}

__global__ void k_free_total(kvc_pool p, int64_t *totals) {
  grid_dep_wait();
  grid_dep_trigger();
  using Red = cub::BlockReduce<int64_t, 1024>;
  __shared__ typename Red::TempStorage tmp;
  int64_t s = 0;
  for (int t = threadIdx.x; t < num_tiles(&p); t += 1024) s += p.free_tile[t];
  s = Red(tmp).Sum(s);
  if (threadIdx.x == 0) totals[3] = s;
}

// Threads per head for the histogram passes and the compaction: heads of at
// most 8192 slots (the decode-time batch) use small CTAs / one warp so more
// heads are resident at once; long prefill heads use wide CTAs.
static bool small_heads(const EvictState &S) { return S.max_slots <= 8192; }

int setup_state(const kvc_pool *pool, const kvc_evict_args *a, Scratch &sc, EvictState &S) {
  S.hp = pool->num_layers * pool->num_kv_heads;
  S.trace = nullptr;
  S.max_slots = (a->max_slots_per_head + 3) & ~int64_t(3);  // uint4 key rows
  S.status = pool->status;
  const int64_t T = (int64_t)a->n_seqs * S.hp;
  S.keys = sc.take<uint32_t>(T * S.max_slots);
  S.cap = sc.take<int32_t>(T);
  S.lo = sc.take<int32_t>(T);
  S.hi = sc.take<int32_t>(T);
  S.ltc = sc.take<int32_t>(T);
  S.lec = sc.take<int32_t>(T);
  S.lt1 = sc.take<int32_t>(T);
  S.lt2 = sc.take<int32_t>(T);
  // zero-initialised block: digit deltas, arrival counters, K/V copy claims
  S.zero_n = (int64_t)a->n_seqs * kBins + a->n_seqs + 1 + T + 1 + 3;
  S.max_chunks = a->moves_capacity / 32 + T + 1;
  S.zero_n += 2 * S.max_chunks + 1;  // the chunk queue (u64, 8-byte aligned below)
  S.zero = sc.take<int32_t>(S.zero_n);
  S.R = S.zero;
  S.done = S.zero ? S.R + (int64_t)a->n_seqs * kBins : nullptr;
  S.done_all = S.zero ? S.done + a->n_seqs : nullptr;
  S.kv_ready = S.zero ? S.done_all + 1 : nullptr;
  S.c16_done = S.zero ? S.kv_ready + T : nullptr;
  S.pub_count = S.zero ? S.c16_done + 1 : nullptr;
  S.chunk_tail = S.zero ? S.pub_count + 1 : nullptr;
  S.claim_next = S.zero ? S.chunk_tail + 1 : nullptr;
  S.chunks = S.zero ? reinterpret_cast<unsigned long long *>(
                          (reinterpret_cast<uintptr_t>(S.claim_next + 1) + 7) & ~uintptr_t(7))
                    : nullptr;
  S.totals = a->totals;
  S.cum1 = small_heads(S) ? nullptr : sc.take<int32_t>(T * kBins);
  S.cum2 = small_heads(S) ? nullptr : sc.take<int32_t>(T * kBins);
  S.cum3 = small_heads(S) ? nullptr : sc.take<int32_t>(T * 1024);
  S.below3 = small_heads(S) ? nullptr : sc.take<int32_t>(T);
  S.lt1p = small_heads(S) ? nullptr : sc.take<int32_t>(T);
  if (!small_heads(S) && (!S.cum1 || !S.cum2 || !S.cum3 || !S.below3 || !S.lt1p)) return KVC_ERR_INVALID;
  S.prefix = sc.take<uint32_t>(a->n_seqs);
  S.E = sc.take<int64_t>(a->n_seqs);
  S.seq_moves = sc.take<int64_t>(a->n_seqs);
  // candidate lists for the warp-per-head compaction of short heads
  S.cand = small_heads(S) && pool->block_size == 16 ? sc.take<unsigned long long>(T * 2 * kCand) : nullptr;
  if (!S.keys || !S.cap || !S.lo || !S.hi || !S.ltc || !S.lec || !S.lt1 || !S.lt2 || !S.R || !S.done || !S.prefix || !S.E || !S.seq_moves ||
      (small_heads(S) && pool->block_size == 16 && !S.cand))
    return KVC_ERR_INVALID;
  return KVC_OK;
}

int validate(const kvc_pool *pool, const kvc_evict_args *a) {
  if (!pool || !a || a->n_seqs < 0 || !pool->metric || !pool->tables) return KVC_ERR_INVALID;
  if (a->n_seqs && (!a->seq_rows || !a->budgets || !a->evict || !a->clamped || !a->move_offsets))
    return KVC_ERR_INVALID;
  if (a->max_slots_per_head < 1) return KVC_ERR_INVALID;
  return KVC_OK;
}

int run_schedule(const kvc_pool *pool, const kvc_evict_args *a, EvictState &S, cudaStream_t s) {
  const int64_t T = (int64_t)a->n_seqs * S.hp;
  cudaMemsetAsync(S.zero, 0, S.zero_n * sizeof(int32_t), s);
  // three radix levels (11 + 11 + 10 bits); the last head CTA of each
  // sequence finds that level's digit inside the histogram kernel; the last
  // one of k_bounds selects the tie rows and the move offsets
  if (small_heads(S)) {
    constexpr int NT = 256;
    launch_pdl(k_load<NT>, dim3((unsigned)T), dim3(NT), 0, s, *pool, a->seq_rows, a->budgets, S, 1, a->clamped);
    launch_pdl(k_hist<NT>, dim3((unsigned)T), dim3(NT), 0, s, *pool, a->seq_rows, S, 21, 10, 11, a->budgets, 2,
               a->clamped);
    launch_pdl(k_hist<NT>, dim3((unsigned)T), dim3(NT), 0, s, *pool, a->seq_rows, S, 10, 0, 10, a->budgets, 3,
               a->clamped);
    launch_pdl(k_bounds<NT>, dim3((unsigned)T), dim3(NT), 0, s, *pool, a->seq_rows, S, a->n_seqs, pool->block_size,
               a->evict, a->move_offsets);
    launch_pdl(k_select, dim3((unsigned)a->n_seqs), dim3(1024), 0, s, S, pool->block_size, a->evict,
               a->move_offsets, pool->status);
    launch_pdl(k_offsets, dim3(1), dim3(1024), 0, s, S, a->n_seqs, a->move_offsets);
  } else {
    constexpr int NT = kThreads;
    launch_pdl(k_load<NT>, dim3((unsigned)T), dim3(NT), 0, s, *pool, a->seq_rows, a->budgets, S, 1, a->clamped);
    launch_pdl(k_hist<NT>, dim3((unsigned)T), dim3(NT), 0, s, *pool, a->seq_rows, S, 21, 10, 11, a->budgets, 2,
               a->clamped);
    launch_pdl(k_hist_final<NT>, dim3((unsigned)T), dim3(NT), 0, s, *pool, a->seq_rows, S, a->budgets, a->clamped,
               a->n_seqs, pool->block_size, a->evict, a->move_offsets);
  }
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

void launch_copy_published(int n_sm, cudaStream_t s, const kvc_pool &pool, const EvictState &S, const MoveArgs &M) {
  // 4 CTAs per SM: they take the SMs as k_compact16's CTAs leave them
  launch_pdl(k_copy_published<8>, dim3(4 * n_sm), dim3(256), 0, s, pool, S, M);
}

int run_compact(const kvc_pool *pool, const kvc_evict_args *a, EvictState &S, cudaStream_t s, bool copy_kv = true) {
  const int64_t T = (int64_t)a->n_seqs * S.hp;
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  // long heads: k_compact16 moves the K/V rows itself, its copier warps
  // helping other heads when the round is one wave of CTAs
  const bool c16 = pool->block_size == 16 && !small_heads(S);
  const bool fuse = c16 && copy_kv && pool->k_cache && pool->head_dim % 8 == 0 && !getenv("KVC_K4_UNFUSED");
  MoveArgs M{a->evict, a->evicted_kvs, a->freed, a->moves, a->move_offsets, a->move_counts, a->totals,
             copy_kv ? nullptr : a->src_pos, S.max_slots, fuse ? 1 : 0, T};
  const int words = (int)((S.max_slots + 31) / 32);
  const int dyn = words * 8;  // bitmap + word prefixes
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_compact, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_compact16<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    configured = true;
  }
  if (dyn > 200 * 1024) return KVC_ERR_UNSUPPORTED;
  bool totals_done = false;
  if (pool->block_size == 16) {
    if (small_heads(S)) {
      launch_pdl(k_compact_warp, dim3((unsigned)((T + kWC - 1) / kWC)), dim3(kWC * 32), 0, s, *pool, a->seq_rows, S,
                 M, T);
    } else if (getenv("KVC_K4_TRACE")) {
      // debug: per-phase time of k_compact16 averaged over the heads (synchronises)
      unsigned long long *tr = nullptr;
      cudaMalloc(&tr, T * 64);
      cudaMemsetAsync(tr, 0, T * 64, s);
      S.trace = tr;
      k_compact16<512><<<(int)T, 512, dyn, s>>>(*pool, a->seq_rows, S, M);
      S.trace = nullptr;
      unsigned long long *h = (unsigned long long *)malloc(T * 64);
      cudaStreamSynchronize(s);
      cudaMemcpy(h, tr, T * 64, cudaMemcpyDeviceToHost);
      double acc[7] = {0};
      unsigned long long t0 = ~0ull, t1 = 0, pub_max = 0, pub_min = ~0ull;
      int n = 0;
      for (int64_t g = 0; g < T; ++g) {
        if (!h[g * 8 + 6]) continue;
        ++n;
        t0 = h[g * 8] < t0 ? h[g * 8] : t0;
        t1 = h[g * 8 + 7] > t1 ? h[g * 8 + 7] : t1;
        pub_max = h[g * 8 + 3] > pub_max ? h[g * 8 + 3] : pub_max;
        pub_min = h[g * 8 + 3] < pub_min ? h[g * 8 + 3] : pub_min;
        for (int k = 0; k < 7; ++k) acc[k] += (double)(h[g * 8 + k + 1] - h[g * 8 + k]) / 1e3;
      }
      fprintf(stderr, "[k4 trace] heads %d span %.1f us (move lists published %.1f-%.1f us); per head: T_h %.1f tie %.1f "
              "pairing %.1f meta %.1f free %.1f renumber %.1f, then K/V copy to CTA end %.1f us\n",
              n, (t1 - t0) / 1e3, (pub_min - t0) / 1e3, (pub_max - t0) / 1e3, acc[0] / n, acc[1] / n, acc[2] / n,
              acc[3] / n, acc[4] / n, acc[5] / n, acc[6] / n);
      free(h);
      cudaFree(tr);
      if (fuse) launch_copy_published(n_sm, s, *pool, S, M);
    }
    else if (dyn <= 100 * 1024) launch_pdl(k_compact16<512>, dim3((unsigned)T), dim3(512), dyn, s, *pool, a->seq_rows, S, M);
    else return KVC_ERR_UNSUPPORTED;
    // K/V moves beside the compaction, in publication order
    if (fuse) launch_copy_published(n_sm, s, *pool, S, M);
    totals_done = !small_heads(S) && !getenv("KVC_K4_TRACE");  // k_compact16's last CTA
  } else {
    launch_pdl(k_compact, dim3((unsigned)T), dim3(kThreads), dyn, s, *pool, a->seq_rows, S, M);
  }
  if (copy_kv && pool->k_cache && T > 0 && !fuse) {
    // short heads (few moves each): one flat grid; long heads: a CTA row per head
    if (small_heads(S))
      launch_pdl(k_copy_kv, dim3(n_sm * 8), dim3(256), 0, s, *pool, a->moves, a->move_offsets, a->move_counts, T);
    else
      launch_pdl(k_copy_kv_heads, dim3((unsigned)T, 8), dim3(256), 0, s, *pool, a->moves, a->move_offsets,
                 a->move_counts);
  }
  if (a->totals && !totals_done) launch_pdl(k_free_total, dim3(1), dim3(1024), 0, s, *pool, a->totals);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

}  // namespace

extern "C" {

int kvc_schedule_evictions(const kvc_pool *pool, const kvc_evict_args *a, void *stream) {
  int rc = validate(pool, a);
  if (rc || a->n_seqs == 0) return rc;
  Scratch sc(pool);
  EvictState S;
  if ((rc = setup_state(pool, a, sc, S))) return rc;
  return run_schedule(pool, a, S, (cudaStream_t)stream);
}

int kvc_execute_moves(const kvc_pool *pool, const kvc_evict_args *a, void *stream) {
  int rc = validate(pool, a);
  if (rc || a->n_seqs == 0) return rc;
  if (!a->moves || !pool->k_cache) return KVC_ERR_INVALID;
  Scratch sc(pool);
  EvictState S;
  if ((rc = setup_state(pool, a, sc, S))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  // keys are recomputed so the call is self-contained
  const int64_t T = (int64_t)a->n_seqs * S.hp;
  cudaMemsetAsync(S.zero, 0, S.zero_n * sizeof(int32_t), s);
  if (small_heads(S))
    launch_pdl(k_load<256>, dim3((unsigned)T), dim3(256), 0, s, *pool, a->seq_rows, a->budgets, S, 0, a->clamped);
  else
    launch_pdl(k_load<kThreads>, dim3((unsigned)T), dim3(kThreads), 0, s, *pool, a->seq_rows, a->budgets, S, 0,
               a->clamped);
  return run_compact(pool, a, S, s);
}

int kvc_prefill_compress(const kvc_pool *pool, const kvc_evict_args *a, const void *k, const void *v, int32_t L,
                         void *stream) {
  int rc = validate(pool, a);
  if (rc) return rc;
  if (a->n_seqs != 1 || !a->moves || !a->src_pos || !k || !v || L < 1 || !pool->k_cache || pool->head_dim % 8 != 0 ||
      pool->block_size != 16)
    return KVC_ERR_INVALID;
  Scratch sc(pool);
  EvictState S;
  if ((rc = setup_state(pool, a, sc, S))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if ((rc = run_schedule(pool, a, S, s))) return rc;
  if ((rc = run_compact(pool, a, S, s, /*copy_kv=*/false))) return rc;
  launch_pdl(k_place_prompt_kv, dim3((unsigned)S.hp, 4), dim3(256), 0, s, *pool, a->seq_rows, S.hp, a->evict,
             a->src_pos, S.max_slots, (const uint4 *)k, (const uint4 *)v, L);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

int kvc_compress(const kvc_pool *pool, const kvc_evict_args *a, void *stream) {
  int rc = validate(pool, a);
  if (rc || a->n_seqs == 0) return rc;
  if (!a->moves || !pool->k_cache) return KVC_ERR_INVALID;
  Scratch sc(pool);
  EvictState S;
  if ((rc = setup_state(pool, a, sc, S))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if ((rc = run_schedule(pool, a, S, s))) return rc;
  return run_compact(pool, a, S, s);
}

}  // extern "C"
