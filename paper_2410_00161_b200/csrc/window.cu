// K2: observation-window importance metric at prefill, on tcgen05 tensor
// cores with TMA-staged operands.
//
// Reference: gqa_attention (pkg/src/pagedkv/attention.py:62-89) builds the
// full causal softmax; window_metrics (metrics.py:68-89) sums f(A[h,i,j])
// over the last w query rows i and the r query heads of KV head h, then
// max-pools along the key axis (metrics.py:57-65) and protects the window;
// write_prompt_pass installs the result per slot (metrics.py:160-175).
//
// Only the r*w window rows of each KV head are ever formed here:
//   S^T[key, row] = K[key,:] . Q_w[row,:]       (M = 128 keys, N = r*w rows)
// is one tcgen05.mma.kind::f16 (bf16 in, fp32 accumulate in TMEM) per
// 16-wide K step; K tiles (128 keys x d) and the Q window are loaded by TMA
// (SWIZZLE_128B, K-major) into a 4-stage shared-memory ring.  Warp roles:
// warp 0 TMA producer, warp 1 MMA issuer + TMEM owner, warps 2-5 epilogue
// (one TMEM lane quadrant each).
//   pass 0: per-row online (max, sum exp) over this CTA's keys  -> partials
//   combine: per row M, 1/Z                                      (tiny)
//   pass 1: recompute the tile, raw[j] = sum_rows f(exp(s-M)/Z)   -> raw
//           (the layer's K is re-read from L2: 64 MB at Llama-8B shapes)
//   pool:  centred max-pool, install metric/logical/protected per slot.
#include <cuda.h>
#include <stdlib.h>
#include <stdio.h>

#include "common.cuh"

using namespace kvc;

namespace {

constexpr int kTileKeys = 128;
template <int D>
constexpr int stages_for() { return D >= 256 ? 2 : D >= 128 ? 3 : 6; }  // 2 CTAs/SM up to d=128

struct WinParams {
  int L, H, r, wq, RW, D, start;
  int tiles_per_head, chunks;  // CTA = (chunk, head)
  float scale;                 // log2(e) / sqrt(d)
  int agg;                     // 1 L1, 2 L2
  int dbg;                     // experiments: bit0 skip pass-0 math
  float2 *partial;             // [H][chunks][N] (m, z)
  float *raw;                  // [H][L]
  int *bar_cnt;                // [2H] fused-path barrier counters
};

// ---- PTX wrappers ---------------------------------------------------------

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  // K-major, SWIZZLE_128B: LBO = 16 B (ignored), SBO = 1024 B (8 rows x 128 B),
  // descriptor version 1 (sm_100), layout type 2.
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// ---- the tile pipeline ------------------------------------------------------

template <int N, int D, int PASS, int EW = 4>
struct WinCfg {
  static constexpr int kEW = PASS == 0 ? EW : 4;  // epilogue warps (EW/4 per lane quadrant in pass 0)
  static constexpr int kThreads = 64 + 32 * kEW;
  static constexpr int kNC = N / (kEW / 4);      // columns per epilogue thread
};

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int N, int D, int PASS, int EW, bool LAZY>
__global__ void __launch_bounds__(WinCfg<N, D, PASS, EW>::kThreads, 1)
    k_window(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmQ, const WinParams P) {
  using Cfg = WinCfg<N, D, PASS, EW>;
  constexpr int kEW = Cfg::kEW, kNC = Cfg::kNC, kThr = Cfg::kThreads;
  constexpr int kStages = stages_for<D>();
  constexpr int kAtoms = D / 64;                      // 128-byte K-major column blocks
  constexpr int kTileBytes = kTileKeys * D * 2;       // one K tile
  constexpr int kQBytes = N * D * 2;
  constexpr int kAcc = 4;                             // TMEM accumulators (MMA runs ahead)
  constexpr uint32_t kCols = kAcc * N;
  constexpr uint32_t kTmemCols = kCols <= 32 ? 32 : kCols <= 64 ? 64 : kCols <= 128 ? 128 : 256;
  constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *ktiles = smem;                                  // kStages x kTileBytes
  uint8_t *qbuf = smem + kStages * kTileBytes;             // kQBytes
  int *lim_s = reinterpret_cast<int *>(qbuf + kQBytes);  // [N] last visible key per column (-1: pad)
  uint64_t *bars = reinterpret_cast<uint64_t *>(lim_s + N);
  uint64_t *full = bars, *empty = bars + kStages, *tfull = bars + 2 * kStages, *tempty = tfull + kAcc,
           *qfull = tempty + kAcc;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(qfull + 1);
  float *stat_s = reinterpret_cast<float *>(tmem_slot + 4);  // pass 1: M[N], invZ[N]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int chunk = blockIdx.x, head = blockIdx.y;
  const int t_lo = (int)((int64_t)chunk * P.tiles_per_head / P.chunks);
  const int t_hi = (int)((int64_t)(chunk + 1) * P.tiles_per_head / P.chunks);
  const int ntiles = t_hi - t_lo;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < kAcc; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 32 * kEW); }
    mbar_init(qfull, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) { prefetch_tmap(&tmK); prefetch_tmap(&tmQ); }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int c = threadIdx.x; c < N; c += kThr) {
    const bool real = c < P.RW;
    lim_s[c] = real ? P.start + c % P.wq : -1;
    if (PASS == 1) {
      // fold the statistics partials of every chunk of this head (log-sum-exp)
      float mm = -INFINITY, zz = 0.f;
      for (int k = 0; k < P.chunks; ++k) {
        const float2 q = P.partial[((int64_t)head * P.chunks + k) * N + c];
        if (q.x == -INFINITY) continue;
        const float mn = fmaxf(mm, q.x);
        zz = (mm == -INFINITY ? 0.f : zz * exp2f(mm - mn)) + q.y * exp2f(q.x - mn);
        mm = mn;
      }
      stat_s[c] = real ? mm : INFINITY;  // padded columns contribute exp2(-inf) * 0
      stat_s[N + c] = (real && zz > 0.f) ? 1.f / zz : 0.f;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0 && ntiles > 0) {
      mbar_expect_tx(qfull, kQBytes);
      for (int a = 0; a < kAtoms; ++a)
        tma_load_2d(qbuf + a * N * 128, &tmQ, a * 64, head * P.RW, qfull);
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kStages;
        if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        mbar_expect_tx(&full[s], kTileBytes);
        const int row = head * P.L + (t_lo + i) * kTileKeys;
        // one 3-D box = the whole tile (kTileKeys contiguous rows, all atoms)
        tma_load_3d(ktiles + s * kTileBytes, &tmK, 0, row, 0, &full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (ntiles > 0) {
      mbar_wait(qfull, 0);
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kStages, acc = i % kAcc;
        mbar_wait(&full[s], (i / kStages) & 1);
        if (i >= kAcc) mbar_wait(&tempty[acc], ((i / kAcc) - 1) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t abase = smem_u32(ktiles + s * kTileBytes);
          const uint32_t bbase = smem_u32(qbuf);
#pragma unroll
          for (int kk = 0; kk < ((P.dbg & 2) ? 0 : D / 16); ++kk) {
            const int atom = kk / 4, sub = kk % 4;
            const uint64_t ad = sw128_desc(abase + atom * kTileKeys * 128 + sub * 32);
            const uint64_t bd = sw128_desc(bbase + atom * N * 128 + sub * 32);
            mma_bf16(tmem + acc * N, ad, bd, kIdesc, kk > 0 ? 1u : 0u);
          }
          mma_commit(&empty[s]);   // smem stage reusable once these MMAs finish
          mma_commit(&tfull[acc]); // accumulator ready for the epilogue
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue: warp w covers TMEM lane quadrant w%4 and
    // columns [half*kNC, half*kNC + kNC) ------------------------------------
    const int quad = warp & 3;
    const int half = (warp - 2) / 4;
    const int c0 = half * kNC;
    const int et = threadIdx.x - 64;
    const int key_local = quad * 32 + lane;
    float m[kNC], z[kNC];
#pragma unroll
    for (int c = 0; c < kNC; ++c) {
      m[c] = PASS == 0 ? -INFINITY : stat_s[c0 + c];
      z[c] = PASS == 0 ? 0.f : stat_s[N + c0 + c];
    }
    for (int i = 0; i < ntiles; ++i) {
      const int acc = i % kAcc;
      mbar_wait(&tfull[acc], (i / kAcc) & 1);
      tc_fence_after();
      float v[kNC];
      const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + acc * N + c0;
      if constexpr (kNC == 16) {
        tmem_ld16(tbase, v);
      } else {
#pragma unroll
        for (int g = 0; g < kNC / 32; ++g) tmem_ld32(tbase + g * 32, v + g * 32);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);  // all epilogue threads arrive: accumulator free
      const int tile0 = (t_lo + i) * kTileKeys;
      const int j = tile0 + key_local;  // key position within the head
      // every window row sees every key of this tile and the tile is inside L
      const bool fast = tile0 + kTileKeys - 1 <= P.start && tile0 + kTileKeys <= P.L;
      if (PASS == 0 && (P.dbg & 1)) {
        m[0] = fmaxf(m[0], v[0]);
      } else if (PASS == 0) {
        // online (max, sum exp2): the max only moves a few times per column,
        // so the rescaling branch is rare and most elements cost one exp2
#pragma unroll
        for (int c = 0; c < kNC; ++c) {
          if (fast || (j < P.L && j <= lim_s[c0 + c])) {
            const float s = v[c] * P.scale;
            if (LAZY) {
              if (s > m[c]) {
                z[c] = z[c] * exp2f(m[c] - s) + 1.f;
                m[c] = s;
              } else {
                z[c] += exp2f(s - m[c]);
              }
            } else {
              const float mn = fmaxf(m[c], s);
              z[c] = z[c] * exp2f(m[c] - mn) + exp2f(s - mn);
              m[c] = mn;
            }
          }
        }
      } else {
        float contrib = 0.f;
#pragma unroll
        for (int c = 0; c < kNC; ++c) {
          const float pr = exp2f(v[c] * P.scale - m[c]) * z[c];  // columns >= RW: M=+inf, 1/Z=0
          const float f = P.agg == 2 ? pr * pr : pr;
          contrib += (fast || j <= lim_s[c0 + c]) ? f : 0.f;
        }
        if (j < P.L) P.raw[(int64_t)head * P.L + j] = contrib;
      }
    }
    if (PASS == 0) {
      // combine the (m, z) of all key lanes per column through the idle ring
      named_sync(1, 32 * kEW);
      float *rm = reinterpret_cast<float *>(ktiles);
      float *rz = rm + 128 * (N + 1);
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        rm[key_local * (N + 1) + c0 + c] = m[c];
        rz[key_local * (N + 1) + c0 + c] = z[c];
      }
      named_sync(1, 32 * kEW);
      // every epilogue thread folds a slice of one column's 128 entries,
      // then one thread per column folds the slices
      constexpr int kSl = 32 * kEW / N;  // slices per column
      constexpr int kPer = 128 / kSl;
      float mm = -INFINITY, zz = 0.f;
      {
        const int col = et % N, sl = et / N;
        for (int k = sl * kPer; k < (sl + 1) * kPer; ++k) {
          const float qm = rm[k * (N + 1) + col], qz = rz[k * (N + 1) + col];
          if (qm == -INFINITY) continue;
          const float mn = fmaxf(mm, qm);
          zz = (mm == -INFINITY ? 0.f : zz * exp2f(mm - mn)) + qz * exp2f(qm - mn);
          mm = mn;
        }
      }
      named_sync(1, 32 * kEW);
      float2 *sl2 = reinterpret_cast<float2 *>(rm);
      sl2[et] = make_float2(mm, zz);
      named_sync(1, 32 * kEW);
      if (et < N) {
        float m2 = -INFINITY, z2 = 0.f;
        for (int k = 0; k < kSl; ++k) {
          const float2 q = sl2[k * N + et];
          if (q.x == -INFINITY) continue;
          const float mn = fmaxf(m2, q.x);
          z2 = (m2 == -INFINITY ? 0.f : z2 * exp2f(m2 - mn)) + q.y * exp2f(q.x - mn);
          m2 = mn;
        }
        P.partial[((int64_t)head * P.chunks + chunk) * N + et] = make_float2(m2, z2);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

// ---------------------------------------------------------------------------
// Fused single-pass K2 (cooperative launch): every CTA owns <= kMaxT tiles of
// one head and keeps their score tiles resident in TMEM, so K is read from
// HBM exactly once.  Per-head grid barriers separate (1) the softmax
// statistics, (2) the metric of the resident tiles and (3) pooling, which
// needs its neighbours' raw metrics.
// ---------------------------------------------------------------------------

struct FusedParams {
  WinParams w;
  int cph;            // CTAs per head
  int tiles_per_cta;  // <= kMaxT
  int *bar_cnt;       // [2][H] arrival counters (zeroed before launch)
  kvc_pool p;
  int row, layer, pool, protect;
  float *out;
};

__device__ __forceinline__ void head_barrier(int *cnt, int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(cnt, 1);
    while (atomicAdd(cnt, 0) < target) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}

template <int D>
constexpr int fused_stages() { return D >= 256 ? 2 : D >= 128 ? 5 : 10; }

// tcgen05 kernels run one CTA per SM here (EIATTR_RESERVED_SMEM_USED), so a
// CTA owns the whole 512-column TMEM: 16 resident 128x32 score tiles.
constexpr int kFusedEW = 16;  // epilogue warps: 4 per TMEM lane quadrant

template <int N, int D>
__global__ void __launch_bounds__(64 + 32 * kFusedEW, 1)
    k_window_fused(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmQ,
                   const __grid_constant__ CUtensorMap tmK16, const FusedParams F) {
  constexpr int kEW = kFusedEW, kGroups = kEW / 4, kNC = N / kGroups;
  constexpr int kStages = fused_stages<D>();
  constexpr int kAtoms = D / 64;
  constexpr int kTileBytes = kTileKeys * D * 2;
  constexpr int kQBytes = N * D * 2;
  constexpr int kMaxT = 512 / N;  // resident score tiles (all 512 TMEM columns)
  constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  const WinParams &P = F.w;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *ktiles = smem;
  uint8_t *qbuf = smem + kStages * kTileBytes;
  int *lim_s = reinterpret_cast<int *>(qbuf + kQBytes);
  uint64_t *bars = reinterpret_cast<uint64_t *>(lim_s + N);
  uint64_t *full = bars, *empty = bars + kStages, *tfull = bars + 2 * kStages, *qfull = tfull + kMaxT;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(qfull + 1);
  float *stat_s = reinterpret_cast<float *>(tmem_slot + 4);  // M[N], invZ[N]
  float *halfsum = stat_s + 2 * N;  // [kGroups-1][kMaxT][128] contributions of column groups >= 1

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int head = blockIdx.x / F.cph, cidx = blockIdx.x % F.cph;
  const int t_lo = cidx * F.tiles_per_cta;
  const int t_hi = min(P.tiles_per_head, t_lo + F.tiles_per_cta);
  const int ntiles = max(0, t_hi - t_lo);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < kMaxT; ++a) mbar_init(&tfull[a], 1);
    mbar_init(qfull, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) { prefetch_tmap(&tmK); prefetch_tmap(&tmQ); }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int c = threadIdx.x; c < N; c += blockDim.x) lim_s[c] = c < P.RW ? P.start + c % P.wq : -1;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int quad = warp & 3;
  const int half = (warp - 2) / 4;
  const int c0 = half * kNC;
  const int et = threadIdx.x - 64;
  const int key_local = quad * 32 + lane;

  // ================= phase 1: stream K once, scores -> TMEM, statistics =====
  if (warp == 0) {
    if (lane == 0 && ntiles > 0) {
      mbar_expect_tx(qfull, kQBytes);
      for (int a = 0; a < kAtoms; ++a) tma_load_2d(qbuf + a * N * 128, &tmQ, a * 64, head * P.RW, qfull);
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kStages;
        if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        mbar_expect_tx(&full[s], kTileBytes);
        const int row0 = head * P.L + (t_lo + i) * kTileKeys;
        if (P.dbg & 4) {
          // 16-row boxes (many small ops in flight) into the same [atom][row] layout
          for (int rg = 0; rg < kTileKeys / 16; ++rg)
            for (int a = 0; a < kAtoms; ++a)
              tma_load_2d(ktiles + s * kTileBytes + a * kTileKeys * 128 + rg * 16 * 128, &tmK16, a * 64,
                          row0 + rg * 16, &full[s]);
        } else {
          tma_load_3d(ktiles + s * kTileBytes, &tmK, 0, row0, 0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (ntiles > 0) {
      mbar_wait(qfull, 0);
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kStages;
        mbar_wait(&full[s], (i / kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t abase = smem_u32(ktiles + s * kTileBytes);
          const uint32_t bbase = smem_u32(qbuf);
#pragma unroll
          for (int kk = 0; kk < ((P.dbg & 2) ? 0 : D / 16); ++kk) {
            const int atom = kk / 4, sub = kk % 4;
            mma_bf16(tmem + i * N, sw128_desc(abase + atom * kTileKeys * 128 + sub * 32),
                     sw128_desc(bbase + atom * N * 128 + sub * 32), kIdesc, kk > 0 ? 1u : 0u);
          }
          mma_commit(&empty[s]);
          mma_commit(&tfull[i]);
        }
        __syncwarp();
      }
    }
  } else {
    float m[kNC], z[kNC];
#pragma unroll
    for (int c = 0; c < kNC; ++c) { m[c] = -INFINITY; z[c] = 0.f; }
    for (int i = 0; i < ntiles; ++i) {
      mbar_wait(&tfull[i], 0);
      tc_fence_after();
      float v[kNC];
      const uint32_t tb = tmem + ((uint32_t)(quad * 32) << 16) + i * N + c0;
      if constexpr (kNC == 16) tmem_ld16(tb, v);
      else tmem_ld32(tb, v);
      const int tile0 = (t_lo + i) * kTileKeys;
      const int j = tile0 + key_local;
      const bool fast = tile0 + kTileKeys - 1 <= P.start && tile0 + kTileKeys <= P.L;
      if (P.dbg & 1) { m[0] = fmaxf(m[0], v[0]); continue; }
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        if (fast || (j < P.L && j <= lim_s[c0 + c])) {
          const float s = v[c] * P.scale;
          const float mn = fmaxf(m[c], s);
          z[c] = z[c] * exp2f(m[c] - mn) + exp2f(s - mn);
          m[c] = mn;
        }
      }
    }
    // CTA combine through the idle ring, then one partial per column
    named_sync(1, 32 * kEW);
    float *rm = reinterpret_cast<float *>(ktiles);
    float *rz = rm + 128 * (N + 1);
#pragma unroll
    for (int c = 0; c < kNC; ++c) {
      rm[key_local * (N + 1) + c0 + c] = m[c];
      rz[key_local * (N + 1) + c0 + c] = z[c];
    }
    named_sync(1, 32 * kEW);
    constexpr int kSl = 32 * kEW / N, kPer = 128 / kSl;
    float mm = -INFINITY, zz = 0.f;
    {
      const int col = et % N, sl = et / N;
      for (int k = sl * kPer; k < (sl + 1) * kPer; ++k) {
        const float qm = rm[k * (N + 1) + col], qz = rz[k * (N + 1) + col];
        if (qm == -INFINITY) continue;
        const float mn = fmaxf(mm, qm);
        zz = (mm == -INFINITY ? 0.f : zz * exp2f(mm - mn)) + qz * exp2f(qm - mn);
        mm = mn;
      }
    }
    named_sync(1, 32 * kEW);
    float2 *sl2 = reinterpret_cast<float2 *>(rm);
    sl2[et] = make_float2(mm, zz);
    named_sync(1, 32 * kEW);
    if (et < N) {
      float m2 = -INFINITY, z2 = 0.f;
      for (int k = 0; k < kSl; ++k) {
        const float2 q = sl2[k * N + et];
        if (q.x == -INFINITY) continue;
        const float mn = fmaxf(m2, q.x);
        z2 = (m2 == -INFINITY ? 0.f : z2 * exp2f(m2 - mn)) + q.y * exp2f(q.x - mn);
        m2 = mn;
      }
      P.partial[((int64_t)head * F.cph + cidx) * N + et] = make_float2(m2, z2);
    }
  }
  head_barrier(&F.bar_cnt[head], F.cph);

  // ================= phase 2: head statistics, metric of resident tiles =======
  for (int c = threadIdx.x; c < N; c += blockDim.x) {
    float mm = -INFINITY, zz = 0.f;
    for (int k = 0; k < F.cph; ++k) {
      const float2 q = __ldcg(P.partial + ((int64_t)head * F.cph + k) * N + c);  // written by other CTAs
      if (q.x == -INFINITY) continue;
      const float mn = fmaxf(mm, q.x);
      zz = (mm == -INFINITY ? 0.f : zz * exp2f(mm - mn)) + q.y * exp2f(q.x - mn);
      mm = mn;
    }
    const bool real = c < P.RW;
    stat_s[c] = real ? mm : INFINITY;
    stat_s[N + c] = (real && zz > 0.f) ? 1.f / zz : 0.f;
  }
  __syncthreads();
  if (warp >= 2) {
    tc_fence_after();
    for (int i = 0; i < ntiles; ++i) {
      float v[kNC];
      const uint32_t tb = tmem + ((uint32_t)(quad * 32) << 16) + i * N + c0;
      if constexpr (kNC == 16) tmem_ld16(tb, v);
      else tmem_ld32(tb, v);
      const int tile0 = (t_lo + i) * kTileKeys;
      const int j = tile0 + key_local;
      const bool fast = tile0 + kTileKeys - 1 <= P.start;
      float contrib = 0.f;
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        const float pr = exp2f(v[c] * P.scale - stat_s[c0 + c]) * stat_s[N + c0 + c];
        const float f = P.agg == 2 ? pr * pr : pr;
        contrib += (fast || j <= lim_s[c0 + c]) ? f : 0.f;
      }
      if (half > 0) halfsum[((half - 1) * kMaxT + i) * 128 + key_local] = contrib;
      named_sync(2, 32 * kEW);
      if (half == 0 && j < P.L) {
        for (int gq = 1; gq < kGroups; ++gq) contrib += halfsum[((gq - 1) * kMaxT + i) * 128 + key_local];
        P.raw[(int64_t)head * P.L + j] = contrib;
      }
    }
  }
  head_barrier(&F.bar_cnt[P.H + head], F.cph);

  // ================= phase 3: centred max-pool + per-slot install ===========
  {
    const int half_p = F.pool / 2;
    const float *raw = P.raw + (int64_t)head * P.L;
    const int64_t hidx = F.row >= 0 ? head_index(F.p, F.row, F.layer, head) : 0;
    const int C = F.row >= 0 ? F.p.ctx[hidx] : 0;
    const int b = F.p.block_size;
    const int j_lo = t_lo * kTileKeys, j_hi = min(P.L, t_hi * kTileKeys);
    // stage this CTA's raw range plus the pooling halo in (idle) shared memory
    float *rs = reinterpret_cast<float *>(ktiles);
    const int s_lo = max(0, j_lo - half_p), s_hi = min(P.L, j_hi + half_p);
    for (int t = s_lo + threadIdx.x; t < s_hi; t += blockDim.x) rs[t - s_lo] = __ldcg(raw + t);
    __syncthreads();
    for (int j = j_lo + threadIdx.x; j < j_hi; j += blockDim.x) {
      float mx = rs[j - s_lo];
      const int lo = j - half_p < 0 ? 0 : j - half_p;
      const int hi = j + half_p >= P.L ? P.L - 1 : j + half_p;
      for (int t = lo; t <= hi; ++t) mx = fmaxf(mx, rs[t - s_lo]);
      if (F.out) F.out[(int64_t)head * P.L + j] = mx;
      if (F.row >= 0 && j < C) {
        const int64_t f = (int64_t)head_table(F.p, hidx)[j / b] * b + j % b;
        F.p.metric[f] = mx;
        F.p.logical[f] = j;
        F.p.protected_[f] = (F.protect && j >= P.start) ? 1 : 0;
        F.p.fresh[f] = 0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Centred max-pool (truncated at the edges) + per-slot install.
__global__ void k_win_pool(kvc_pool p, WinParams P, int row, int layer, int pool, int protect, float *out) {
  const int head = blockIdx.y;
  const int half = pool / 2;
  const float *raw = P.raw + (int64_t)head * P.L;
  const int64_t hidx = row >= 0 ? head_index(p, row, layer, head) : 0;
  const int C = row >= 0 ? p.ctx[hidx] : 0;
  const int b = p.block_size;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P.L; j += gridDim.x * blockDim.x) {
    float m = raw[j];
    const int lo = j - half < 0 ? 0 : j - half;
    const int hi = j + half >= P.L ? P.L - 1 : j + half;
    for (int t = lo; t <= hi; ++t) m = fmaxf(m, raw[t]);
    if (out) out[(int64_t)head * P.L + j] = m;
    if (row >= 0 && j < C) {
      const int64_t f = (int64_t)head_table(p, hidx)[j / b] * b + j % b;
      p.metric[f] = m;
      p.logical[f] = j;
      p.protected_[f] = (protect && j >= P.start) ? 1 : 0;
      p.fresh[f] = 0;
    }
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
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

// 2-D bf16 map over [rows][D] with a {64, box_rows} SWIZZLE_128B box.
// 3-D view {64 elems, rows, D/64 atoms} with a {64, box_rows, D/64} box: one
// op per tile, contiguous source rows, smem laid out [atom][row][128 B].
bool make_map3(CUtensorMap *map, const void *base, int64_t rows, int D, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(D / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)(D / 64)};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map(CUtensorMap *map, const void *base, int64_t rows, int D, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int N, int D>
int run_fused(const kvc_pool *pool, const kvc_window_args *a, WinParams &P, cudaStream_t s, int *bar_cnt) {
  constexpr int kMaxT = 512 / N;
  auto fn = k_window_fused<N, D>;
  const int smem = fused_stages<D>() * kTileKeys * D * 2 + N * D * 2 + N * 4 + 256 + 2 * N * 4 + (kFusedEW / 4) * kMaxT * 128 * 4 + 1024;
  static bool configured = false;
  static int capacity = 0;
  if (!configured) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int per_sm = 0, dev = 0, nsm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 64 + 32 * kFusedEW, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    per_sm = per_sm > 1 ? 1 : per_sm;  // 512 TMEM columns per CTA
    capacity = per_sm * nsm;
    configured = true;
  }
  if (getenv("KVC_DEBUG")) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 64 + 32 * kFusedEW, smem);
    cudaFuncAttributes at;
    cudaFuncGetAttributes(&at, fn);
    for (int sm2 : {100000, 90000, 60000, 30000}) {
      int ps = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, fn, 64 + 32 * 8, sm2);
      int ps2 = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps2, fn, 64, sm2);
      fprintf(stderr, "[kvc]   smem %d -> per_sm %d (64 thr: %d)\n", sm2, ps, ps2);
    }
    fprintf(stderr, "[kvc] fused K2: smem %d capacity %d per_sm %d regs %d static %zu maxdyn %d maxthr %d\n", smem,
            capacity, per_sm, at.numRegs, at.sharedSizeBytes, at.maxDynamicSharedSizeBytes, at.maxThreadsPerBlock);
  }
  if (capacity < 1 || smem > 227 * 1024) return KVC_ERR_UNSUPPORTED;
  const int total = P.H * P.tiles_per_head;
  int tpc = (total + capacity - 1) / capacity;
  if (tpc < 1) tpc = 1;
  while (tpc <= kMaxT && P.H * ((P.tiles_per_head + tpc - 1) / tpc) > capacity) ++tpc;
  if (tpc > kMaxT) return KVC_ERR_UNSUPPORTED;  // scores do not fit in TMEM: two-pass path
  const int cph = (P.tiles_per_head + tpc - 1) / tpc;
  CUtensorMap tmK, tmQ;
  if (!make_map3(&tmK, a->k, (int64_t)P.H * P.L, D, kTileKeys)) return KVC_ERR_CUDA;
  if (!make_map(&tmQ, a->q_win, (int64_t)a->num_query_heads * P.wq, D, N)) return KVC_ERR_CUDA;
  CUtensorMap tmK16;
  if (!make_map(&tmK16, a->k, (int64_t)P.H * P.L, D, 16)) return KVC_ERR_CUDA;
  FusedParams F;
  F.w = P;
  F.cph = cph;
  F.tiles_per_cta = tpc;
  F.bar_cnt = bar_cnt;
  F.p = *pool;
  F.row = a->seq_row;
  F.layer = a->layer;
  F.pool = a->pool;
  F.protect = a->protect_window;
  F.out = a->metrics_out;
  cudaMemsetAsync(bar_cnt, 0, 2 * P.H * sizeof(int), s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.H * cph);
  cfg.blockDim = dim3(64 + 32 * kFusedEW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: per-head grid barriers
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, tmK, tmQ, tmK16, F) == cudaSuccess ? KVC_OK : KVC_ERR_CUDA;
}

template <int N, int D>
int run_window(const kvc_pool *pool, const kvc_window_args *a, WinParams &P, cudaStream_t s) {
  {
    static int fused_off = -1;
    if (fused_off < 0) {
      const char *e = getenv("KVC_K2_TWOPASS");
      fused_off = (e && atoi(e) == 1) ? 1 : 0;
    }
    if (!fused_off && D <= 128 && P.bar_cnt) {
      const int rc = run_fused<N, D>(pool, a, P, s, P.bar_cnt);
      if (rc != KVC_ERR_UNSUPPORTED) return rc;
    }
  }
  CUtensorMap tmK, tmQ;
  if (!make_map3(&tmK, a->k, (int64_t)P.H * P.L, D, kTileKeys)) return KVC_ERR_CUDA;
  if (!make_map(&tmQ, a->q_win, (int64_t)a->num_query_heads * P.wq, D, N)) return KVC_ERR_CUDA;
  const int smem = stages_for<D>() * kTileKeys * D * 2 + N * D * 2 + N * 4 + 256 + 2 * N * 4 + 1024;
  // variant (experiments): KVC_K2_EW = 4|8 epilogue warps in pass 0, KVC_K2_LAZY = 0|1
  static int ew = -1, lazy = -1;
  if (ew < 0) {
    const char *e1 = getenv("KVC_K2_EW");
    const char *e2 = getenv("KVC_K2_LAZY");
    ew = (e1 && atoi(e1) == 8) ? 8 : 4;
    lazy = (e2 && atoi(e2) == 1) ? 1 : 0;
  }
  auto k1 = k_window<N, D, 1, 4, false>;
  auto k0 = ew == 8 ? (lazy ? k_window<N, D, 0, 8, true> : k_window<N, D, 0, 8, false>)
                    : (lazy ? k_window<N, D, 0, 4, true> : k_window<N, D, 0, 4, false>);
  const int t0 = ew == 8 ? WinCfg<N, D, 0, 8>::kThreads : WinCfg<N, D, 0, 4>::kThreads;
  static bool configured = false;
  if (!configured) {
    for (auto f : {k_window<N, D, 0, 8, true>, k_window<N, D, 0, 8, false>, k_window<N, D, 0, 4, true>,
                   k_window<N, D, 0, 4, false>, k1})
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  if (smem > 227 * 1024) return KVC_ERR_UNSUPPORTED;
  dim3 grid(P.chunks, P.H);
  k0<<<grid, t0, smem, s>>>(tmK, tmQ, P);
  k1<<<grid, WinCfg<N, D, 1>::kThreads, smem, s>>>(tmK, tmQ, P);
  const int gx = (P.L + 255) / 256 < 1184 ? (P.L + 255) / 256 : 1184;
  k_win_pool<<<dim3(gx, P.H), 256, 0, s>>>(*pool, P, a->seq_row, a->layer, a->pool, a->protect_window,
                                           a->metrics_out);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

}  // namespace

extern "C" int kvc_window_metric(const kvc_pool *pool, const kvc_window_args *a, void *stream) {
  if (!pool || !a || !a->q_win || !a->k || a->L < 1 || a->window < 1 || a->pool < 1 || a->pool % 2 == 0)
    return KVC_ERR_INVALID;
  const int H = pool->num_kv_heads;
  const int D = pool->head_dim;
  if (a->num_query_heads % H) return KVC_ERR_INVALID;
  if (a->seq_row >= 0 && (!pool->metric || !pool->tables)) return KVC_ERR_INVALID;
  WinParams P;
  P.L = a->L;
  P.H = H;
  P.r = a->num_query_heads / H;
  P.wq = a->window < a->L ? a->window : a->L;
  P.RW = P.r * P.wq;
  P.D = D;
  P.start = a->L - P.wq;
  P.tiles_per_head = (a->L + kTileKeys - 1) / kTileKeys;
  // one wave of CTAs (2 per SM when the ring fits twice in shared memory)
  const int per_sm = D <= 128 ? 2 : 1;
  int chunks = per_sm * 148 / H > 0 ? per_sm * 148 / H : 1;
  if (chunks > P.tiles_per_head) chunks = P.tiles_per_head;
  P.chunks = chunks;
  P.scale = 1.4426950408889634f / sqrtf((float)D);
  P.agg = a->aggregation == 2 ? 2 : 1;
  {
    const char *e = getenv("KVC_K2_DBG");
    P.dbg = e ? atoi(e) : 0;
  }
  const int N = P.RW <= 32 ? 32 : P.RW <= 64 ? 64 : 0;
  if (!N) return KVC_ERR_UNSUPPORTED;
  Scratch sc(pool);
  P.partial = sc.take<float2>((int64_t)H * (chunks > 304 ? chunks : 304) * N);
  P.raw = sc.take<float>((int64_t)H * a->L);
  P.bar_cnt = sc.take<int>(2 * H);
  if (!P.partial || !P.raw) return KVC_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const int nl = a->n_layers > 1 ? a->n_layers : 1;
  if (a->layer < 0 || (a->seq_row >= 0 && a->layer + nl > pool->num_layers)) return KVC_ERR_INVALID;
  // one layer at a time: the layer's K (64 MB at Llama-8B shapes) stays in L2
  // between the statistics pass and the metric pass
  for (int li = 0; li < nl; ++li) {
    kvc_window_args al = *a;
    al.layer = a->layer + li;
    al.q_win = reinterpret_cast<const uint16_t *>(a->q_win) + li * a->q_layer_stride;
    al.k = reinterpret_cast<const uint16_t *>(a->k) + li * a->k_layer_stride;
    al.metrics_out = a->metrics_out ? a->metrics_out + li * a->out_layer_stride : nullptr;
    int rc = KVC_ERR_UNSUPPORTED;
    if (N == 32 && D == 64) rc = run_window<32, 64>(pool, &al, P, s);
    else if (N == 32 && D == 128) rc = run_window<32, 128>(pool, &al, P, s);
    else if (N == 32 && D == 256) rc = run_window<32, 256>(pool, &al, P, s);
    else if (N == 64 && D == 64) rc = run_window<64, 64>(pool, &al, P, s);
    else if (N == 64 && D == 128) rc = run_window<64, 128>(pool, &al, P, s);
    if (rc != KVC_OK) return rc;
  }
  return KVC_OK;
}
