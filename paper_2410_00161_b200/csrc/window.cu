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
#include "tc.cuh"

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
// Persistent K2 over every layer of a prompt (cooperative launch, one CTA per
// SM).  CTA c owns the K tiles [t_lo, t_hi) of head h = c / cph in every
// layer, so each layer's K is read from HBM exactly once.  Score tiles live
// in a TMEM slot ring (S = 512 / N slots of 128 keys x N columns) that runs
// across layers: while the epilogue warps finish layer l
//     A  online (max, sum exp2) per column over the CTA's resident tiles
//        -> one partial per column               -> head barrier 1
//     B  head statistics; raw[j] = sum_col f(exp2(s - M) / Z), releasing
//        each TMEM slot after its last read      -> head barrier 2
//     C  centred max-pool of raw (halo from the neighbours) + per-slot
//        install through the block table (metrics.py:57-65, 160-175)
// the TMA warp already streams layer l+1 into the shared-memory ring and the
// MMA warp into the slots that B frees.  Epilogue group g (4 warps, one per
// TMEM lane quadrant) owns the tiles i with i % kGroups == g in A and B.
// Head barriers are monotonic per-head counters (zeroed before launch).
// ---------------------------------------------------------------------------

struct PersistParams {
  int L, Lp, H, RW, wq, start, nl, n_q;
  int tiles_per_head, cph;
  int rs_len;       // pooling stage floats (persist_rs_len of the largest tile range)
  float scale;      // log2(e) / sqrt(d)
  int agg;          // 1 L1, 2 L2
  float2 *partial;  // [H][cph][N] (m, z) per CTA and column
  float *raw;       // [2][H][Lp] (Lp = L rounded up to 4) unpooled metric of layers l (l & 1) and l - 1
  int *bar_cnt;     // [H] arrivals (monotonic over the launch)
  kvc_pool p;
  int row, layer0, pool, protect;
  float *out;       // [nl][H][L] pooled metrics (optional)
  int64_t out_layer_stride;
  unsigned long long *trace;  // debug (KVC_K2_TRACE): [grid][nl][8] globaltimer stamps
  int dbg;                    // debug (KVC_K2_DBG): bit0 treat every tile as unmasked
  int write_k;                // also store the prompt K rows of every whole 16-key block into the pool
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int kPEW = 8;                // epilogue warps
constexpr int kPGroups = kPEW / 4;     // tile groups (4 warps cover the 4 TMEM lane quadrants)
constexpr int kPThreads = 96 + 32 * kPEW;  // TMA, MMA, epilogue warps, K-row writer

template <int D>
constexpr int persist_stages() { return D >= 128 ? 5 : 10; }

// pooling stage length (floats): a CTA's own key range + halo, 16-byte rows
__host__ __device__ constexpr int persist_rs_len(int ntiles, int pool) {
  return (ntiles * kTileKeys + pool + 8 + 3) & ~3;
}

template <int N, int D>
constexpr int persist_smem(int pool, int ntiles) {
  return persist_stages<D>() * kTileKeys * D * 2   // K ring
         + 2 * N * D * 2                           // Q window, double-buffered over layers
         + persist_rs_len(ntiles, pool) * 4         // pooling stage (own range + halo)
         + kPEW * N * 8                            // per-warp statistics
         + 2 * N * 4 + N * 4                       // M, 1/Z, column limits
         + 512 + 1024;                             // barriers, TMEM slot, alignment
}

constexpr float kNegBig = -1e30f;  // running-max sentinel: finite, so no inf - inf
constexpr int kMaxHalf = 7;         // pool widths up to 15 take the register path in phase C


// One element of the online (max, sum exp2) with lazy rescaling, branch-free:
// one MUFU per element; s = -inf (masked) leaves (m, z) unchanged.
__device__ __forceinline__ void lse_step(float &m, float &z, float s) {
  const bool up = s > m;
  const float e = ex2_approx(up ? m - s : s - m);
  z = up ? fmaf(z, e, 1.f) : z + e;
  m = up ? s : m;
}

// Bit c: column h*32 + c (query head (h*32+c) / wq, window row start +
// (h*32+c) % wq) sees key j causally; padding columns (>= RW) never do.
__device__ __forceinline__ uint32_t window_mask(const PersistParams &P, int j, int h) {
  uint32_t vm = 0;
  if (j < P.L) {
    const int dj = j - P.start;
    int rr = (h * 32) % P.wq;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      if (h * 32 + c < P.RW && rr >= dj) vm |= 1u << c;
      rr = rr + 1 == P.wq ? 0 : rr + 1;
    }
  }
  return vm;
}

// (m, z) <- log-sum-exp merge of (m, z) and (m2, z2) in base 2.
__device__ __forceinline__ void lse2_merge(float &m, float &z, float m2, float z2) {
  const float mn = fmaxf(m, m2);
  const float a = m == -INFINITY ? 0.f : z * ex2_approx(m - mn);
  const float b = m2 == -INFINITY ? 0.f : z2 * ex2_approx(m2 - mn);
  m = mn;
  z = a + b;
}

// Warp reduce-scatter of 32 per-lane (m, z) columns: afterwards lane l holds
// the merge over all 32 lanes of column l in m[0], z[0].
__device__ __forceinline__ void warp_lse_scatter32(float *m, float *z, int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int c = 0; c < o; ++c) {
      const float sm = up ? m[c] : m[c + o], sz = up ? z[c] : z[c + o];
      const float km = up ? m[c + o] : m[c], kz = up ? z[c + o] : z[c];
      const float rm = __shfl_xor_sync(0xffffffffu, sm, o);
      const float rz = __shfl_xor_sync(0xffffffffu, sz, o);
      float mm = km, zz = kz;
      lse2_merge(mm, zz, rm, rz);
      m[c] = mm;
      z[c] = zz;
    }
  }
}

// Epilogue-only head barrier: named barrier over the epilogue warps, one
// thread publishes the CTA's arrival and waits for `target` arrivals.
__device__ __forceinline__ void epi_head_barrier(int *cnt, int target, bool leader) {
  named_sync(1, 32 * kPEW);
  if (leader) {
    // release/acquire instead of two fence.sc: the named barrier orders the
    // other epilogue threads' partial/raw writes before this release, and the
    // acquire poll (with the named barrier after it) orders their reads after
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(cnt) : "memory");
    while (ld_acquire_gpu(cnt) < target) __nanosleep(32);
  }
  named_sync(1, 32 * kPEW);
}

// RECOMP: a CTA's tiles of a layer exceed the TMEM slots (long prompts, e.g.
// 128k); each layer's tiles are then streamed twice - statistics, then the
// metric - through a rolling slot ring (K read twice from HBM).
template <int N, int D, bool RECOMP>
__global__ void __launch_bounds__(kPThreads, 1)
    k_window_persist(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmQ,
                     const __grid_constant__ CUtensorMap tmP, const PersistParams P) {
  constexpr int kS = 512 / N;  // TMEM slots
  constexpr int kPasses = RECOMP ? 2 : 1;
  constexpr int kStages = persist_stages<D>();
  constexpr int kAtoms = D / 64;
  constexpr int kTileBytes = kTileKeys * D * 2;
  constexpr int kQBytes = N * D * 2;
  constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *ktiles = smem;
  uint8_t *qbuf = smem + kStages * kTileBytes;                      // [2][kQBytes]
  float *rs = reinterpret_cast<float *>(qbuf + 2 * kQBytes);        // pooling stage
  float2 *wred = reinterpret_cast<float2 *>(rs + P.rs_len);         // [kPEW][N]
  float *stat_s = reinterpret_cast<float *>(wred + kPEW * N);       // M[N], 1/Z[N]
  int *lim_s = reinterpret_cast<int *>(stat_s + 2 * N);             // [N]
  uint64_t *bars = reinterpret_cast<uint64_t *>(lim_s + N);
  uint64_t *full = bars, *empty = bars + kStages, *tfull = empty + kStages, *tempty = tfull + kS;
  uint64_t *qfull = tempty + kS, *qempty = qfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(qempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int head = blockIdx.x / P.cph, cidx = blockIdx.x % P.cph;
  // the first (tiles % cph) CTAs take one extra tile; the last CTA, which
  // holds the masked observation-window tile, never does
  const int q_t = P.tiles_per_head / P.cph, rem_t = P.tiles_per_head % P.cph;
  const int t_lo = cidx * q_t + min(cidx, rem_t);
  const int t_hi = t_lo + q_t + (cidx < rem_t ? 1 : 0);
  const int ntiles = t_hi - t_lo;  // >= 1; <= kS unless RECOMP (checked on the host)

  if (threadIdx.x == 0) {
    // write_k: a stage is free again once its MMAs have read it (tcgen05.commit) and
    // its K-row stores have read it (the MMA warp's arrival after wait_group.read)
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], P.write_k ? 2 : 1); }
    for (int a = 0; a < kS; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    for (int b = 0; b < 2; ++b) { mbar_init(&qfull[b], 1); mbar_init(&qempty[b], 1); }
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

  if (warp == 0) {
    // ---------------- TMA producer: Q window per layer, K tiles ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int l = 0; l < P.nl; ++l) {
        const int qb = l & 1;
        if (l >= 2) mbar_wait(&qempty[qb], ((l >> 1) - 1) & 1);
        mbar_expect_tx(&qfull[qb], kQBytes);
        for (int a = 0; a < kAtoms; ++a)
          tma_load_2d(qbuf + qb * kQBytes + a * N * 128, &tmQ, a * 64, (l * P.n_q) * P.wq + head * P.RW, &qfull[qb]);
        for (int gi = 0; gi < kPasses * ntiles; ++gi) {
          const int i = gi % ntiles;
          const uint32_t g = (uint32_t)(l * kPasses * ntiles + gi);
          const int s = g % kStages;
          if (g >= (uint32_t)kStages) mbar_wait(&empty[s], ((g / kStages) - 1) & 1);
          mbar_expect_tx(&full[s], kTileBytes);
          const int row0 = (l * P.H + head) * P.L + (t_lo + i) * kTileKeys;
          tma_load_3d_hint(ktiles + s * kTileBytes, &tmK, 0, row0, 0, &full[s], pol);
          if (P.trace && i == 0) P.trace[((int64_t)blockIdx.x * P.nl + l) * 8 + 6] = gtimer();
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: S^T[key, col] = K . Q_w^T into TMEM slots ----------------
    for (int l = 0; l < P.nl; ++l) {
      const int qb = l & 1;
      mbar_wait(&qfull[qb], (l >> 1) & 1);
      for (int gi = 0; gi < kPasses * ntiles; ++gi) {
        const uint32_t g = (uint32_t)(l * kPasses * ntiles + gi);
        const int s = g % kStages, slot = g % kS;
        mbar_wait(&full[s], (g / kStages) & 1);
        if (g >= (uint32_t)kS) mbar_wait(&tempty[slot], ((g / kS) - 1) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t abase = smem_u32(ktiles + s * kTileBytes);
          const uint32_t bbase = smem_u32(qbuf + qb * kQBytes);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const int atom = kk / 4, sub = kk % 4;
            mma_bf16(tmem + slot * N, sw128_desc(abase + atom * kTileKeys * 128 + sub * 32),
                     sw128_desc(bbase + atom * N * 128 + sub * 32), kIdesc, kk > 0 ? 1u : 0u);
          }
          mma_commit(&empty[s]);
          mma_commit(&tfull[slot]);
          if (gi == kPasses * ntiles - 1) mma_commit(&qempty[qb]);
          if (P.trace && gi == kPasses * ntiles - 1) P.trace[((int64_t)blockIdx.x * P.nl + l) * 8 + 7] = gtimer();
        }
        __syncwarp();
      }
    }
  } else if (warp == 2 + kPEW) {
    // ---------------- K-row writer (write_k: the unfused prefill) ----------------
    // Each staged K tile also goes to the paged cache, one TMA store per
    // (16-key block, 64-column atom), so the prompt's K is read from HBM once
    // for the metric and the write.  Lane b < 8 holds block b's pool id of
    // the current tile, loaded a tile ahead (-1: recompute pass, or a block
    // not whole inside the prompt: the scatter writes that one).  A stage is
    // released (its second arrival) once its stores have read it.
    if (P.write_k) {
      const uint32_t gtot = (uint32_t)(P.nl * kPasses * ntiles);
      auto tile_blk = [&](uint32_t g) -> int32_t {
        const int l = (int)(g / (uint32_t)(kPasses * ntiles)), gi = (int)(g % (uint32_t)(kPasses * ntiles));
        if (gi >= ntiles || lane >= kTileKeys / 16) return -1;
        const int key0 = (t_lo + gi) * kTileKeys + lane * 16;
        if (key0 + 16 > P.L) return -1;
        return head_table(P.p, head_index(P.p, P.row, P.layer0 + l, head))[key0 / 16];
      };
      int32_t blk_nxt = tile_blk(0);
      int prev_s = -1;
      for (uint32_t g = 0; g < gtot; ++g) {
        const int s = g % kStages;
        const int32_t blk_cur = blk_nxt;
        blk_nxt = g + 1 < gtot ? tile_blk(g + 1) : -1;
        int32_t blks[kTileKeys / 16];
#pragma unroll
        for (int b = 0; b < kTileKeys / 16; ++b) blks[b] = __shfl_sync(0xffffffffu, blk_cur, b);
        mbar_wait(&full[s], (g / kStages) & 1);
        if (lane == 0) {
          const uint8_t *tile = ktiles + s * kTileBytes;
#pragma unroll
          for (int b = 0; b < kTileKeys / 16; ++b)
            if (blks[b] >= 0)
#pragma unroll
              for (int a = 0; a < kAtoms; ++a)
                tma_store_3d(&tmP, tile + a * kTileKeys * 128 + b * 16 * 128, 0, blks[b] * 16, a);
          bulk_commit();
          if (prev_s >= 0) {  // the previous stage's stores have read it
            bulk_wait_read<1>();
            mbar_arrive(&empty[prev_s]);
          }
          prev_s = s;
        }
        __syncwarp();
      }
      if (lane == 0) {
        bulk_wait_read<0>();
        if (prev_s >= 0) mbar_arrive(&empty[prev_s]);
        bulk_wait<0>();  // the K rows are in the pool before the grid completes
      }
    }
  } else {
    // ---------------- epilogue ----------------
    const int ew = warp - 2;                // 0 .. kPEW-1
    const int quad = warp & 3;              // TMEM lane quadrant this warp may access
    const int grp = ew / 4;                 // tile group
    const int key_local = quad * 32 + lane;
    const int et = threadIdx.x - 64;
    int phase_k = 0;                        // head barriers passed
    const float scale_b = P.agg == 2 ? 2.f * P.scale : P.scale;
    for (int l = 0; l <= P.nl; ++l) {
      unsigned long long *tr = (P.trace && l < P.nl) ? P.trace + ((int64_t)blockIdx.x * P.nl + l) * 8 : nullptr;
      if (tr && et == 0) tr[0] = gtimer();
      float m[N], z[N];
      if (l < P.nl) {
        const uint32_t gbase = (uint32_t)(l * kPasses * ntiles);
        // ---- A: online (max, sum exp2) per column, branch-free lazy rescale ----
#pragma unroll
        for (int c = 0; c < N; ++c) { m[c] = kNegBig; z[c] = 0.f; }
        for (int i = grp; i < ntiles; i += kPGroups) {
          const uint32_t g = gbase + i;
          const int slot = g % kS;
          mbar_wait(&tfull[slot], (g / kS) & 1);
          tc_fence_after();
          const int tile0 = (t_lo + i) * kTileKeys;
          const int j = tile0 + key_local;
          const bool fast = (tile0 + kTileKeys - 1 <= P.start && tile0 + kTileKeys <= P.L) || (P.dbg & 1);
          const uint32_t tb = tmem + ((uint32_t)(quad * 32) << 16) + slot * N;
#pragma unroll
          for (int h = 0; h < N / 32; ++h) {
            float v[32];
            tmem_ld32(tb + h * 32, v);
            if (fast) {  // every window row sees every key (padded columns are discarded later)
#pragma unroll
              for (int c = 0; c < 32; ++c) lse_step(m[h * 32 + c], z[h * 32 + c], v[c] * P.scale);
            } else {
              const uint32_t vm = window_mask(P, j, h);
#pragma unroll
              for (int c = 0; c < 32; ++c)
                lse_step(m[h * 32 + c], z[h * 32 + c], ((vm >> c) & 1u) ? v[c] * P.scale : -INFINITY);
            }
          }
          if (RECOMP) {  // the metric pass recomputes this tile: free the slot now
            tc_fence_before();
            mbar_arrive(&tempty[slot]);
          }
        }
        // CTA partial per column: warp reduce-scatter, then fold the warps
#pragma unroll
        for (int h = 0; h < N / 32; ++h) {
          warp_lse_scatter32(m + h * 32, z + h * 32, lane);
          wred[ew * N + h * 32 + lane] = make_float2(m[h * 32], z[h * 32]);
        }
        if (tr && et == 0) tr[1] = gtimer();
        named_sync(1, 32 * kPEW);
        if (et < N) {
          float2 acc = wred[et];
#pragma unroll
          for (int w = 1; w < kPEW; ++w) {
            const float2 q = wred[w * N + et];
            lse2_merge(acc.x, acc.y, q.x, q.y);
          }
          P.partial[((int64_t)head * P.cph + cidx) * N + et] = acc;
        }
      }
      // one head barrier per layer: after it, layer l's partials and layer
      // l-1's raw metrics of the whole head are visible
      epi_head_barrier(&P.bar_cnt[head], P.cph * (++phase_k), et == 0);
      if (tr && et == 0) tr[2] = gtimer();

      if (l < P.nl) {
        const uint32_t gbase = (uint32_t)((l * kPasses + kPasses - 1) * ntiles);  // the metric pass's tiles
        // ---- B: head statistics (8 partial folds per column in parallel) ----
        {
          constexpr int kParts = 32 * kPEW / N;
          const int col = et % N, part = et / N;
          float mm = kNegBig, zz = 0.f;
          for (int k = part; k < P.cph; k += kParts) {
            const float2 q = __ldcg(P.partial + ((int64_t)head * P.cph + k) * N + col);  // other CTAs' partials
            lse2_merge(mm, zz, q.x, q.y);
          }
          named_sync(1, 32 * kPEW);  // wred reuse
          wred[part * N + col] = make_float2(mm, zz);
          named_sync(1, 32 * kPEW);
          if (et < N) {
            float2 acc = wred[et];
#pragma unroll
            for (int w = 1; w < kParts; ++w) {
              const float2 q = wred[w * N + et];
              lse2_merge(acc.x, acc.y, q.x, q.y);
            }
            const bool real = et < P.RW;
            const float iz = (real && acc.y > 0.f) ? 1.f / acc.y : 0.f;
            // f(p) = p (L1) or p^2 = exp2(2(s - M)) / Z^2 (L2)
            stat_s[et] = real ? (P.agg == 2 ? 2.f * acc.x : acc.x) : INFINITY;
            stat_s[N + et] = P.agg == 2 ? iz * iz : iz;
          }
          named_sync(1, 32 * kPEW);
        }
#pragma unroll
        for (int c = 0; c < N; ++c) { m[c] = stat_s[c]; z[c] = stat_s[N + c]; }
        // ---- B: raw metric of the resident tiles; each slot is released after its last read ----
        float *raw = P.raw + ((int64_t)(l & 1) * P.H + head) * P.Lp;
        for (int i = grp; i < ntiles; i += kPGroups) {
          const uint32_t g = gbase + i;
          const int slot = g % kS;
          if (RECOMP) {  // recomputed tile of the metric pass
            mbar_wait(&tfull[slot], (g / kS) & 1);
            tc_fence_after();
          }
          const int tile0 = (t_lo + i) * kTileKeys;
          const int j = tile0 + key_local;
          const bool fast = tile0 + kTileKeys - 1 <= P.start;
          const uint32_t tb = tmem + ((uint32_t)(quad * 32) << 16) + slot * N;
          float contrib = 0.f;
#pragma unroll
          for (int h = 0; h < N / 32; ++h) {
            float v[32];
            tmem_ld32(tb + h * 32, v);
            if (h == N / 32 - 1) {
              tc_fence_before();
              mbar_arrive(&tempty[slot]);  // slot free for the next layer's tiles
            }
            if (fast) {
#pragma unroll
              for (int c = 0; c < 32; ++c)
                contrib = fmaf(ex2_approx(fmaf(v[c], scale_b, -m[h * 32 + c])), z[h * 32 + c], contrib);
            } else {
              const uint32_t vm = window_mask(P, j, h);
#pragma unroll
              for (int c = 0; c < 32; ++c) {
                const float f = ex2_approx(fmaf(v[c], scale_b, -m[h * 32 + c])) * z[h * 32 + c];
                contrib += ((vm >> c) & 1u) ? f : 0.f;
              }
            }
          }
          if (j < P.L) raw[j] = contrib;
        }
        if (tr && et == 0) tr[3] = gtimer();
      }

      // ---- C: pooling + install of the PREVIOUS layer (its raw metrics of
      // the whole head became visible at this layer's barrier).  Four keys
      // per step: their slots are contiguous (block_size % 4 == 0). ----
      if (l >= 1) {
        const int lp = l - 1;
        const int half_p = P.pool / 2;
        const float *raw = P.raw + ((int64_t)(lp & 1) * P.H + head) * P.Lp;
        const int layer = P.layer0 + lp;
        const int64_t hidx = P.row >= 0 ? head_index(P.p, P.row, layer, head) : 0;
        const int b = P.row >= 0 ? P.p.block_size : 16;
        const int j_lo = t_lo * kTileKeys, j_hi = min(P.L, t_hi * kTileKeys);
        const int s_lo = j_lo - half_p;  // rs[t - s_lo] = raw[t]; outside [0, L): -inf
        const int n_own = (j_hi - j_lo + 3) / 4;
        // own range as float4 (j_lo is 128-aligned), halo as scalars, table slice
        for (int t = et; t < n_own; t += 32 * kPEW) {
          const int j = j_lo + 4 * t;
          float4 v4;
          if (j + 3 < P.L) v4 = __ldcg(reinterpret_cast<const float4 *>(raw + j));
          else {
            v4.x = raw[j];
            v4.y = j + 1 < P.L ? __ldcg(raw + j + 1) : -INFINITY;
            v4.z = j + 2 < P.L ? __ldcg(raw + j + 2) : -INFINITY;
            v4.w = -INFINITY;
          }
          rs[half_p + 4 * t] = v4.x; rs[half_p + 4 * t + 1] = v4.y;
          rs[half_p + 4 * t + 2] = v4.z; rs[half_p + 4 * t + 3] = v4.w;
        }
        if (et < 2 * half_p) {
          const int k = et < half_p ? et : half_p + 4 * n_own + (et - half_p);
          const int t = s_lo + k;
          rs[k] = (t >= 0 && t < P.L) ? __ldcg(raw + t) : -INFINITY;
        }
        const int nb_rng = (j_hi - j_lo + b - 1) / b;
        int *tab_s = reinterpret_cast<int *>(wred);  // idle here: kPEW*N*2 ints >= 16 tiles of blocks
        const int C = P.row >= 0 ? P.p.ctx[hidx] : 0;
        if (P.row >= 0)
          for (int t = et; t < nb_rng; t += 32 * kPEW) tab_s[t] = __ldg(head_table(P.p, hidx) + j_lo / b + t);
        named_sync(1, 32 * kPEW);
        float *out = P.out ? P.out + lp * P.out_layer_stride + (int64_t)head * P.L : nullptr;
        for (int t = et; t < n_own; t += 32 * kPEW) {
          const int j = j_lo + 4 * t;
          float w[4 + 2 * kMaxHalf];
          float mx[4];
          if (half_p <= kMaxHalf) {
#pragma unroll
            for (int k = 0; k < 4 + 2 * kMaxHalf; ++k) w[k] = k < 4 + 2 * half_p ? rs[4 * t + k] : -INFINITY;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float v = -INFINITY;
#pragma unroll
              for (int k = 0; k <= 2 * kMaxHalf; ++k) v = k <= 2 * half_p ? fmaxf(v, w[e + k]) : v;
              mx[e] = v;
            }
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float v = -INFINITY;
              for (int k = 0; k <= 2 * half_p; ++k) v = fmaxf(v, rs[4 * t + e + k]);
              mx[e] = v;
            }
          }
          if (out) {
            if (j + 3 < P.L && (reinterpret_cast<uintptr_t>(out + j) & 15) == 0)
              *reinterpret_cast<float4 *>(out + j) = make_float4(mx[0], mx[1], mx[2], mx[3]);
            else
              for (int e = 0; e < 4 && j + e < P.L; ++e) out[j + e] = mx[e];
          }
          if (P.row >= 0 && j < C) {
            const int64_t f = (int64_t)tab_s[(j - j_lo) / b] * b + j % b;
            const uint8_t pr[4] = {(uint8_t)(P.protect && j >= P.start), (uint8_t)(P.protect && j + 1 >= P.start),
                                   (uint8_t)(P.protect && j + 2 >= P.start), (uint8_t)(P.protect && j + 3 >= P.start)};
            if (j + 3 < C) {
              *reinterpret_cast<float4 *>(P.p.metric + f) = make_float4(mx[0], mx[1], mx[2], mx[3]);
              *reinterpret_cast<int4 *>(P.p.logical + f) = make_int4(j, j + 1, j + 2, j + 3);
              *reinterpret_cast<uint32_t *>(P.p.protected_ + f) =
                  pr[0] | (uint32_t)pr[1] << 8 | (uint32_t)pr[2] << 16 | (uint32_t)pr[3] << 24;
              *reinterpret_cast<uint32_t *>(P.p.fresh + f) = 0u;
            } else {
              for (int e = 0; e < 4 && j + e < C; ++e) {
                P.p.metric[f + e] = mx[e];
                P.p.logical[f + e] = j + e;
                P.p.protected_[f + e] = pr[e];
                P.p.fresh[f + e] = 0;
              }
            }
          }
        }
        named_sync(1, 32 * kPEW);  // rs / tab_s are refilled by the next layer
        if (P.trace && et == 0) P.trace[((int64_t)blockIdx.x * P.nl + lp) * 8 + 5] = gtimer();
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

// The pool as {64 elems, rows = blocks * 16, D/64 atoms}, box {64, 16, 1}
// SWIZZLE_128B: one 16-row, 64-column slice of a staged K tile per store.
bool make_pool_store_map(CUtensorMap *map, const void *base, int64_t rows, int D) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(D / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, 128};
  cuuint32_t box[3] = {64, 16, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
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
int run_persist(const kvc_pool *pool, const kvc_window_args *a, const WinParams &W, int nl, cudaStream_t s) {
  constexpr int kS = 512 / N;
  if (a->pool > 1023 || !W.bar_cnt) return KVC_ERR_UNSUPPORTED;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  // one CTA per SM: it owns all 512 TMEM columns
  int cph = nsm / W.H;
  if (cph > W.tiles_per_head) cph = W.tiles_per_head;
  if (cph < 1) return KVC_ERR_UNSUPPORTED;
  const int ntiles_max = (W.tiles_per_head + cph - 1) / cph;
  // scores of a CTA's tiles fit in TMEM: one pass; else stream each layer twice
  const bool recomp = ntiles_max > kS;
  if (recomp && ntiles_max > 2 * kPEW * N * 16 / kTileKeys) return KVC_ERR_UNSUPPORTED;  // phase C table stage
  auto fn = recomp ? k_window_persist<N, D, true> : k_window_persist<N, D, false>;
  // phase C installs four contiguous slots at a time and stages the table slice in 2*kPEW*N ints
  if (a->seq_row >= 0 && (pool->block_size % 4 != 0 || ntiles_max * kTileKeys / pool->block_size > 2 * kPEW * N))
    return KVC_ERR_UNSUPPORTED;
  const int smem = persist_smem<N, D>(a->pool, ntiles_max);
  if (smem > 227 * 1024) return KVC_ERR_UNSUPPORTED;
  static bool configured[2] = {false, false};
  if (!configured[recomp]) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured[recomp] = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPThreads, smem);
  if (per_sm < 1) return KVC_ERR_UNSUPPORTED;
  CUtensorMap tmK, tmQ, tmP;
  if (!make_map3(&tmK, a->k, (int64_t)nl * W.H * W.L, D, kTileKeys)) return KVC_ERR_CUDA;
  if (!make_map(&tmQ, a->q_win, (int64_t)nl * a->num_query_heads * W.wq, D, N)) return KVC_ERR_CUDA;
  tmP = tmK;  // unused unless write_k
  if (a->write_k && !make_pool_store_map(&tmP, pool->k_cache, (int64_t)pool->num_blocks * 16, D)) return KVC_ERR_CUDA;
  PersistParams P;
  P.L = W.L; P.Lp = (W.L + 3) & ~3; P.H = W.H; P.RW = W.RW; P.wq = W.wq; P.start = W.start; P.nl = nl; P.n_q = a->num_query_heads;
  P.tiles_per_head = W.tiles_per_head; P.cph = cph;
  P.rs_len = persist_rs_len(ntiles_max, a->pool);
  P.scale = W.scale; P.agg = W.agg;
  P.partial = W.partial; P.raw = W.raw; P.bar_cnt = W.bar_cnt;
  P.p = *pool;
  P.row = a->seq_row; P.layer0 = a->layer; P.pool = a->pool; P.protect = a->protect_window;
  P.out = a->metrics_out;
  P.out_layer_stride = a->out_layer_stride;
  P.trace = nullptr;
  P.dbg = getenv("KVC_K2_DBG") ? atoi(getenv("KVC_K2_DBG")) : 0;
  P.write_k = a->write_k ? 1 : 0;
  static const bool trace = getenv("KVC_K2_TRACE") != nullptr;
  if (trace) cudaMalloc(&P.trace, (size_t)W.H * cph * nl * 8 * 8);
  cudaMemsetAsync(W.bar_cnt, 0, W.H * sizeof(int), s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(W.H * cph);
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: per-head barriers
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int rc = cudaLaunchKernelEx(&cfg, fn, tmK, tmQ, tmP, P) == cudaSuccess ? KVC_OK : KVC_ERR_CUDA;
  if (trace) {
    // debug: per layer, average over CTAs of each phase's duration (us), relative to the CTA's A start
    const int G = W.H * cph;
    unsigned long long *h = (unsigned long long *)malloc((size_t)G * nl * 64);
    cudaStreamSynchronize(s);
    cudaMemcpy(h, P.trace, (size_t)G * nl * 64, cudaMemcpyDeviceToHost);
    unsigned long long t00 = ~0ull;
    for (int c = 0; c < G; ++c) t00 = h[(size_t)c * nl * 8] < t00 ? h[(size_t)c * nl * 8] : t00;
    for (int l = 0; l < nl; ++l) {
      double acc[8] = {0};
      for (int c = 0; c < G; ++c)
        for (int k = 0; k < 8; ++k) acc[k] += (double)(h[((size_t)c * nl + l) * 8 + k] - t00) / 1e3 / G;
      // per head: spread of the A-finish times and barrier exit minus the last arrival
      double skew = 0, lat = 0;
      for (int hd = 0; hd < W.H; ++hd) {
        double mn = 1e30, mx = 0, bx = 0;
        for (int c = hd * cph; c < (hd + 1) * cph; ++c) {
          const double a1 = (double)(h[((size_t)c * nl + l) * 8 + 1] - t00) / 1e3;
          const double b1 = (double)(h[((size_t)c * nl + l) * 8 + 2] - t00) / 1e3;
          mn = a1 < mn ? a1 : mn; mx = a1 > mx ? a1 : mx; bx += b1 / cph;
        }
        skew += (mx - mn) / W.H; lat += (bx - mx) / W.H;
      }
      fprintf(stderr, "[k2 trace] layer %2d: A0 %.2f A1 %.2f bar %.2f B %.2f C(next) %.2f | tma_first %.2f mma_last %.2f | A1 skew %.2f bar-lastA1 %.2f\n", l,
              acc[0], acc[1], acc[2], acc[3], acc[5], acc[6], acc[7], skew, lat);
    }
    // per CTA index within a head: mean A1 relative to the head's earliest A1 (layers >= 1)
    for (int ci = 0; ci < cph; ++ci) {
      double d = 0;
      for (int l = 1; l < nl; ++l)
        for (int hd = 0; hd < W.H; ++hd) {
          double mn = 1e30;
          for (int c = hd * cph; c < (hd + 1) * cph; ++c) {
            const double a1 = (double)(h[((size_t)c * nl + l) * 8 + 1] - t00) / 1e3;
            mn = a1 < mn ? a1 : mn;
          }
          d += ((double)(h[((size_t)(hd * cph + ci) * nl + l) * 8 + 1] - t00) / 1e3 - mn) / ((nl - 1) * W.H);
        }
      fprintf(stderr, "[k2 trace] cidx %2d tiles %d: A1 - head min %.2f us\n", ci,
              (int)((int64_t)(ci + 1) * W.tiles_per_head / cph - (int64_t)ci * W.tiles_per_head / cph), d);
    }
    free(h);
    cudaFree(P.trace);
  }
  return rc;
}

template <int N, int D>
int run_window(const kvc_pool *pool, const kvc_window_args *a, WinParams &P, cudaStream_t s) {
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
  P.raw = sc.take<float>((int64_t)2 * H * ((a->L + 3) & ~3));  // two layers in flight (persistent kernel)
  P.bar_cnt = sc.take<int>(2 * H);
  if (!P.partial || !P.raw) return KVC_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const int nl = a->n_layers > 1 ? a->n_layers : 1;
  if (a->layer < 0 || (a->seq_row >= 0 && a->layer + nl > pool->num_layers)) return KVC_ERR_INVALID;
  static int twopass = -1;  // KVC_K2_TWOPASS=1: per-layer two-pass kernels (experiments)
  if (twopass < 0) {
    const char *e = getenv("KVC_K2_TWOPASS");
    twopass = (e && atoi(e) == 1) ? 1 : 0;
  }
  // persistent kernel over all layers when the layers are packed back to back
  const bool packed = nl == 1 || (a->k_layer_stride == (int64_t)H * a->L * D &&
                                  a->q_layer_stride == (int64_t)a->num_query_heads * P.wq * D);
  if (a->write_k && (a->seq_row < 0 || !pool->k_cache || pool->block_size != 16 || twopass || !packed || D > 128))
    return KVC_ERR_UNSUPPORTED;
  if (!twopass && packed && D <= 128) {
    int rc = KVC_ERR_UNSUPPORTED;
    if (N == 32 && D == 64) rc = run_persist<32, 64>(pool, a, P, nl, s);
    else if (N == 32 && D == 128) rc = run_persist<32, 128>(pool, a, P, nl, s);
    else if (N == 64 && D == 64) rc = run_persist<64, 64>(pool, a, P, nl, s);
    else if (N == 64 && D == 128) rc = run_persist<64, 128>(pool, a, P, nl, s);
    if (rc != KVC_ERR_UNSUPPORTED || a->write_k) return rc;  // write_k: the per-layer kernels do not store K
  }
  // otherwise one layer at a time, two passes: the layer's K (64 MB at
  // Llama-8B shapes) stays in L2 between the statistics and the metric pass
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
