// KVC-full prefill metric on tcgen05 tensor cores.
//
// Reference: full_metrics (pkg/src/pagedkv/metrics.py:92-109) over the causal
// softmax of gqa_attention (attention.py:62-89): for key j of KV head h_k,
//   M[h_k, j] = sum_{h in group(h_k)} sum_{i >= j + v, i < L} f(A[h, i, j]),
//   A[h, i, :] = softmax(q_{h,i} . K[:i+1]^T / sqrt(d)),  f = x (L1) or x^2 (L2).
// No pooling, no protection.  This is the only compute-bound contraction of
// the path (2 * L^2/2 * d * 2 flops per query head), so both passes run on
// tcgen05 with TMA-staged SW128 operands and fp32 accumulators in TMEM:
//   F1 k_full_stats:  S = Q_tile (128 rows) . K_tile^T over the causal key
//                     tiles; TMEM lane = query row, so each epilogue thread
//                     keeps its row's online (max, sum exp2) -> c_i = m_i +
//                     log2(l_i), i.e. A[h,i,j] = exp2(s_ij - c_i).
//   F2 k_full_colsum: S^T = K_tile (128 keys) . Q_tile^T for the r heads of
//                     the group and every query tile with rows >= j0 + v;
//                     TMEM lane = key, so each thread sums f(exp2(s - c_i))
//                     down its own column - no cross-lane reduction.
// Both passes issue one exp2 per score (MUFU) next to 2*d MMA flops.
#include <cuda.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc.cuh"

using namespace kvc;

namespace {

constexpr int kT = 128;        // rows / keys per tile
// warp 0 TMA, warp 1 MMA, 8 epilogue warps: two per TMEM lane quadrant, each
// taking half of a tile's 128 columns (more exp2 in flight per SM)
constexpr int kEpiW = 8;
constexpr int kFThreads = 64 + 32 * kEpiW;

template <int D>
constexpr int full_stages() { return D >= 128 ? 2 : 4; }  // 2 CTAs per SM (2 x 256 TMEM columns)

struct FullParams {
  int L, n_q, H, r, v;  // v = excluded query window
  int nt;               // tiles along L
  float scale;          // log2(e) / sqrt(d)
  int agg;              // 1 L1, 2 L2
  float *cst;           // [n_q][nt*128] per-row log2 normalisers x f's power (F1 out, F2 in)
  float *out;           // [H][L] metrics
};

// idesc for kind::f16: D f32, A/B bf16, K-major both, N = 128, M = 128
constexpr uint32_t kIdesc128 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kT >> 3) << 17) | ((uint32_t)(kT >> 4) << 24);

// One online (max, sum exp2) element, lazy rescale, branch-free.
__device__ __forceinline__ void lse_elem(float &m, float &z, float s) {
  const bool up = s > m;
  const float e = ex2_approx(up ? m - s : s - m);
  z = up ? fmaf(z, e, 1.f) : z + e;
  m = up ? s : m;
}

// Issue the D/16 MMAs of one 128x128 tile pair (both operands K-major SW128,
// smem laid out [atom][128 rows][128 B]).
template <int D>
__device__ __forceinline__ void mma_tile(uint32_t tmem_d, uint32_t abase, uint32_t bbase) {
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    const int atom = kk / 4, sub = kk % 4;
    mma_bf16(tmem_d, sw128_desc(abase + atom * kT * 128 + sub * 32), sw128_desc(bbase + atom * kT * 128 + sub * 32),
             kIdesc128, kk > 0 ? 1u : 0u);
  }
}

// ---------------------------------------------------------------------------
// F1: row statistics.  CTA = (query tile, query head), heaviest tiles first.
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kFThreads, 2)
    k_full_stats(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK, const FullParams P) {
  constexpr int kStages = full_stages<D>();
  constexpr int kTileBytes = kT * D * 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *qbuf = smem;
  uint8_t *ring = smem + kTileBytes;
  uint64_t *bars = reinterpret_cast<uint64_t *>(ring + kStages * kTileBytes);
  uint64_t *full = bars, *empty = full + kStages, *tfull = empty + kStages, *tempty = tfull + 2, *qfull = tempty + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(qfull + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qt = P.nt - 1 - (int)blockIdx.x;  // heavy (long causal range) first
  const int h = blockIdx.y;
  const int hk = h / P.r;
  const int ntk = qt + 1;  // causal key tiles

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 32 * kEpiW); }
    mbar_init(qfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(qfull, kTileBytes);
      tma_load_3d(qbuf, &tmQ, 0, h * P.L + qt * kT, 0, qfull);
      for (int t = 0; t < ntk; ++t) {
        const int s = t % kStages;
        if (t >= kStages) mbar_wait(&empty[s], ((t / kStages) - 1) & 1);
        mbar_expect_tx(&full[s], kTileBytes);
        tma_load_3d(ring + s * kTileBytes, &tmK, 0, hk * P.L + t * kT, 0, &full[s]);
      }
    }
  } else if (warp == 1) {
    mbar_wait(qfull, 0);
    for (int t = 0; t < ntk; ++t) {
      const int s = t % kStages, acc = t & 1;
      mbar_wait(&full[s], (t / kStages) & 1);
      if (t >= 2) mbar_wait(&tempty[acc], ((t >> 1) - 1) & 1);
      tc_fence_after();
      if (lane == 0) {
        mma_tile<D>(tmem + acc * kT, smem_u32(qbuf), smem_u32(ring + s * kTileBytes));
        mma_commit(&empty[s]);
        mma_commit(&tfull[acc]);
      }
      __syncwarp();
    }
  } else {
    const int quad = warp & 3, half = (warp - 2) / 4;
    const int row = quad * 32 + lane;
    const int i = qt * kT + row;  // query position
    // four independent (max, sum) chains per thread (columns e % 4)
    float m[4] = {-1e30f, -1e30f, -1e30f, -1e30f}, z[4] = {0.f, 0.f, 0.f, 0.f};
    for (int t = 0; t < ntk; ++t) {
      const int acc = t & 1;
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      const bool diag = t == qt;
#pragma unroll
      for (int c = 0; c < kT / 64; ++c) {
        const int col0 = half * (kT / 2) + c * 32;
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + acc * kT + col0, v);
        if (!diag) {
          // chunk max first (one FMNMX per score), one rescale per chunk and
          // chain, then exp2 + add per score: ~4 instructions per score
          float cmax[4] = {v[0], v[1], v[2], v[3]};
#pragma unroll
          for (int e = 4; e < 32; ++e) cmax[e & 3] = fmaxf(cmax[e & 3], v[e]);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float mn = fmaxf(m[q], cmax[q] * P.scale);
            z[q] *= ex2_approx(m[q] - mn);
            m[q] = mn;
          }
#pragma unroll
          for (int e = 0; e < 32; ++e) z[e & 3] += ex2_approx(fmaf(v[e], P.scale, -m[e & 3]));
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int j = t * kT + col0 + e;
            lse_elem(m[e & 3], z[e & 3], (j <= i) ? v[e] * P.scale : -INFINITY);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
    // merge the chains, then the two column halves of the row through smem
    float mm = fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
    float zz = z[0] * ex2_approx(m[0] - mm) + z[1] * ex2_approx(m[1] - mm) + z[2] * ex2_approx(m[2] - mm) +
               z[3] * ex2_approx(m[3] - mm);
    float2 *xs = reinterpret_cast<float2 *>(ring);  // the ring is idle now (all MMAs consumed)
    if (half == 1) xs[row] = make_float2(mm, zz);
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kEpiW) : "memory");
    if (half == 0) {
      const float2 o = xs[row];
      const float mn = fmaxf(mm, o.x);
      zz = zz * ex2_approx(mm - mn) + o.y * ex2_approx(o.x - mn);
      // stored pre-multiplied by f's power (2 for L2): F2 computes exp2(pow*s - cst)
      if (i < P.L) P.cst[(int64_t)h * P.nt * kT + i] = (P.agg == 2 ? 2.f : 1.f) * (mn + __log2f(zz));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// ---------------------------------------------------------------------------
// F2: column sums.  CTA = (key tile, KV head), heaviest (earliest) first; the
// stream is the group's r query heads x query tiles with rows >= j0 + v.
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kFThreads, 2)
    k_full_colsum(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK, const FullParams P) {
  constexpr int kStages = full_stages<D>();
  constexpr int kTileBytes = kT * D * 2;
  constexpr int kStageBytes = kTileBytes + 1024;  // Q tile + its rows' c_i (keeps stages 1024-aligned)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *kbuf = smem;
  uint8_t *ring = smem + kTileBytes;  // stage s: Q tile at s*kStageBytes (1024-aligned), c_i after it
  uint64_t *bars = reinterpret_cast<uint64_t *>(ring + kStages * kStageBytes);
  uint64_t *full = bars, *empty = full + kStages, *tfull = empty + kStages, *tempty = tfull + 2, *kfull = tempty + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(kfull + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int kt = blockIdx.x;
  const int hk = blockIdx.y;
  const int j0 = kt * kT;
  const int qt0 = min(P.nt, (j0 + P.v) / kT);
  const int nq_t = P.nt - qt0;           // query tiles per head
  const int nwork = P.r * nq_t;          // (head, query tile) pairs

  if (threadIdx.x == 0) {
    // empty[s]: all 128 epilogue threads have read the stage's c_i (the MMA's
    // read of its Q tile completed before tfull)
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 32 * kEpiW); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 32 * kEpiW); }
    mbar_init(kfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && nwork > 0) {
      mbar_expect_tx(kfull, kTileBytes);
      tma_load_3d(kbuf, &tmK, 0, hk * P.L + j0, 0, kfull);
      for (int w = 0; w < nwork; ++w) {
        const int hq = hk * P.r + w / nq_t, qt = qt0 + w % nq_t;
        const int s = w % kStages;
        if (w >= kStages) mbar_wait(&empty[s], ((w / kStages) - 1) & 1);
        mbar_expect_tx(&full[s], kTileBytes + kT * 4);
        tma_load_3d(ring + s * kStageBytes, &tmQ, 0, hq * P.L + qt * kT, 0, &full[s]);
        // c_i of the tile's rows (the array is padded to whole tiles)
        bulk_g2s(ring + s * kStageBytes + kTileBytes, P.cst + (int64_t)hq * P.nt * kT + qt * kT, kT * 4, &full[s],
                 policy_evict_first());
      }
    }
  } else if (warp == 1) {
    if (nwork > 0) {
      mbar_wait(kfull, 0);
      for (int w = 0; w < nwork; ++w) {
        const int s = w % kStages, acc = w & 1;
        mbar_wait(&full[s], (w / kStages) & 1);
        if (w >= 2) mbar_wait(&tempty[acc], ((w >> 1) - 1) & 1);
        tc_fence_after();
        if (lane == 0) {
          mma_tile<D>(tmem + acc * kT, smem_u32(kbuf), smem_u32(ring + s * kStageBytes));
          mma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else {
    const int quad = warp & 3, half = (warp - 2) / 4;
    const int key = quad * 32 + lane;
    const int j = j0 + key;
    const float sc = P.agg == 2 ? 2.f * P.scale : P.scale;
    float acc_sum = 0.f, acc_b = 0.f;  // two FADD chains
    for (int w = 0; w < nwork; ++w) {
      const int s = w % kStages, acc = w & 1;
      const int qt = qt0 + w % nq_t;
      mbar_wait(&tfull[acc], (w >> 1) & 1);
      tc_fence_after();
      const float *cs = reinterpret_cast<const float *>(ring + s * kStageBytes + kTileBytes);
      // every row of the tile is >= j + v and < L: no masks
      const bool inner = qt * kT >= j0 + kT - 1 + P.v && qt * kT + kT <= P.L;
#pragma unroll
      for (int c = 0; c < kT / 64; ++c) {
        const int col0 = half * (kT / 2) + c * 32;
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + acc * kT + col0, v);
        if (inner) {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            acc_sum += ex2_approx(fmaf(v[e], sc, -cs[col0 + e]));
            acc_b += ex2_approx(fmaf(v[e + 1], sc, -cs[col0 + e + 1]));
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int i = qt * kT + col0 + e;
            const float f = ex2_approx(fmaf(v[e], sc, -cs[col0 + e]));
            acc_sum += (i >= j + P.v && i < P.L) ? f : 0.f;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      mbar_arrive(&empty[s]);
    }
    // the two halves of the key's query rows: sum through smem (ring idle now)
    float *xs = reinterpret_cast<float *>(kbuf);
    acc_sum += acc_b;
    if (half == 1) xs[key] = acc_sum;
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kEpiW) : "memory");
    if (half == 0 && j < P.L) P.out[(int64_t)hk * P.L + j] = acc_sum + xs[key];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 3-D view {64 elems, rows, D/64 atoms} of a [rows][D] bf16 array, 128-row box.
bool tile_map(CUtensorMap *map, const void *base, int64_t rows, int D) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(D / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)kT, (cuuint32_t)(D / 64)};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
int run_full(const kvc_full_args *a, FullParams &P, cudaStream_t s) {
  CUtensorMap tmQ, tmK;
  if (!tile_map(&tmQ, a->q, (int64_t)a->num_query_heads * a->L, D)) return KVC_ERR_CUDA;
  if (!tile_map(&tmK, a->k, (int64_t)P.H * a->L, D)) return KVC_ERR_CUDA;
  constexpr int kTileBytes = kT * D * 2;
  const int smem1 = kTileBytes + full_stages<D>() * kTileBytes + 512 + 1024;
  const int smem2 = kTileBytes + full_stages<D>() * (kTileBytes + 1024) + 512 + 1024;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_full_stats<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1);
    cudaFuncSetAttribute(k_full_colsum<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    configured = true;
  }
  k_full_stats<D><<<dim3(P.nt, P.n_q), kFThreads, smem1, s>>>(tmQ, tmK, P);
  k_full_colsum<D><<<dim3(P.nt, P.H), kFThreads, smem2, s>>>(tmQ, tmK, P);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

}  // namespace

extern "C" int kvc_full_metric(const kvc_pool *pool, const kvc_full_args *a, void *stream) {
  if (!pool || !a || !a->q || !a->k || !a->metrics_out || a->L < 1 || a->excluded < 0) return KVC_ERR_INVALID;
  const int H = pool->num_kv_heads, D = pool->head_dim;
  if (H < 1 || a->num_query_heads % H) return KVC_ERR_INVALID;
  if (D != 64 && D != 128) return KVC_ERR_UNSUPPORTED;
  FullParams P;
  P.L = a->L;
  P.n_q = a->num_query_heads;
  P.H = H;
  P.r = a->num_query_heads / H;
  P.v = a->excluded;
  P.nt = (a->L + kT - 1) / kT;
  P.scale = 1.4426950408889634f / sqrtf((float)D);
  P.agg = a->aggregation == 2 ? 2 : 1;
  Scratch sc(pool);
  P.cst = sc.take<float>((int64_t)P.n_q * P.nt * kT);  // rows padded to whole tiles
  P.out = a->metrics_out;
  if (!P.cst) return KVC_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  // padded rows (>= L) must read as +inf normalisers: exp2(s - inf) = 0
  cudaMemsetAsync(P.cst, 0x7f, (size_t)P.n_q * P.nt * kT * 4, s);  // 0x7f7f7f7f: a huge finite value
  return D == 64 ? run_full<64>(a, P, s) : run_full<128>(a, P, s);
}
