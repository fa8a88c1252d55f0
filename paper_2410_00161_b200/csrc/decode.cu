// K1: paged GQA decode over ragged per-KV-head block tables, with the new
// token's append and the eviction-metric accumulation fused in.
//
// Reference: paged_attention (pkg/src/pagedkv/attention.py:92-127) gathers a
// head's C live KVs in table order, softmaxes q_group.K^T / sqrt(d) and
// returns out = P.V plus the (r, C) weights; accumulate_decode
// (metrics.py:189-211) then adds sum_h f(p_hj) to each key's metric; the
// engine appends the step's K/V (cache.py:163-184, metrics.py:153-158)
// before attending (engine.py:426-444).
//
// Design (one launch per layer, grid = splits x kv_heads x batch):
//  * a thread-block CLUSTER of `splits` CTAs owns one (seq, kv_head); CTA i
//    takes a block-aligned chunk of the head's positions;
//  * each warp streams its 16-token KV blocks (b*d*2 bytes, 4 KB at d=128)
//    into a private 4-stage shared-memory ring with cp.async.bulk (TMA
//    engine) completing on mbarriers; 16-byte vector LDS, fp32 math;
//  * pass A computes all raw scores of the chunk into shared memory; the
//    cluster exchanges per-head maxima through DSMEM; p = exp2(s - M) is
//    formed in place; pass B streams V and accumulates P.V;
//  * a second DSMEM exchange yields the softmax denominators Z_h, after
//    which every CTA folds f(p/Z) into the metric of its own slots (each
//    slot has exactly one owner: no atomics) and rank 0 writes the output.
//  The scores never leave shared memory, so the fused metric costs only its
//  own 8 B/key read-modify-write.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;
using namespace kvc;

int kvc_decode_mma(const kvc_pool *pool, const kvc_decode_args *a, int splits, int chunk, cudaStream_t s);

namespace {

constexpr int kWarps = 4;
constexpr int kStages = 4;
constexpr int kThreads = kWarps * 32;

struct DecodeParams {
  kvc_pool p;
  const int32_t *rows;
  int layer;
  int r;  // runtime group size (<= RMAX)
  const uint16_t *q;
  const uint16_t *k_new;
  const uint16_t *v_new;
  void *out;
  int out_f32;
  float *rows_out;
  int64_t rows_stride;
  int metric_mode;
  int append_fresh;
  int chunk;  // positions per CTA, multiple of block_size
  int splits;
  float q_scale;  // log2(e) / sqrt(d)
};

struct SmemLayout {
  int ring_bytes, ring_off, bar_off, scores_off, cta_o_off, stat_off, total;
};

template <int D, int RMAX>
__host__ __device__ inline SmemLayout smem_layout(int block_size, int chunk) {
  SmemLayout L;
  const int blk_bytes = block_size * D * 2;
  int ring = kWarps * kStages * blk_bytes;
  const int opart = kWarps * RMAX * D * 4;
  L.ring_bytes = ring > opart ? ring : opart;
  L.ring_off = 0;
  L.bar_off = (L.ring_bytes + 127) & ~127;
  L.scores_off = L.bar_off + kWarps * kStages * 8;
  L.scores_off = (L.scores_off + 15) & ~15;
  L.cta_o_off = L.scores_off + chunk * RMAX * 4;
  L.stat_off = L.cta_o_off + RMAX * D * 4;
  // stats: cta_max[RMAX], cta_sum[RMAX], red[kWarps][RMAX]
  L.total = L.stat_off + (2 + kWarps) * RMAX * 4 + 16;
  return L;
}

template <int D, int RMAX>
__global__ void __launch_bounds__(kThreads) k_paged_decode(const DecodeParams P) {
  constexpr int kVec = D >= 8 ? 8 : D;  // bf16 per lane and vector load (16 B; 8 B at d = 4)
  using VT = typename BfVec<kVec>::T;
  constexpr int LPT = D / kVec;      // lanes per token row
  constexpr int TPP = 32 / LPT;      // tokens per warp pass
  extern __shared__ __align__(128) uint8_t smem[];
  const kvc_pool &p = P.p;
  const int b = p.block_size;
  const int blk_bytes = b * D * 2;
  const SmemLayout L = smem_layout<D, RMAX>(b, P.chunk);
  uint8_t *ring = smem + L.ring_off;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L.bar_off);
  float *scores = reinterpret_cast<float *>(smem + L.scores_off);
  float *cta_o = reinterpret_cast<float *>(smem + L.cta_o_off);
  float *cta_max = reinterpret_cast<float *>(smem + L.stat_off);
  float *cta_sum = cta_max + RMAX;
  float *red = cta_sum + RMAX;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int split = blockIdx.x;
  const int head = blockIdx.y;
  const int bi = blockIdx.z;
  const int heads = p.num_kv_heads;
  const int n_q = heads * P.r;
  const int row = P.rows[bi];
  const int64_t hidx = head_index(p, row, P.layer, head);
  const int32_t *tab = head_table(p, hidx);
  const int c_old = p.ctx[hidx];
  const int nb = p.nblocks[hidx];
  const bool append = P.k_new != nullptr;
  const int cp = c_old + (append ? 1 : 0);
  const bool multi = P.splits > 1;

  // Uniform early exits (identical for every CTA of the cluster).  C beyond
  // the caller's max_ctx bound (chunks x splits) would be silently truncated:
  // reported as cache corruption instead.
  if (cp < 1 || (append && c_old >= nb * b) || cp > nb * b || cp > P.chunk * P.splits) {
    if (split == 0 && threadIdx.x == 0) {
      if (cp < 1) set_status(p.status, KVC_DEV_EMPTY_CONTEXT, (int32_t)hidx, 0);
      else if (append && c_old >= nb * b) set_status(p.status, KVC_DEV_ALLOCATION_ORDER, (int32_t)hidx, c_old);
      else set_status(p.status, KVC_DEV_CACHE_CORRUPTION, (int32_t)hidx, cp);
    }
    return;
  }

  const int t0 = split * P.chunk;
  const int t1 = min(cp, t0 + P.chunk);
  const int ntok = max(0, t1 - t0);
  const int blk0 = t0 / b;
  const int nblk = ntok > 0 ? (t1 - 1) / b - blk0 + 1 : 0;
  const int my_blocks = nblk > warp ? (nblk - warp + kWarps - 1) / kWarps : 0;

  // Barrier init.
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[warp * kStages + s], 1);
  }
  fence_barrier_init();
  __syncwarp();
  const uint64_t pol = policy_evict_first();

  // Query fragment: dims [sub*8, sub*8+8) of every head in the group.
  const int sub = lane % LPT;
  const int grp = lane / LPT;
  float qf[RMAX][kVec];
  bool bad_q = false;
#pragma unroll
  for (int h = 0; h < RMAX; ++h) {
    if (h < P.r) {
      const VT v = *reinterpret_cast<const VT *>(P.q + ((int64_t)bi * n_q + head * P.r + h) * D + sub * kVec);
      BfVec<kVec>::to_f32(v, qf[h]);
#pragma unroll
      for (int i = 0; i < kVec; ++i) {
        bad_q |= !isfinite(qf[h][i]);
        qf[h][i] *= P.q_scale;
      }
    } else {
#pragma unroll
      for (int i = 0; i < kVec; ++i) qf[h][i] = 0.f;
    }
  }
  if (bad_q && split == 0) set_status(p.status, KVC_DEV_NUMERIC, (int32_t)hidx, 0);

  uint8_t *my_ring = ring + warp * kStages * blk_bytes;
  uint64_t *my_bars = bars + warp * kStages;
  const uint16_t *kbase = reinterpret_cast<const uint16_t *>(p.k_cache);
  const uint16_t *vbase = reinterpret_cast<const uint16_t *>(p.v_cache);

  auto issue = [&](int use, int it, const uint16_t *base) {
    const int stage = use % kStages;
    const int blk = blk0 + warp + it * kWarps;
    const int64_t phys = tab[blk];
    mbar_expect_tx(&my_bars[stage], blk_bytes);
    bulk_g2s(my_ring + stage * blk_bytes, base + phys * b * D, blk_bytes, &my_bars[stage], pol);
  };

  int use = 0;  // ring uses issued so far by this warp (waits mirror it)
  // ---------------- pass A: scores ----------------
  if (lane == 0) {
    for (int it = 0; it < my_blocks && it < kStages; ++it) issue(it, it, kbase);
  }
  float mloc[RMAX];
#pragma unroll
  for (int h = 0; h < RMAX; ++h) mloc[h] = -INFINITY;

  for (int it = 0; it < my_blocks; ++it, ++use) {
    const int stage = use % kStages;
    mbar_wait(&my_bars[stage], (use / kStages) & 1);
    uint8_t *buf = my_ring + stage * blk_bytes;
    const int blk = blk0 + warp + it * kWarps;
    const int tb0 = blk * b;
    const int valid = min(b, t1 - tb0);
    if (append && c_old >= tb0 && c_old < tb0 + b) {
      // the step's new key: patch the staged row and persist it to the pool
      const int off = c_old - tb0;
      const int64_t slot = (int64_t)tab[blk] * b + off;
      const uint16_t *kn = P.k_new + ((int64_t)bi * heads + head) * D;
      const uint16_t *vn = P.v_new + ((int64_t)bi * heads + head) * D;
      for (int i = lane; i < D / kVec; i += 32) {
        const VT kv = reinterpret_cast<const VT *>(kn)[i];
        reinterpret_cast<VT *>(buf + off * D * 2)[i] = kv;
        reinterpret_cast<VT *>(const_cast<uint16_t *>(kbase) + slot * D)[i] = kv;
        reinterpret_cast<VT *>(const_cast<uint16_t *>(vbase) + slot * D)[i] = reinterpret_cast<const VT *>(vn)[i];
      }
      __syncwarp();
    }
    for (int tp = 0; tp < b; tp += TPP) {  // warp-uniform trip count (shuffles inside)
      const int t = tp + grp;
      float acc[RMAX];
#pragma unroll
      for (int h = 0; h < RMAX; ++h) acc[h] = 0.f;
      if (t < valid) {
        const VT kv = *reinterpret_cast<const VT *>(buf + t * D * 2 + sub * kVec * 2);
        float kf[kVec];
        BfVec<kVec>::to_f32(kv, kf);
#pragma unroll
        for (int h = 0; h < RMAX; ++h)
#pragma unroll
          for (int i = 0; i < kVec; ++i) acc[h] = fmaf(qf[h][i], kf[i], acc[h]);
      }
#pragma unroll
      for (int h = 0; h < RMAX; ++h) {
#pragma unroll
        for (int o = LPT / 2; o > 0; o >>= 1) acc[h] += __shfl_xor_sync(0xffffffffu, acc[h], o);
      }
      if (t < valid) {
        float *srow = scores + (tb0 - t0 + t) * RMAX;
#pragma unroll
        for (int h = 0; h < RMAX; ++h) {
          if (h < P.r) mloc[h] = fmaxf(mloc[h], acc[h]);
          if ((h % LPT) == sub) srow[h] = acc[h];
        }
      }
    }
    __syncwarp();
    if (lane == 0 && it + kStages < my_blocks) {
      fence_proxy_async();
      issue(use + kStages, it + kStages, kbase);
    }
  }
  // prefetch the first V blocks while the cluster agrees on the maxima
  if (lane == 0) {
    fence_proxy_async();
    for (int it = 0; it < my_blocks && it < kStages; ++it) issue(use + it, it, vbase);
  }
#pragma unroll
  for (int h = 0; h < RMAX; ++h) {
    float m = warp_max(mloc[h]);
    if (lane == 0) red[warp * RMAX + h] = m;
  }
  __syncthreads();
  if (threadIdx.x < RMAX) {
    float m = -INFINITY;
    for (int w = 0; w < kWarps; ++w) m = fmaxf(m, red[w * RMAX + threadIdx.x]);
    cta_max[threadIdx.x] = m;
  }
  cg::cluster_group cluster = cg::this_cluster();
  if (multi) cluster.sync(); else __syncthreads();
  float M[RMAX];
#pragma unroll
  for (int h = 0; h < RMAX; ++h) {
    float m = cta_max[h];
    if (multi) {
      for (int rk = 0; rk < P.splits; ++rk) {
        if (rk == split) continue;
        const float *peer = cluster.map_shared_rank(cta_max, rk);
        m = fmaxf(m, peer[h]);
      }
    }
    M[h] = m;
  }
  // p = exp2(s - M) in place, partial row sums
  float lsum[RMAX];
#pragma unroll
  for (int h = 0; h < RMAX; ++h) lsum[h] = 0.f;
  for (int t = threadIdx.x; t < ntok; t += kThreads) {
    float *srow = scores + t * RMAX;
#pragma unroll
    for (int h = 0; h < RMAX; ++h) {
      if (h < P.r) {
        const float e = exp2f(srow[h] - M[h]);
        srow[h] = e;
        lsum[h] += e;
      }
    }
  }
#pragma unroll
  for (int h = 0; h < RMAX; ++h) {
    float s = warp_sum(lsum[h]);
    if (lane == 0) red[warp * RMAX + h] = s;
  }
  __syncthreads();  // p visible to every warp; red complete
  if (threadIdx.x < RMAX) {
    float s = 0.f;
    for (int w = 0; w < kWarps; ++w) s += red[w * RMAX + threadIdx.x];
    cta_sum[threadIdx.x] = s;
  }

  // ---------------- pass B: P.V ----------------
  float acc[RMAX][kVec];
#pragma unroll
  for (int h = 0; h < RMAX; ++h)
#pragma unroll
    for (int i = 0; i < kVec; ++i) acc[h][i] = 0.f;
  for (int it = 0; it < my_blocks; ++it, ++use) {
    const int stage = use % kStages;
    mbar_wait(&my_bars[stage], (use / kStages) & 1);
    uint8_t *buf = my_ring + stage * blk_bytes;
    const int blk = blk0 + warp + it * kWarps;
    const int tb0 = blk * b;
    const int valid = min(b, t1 - tb0);
    if (append && c_old >= tb0 && c_old < tb0 + b) {
      const int off = c_old - tb0;
      const uint16_t *vn = P.v_new + ((int64_t)bi * heads + head) * D;
      for (int i = lane; i < D / kVec; i += 32)
        reinterpret_cast<VT *>(buf + off * D * 2)[i] = reinterpret_cast<const VT *>(vn)[i];
      __syncwarp();
    }
    for (int t = grp; t < valid; t += TPP) {
      const VT vv = *reinterpret_cast<const VT *>(buf + t * D * 2 + sub * kVec * 2);
      float vf[kVec];
      BfVec<kVec>::to_f32(vv, vf);
      const float *prow = scores + (tb0 - t0 + t) * RMAX;
#pragma unroll
      for (int h = 0; h < RMAX; ++h) {
        const float pw = h < P.r ? prow[h] : 0.f;
#pragma unroll
        for (int i = 0; i < kVec; ++i) acc[h][i] = fmaf(pw, vf[i], acc[h][i]);
      }
    }
    __syncwarp();
    if (lane == 0 && it + kStages < my_blocks) {
      fence_proxy_async();
      issue(use + kStages, it + kStages, vbase);
    }
  }
  // reduce across token groups (lanes sharing `sub`)
#pragma unroll
  for (int h = 0; h < RMAX; ++h)
#pragma unroll
    for (int i = 0; i < kVec; ++i)
#pragma unroll
      for (int o = LPT; o < 32; o <<= 1) acc[h][i] += __shfl_xor_sync(0xffffffffu, acc[h][i], o);
  __syncthreads();  // ring no longer in use by any warp
  float *opart = reinterpret_cast<float *>(ring);
  if (grp == 0) {
#pragma unroll
    for (int h = 0; h < RMAX; ++h)
#pragma unroll
      for (int i = 0; i < kVec; ++i) opart[(warp * RMAX + h) * D + sub * kVec + i] = acc[h][i];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < RMAX * D; e += kThreads) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += opart[w * RMAX * D + e];
    cta_o[e] = s;
  }
  if (multi) cluster.sync(); else __syncthreads();

  float Z[RMAX];
#pragma unroll
  for (int h = 0; h < RMAX; ++h) {
    float z = cta_sum[h];
    if (multi) {
      for (int rk = 0; rk < P.splits; ++rk) {
        if (rk == split) continue;
        z += cluster.map_shared_rank(cta_sum, rk)[h];
      }
    }
    Z[h] = z;
  }
  if (split == 0) {
    for (int e = threadIdx.x; e < P.r * D; e += kThreads) {
      const int h = e / D;
      float s = cta_o[e];
      if (multi) {
        for (int rk = 1; rk < P.splits; ++rk) s += cluster.map_shared_rank(cta_o, rk)[e];
      }
      const float o = s / Z[h];
      const int64_t oi = ((int64_t)bi * n_q + head * P.r) * D + e;
      if (P.out_f32) reinterpret_cast<float *>(P.out)[oi] = o;
      else reinterpret_cast<__nv_bfloat16 *>(P.out)[oi] = __float2bfloat16(o);
    }
  }
  // metric accumulation / row export over this CTA's positions
  float invZ[RMAX];
#pragma unroll
  for (int h = 0; h < RMAX; ++h) invZ[h] = 1.f / Z[h];
  if (P.metric_mode || P.rows_out) {
    for (int t = threadIdx.x; t < ntok; t += kThreads) {
      const int pos = t0 + t;
      const float *prow = scores + t * RMAX;
      float contrib = 0.f;
#pragma unroll
      for (int h = 0; h < RMAX; ++h) {
        if (h < P.r) {
          const float w = prow[h] * invZ[h];
          contrib += P.metric_mode == 2 ? w * w : w;
          if (P.rows_out)
            P.rows_out[(((int64_t)bi * heads + head) * P.r + h) * P.rows_stride + pos] = w;
        }
      }
      if (P.metric_mode) {
        const int64_t slot = (int64_t)tab[pos / b] * b + pos % b;
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
  if (append && !P.metric_mode && p.metric && threadIdx.x == 0 && c_old >= t0 && c_old < t1) {
    const int64_t slot = (int64_t)tab[c_old / b] * b + c_old % b;
    p.metric[slot] = 0.f;
    p.logical[slot] = c_old;
    p.protected_[slot] = 0;
    p.fresh[slot] = P.append_fresh ? 1 : 0;
  }
  if (multi) cluster.sync();  // peers' smem stays alive until rank 0 is done
  if (append && split == 0 && threadIdx.x == 0) p.ctx[hidx] = c_old + 1;
}

template <int D, int RMAX>
int launch_decode(const DecodeParams &P, int batch, cudaStream_t s) {
  const SmemLayout L = smem_layout<D, RMAX>(P.p.block_size, P.chunk);
  auto fn = k_paged_decode<D, RMAX>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    configured = true;
  }
  if (L.total > 227 * 1024) return KVC_ERR_UNSUPPORTED;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.splits, P.p.num_kv_heads, batch);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P.splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fn, P);
  return e == cudaSuccess ? KVC_OK : KVC_ERR_CUDA;
}

template <int D>
int dispatch_r(const DecodeParams &P, int batch, cudaStream_t s) {
  if (P.r <= 1) return launch_decode<D, 1>(P, batch, s);
  if (P.r <= 2) return launch_decode<D, 2>(P, batch, s);
  if (P.r <= 4) return launch_decode<D, 4>(P, batch, s);
  if (P.r <= 8) return launch_decode<D, 8>(P, batch, s);
  return KVC_ERR_UNSUPPORTED;
}

int rmax_of(int r) { return r <= 1 ? 1 : r <= 2 ? 2 : r <= 4 ? 4 : 8; }

// ---------------------------------------------------------------------------
// Small kernels: append, accumulate rows, clear fresh, prefill writes
// ---------------------------------------------------------------------------

__global__ void k_append(kvc_pool p, const int32_t *heads3, const uint16_t *k, const uint16_t *v,
                         int n, int fresh) {
  const int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (i >= n) return;
  const int64_t hidx = head_index(p, heads3[3 * i], heads3[3 * i + 1], heads3[3 * i + 2]);
  const int c = p.ctx[hidx];
  const int b = p.block_size, D = p.head_dim;
  if (c >= p.nblocks[hidx] * b) {
    if (lane == 0) set_status(p.status, KVC_DEV_ALLOCATION_ORDER, (int32_t)hidx, c);
    return;
  }
  const int64_t slot = (int64_t)head_table(p, hidx)[c / b] * b + c % b;
  uint16_t *kc = reinterpret_cast<uint16_t *>(p.k_cache) + slot * D;
  uint16_t *vc = reinterpret_cast<uint16_t *>(p.v_cache) + slot * D;
  for (int e = lane; e < D; e += 32) {
    kc[e] = k[(int64_t)i * D + e];
    vc[e] = v[(int64_t)i * D + e];
  }
  if (lane == 0) {
    if (p.metric) {  // on_append fused (metrics.py:153-158) when a store is bound
      p.metric[slot] = 0.f;
      p.logical[slot] = c;
      p.protected_[slot] = 0;
      p.fresh[slot] = fresh ? 1 : 0;
    }
    p.ctx[hidx] = c + 1;
  }
}

__global__ void k_accumulate_rows(kvc_pool p, int row, int layer, const float *rows, int r,
                                  int64_t stride, int mode) {
  const int head = blockIdx.y;
  const int64_t hidx = head_index(p, row, layer, head);
  const int c = p.ctx[hidx];
  const int b = p.block_size;
  const int32_t *tab = head_table(p, hidx);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < c; j += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int h = 0; h < r; ++h) {
      const float w = rows[((int64_t)head * r + h) * stride + j];
      s += mode == 2 ? w * w : w;
    }
    p.metric[(int64_t)tab[j / b] * b + j % b] += s;
  }
}

__global__ void k_clear_fresh_all(uint4 *fresh, int64_t n16, uint8_t *tail, int64_t ntail) {
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    fresh[i] = z;
  if (blockIdx.x == 0 && threadIdx.x < ntail) tail[threadIdx.x] = 0;
}

__global__ void k_clear_fresh_rows(kvc_pool p, const int32_t *rows, int n_rows) {
  const int hp = p.num_layers * p.num_kv_heads;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n_rows * hp) return;
  const int64_t hidx = (int64_t)rows[i / hp] * hp + i % hp;
  const int c = p.ctx[hidx];
  if (c < 1) return;
  const int b = p.block_size;
  const int64_t slot = (int64_t)head_table(p, hidx)[(c - 1) / b] * b + (c - 1) % b;
  p.fresh[slot] = 0;
}

// K/V scatter of a prompt: a warp copies one table block (b rows, contiguous
// on both sides: the prompt's rows [blk*b, blk*b + b) and the pool block),
// 16 bytes per lane, four chunks in flight; 32-bit index math per block.
// k_tail_only: V rows, and K rows of the partial last block only (K2 with
// write_k stores the whole blocks' K rows).
__global__ void __launch_bounds__(256) k_write_prefill_kv(kvc_pool p, int row, int layer0, const uint4 *k,
                                                          const uint4 *v, int L, int k_tail_only) {
  const int head = blockIdx.y;
  const int layer = layer0 + blockIdx.z;
  k += (int64_t)blockIdx.z * gridDim.y * L * (p.head_dim / 8);  // [layer][heads][L][d]
  v += (int64_t)blockIdx.z * gridDim.y * L * (p.head_dim / 8);
  const int64_t hidx = head_index(p, row, layer, head);
  const int b = p.block_size;
  const int vec = p.head_dim / 8;  // 16-byte chunks per row
  const int nblk = (L + b - 1) / b;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int32_t *tab = head_table(p, hidx);
  const uint4 *ks = k + (int64_t)head * L * vec;
  const uint4 *vs = v + (int64_t)head * L * vec;
  uint4 *kc = reinterpret_cast<uint4 *>(p.k_cache);
  uint4 *vc = reinterpret_cast<uint4 *>(p.v_cache);
  for (int bl = blockIdx.x * 8 + warp; bl < nblk; bl += gridDim.x * 8) {
    const int rows = min(b, L - bl * b);
    const int n = rows * vec;  // chunks of this block
    const uint4 *sk = ks + (int64_t)bl * b * vec, *sv = vs + (int64_t)bl * b * vec;
    const int64_t d0 = (int64_t)tab[bl] * b * vec;
    const bool with_k = !k_tail_only || rows < b;
    for (int c0 = 0; c0 < n; c0 += 4 * 32) {
      uint4 tk[4], tv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c < n) {
          if (with_k) tk[u] = __ldcs(sk + c);
          tv[u] = __ldcs(sv + c);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + u * 32 + lane;
        if (c < n) {
          if (with_k) kc[d0 + c] = tk[u];
          vc[d0 + c] = tv[u];
        }
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) p.ctx[hidx] = L;
}

__global__ void k_write_prompt_pass(kvc_pool p, int row, int layer, const float *metrics, int64_t stride,
                                    const uint8_t *prot, int L) {
  const int head = blockIdx.y;
  const int64_t hidx = head_index(p, row, layer, head);
  const int b = p.block_size;
  const int c = min(L, p.ctx[hidx]);
  const int32_t *tab = head_table(p, hidx);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < c; j += gridDim.x * blockDim.x) {
    const int64_t slot = (int64_t)tab[j / b] * b + j % b;
    p.metric[slot] = metrics[(int64_t)head * stride + j];
    p.logical[slot] = j;
    p.protected_[slot] = (prot && prot[j]) ? 1 : 0;
    p.fresh[slot] = 0;
  }
}

}  // namespace

extern "C" {

int kvc_paged_decode(const kvc_pool *pool, const kvc_decode_args *a, void *stream) {
  if (!pool || !a || a->batch < 0 || !a->q || !a->out || !a->seq_rows) return KVC_ERR_INVALID;
  if (a->batch == 0) return KVC_OK;
  const int H = pool->num_kv_heads;
  if (a->num_query_heads % H != 0) return KVC_ERR_INVALID;
  const int r = a->num_query_heads / H;
  const int D = pool->head_dim;
  const int b = pool->block_size;
  if (r < 1 || r > 8) return KVC_ERR_UNSUPPORTED;
  if ((a->k_new == nullptr) != (a->v_new == nullptr)) return KVC_ERR_INVALID;
  if (a->layer < 0 || a->layer >= pool->num_layers) return KVC_ERR_INVALID;
  if ((b * D * 2) % 16 != 0) return KVC_ERR_UNSUPPORTED;
  const int max_ctx = a->max_ctx > 0 ? a->max_ctx : 1;
  const int rm = rmax_of(r);
  // splits: enough CTAs to fill 148 SMs ~4 deep, >= 256 positions per CTA,
  // and a score buffer that fits shared memory.
  // tensor-core persistent fast path (block_size 16, d in {64,128,256}, r <= 8)
  {
    const int rc = kvc_decode_mma(pool, a, 0, 0, (cudaStream_t)stream);
    if (rc != KVC_ERR_UNSUPPORTED) return rc;
  }
  int splits = a->splits;
  if (splits <= 0) {
    const int64_t pairs = (int64_t)a->batch * H;
    splits = 1;
    while (splits < 16 && pairs * splits < 148 * 4 && (max_ctx + splits * 2 - 1) / (splits * 2) >= 256)
      splits *= 2;
  }
  auto chunk_for = [&](int sp) {
    int c = (max_ctx + sp - 1) / sp;
    return ((c + b - 1) / b) * b;
  };
  while (splits < 16 && chunk_for(splits) * rm * 4 > 96 * 1024) splits *= 2;
  if (splits > 16) return KVC_ERR_UNSUPPORTED;
  DecodeParams P;
  P.p = *pool;
  P.rows = a->seq_rows;
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
  P.chunk = chunk_for(splits);
  P.splits = splits;
  P.q_scale = 1.4426950408889634f / sqrtf((float)D);
  cudaStream_t s = (cudaStream_t)stream;
  switch (D) {
    case 4: return dispatch_r<4>(P, a->batch, s);
    case 8: return dispatch_r<8>(P, a->batch, s);
    case 16: return dispatch_r<16>(P, a->batch, s);
    case 32: return dispatch_r<32>(P, a->batch, s);
    case 64: return dispatch_r<64>(P, a->batch, s);
    case 128: return dispatch_r<128>(P, a->batch, s);
    case 256: return dispatch_r<256>(P, a->batch, s);
    default: return KVC_ERR_UNSUPPORTED;
  }
}

int kvc_append_kv(const kvc_pool *pool, const int32_t *heads, const void *k, const void *v, int32_t n,
                  int32_t fresh, void *stream) {
  if (!pool || n < 0 || (n && (!heads || !k || !v))) return KVC_ERR_INVALID;
  if (n == 0) return KVC_OK;
  k_append<<<(n + 3) / 4, 128, 0, (cudaStream_t)stream>>>(*pool, heads, (const uint16_t *)k,
                                                         (const uint16_t *)v, n, fresh);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

int kvc_accumulate_rows(const kvc_pool *pool, int32_t seq_row, int32_t layer, const float *rows, int32_t r,
                        int64_t rows_stride, int32_t metric_mode, void *stream) {
  if (!pool || !rows || r < 1 || metric_mode < 1 || metric_mode > 2) return KVC_ERR_INVALID;
  dim3 grid(8, pool->num_kv_heads);
  k_accumulate_rows<<<grid, 256, 0, (cudaStream_t)stream>>>(*pool, seq_row, layer, rows, r, rows_stride,
                                                            metric_mode);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

int kvc_clear_fresh(const kvc_pool *pool, const int32_t *seq_rows, int32_t n_rows, void *stream) {
  if (!pool) return KVC_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (!seq_rows) {
    const int64_t n = pool->num_blocks * pool->block_size;
    // fresh is a torch/cudaMalloc allocation: 256-byte aligned, uint4 stores
    k_clear_fresh_all<<<1184, 256, 0, s>>>(reinterpret_cast<uint4 *>(pool->fresh), n / 16,
                                            pool->fresh + (n / 16) * 16, n % 16);
  } else if (n_rows > 0) {
    const int64_t n = (int64_t)n_rows * pool->num_layers * pool->num_kv_heads;
    k_clear_fresh_rows<<<(int)((n + 255) / 256), 256, 0, s>>>(*pool, seq_rows, n_rows);
  }
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

static int write_prefill(const kvc_pool *pool, int32_t seq_row, int32_t layer, int32_t n_layers, const void *k,
                         const void *v, int32_t L, void *stream, int k_tail_only) {
  if (!pool || !k || !v || L < 0 || n_layers < 1 || pool->head_dim % 8 != 0 || pool->block_size < 1)
    return KVC_ERR_INVALID;
  if (layer < 0 || layer + n_layers > pool->num_layers) return KVC_ERR_INVALID;
  if (L == 0) return KVC_OK;
  const int nblk = (L + pool->block_size - 1) / pool->block_size;
  int gx = (nblk + 7) / 8;  // 8 warps per CTA, one block per warp
  const int H = pool->num_kv_heads > 0 ? pool->num_kv_heads : 1;
  int cap = 148 * 16 / (H * n_layers);
  if (cap < 1) cap = 1;
  if (gx > cap) gx = cap;
  dim3 grid(gx, pool->num_kv_heads, n_layers);
  k_write_prefill_kv<<<grid, 256, 0, (cudaStream_t)stream>>>(*pool, seq_row, layer, (const uint4 *)k,
                                                             (const uint4 *)v, L, k_tail_only);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

int kvc_write_prefill_kv_layers(const kvc_pool *pool, int32_t seq_row, int32_t layer, int32_t n_layers,
                                const void *k, const void *v, int32_t L, void *stream) {
  return write_prefill(pool, seq_row, layer, n_layers, k, v, L, stream, 0);
}

int kvc_write_prefill_v_layers(const kvc_pool *pool, int32_t seq_row, int32_t layer, int32_t n_layers,
                               const void *k, const void *v, int32_t L, void *stream) {
  if (pool && pool->block_size != 16) return KVC_ERR_INVALID;  // pairs with K2's 16-key block stores
  return write_prefill(pool, seq_row, layer, n_layers, k, v, L, stream, 1);
}

int kvc_write_prefill_kv(const kvc_pool *pool, int32_t seq_row, int32_t layer, const void *k, const void *v,
                         int32_t L, void *stream) {
  return kvc_write_prefill_kv_layers(pool, seq_row, layer, 1, k, v, L, stream);
}

int kvc_write_prompt_pass(const kvc_pool *pool, int32_t seq_row, int32_t layer, const float *metrics,
                          int64_t metrics_stride, const uint8_t *protected_mask, int32_t L, void *stream) {
  if (!pool || !metrics || L < 0) return KVC_ERR_INVALID;
  if (L == 0) return KVC_OK;
  int gx = (L + 255) / 256;
  if (gx > 1184) gx = 1184;
  dim3 grid(gx, pool->num_kv_heads);
  k_write_prompt_pass<<<grid, 256, 0, (cudaStream_t)stream>>>(*pool, seq_row, layer, metrics, metrics_stride,
                                                              protected_mask, L);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

}  // extern "C"
