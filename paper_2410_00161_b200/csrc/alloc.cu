// K0: on-device block allocator + frees (smallest free ids first).
//
// Reference semantics (pkg/src/pagedkv/block_manager.py): the free pool is a
// min-heap, so every allocation hands out the smallest free ids, and a batch
// request is served in a fixed request order (prefill: layer-major heads,
// per_head consecutive ids, :56-72; decode: sorted(seq), (layer, head),
// :74-97).  Equivalently the k-th request receives the k-th smallest free
// id.  Here the free pool is a byte flag per block plus a free count per
// 1024-block tile; an allocation is (1) an exclusive scan of the tile counts,
// (2) per-tile block scans that hand the ids of rank < demand to their
// requests, (3) a bind pass that appends ids to the block tables.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"

using namespace kvc;

namespace {

constexpr int kTile = KVC_FREE_TILE;

__global__ void k_init_tiles(kvc_pool p) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  int nt = num_tiles(&p);
  if (t < nt) {
    int64_t lo = (int64_t)t * kTile;
    int64_t hi = lo + kTile < p.num_blocks ? lo + kTile : p.num_blocks;
    p.free_tile[t] = (int32_t)(hi - lo);
  }
}

__global__ void k_fill_u8(uint8_t *ptr, int64_t n, uint8_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    ptr[i] = v;
}

// One CTA: scan tile free counts -> tile_prefix; check demand (all-or-nothing).
// demand_in: device scalar (or -1 and use demand_host).
__global__ void __launch_bounds__(1024) k_tile_scan(kvc_pool p, const int64_t *demand_dev,
                                                   int64_t demand_host, int64_t *demand_eff,
                                                   int64_t *tile_prefix) {
  using Scan = cub::BlockScan<int64_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t carry;
  int nt = num_tiles(&p);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nt; base += 1024) {
    int t = base + threadIdx.x;
    int64_t v = t < nt ? p.free_tile[t] : 0;
    int64_t excl, total;
    Scan(tmp).ExclusiveSum(v, excl, total);
    if (t < nt) tile_prefix[t] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int64_t demand = demand_dev ? *demand_dev : demand_host;
    if (demand > carry) {
      set_status(p.status, KVC_DEV_PREEMPTION, (int32_t)(demand - carry), 0);
      *demand_eff = 0;
    } else {
      *demand_eff = demand;
    }
  }
}

// Per tile: hand out free ids of global rank < demand.
__global__ void __launch_bounds__(256) k_tile_take(kvc_pool p, const int64_t *demand_eff,
                                                  const int64_t *tile_prefix, int32_t *ids) {
  using Scan = cub::BlockScan<int32_t, 256>;
  __shared__ typename Scan::TempStorage tmp;
  const int t = blockIdx.x;
  const int64_t demand = *demand_eff;
  const int64_t base_rank = tile_prefix[t];
  if (base_rank >= demand || p.free_tile[t] == 0) return;
  const int64_t lo = (int64_t)t * kTile;
  constexpr int kPer = kTile / 256;  // 4 blocks per thread, contiguous
  int32_t f[kPer];
  int32_t cnt = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    int64_t blk = lo + threadIdx.x * kPer + i;
    f[i] = (blk < p.num_blocks) ? p.free_flag[blk] : 0;
    cnt += f[i];
  }
  int32_t excl;
  int32_t total;
  Scan(tmp).ExclusiveSum(cnt, excl, total);
  int32_t taken_local = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    if (f[i]) {
      int64_t rank = base_rank + excl;
      if (rank < demand) {
        int64_t blk = lo + threadIdx.x * kPer + i;
        ids[rank] = (int32_t)blk;
        p.free_flag[blk] = 0;
        ++taken_local;
      }
      ++excl;
    }
  }
  using Red = cub::BlockReduce<int32_t, 256>;
  __shared__ typename Red::TempStorage rtmp;
  __syncthreads();
  int32_t taken = Red(rtmp).Sum(taken_local);
  if (threadIdx.x == 0) p.free_tile[t] -= taken;
}

// Prefill bind: head i (layer-major) gets ids[i*per_head .. +per_head).
__global__ void k_bind_runs(kvc_pool p, int32_t row, const int64_t *demand_eff,
                            const int32_t *ids, const int32_t *counts, const int64_t *offsets,
                            int32_t per_head) {
  if (*demand_eff <= 0) return;
  const int heads = p.num_layers * p.num_kv_heads;
  const int h = blockIdx.x;
  if (h >= heads) return;
  const int64_t hidx = (int64_t)row * heads + h;
  const int32_t n = counts ? counts[h] : per_head;
  const int64_t off = counts ? offsets[h] : (int64_t)h * per_head;
  const int32_t nb = p.nblocks[hidx];
  if (nb + n > p.max_blocks) {
    if (threadIdx.x == 0) set_status(p.status, KVC_DEV_CAPACITY, (int32_t)hidx, nb + n);
    return;
  }
  int32_t *tab = head_table(p, hidx);
  for (int j = threadIdx.x; j < n; j += blockDim.x) tab[nb + j] = ids[off + j];
  __syncthreads();
  if (threadIdx.x == 0) p.nblocks[hidx] = nb + n;
}

// Exclusive scan of per-head counts for kvc_alloc_heads (one CTA).
__global__ void __launch_bounds__(1024) k_scan_counts(const int32_t *counts, int n,
                                                     int64_t *offsets, int64_t *demand) {
  using Scan = cub::BlockScan<int64_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 1024) {
    int i = base + threadIdx.x;
    int64_t v = i < n ? counts[i] : 0;
    int64_t excl, total;
    Scan(tmp).ExclusiveSum(v, excl, total);
    if (i < n) offsets[i] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *demand = carry;
}

// Decode demand: heads (row order given, then layer-major) with C % b == 0.
// One CTA: head i (row-major over the batch rows, then layer x head) needs a
// block iff its C is a multiple of the block size; its rank is the
// exclusive count of needing heads before it (the reference's order).  Each
// thread takes 16 consecutive heads (16 independent C loads in flight), one
// block scan per 16K-head tile.
__global__ void __launch_bounds__(1024) k_decode_demand(kvc_pool p, const int32_t *rows, int n_rows,
                                                       int32_t *head_rank, int32_t *out_counts,
                                                       int64_t *demand) {
  constexpr int kPer = 16;
  using Scan = cub::BlockScan<int32_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int32_t carry;
  const int heads = p.num_layers * p.num_kv_heads;
  const int64_t total_heads = (int64_t)n_rows * heads;
  if (threadIdx.x == 0) carry = 0;
  for (int i = threadIdx.x; i < n_rows; i += blockDim.x) out_counts[i] = 0;
  __syncthreads();
  for (int64_t base = 0; base < total_heads; base += 1024 * kPer) {
    const int64_t i0 = base + (int64_t)threadIdx.x * kPer;
    uint32_t needm = 0;  // bit j: head i0 + j needs a block
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int64_t i = i0 + j;
      if (i < total_heads) {
        const int rix = (int)(i / heads);
        const int64_t hidx = (int64_t)rows[rix] * heads + (i % heads);
        needm |= ((p.ctx[hidx] % p.block_size) == 0 ? 1u : 0u) << j;
      }
    }
    int32_t excl, total;
    Scan(tmp).ExclusiveSum(__popc(needm), excl, total);
    const int32_t c0 = carry;
    int32_t rank = c0 + excl;
    int cur_r = -1, cur_n = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int64_t i = i0 + j;
      if (i < total_heads) {
        const bool need = (needm >> j) & 1u;
        head_rank[i] = need ? rank : -1;
        rank += need ? 1 : 0;
        const int rix = (int)(i / heads);
        if (rix != cur_r) {
          if (cur_n) atomicAdd(&out_counts[cur_r], cur_n);
          cur_r = rix;
          cur_n = 0;
        }
        cur_n += need ? 1 : 0;
      }
    }
    if (cur_n) atomicAdd(&out_counts[cur_r], cur_n);
    __syncthreads();
    if (threadIdx.x == 0) carry = c0 + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *demand = carry;
}

__global__ void k_decode_bind(kvc_pool p, const int32_t *rows, int n_rows, const int32_t *head_rank,
                              const int64_t *demand_eff, const int32_t *ids) {
  if (*demand_eff <= 0) return;
  const int heads = p.num_layers * p.num_kv_heads;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n_rows * heads) return;
  int32_t rank = head_rank[i];
  if (rank < 0) return;
  int64_t hidx = (int64_t)rows[i / heads] * heads + (i % heads);
  int32_t nb = p.nblocks[hidx];
  if (nb >= p.max_blocks) {
    set_status(p.status, KVC_DEV_CAPACITY, (int32_t)hidx, nb + 1);
    return;
  }
  head_table(p, hidx)[nb] = ids[rank];
  p.nblocks[hidx] = nb + 1;
}

// Free trailing table entries of listed heads; reset their slots.
__global__ void k_free_trailing(kvc_pool p, const int32_t *heads3, const int32_t *drop,
                                int32_t row_all, int32_t n) {
  const int hp = p.num_layers * p.num_kv_heads;
  int i = blockIdx.x;
  int64_t hidx;
  int32_t d;
  if (heads3) {
    if (i >= n) return;
    hidx = head_index(p, heads3[3 * i], heads3[3 * i + 1], heads3[3 * i + 2]);
    d = drop[i];
  } else {
    if (i >= hp) return;
    hidx = (int64_t)row_all * hp + i;
    d = p.nblocks[hidx];
  }
  const int32_t nb = p.nblocks[hidx];
  if (d > nb) d = nb;
  const int32_t keep = nb - d;
  const int b = p.block_size;
  const int32_t *tab = head_table(p, hidx);
  for (int64_t e = threadIdx.x; e < (int64_t)d * b; e += blockDim.x) {
    int32_t blk = tab[keep + e / b];
    int64_t f = (int64_t)blk * b + e % b;
    if (p.metric) {  // clear_blocks fused (metrics.py:177-183) when a store is bound
      p.metric[f] = 0.f;
      p.logical[f] = -1;
      p.protected_[f] = 0;
      p.fresh[f] = 0;
    }
    if (e % b == 0) {
      p.free_flag[blk] = 1;
      atomicAdd(&p.free_tile[blk / kTile], 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    p.nblocks[hidx] = keep;
    int32_t c = p.ctx[hidx];
    int32_t cap = keep * b;
    p.ctx[hidx] = c < cap ? c : cap;
  }
}

int alloc_common(const kvc_pool *pool, Scratch &sc, const int64_t *demand_dev, int64_t demand_host,
                 int64_t max_demand, int32_t **ids_out, int64_t **demand_eff_out, cudaStream_t s) {
  const int nt = num_tiles(pool);
  int64_t *tile_prefix = sc.take<int64_t>(nt);
  int64_t *demand_eff = sc.take<int64_t>(1);
  int32_t *ids = sc.take<int32_t>(max_demand > 0 ? max_demand : 1);
  if (!tile_prefix || !demand_eff || !ids) return KVC_ERR_INVALID;
  k_tile_scan<<<1, 1024, 0, s>>>(*pool, demand_dev, demand_host, demand_eff, tile_prefix);
  k_tile_take<<<nt, 256, 0, s>>>(*pool, demand_eff, tile_prefix, ids);
  *ids_out = ids;
  *demand_eff_out = demand_eff;
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

}  // namespace

extern "C" {

int kvc_abi_version(void) { return KVC_ABI_VERSION; }

const char *kvc_status_name(int status) {
  switch (status) {
    case KVC_OK: return "ok";
    case KVC_ERR_INVALID: return "invalid argument";
    case KVC_ERR_UNSUPPORTED: return "unsupported shape";
    case KVC_ERR_CUDA: return "cuda error";
    case KVC_DEV_PREEMPTION: return "PreemptionNeeded";
    case KVC_DEV_ALLOCATION_ORDER: return "AllocationOrderError";
    case KVC_DEV_EMPTY_CONTEXT: return "EmptyContextError";
    case KVC_DEV_NUMERIC: return "NumericError";
    case KVC_DEV_SCHEDULE_CORRUPTION: return "ScheduleCorruptionError";
    case KVC_DEV_CACHE_CORRUPTION: return "CacheCorruptionError";
    case KVC_DEV_CAPACITY: return "table capacity exceeded";
    default: return "unknown";
  }
}

int kvc_pool_init(const kvc_pool *pool, void *stream) {
  if (!pool || pool->num_blocks < 1 || pool->block_size < 1) return KVC_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t slots = pool->num_blocks * pool->block_size;
  const int64_t heads = (int64_t)pool->max_seqs * pool->num_layers * pool->num_kv_heads;
  cudaMemsetAsync(pool->metric, 0, slots * sizeof(float), s);
  cudaMemsetAsync(pool->logical, 0xff, slots * sizeof(int32_t), s);
  cudaMemsetAsync(pool->protected_, 0, slots, s);
  cudaMemsetAsync(pool->fresh, 0, slots, s);
  cudaMemsetAsync(pool->nblocks, 0, heads * sizeof(int32_t), s);
  cudaMemsetAsync(pool->ctx, 0, heads * sizeof(int32_t), s);
  cudaMemsetAsync(pool->status, 0, 4 * sizeof(int32_t), s);
  k_fill_u8<<<1184, 256, 0, s>>>(pool->free_flag, pool->num_blocks, 1);
  int nt = num_tiles(pool);
  k_init_tiles<<<(nt + 255) / 256, 256, 0, s>>>(*pool);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

int64_t kvc_scratch_bytes(const kvc_pool *pool, int64_t max_heads, int64_t max_slots,
                          int32_t max_batch) {
  const int64_t nt = num_tiles(pool);
  const int64_t hp = (int64_t)pool->num_layers * pool->num_kv_heads;
  int64_t alloc = nt * 8 + 8 + (int64_t)hp * pool->max_blocks * 4 + hp * 16 + 4096;
  int64_t decode = (int64_t)max_batch * hp * 8 + 4096;
  // K3/K4: u32 keys (rows padded to 4), 9 per-head ints, the short-head
  // candidate lists (2 x 256 u64), per-sequence digit deltas (n_seqs <= heads)
  // and the K/V copy queue (a u64 per 32 moves; moves <= slots)
  int64_t evict = max_slots * 4 + max_slots / 2 + max_heads * (12 + 36 + 4096 + 2048 * 4 + 44 + 8 + 4104 + 16384) + 65536;
  int64_t m = alloc > decode ? alloc : decode;
  m = m > evict ? m : evict;
  return m + (1 << 20);
}

int kvc_alloc_prefill(const kvc_pool *pool, int32_t seq_row, int32_t blocks_per_head, void *stream) {
  if (!pool || seq_row < 0 || seq_row >= pool->max_seqs || blocks_per_head < 0) return KVC_ERR_INVALID;
  if (blocks_per_head > pool->max_blocks) return KVC_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sc(pool);
  const int hp = pool->num_layers * pool->num_kv_heads;
  const int64_t demand = (int64_t)blocks_per_head * hp;
  int32_t *ids;
  int64_t *demand_eff;
  int rc = alloc_common(pool, sc, nullptr, demand, demand, &ids, &demand_eff, s);
  if (rc) return rc;
  k_bind_runs<<<hp, 256, 0, s>>>(*pool, seq_row, demand_eff, ids, nullptr, nullptr, blocks_per_head);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

int kvc_alloc_heads(const kvc_pool *pool, int32_t seq_row, const int32_t *counts, int64_t total,
                    void *stream) {
  if (!pool || !counts || seq_row < 0 || seq_row >= pool->max_seqs || total < 0) return KVC_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sc(pool);
  const int hp = pool->num_layers * pool->num_kv_heads;
  int64_t *offsets = sc.take<int64_t>(hp);
  int64_t *demand = sc.take<int64_t>(1);
  if (!offsets || !demand) return KVC_ERR_INVALID;
  k_scan_counts<<<1, 1024, 0, s>>>(counts, hp, offsets, demand);
  int32_t *ids;
  int64_t *demand_eff;
  int rc = alloc_common(pool, sc, demand, 0, total, &ids, &demand_eff, s);
  if (rc) return rc;
  k_bind_runs<<<hp, 256, 0, s>>>(*pool, seq_row, demand_eff, ids, counts, offsets, 0);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

int kvc_alloc_decode(const kvc_pool *pool, const int32_t *seq_rows, int32_t n_rows, int32_t *out_counts,
                     void *stream) {
  if (!pool || n_rows < 0 || (n_rows && (!seq_rows || !out_counts))) return KVC_ERR_INVALID;
  if (n_rows == 0) return KVC_OK;
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sc(pool);
  const int hp = pool->num_layers * pool->num_kv_heads;
  const int64_t nh = (int64_t)n_rows * hp;
  int32_t *head_rank = sc.take<int32_t>(nh);
  int64_t *demand = sc.take<int64_t>(1);
  if (!head_rank || !demand) return KVC_ERR_INVALID;
  k_decode_demand<<<1, 1024, 0, s>>>(*pool, seq_rows, n_rows, head_rank, out_counts, demand);
  int32_t *ids;
  int64_t *demand_eff;
  int rc = alloc_common(pool, sc, demand, 0, nh, &ids, &demand_eff, s);
  if (rc) return rc;
  k_decode_bind<<<(int)((nh + 255) / 256), 256, 0, s>>>(*pool, seq_rows, n_rows, head_rank, demand_eff, ids);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

int kvc_free_trailing(const kvc_pool *pool, const int32_t *heads, const int32_t *drop, int32_t n,
                      void *stream) {
  if (!pool || n < 0 || (n && (!heads || !drop))) return KVC_ERR_INVALID;
  if (n == 0) return KVC_OK;
  k_free_trailing<<<n, 256, 0, (cudaStream_t)stream>>>(*pool, heads, drop, 0, n);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

int kvc_free_sequence(const kvc_pool *pool, int32_t seq_row, void *stream) {
  if (!pool || seq_row < 0 || seq_row >= pool->max_seqs) return KVC_ERR_INVALID;
  const int hp = pool->num_layers * pool->num_kv_heads;
  k_free_trailing<<<hp, 256, 0, (cudaStream_t)stream>>>(*pool, nullptr, nullptr, seq_row, hp);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

}  // extern "C"
