// Shared device helpers for libkvc (sm_100a).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "kvc.h"

#define KVC_CHECK_LAUNCH()                                  \
  do {                                                      \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return KVC_ERR_CUDA;             \
  } while (0)

namespace kvc {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// Pool addressing
// ---------------------------------------------------------------------------

__host__ __device__ inline int64_t head_index(const kvc_pool &p, int row, int layer, int head) {
  return ((int64_t)row * p.num_layers + layer) * p.num_kv_heads + head;
}

__host__ __device__ inline int32_t *head_table(const kvc_pool &p, int64_t hidx) {
  return p.tables + hidx * p.max_blocks;
}

// Programmatic dependent launch: wait for the preceding kernel of the stream
// (no-op without the launch attribute) / let the next one's CTAs launch.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// First error wins; payload words written by the winner only.
__device__ inline void set_status(int32_t *status, int code, int32_t a = 0, int32_t b = 0) {
  if (atomicCAS(status, 0, code) == 0) {
    status[1] = a;
    status[2] = b;
  }
}

// ---------------------------------------------------------------------------
// bf16 helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ void bf16x8_to_f32(const uint4 &v, float *f) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

__device__ __forceinline__ void bf16x4_to_f32(const uint2 &v, float *f) {
  f[0] = __uint_as_float(v.x << 16);
  f[1] = __uint_as_float(v.x & 0xffff0000u);
  f[2] = __uint_as_float(v.y << 16);
  f[3] = __uint_as_float(v.y & 0xffff0000u);
}

// V consecutive bf16 values as one vector load (V = 8: 16 bytes, 4: 8 bytes)
template <int V> struct BfVec;
template <> struct BfVec<8> {
  using T = uint4;
  static __device__ __forceinline__ void to_f32(const T &v, float *f) { bf16x8_to_f32(v, f); }
};
template <> struct BfVec<4> {
  using T = uint2;
  static __device__ __forceinline__ void to_f32(const T &v, float *f) { bf16x4_to_f32(v, f); }
};

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t b) {
  return __uint_as_float(((uint32_t)b) << 16);
}

// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (cp.async.bulk, TMA engine, non-tensor form)
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Global -> shared bulk copy of `bytes` (multiple of 16, 16B-aligned) that
// completes a transaction on `bar`.  Evict-first: KV blocks are streamed.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// store with an L2 eviction-priority hint (scratch that is read back soon)
__device__ __forceinline__ void st_hint(float *a, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}

// drop a 128-byte L2 line without writing it back (scratch fully consumed;
// `a` 128-byte aligned)
__device__ __forceinline__ void discard_l2(const void *a) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
}

// ---------------------------------------------------------------------------
// Warp reductions
// ---------------------------------------------------------------------------

template <int WIDTH = 32>
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int WIDTH = 32>
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Order-preserving map of an fp32 value to uint32 (total order for non-NaN).
__host__ __device__ __forceinline__ uint32_t f32_order_key(float f) {
  uint32_t u;
#ifdef __CUDA_ARCH__
  u = __float_as_uint(f);
#else
  memcpy(&u, &f, 4);
#endif
  if (u == 0x80000000u) u = 0;  // -0.0 == +0.0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Scratch bump allocator (host side).
struct Scratch {
  char *base;
  int64_t size;
  int64_t used = 0;
  Scratch(const kvc_pool *p) : base(reinterpret_cast<char *>(p->scratch)), size(p->scratch_bytes) {}
  template <typename T>
  T *take(int64_t count) {
    int64_t off = (used + 255) & ~int64_t(255);
    int64_t bytes = count * (int64_t)sizeof(T);
    if (off + bytes > size) return nullptr;
    used = off + bytes;
    return reinterpret_cast<T *>(base + off);
  }
};

__host__ __device__ inline int num_tiles(const kvc_pool *p) {
  return (int)((p->num_blocks + KVC_FREE_TILE - 1) / KVC_FREE_TILE);
}

}  // namespace kvc
