// Read-bandwidth ceiling on this B200 for the load paths the kernels use:
// LDG.128, cp.async.bulk (1-D TMA) and cp.async.bulk.tensor 3-D boxes (the
// K1 {64,16,2} and K2 {64,128,2} SWIZZLE_128B boxes).  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/readbw tools/microbench/readbw.cu -lcuda && /tmp/readbw
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ldg_read(const uint4 *p, int64_t n, uint32_t *out) {
  uint32_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n; i += stride) { uint4 v = __ldcs(p + i); acc ^= v.x ^ v.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

// mode 0: 1-D bulk chunks of CH bytes; mode 1: 3-D tensor boxes (rows x 256 B)
template <int MODE>
__global__ void tma_read(const char *base, int64_t bytes, const __grid_constant__ CUtensorMap tm, int box_rows,
                         int stages, int ch, uint32_t *out) {
  extern __shared__ __align__(1024) char sm[];
  char *buf = (char *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(buf + (size_t)stages * ch);
  uint64_t *empty = full + stages;
  const int64_t nchunks = bytes / ch;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int64_t my = 0;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) ++my;
  if (warp == 0 && lane == 0) {
    int64_t k = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
      const int s = k % stages;
      if (k >= stages) {
        const uint32_t par = ((k / stages) - 1) & 1;
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(&empty[s])), "r"(par) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(ch) : "memory");
      if (MODE == 0) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(buf + (size_t)s * ch)),
                     "l"(base + c * ch), "r"(ch), "r"(su32(&full[s])) : "memory");
      } else {
        const int per = ch / (box_rows * 256);
        for (int q = 0; q < per; ++q) {
          const int row = (int)((c * per + q) * box_rows);
          asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(buf + (size_t)s * ch + q * box_rows * 256)),
                       "l"(&tm), "r"(0), "r"(row), "r"(0), "r"(su32(&full[s])) : "memory");
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    uint32_t acc = 0;
    for (int64_t k = 0; k < my; ++k) {
      const int s = k % stages;
      const uint32_t par = (k / stages) & 1;
      asm volatile("{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}" ::"r"(su32(&full[s])), "r"(par) : "memory");
      acc ^= *(volatile uint32_t *)(buf + (size_t)s * ch);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
    if (acc == 0x12345678u) out[0] = acc;
  }
}

typedef CUresult (*Enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                        const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int64_t bytes = 8LL << 30;
  char *buf;
  uint32_t *out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 64);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char *name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s %8.1f GB/s  (%s)\n", name, 3.0 * bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (int cps : {4, 8, 16})
    for (int thr : {256, 512}) {
      char nm[64];
      snprintf(nm, 64, "LDG.128 x8 in flight, %d CTA/SM x %d", cps, thr);
      timeit(nm, [&] { ldg_read<<<148 * cps, thr>>>((const uint4 *)buf, bytes / 16, out); });
    }
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  for (int box : {16, 128}) {
    CUtensorMap tm;
    cuuint64_t dims[3] = {64, (cuuint64_t)(bytes / 256), 2};
    cuuint64_t str[2] = {256, 128};
    cuuint32_t bx[3] = {64, (cuuint32_t)box, 2};
    cuuint32_t es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int cps : {1, 2})
      for (int stages : {4, 8}) {
        const int ch = 32768 / cps;
        if (ch < box * 256) continue;  // a stage must hold whole boxes
        const int smem = stages * ch + 2048;
        cudaFuncSetAttribute(tma_read<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        char nm[80];
        snprintf(nm, 80, "TMA 3-D box {64,%d,2}, %d CTA/SM, %d x %d KB", box, cps, stages, ch / 1024);
        timeit(nm, [&] { tma_read<1><<<148 * cps, 64, smem>>>(buf, bytes, tm, box, stages, ch, out); });
      }
  }
  for (int cps : {1, 2})
    for (int stages : {4, 8}) {
      const int ch = 32768 / cps;
      const int smem = stages * ch + 2048;
      cudaFuncSetAttribute(tma_read<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      CUtensorMap dummy;
      char nm[80];
      snprintf(nm, 80, "TMA 1-D bulk, %d CTA/SM, %d x %d KB", cps, stages, ch / 1024);
      timeit(nm, [&] { tma_read<0><<<148 * cps, 64, smem>>>(buf, bytes, dummy, 16, stages, ch, out); });
    }
  return 0;
}
