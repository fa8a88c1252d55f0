// Reference-signature prompt-metric entry points on an explicit attention
// tensor (the drop-in surface of pagedkv.metrics / pagedkv.attention for
// callers that already hold the (n_q, L, L) attention):
//
//   kvc_gqa_attention  gqa_attention   attention.py:62-89   dense causal GQA, f32
//   kvc_attn_metrics   window_metrics  metrics.py:68-89     (+ _group_sum :50-54,
//                      full_metrics    metrics.py:92-109      _pool_max :57-65)
//
// These materialise O(n_q L^2) data exactly like the reference; the serving
// path never does (K2 window.cu and F1/F2 fullmetric.cu compute the same
// metrics from Q and K on tcgen05 without the attention tensor).  Both are
// HBM-streaming kernels: one CTA per attention row, and one thread per key
// column walking the rows (coalesced across keys).
#include "common.cuh"

using namespace kvc;

namespace {

// One CTA per (query head h, query row i): s_j = q_i . k_j / sqrt(d) for
// j <= i, row softmax (max-subtracted, fp32), attn row (zeros above the
// diagonal), out_i = sum_j p_j v_j.  Scores live in dynamic shared memory.
__global__ void __launch_bounds__(256) k_gqa_dense(const float *__restrict__ q, const float *__restrict__ k,
                                                   const float *__restrict__ v, float *__restrict__ out,
                                                   float *__restrict__ attn, int L, int d, int r, float scale,
                                                   int32_t *status) {
  extern __shared__ float sc[];  // [L] scores, then [32] reduction
  float *red = sc + L;
  const int i = blockIdx.x, h = blockIdx.y, kv = h / r;
  const float *qi = q + ((int64_t)h * L + i) * d;
  const float *kh = k + (int64_t)kv * L * d;
  const float *vh = v ? v + (int64_t)kv * L * d : nullptr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  bool bad = false;
  float mloc = -INFINITY;
  for (int j = threadIdx.x; j <= i; j += blockDim.x) {
    float s = 0.f;
    for (int e = 0; e < d; ++e) s = fmaf(qi[e], kh[(int64_t)j * d + e], s);
    s *= scale;
    bad |= !isfinite(s);
    sc[j] = s;
    mloc = fmaxf(mloc, s);
  }
  if (bad) set_status(status, KVC_DEV_NUMERIC, h, i);
  for (int o = 16; o > 0; o >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, o));
  if (lane == 0) red[warp] = mloc;
  __syncthreads();
  float M = -INFINITY;
  for (int w = 0; w < nw; ++w) M = fmaxf(M, red[w]);
  __syncthreads();
  float zloc = 0.f;
  for (int j = threadIdx.x; j <= i; j += blockDim.x) {
    const float e = expf(sc[j] - M);
    sc[j] = e;
    zloc += e;
  }
  for (int o = 16; o > 0; o >>= 1) zloc += __shfl_xor_sync(0xffffffffu, zloc, o);
  if (lane == 0) red[warp] = zloc;
  __syncthreads();
  float Z = 0.f;
  for (int w = 0; w < nw; ++w) Z += red[w];
  const float iz = 1.f / Z;
  float *arow = attn + ((int64_t)h * L + i) * L;
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    const float p = j <= i ? sc[j] * iz : 0.f;
    if (j <= i) sc[j] = p;
    arow[j] = p;
  }
  if (!out || !vh) return;
  __syncthreads();
  float *orow = out + ((int64_t)h * L + i) * d;
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j <= i; ++j) acc = fmaf(sc[j], vh[(int64_t)j * d + e], acc);
    orow[e] = acc;
  }
}

// raw[kv][j] = sum_{h in group(kv)} sum_{i in rows(j)} f(attn[h][i][j]);
// rows = [max(L - window, 0), L) (window) or [j + excluded, L) (full).
__global__ void k_attn_colsum(const float *__restrict__ attn, float *__restrict__ raw, int L, int r, int full,
                              int window, int excluded, int agg) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, kv = blockIdx.y;
  if (j >= L) return;
  const int i0 = full ? j + excluded : max(L - window, 0);
  float acc = 0.f;
  for (int h = kv * r; h < (kv + 1) * r; ++h) {
    const float *col = attn + (int64_t)h * L * L + j;
    for (int i = i0; i < L; ++i) {
      const float a = __ldg(col + (int64_t)i * L);
      acc += agg == 2 ? a * a : a;
    }
  }
  raw[(int64_t)kv * L + j] = acc;
}

// centred max-pool of odd width, truncated at the edges (metrics.py:57-65)
__global__ void k_pool_max(const float *__restrict__ raw, float *__restrict__ out, int L, int pool) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, kv = blockIdx.y;
  if (j >= L) return;
  const int half = pool / 2;
  const float *row = raw + (int64_t)kv * L;
  float m = row[j];
  for (int t = max(0, j - half); t <= min(L - 1, j + half); ++t) m = fmaxf(m, row[t]);
  out[(int64_t)kv * L + j] = m;
}

}  // namespace

extern "C" {

int kvc_gqa_attention(const kvc_pool *pool, const kvc_dense_args *a, void *stream) {
  if (!pool || !a || !a->q || !a->k || !a->attn || a->L < 1) return KVC_ERR_INVALID;
  const int H = pool->num_kv_heads, d = pool->head_dim;
  if (H < 1 || d < 1 || a->num_query_heads % H) return KVC_ERR_INVALID;
  const size_t smem = ((size_t)a->L + 32) * 4;
  if (smem > 227 * 1024) return KVC_ERR_UNSUPPORTED;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_gqa_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = true;
  }
  dim3 grid(a->L, a->num_query_heads);
  k_gqa_dense<<<grid, 256, smem, (cudaStream_t)stream>>>(a->q, a->k, a->v, a->out, a->attn, a->L, d,
                                                         a->num_query_heads / H, 1.f / sqrtf((float)d),
                                                         pool->status);
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

int kvc_attn_metrics(const kvc_pool *pool, const kvc_attn_metric_args *a, void *stream) {
  if (!pool || !a || !a->attn || !a->metrics_out || a->L < 1) return KVC_ERR_INVALID;
  const int H = pool->num_kv_heads;
  if (H < 1 || a->num_query_heads % H) return KVC_ERR_INVALID;
  if (a->mode == 0 && (a->window < 1 || a->pool < 1 || a->pool % 2 == 0)) return KVC_ERR_INVALID;
  if (a->mode == 1 && a->excluded < 0) return KVC_ERR_INVALID;
  const int r = a->num_query_heads / H;
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((a->L + 127) / 128, H);
  const int agg = a->aggregation == 2 ? 2 : 1;
  if (a->mode == 1 || a->pool == 1) {
    k_attn_colsum<<<grid, 128, 0, s>>>(a->attn, a->metrics_out, a->L, r, a->mode == 1, a->window, a->excluded, agg);
  } else {
    if (!pool->scratch || pool->scratch_bytes < (int64_t)H * a->L * 4) return KVC_ERR_INVALID;
    float *raw = reinterpret_cast<float *>(pool->scratch);
    k_attn_colsum<<<grid, 128, 0, s>>>(a->attn, raw, a->L, r, 0, a->window, a->excluded, agg);
    k_pool_max<<<grid, 128, 0, s>>>(raw, a->metrics_out, a->L, a->pool);
  }
  KVC_CHECK_LAUNCH();
  return KVC_OK;
}

}  // extern "C"
