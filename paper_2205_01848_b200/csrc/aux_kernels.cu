// aux_kernels.cu -- Eq. 3 balance term of the gate, SURVEY §8(f) N3.
//
//   B = lambda * n * sum_i T_i G_i,   T_i = cnt_i / (T_g k)  (pre-drop counts, stop-gradient,
//   S:347-348),   G_i = (1/T_g) sum_t p[t, i]  (mean gate probability).
// Forward: fixed-order partial column sums of the softmax over 64-token chunks, a fixed-order
// reduction (plus an fp32 all-reduce across EP ranks on the host side), then B and the
// backward coefficients g_i = lambda n T_i / T_g (dB/dl = p (g - <p, g>), applied inside the
// combine-backward kernel).  Deterministic: no atomics.
#include "common.cuh"
#include "kernels.h"

namespace moe {

constexpr int BAL_TOK = 64;

__global__ void __launch_bounds__(256) balance_partial_kernel(const float* __restrict__ logits,
                                                              int Tn, int n,
                                                              float* __restrict__ partial) {
  extern __shared__ float sl[];  // [BAL_TOK][n]
  __shared__ float sm[BAL_TOK], ss[BAL_TOK];
  const int t0 = blockIdx.x * BAL_TOK;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < BAL_TOK * n; i += blockDim.x) {
    const int t = t0 + i / n;
    sl[i] = t < Tn ? logits[(size_t)t0 * n + i] : 0.f;
  }
  __syncthreads();
  for (int tt = warp; tt < BAL_TOK; tt += blockDim.x / 32) {
    float m = -INFINITY;
    for (int e = lane; e < n; e += 32) m = fmaxf(m, sl[tt * n + e]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float s = 0.f;
    for (int e = lane; e < n; e += 32) s += expf(sl[tt * n + e] - m);
    s = __shfl_sync(0xffffffffu, warp_sum(s), 0);
    if (lane == 0) {
      sm[tt] = m;
      ss[tt] = s;
    }
  }
  __syncthreads();
  const int tl = min(BAL_TOK, Tn - t0);
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    float acc = 0.f;
    for (int tt = 0; tt < tl; ++tt) acc += expf(sl[tt * n + e] - sm[tt]) / ss[tt];
    partial[(size_t)blockIdx.x * n + e] = acc;
  }
}

__global__ void balance_reduce_kernel(const float* __restrict__ partial, int nparts, int n,
                                      float* __restrict__ gsum) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  float s = 0.f;
  for (int j = 0; j < nparts; ++j) s += partial[(size_t)j * n + e];
  gsum[e] = s;
}

__global__ void balance_final_kernel(const float* __restrict__ gsum,
                                     const int32_t* __restrict__ counts, int n, int k, float Tg,
                                     float lam, float* __restrict__ g_out,
                                     float* __restrict__ aux_out) {
  __shared__ float terms[MOE_MAX_E];
  const int e = threadIdx.x;
  if (e < n) {
    const float Ti = (float)counts[e] / (Tg * (float)k);
    const float Gi = gsum[e] / Tg;
    g_out[e] = lam * (float)n * Ti / Tg;
    terms[e] = Ti * Gi;
  }
  __syncthreads();
  if (e == 0) {
    float s = 0.f;
    for (int i = 0; i < n; ++i) s += terms[i];  // fixed order
    *aux_out = lam * (float)n * s;
  }
}

cudaError_t launch_balance_partial(const float* logits, int T, int n, float* partial,
                                   float* gsum, cudaStream_t s) {
  const int nparts = (T + BAL_TOK - 1) / BAL_TOK;
  if (nparts > 0) {
    const size_t smem = (size_t)BAL_TOK * n * 4;
    cudaFuncSetAttribute(balance_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    balance_partial_kernel<<<nparts, 256, smem, s>>>(logits, T, n, partial);
  }
  balance_reduce_kernel<<<(n + 255) / 256, 256, 0, s>>>(partial, nparts, n, gsum);
  return cudaGetLastError();
}

cudaError_t launch_balance_final(const float* gsum, const int32_t* counts, int n, int k,
                                 int64_t Tg, float lam, float* g_out, float* aux_out,
                                 cudaStream_t s) {
  balance_final_kernel<<<1, MOE_MAX_E, 0, s>>>(gsum, counts, n, k, (float)(Tg > 0 ? Tg : 1), lam,
                                               g_out, aux_out);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------------------
// Per-sample assignment cache (S4.2 P:245-256; SPEC cache_step S:252-257, cached_route
// S:259-267): a caller-owned table [num_samples x k] int32, -1 = unknown.
// --------------------------------------------------------------------------------------
__global__ void cache_gather_kernel(const int32_t* __restrict__ table, long long num, int k,
                                    const int64_t* __restrict__ ids, int Tn,
                                    int32_t* __restrict__ idx, int32_t* __restrict__ flags) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Tn) return;
  const long long sid = ids[t];
  const bool ok = sid >= 0 && sid < num;
  if (!ok) atomicOr(flags, 4);  // sample id out of range
  for (int r = 0; r < k; ++r) idx[(size_t)t * k + r] = ok ? table[sid * k + r] : -1;
}

__global__ void cache_update_kernel(int32_t* __restrict__ table, long long num, int k,
                                    const int64_t* __restrict__ ids, int Tn,
                                    const int32_t* __restrict__ fresh) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Tn) return;
  const long long sid = ids[t];
  if (sid < 0 || sid >= num) return;
  for (int r = 0; r < k; ++r) table[sid * k + r] = fresh[(size_t)t * k + r];
}

// observe mode: hit = the remembered row equals the fresh top-k as a set (unknown: a miss),
// then remember the fresh row (the metric of P:353 while caching is off)
__global__ void cache_observe_kernel(int32_t* __restrict__ table, long long num, int k,
                                     const int64_t* __restrict__ ids, int Tn,
                                     const int32_t* __restrict__ fresh, int32_t* __restrict__ hit,
                                     int32_t* __restrict__ flags) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Tn) return;
  const long long sid = ids[t];
  if (sid < 0 || sid >= num) {
    atomicOr(flags, 4);
    return;
  }
  int32_t* row = table + sid * k;
  const int32_t* fr = fresh + (size_t)t * k;
  bool same = true;
  for (int r = 0; r < k; ++r) {
    bool found = false;
    for (int q = 0; q < k; ++q) found |= row[r] == fr[q];
    same &= found && row[r] >= 0;
  }
  if (same) atomicAdd(hit, 1);
  for (int r = 0; r < k; ++r) row[r] = fr[r];
}

cudaError_t launch_cache_observe(int32_t* table, int64_t num, int k, const int64_t* ids, int T,
                                 const int32_t* fresh, int32_t* hit, int32_t* flags,
                                 cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  cache_observe_kernel<<<(T + 255) / 256, 256, 0, s>>>(table, num, k, ids, T, fresh, hit, flags);
  return cudaGetLastError();
}

cudaError_t launch_cache_gather(const int32_t* table, int64_t num, int k, const int64_t* ids,
                                int T, int32_t* idx, int32_t* flags, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  cache_gather_kernel<<<(T + 255) / 256, 256, 0, s>>>(table, num, k, ids, T, idx, flags);
  return cudaGetLastError();
}

cudaError_t launch_cache_update(int32_t* table, int64_t num, int k, const int64_t* ids, int T,
                                const int32_t* fresh, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  cache_update_kernel<<<(T + 255) / 256, 256, 0, s>>>(table, num, k, ids, T, fresh);
  return cudaGetLastError();
}

}  // namespace moe
