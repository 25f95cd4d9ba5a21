// route_kernels.cu -- gate/top-k, routing (histogram, scan, stable scatter), combine and
// their backwards for the DynaMoE MoE layer on sm_100a.
//
// Paper passages: Alg. 1 lines 1-3 (gate, argmax_k, normalize) and 5-8
// (weighted combine); P:225 (capacity drop, zero gradient for dropped samples); Eq. 4
// (capacities arrive as integers in CapTable); S4.2 P:238-256 (cached indices).
// Readings: top-k on fp32 logits, IEEE '>', ties -> lower expert
// index; token-major global drop order; relu'(0) = 0; fp32 accumulators everywhere; no
// floating-point atomics (bitwise run-to-run determinism).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace moe {

// =====================================================================================
// K1 (SIMT form): gate logits l = x W_g^T (fp32 accumulate, sequential over d), then
// softmax / top-k / normalize per token.  CTA = 32 tokens x all n experts.
// =====================================================================================
constexpr int GATE_TOK = 32;
constexpr int GATE_DK = 32;

template <typename T, int NJ>
__global__ void __launch_bounds__(256) gate_topk_kernel(
    const T* __restrict__ x, const T* __restrict__ wg, int Tn, int n, int d, int k,
    int renorm, const int32_t* __restrict__ cached, float* __restrict__ logits,
    int32_t* __restrict__ idx_out, float* __restrict__ w_out, int32_t* __restrict__ hit,
    int32_t* __restrict__ flags, int32_t* __restrict__ idx_fix) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  extern __shared__ float smem[];
  float* xs = smem;                              // [GATE_TOK][GATE_DK+1]
  float* ws = xs + GATE_TOK * (GATE_DK + 1);     // [n][GATE_DK+1]
  const int tid = threadIdx.x;
  const int t0 = blockIdx.x * GATE_TOK;
  const int tok = tid >> 3, g = tid & 7;
  float acc[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) acc[j] = 0.f;

  // the next d-slice of x and W_g is loaded into registers while the current one is
  // multiplied out of shared memory (same c order per logit: bitwise identical results)
  static_assert(GATE_TOK * GATE_DK == 4 * 256, "x slice = 4 elements per thread");
  float rx[4], rw[NJ];  // n * GATE_DK <= 8 NJ * 32 = NJ * 256 elements of W_g
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = tid + 256 * q, r = i / GATE_DK, c = i % GATE_DK, t = t0 + r;
      rx[q] = (t < Tn) ? to_f(x[(size_t)t * d + k0 + c]) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < NJ; ++q) {
      const int i = tid + 256 * q;
      if (i < n * GATE_DK) rw[q] = to_f(wg[(size_t)(i / GATE_DK) * d + k0 + i % GATE_DK]);
    }
  };
  load(0);
  for (int k0 = 0; k0 < d; k0 += GATE_DK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = tid + 256 * q;
      xs[(i / GATE_DK) * (GATE_DK + 1) + i % GATE_DK] = rx[q];
    }
#pragma unroll
    for (int q = 0; q < NJ; ++q) {
      const int i = tid + 256 * q;
      if (i < n * GATE_DK) ws[(i / GATE_DK) * (GATE_DK + 1) + i % GATE_DK] = rw[q];
    }
    __syncthreads();
    if (k0 + GATE_DK < d) load(k0 + GATE_DK);
#pragma unroll 4
    for (int c = 0; c < GATE_DK; ++c) {
      float xv = xs[tok * (GATE_DK + 1) + c];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        int e = g + 8 * j;
        if (e < n) acc[j] = fmaf(xv, ws[e * (GATE_DK + 1) + c], acc[j]);
      }
    }
    __syncthreads();
  }
  // logits -> smem [GATE_TOK][n+1] (reuses ws) and global
  float* ls = ws;
  {
    int t = t0 + tok;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      int e = g + 8 * j;
      if (e < n) {
        ls[tok * (n + 1) + e] = acc[j];
        if (t < Tn) logits[(size_t)t * n + e] = acc[j];
      }
    }
  }
  __syncthreads();
  if (tid < GATE_TOK) {
    const int t = t0 + tid;
    if (t < Tn) {
      const float* l = ls + tid * (n + 1);
      // top-k: repeatedly take the first maximum among experts not yet taken (IEEE '>',
      // strict, so equal values -- including -0.0 vs +0.0 -- keep the lower index).
      int sel[MOE_MAX_K];
      bool nan_seen = false;
      for (int r = 0; r < k; ++r) {
        int best = -1;
        float bv = 0.f;
        for (int e = 0; e < n; ++e) {
          bool taken = false;
          for (int q = 0; q < r; ++q) taken |= (sel[q] == e);
          if (taken) continue;
          float v = l[e];
          if (v != v) nan_seen = true;
          if (best < 0 || v > bv) { best = e; bv = v; }
        }
        sel[r] = best;
      }
      if (nan_seen) atomicOr(flags, 1);
      int32_t* orow = idx_out + (size_t)t * k;
      for (int r = 0; r < k; ++r) orow[r] = sel[r];
      // dispatch indices: cached (validated) or fresh
      int use[MOE_MAX_K];
      if (cached) {
        const int32_t* crow = cached + (size_t)t * k;
        bool ok = true, unknown = false;
        for (int r = 0; r < k; ++r) {
          use[r] = crow[r];
          ok &= (use[r] >= 0 && use[r] < n);
          unknown |= use[r] == -1;
          for (int q = 0; q < r; ++q) ok &= (use[q] != use[r]);
        }
        if (!ok) {  // unknown sample in fallback mode: fresh top-k, a miss
          if (!(unknown && idx_fix)) atomicOr(flags, 2);
          for (int r = 0; r < k; ++r) use[r] = sel[r];
          if (idx_fix)
            for (int r = 0; r < k; ++r) idx_fix[(size_t)t * k + r] = sel[r];
        }
        bool same = true;  // set equality of fresh and cached rows
        for (int r = 0; r < k; ++r) {
          bool found = false;
          for (int q = 0; q < k; ++q) found |= (use[r] == sel[q]);
          same &= found;
        }
        if (same && ok) atomicAdd(hit, 1);
      } else {
        for (int r = 0; r < k; ++r) use[r] = sel[r];
      }
      // normalize (Alg. 1 l.3): renorm = softmax over the selected logits; raw = p_i.
      float* wrow = w_out + (size_t)t * k;
      if (renorm) {
        float m = l[use[0]];
        for (int r = 1; r < k; ++r) m = fmaxf(m, l[use[r]]);
        float ev[MOE_MAX_K], s = 0.f;
        for (int r = 0; r < k; ++r) { ev[r] = expf(l[use[r]] - m); s += ev[r]; }
        for (int r = 0; r < k; ++r) wrow[r] = ev[r] / s;
      } else {
        float m = l[0];
        for (int e = 1; e < n; ++e) m = fmaxf(m, l[e]);
        float s = 0.f;
        for (int e = 0; e < n; ++e) s += expf(l[e] - m);
        for (int r = 0; r < k; ++r) wrow[r] = expf(l[use[r]] - m) / s;
      }
    }
  }
}

cudaError_t launch_gate_topk(int dtype, const void* x, const void* wg, int T, int n, int d,
                             int k, int renorm, const int32_t* cached, RouteBufs b,
                             cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  dim3 grid((T + GATE_TOK - 1) / GATE_TOK);
  size_t smem = (size_t)(GATE_TOK * (GATE_DK + 1)) * 4 +
                (size_t)max(n * (GATE_DK + 1), GATE_TOK * (n + 1)) * 4;
  int32_t* idx_out = cached ? b.fresh_idx : b.idx;
#define GATE_CASE(NJ)                                                                      \
  if (n <= 8 * NJ) {                                                                       \
    if (dtype == 1) {                                                                      \
      auto kf = gate_topk_kernel<__nv_bfloat16, NJ>;                                       \
      cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
      launch_pdl(kf, grid, 256, smem, s, (const __nv_bfloat16*)x, (const __nv_bfloat16*)wg, T, n,  \
                                 d, k, renorm, cached, b.logits, idx_out, b.w,             \
                                 b.hit_count, b.flags, cached ? b.idx_fix : nullptr);      \
    } else {                                                                               \
      auto kf = gate_topk_kernel<float, NJ>;                                               \
      cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
      launch_pdl(kf, grid, 256, smem, s, (const float*)x, (const float*)wg, T, n, d, k, renorm,    \
                                 cached, b.logits, idx_out, b.w, b.hit_count, b.flags,     \
                                 cached ? b.idx_fix : nullptr);                            \
    }                                                                                      \
    return cudaGetLastError();                                                             \
  }
  GATE_CASE(1) GATE_CASE(2) GATE_CASE(4) GATE_CASE(8) GATE_CASE(16) GATE_CASE(32)
#undef GATE_CASE
  return cudaErrorInvalidValue;
}

// =====================================================================================
// K2a: per-tile expert histogram of the dispatch indices (order-independent counts).
// =====================================================================================
// src != null (cached mode): the dispatch indices are read from the caller's cached array and
// copied into idx on the way (one pass instead of a device copy + this kernel)
__global__ void route_hist_kernel(int32_t* __restrict__ idx, int Tn, int k, int n,
                                  int32_t* __restrict__ hist, const int32_t* __restrict__ src) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  __shared__ int32_t h[MOE_MAX_E];
  for (int e = threadIdx.x; e < n; e += blockDim.x) h[e] = 0;
  __syncthreads();
  int t = blockIdx.x * MOE_ROUTE_TILE + threadIdx.x;
  if (t < Tn)
    for (int r = 0; r < k; ++r) {
      const size_t i = (size_t)t * k + r;
      const int e = src ? src[i] : idx[i];
      if (src) idx[i] = e;
      if ((unsigned)e < (unsigned)n) atomicAdd(&h[e], 1);  // invalid cached index: flagged
    }
  __syncthreads();
  for (int e = threadIdx.x; e < n; e += blockDim.x) hist[(size_t)blockIdx.x * n + e] = h[e];
}

cudaError_t launch_route_hist(int32_t* idx, int T, int k, int n, int32_t* hist,
                              cudaStream_t s, const int32_t* src) {
  if (T == 0) return cudaSuccess;
  int ntiles = (T + MOE_ROUTE_TILE - 1) / MOE_ROUTE_TILE;
  launch_pdl(route_hist_kernel, ntiles, MOE_ROUTE_TILE, 0, s, idx, T, k, n, hist, src);
  return cudaGetLastError();
}

// =====================================================================================
// K2b: exclusive scan of the tile histograms per expert (one CTA per expert), then the
// last CTA finalises: kept_e = min(cnt_e, C_e), drops = sum(cnt - kept), GEMM m-tile prefix.
// =====================================================================================
__global__ void __launch_bounds__(256) route_scan_kernel(
    const int32_t* __restrict__ hist, int ntiles, int n, CapTable ct,
    int32_t* __restrict__ tile_off, int32_t* __restrict__ counts, int32_t* __restrict__ kept,
    int32_t* __restrict__ mtile_prefix, int64_t* __restrict__ drops,
    uint32_t* __restrict__ ticket, int32_t* __restrict__ drop_cnt, int pad_gemm) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  const int e = blockIdx.x;
  __shared__ int32_t warp_tot[8];
  __shared__ int32_t carry;
  __shared__ bool is_last;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int PER = 4;  // tiles per thread: every load of a chunk is in flight at once
  for (int t0 = 0; t0 < ntiles; t0 += 256 * PER) {
    const int i0 = t0 + threadIdx.x * PER;
    int v[PER], sum = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      v[j] = (i0 + j < ntiles) ? hist[(size_t)(i0 + j) * n + e] : 0;
      sum += v[j];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    int wpre = 0, tot = 0;
    for (int q = 0; q < 8; ++q) {
      if (q < wid) wpre += warp_tot[q];
      tot += warp_tot[q];
    }
    int run = carry + wpre + incl - sum;  // exclusive prefix of this thread's first tile
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (i0 + j < ntiles) tile_off[(size_t)(i0 + j) * n + e] = run;
      run += v[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    counts[e] = carry;
    __threadfence();
    unsigned prev = atomicAdd(ticket, 1u);
    is_last = (prev == (unsigned)(gridDim.x - 1));
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (threadIdx.x < 32) {  // one warp: parallel loads, warp scan for the GEMM m-tile prefix
    const int lane = threadIdx.x;
    long long dr = 0;
    int carry = 0;
    int cq[MOE_MAX_E / 32];  // every expert's count requested before the first use
#pragma unroll
    for (int j = 0; j < MOE_MAX_E / 32; ++j)
      cq[j] = j * 32 + lane < n ? *((volatile int32_t*)counts + j * 32 + lane) : 0;
#pragma unroll
    for (int j = 0; j < MOE_MAX_E / 32; ++j) {
      const int q0 = j * 32;
      if (q0 >= n) break;
      const int q = q0 + lane;
      int kq = 0;
      if (q < n) {
        const int c = cq[j];
        kq = min(c, ct.cap[q]);
        dr += (long long)(c - kq);
        // timing experiment only (MOE_DBG_PAD_GEMM=1): the expert GEMMs run over all C_e
        // rows, as a capacity-padded implementation would -- results are NOT valid
        if (pad_gemm) kq = ct.cap[q];
        kept[q] = kq;
      }
      const int v = (kq + 127) / 128;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (q < n) mtile_prefix[q] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dr += __shfl_xor_sync(0xffffffffu, dr, o);
    if (lane == 0) {
      mtile_prefix[n] = carry;
      *drops = dr;
      *ticket = 0u;  // self-reset for the next launch
      if (drop_cnt) *drop_cnt = 0;  // the combine backward's dropped-token list starts empty
    }
  }
}

cudaError_t launch_route_scan(const int32_t* hist, int ntiles, int n, const CapTable& ct,
                              RouteBufs b, cudaStream_t s) {
  static const int pad_gemm = [] {
    const char* v = getenv("MOE_DBG_PAD_GEMM");
    return v && v[0] == '1' ? 1 : 0;
  }();
  launch_pdl(route_scan_kernel, n, 256, 0, s, hist, ntiles, n, ct, b.tile_off, b.counts, b.kept,
                                      b.mtile_prefix, b.drops, b.ticket, b.drop_cnt, pad_gemm);
  return cudaGetLastError();
}

// =====================================================================================
// K3: stable capacity-bounded scatter.  Per 128-token tile: intra-tile ranks from per-expert
// token bitmasks (popc of lower tokens; exact token-major order since an expert appears at
// most once per token), slot = tile_off + rank; kept iff slot < C_e.  Then each warp
// copies its tokens' rows x[t] -> X_buf[base_e + slot] with 16-byte vectors (row read once,
// written once per kept pair).
// =====================================================================================
// Zero rows [kept_e, min(roundup(kept_e, PAD), region end)) of expert regions e = first,
// first + stride, ... with all threads of the calling block (the token-contraction GEMMs read
// whole 64-row K-blocks).  Fused into the dispatch / combine-backward kernels on one GPU.
// Local region j starts at row ct.base[e0 + j]; regions are 128-row aligned and kept <= cap,
// so roundup(kept, 64) never leaves the region.
template <typename T, int RU, int KM>
__global__ void __launch_bounds__(256) dispatch_kernel(
    const int32_t* __restrict__ idx, const T* __restrict__ x, int Tn, int k, int n, int d,
    long long token_base, CapTable ct, const int32_t* __restrict__ tile_off,
    int32_t* __restrict__ slot_of, int32_t* __restrict__ token_of_slot, T* __restrict__ xbuf,
    const int32_t* __restrict__ pad_kept, int pad_e0, PeerBufs px, PeerBufs ptos,
    const int32_t* __restrict__ pre_dev, T* __restrict__ yz, int dout) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  // px.nl != 0 (peer EP, N1): rows go straight into the owners' X buffers over NVLink, the
  // global slot offsets come from the device plan (pre_dev), token_of_slot is the owner's.
  // xbuf == null (N2 gather fusion): only the routing tables are written -- the expert GEMMs
  // gather the x rows themselves; yz != null (N2 fused combine): y rows of tokens with every
  // pair dropped are zeroed here (the GEMM epilogue writes the others).
  __shared__ uint32_t masks[MOE_MAX_E][MOE_ROUTE_TILE / 32];
  if (pad_kept)
    zero_pads_block(xbuf, d, pad_kept, ct, px.nl ? px.nl : n, pad_e0, blockIdx.x, gridDim.x);
  __shared__ int32_t srow[MOE_ROUTE_TILE * MOE_MAX_K];  // destination row or -1
  __shared__ int32_t sexp[MOE_ROUTE_TILE * MOE_MAX_K];  // its expert
  const int tile = blockIdx.x;
  const int t0 = tile * MOE_ROUTE_TILE;
  for (int i = threadIdx.x; i < n * (MOE_ROUTE_TILE / 32); i += blockDim.x)
    (&masks[0][0])[i] = 0u;
  __syncthreads();
  const int lt = threadIdx.x;  // local token (threads 0..127)
  const int t = t0 + lt;
  int ev[MOE_MAX_K];
  if (lt < MOE_ROUTE_TILE && t < Tn) {
#pragma unroll
    for (int r = 0; r < MOE_MAX_K; ++r) {
      if (r >= k) break;
      ev[r] = idx[(size_t)t * k + r];
      if ((unsigned)ev[r] < (unsigned)n) atomicOr(&masks[ev[r]][lt >> 5], 1u << (lt & 31));
      else ev[r] = -1;  // invalid cached index (device flag raised by the gate): dropped
    }
  }
  __syncthreads();
  if (lt < MOE_ROUTE_TILE) {
#pragma unroll
    for (int r = 0; r < MOE_MAX_K; ++r) {
      if (r >= k) break;
      int row = -1;
      if (t < Tn && ev[r] < 0) {
        slot_of[(size_t)t * k + r] = -1;
      } else if (t < Tn) {
        const int e = ev[r];
        int rank = __popc(masks[e][lt >> 5] & ((1u << (lt & 31)) - 1u));
        for (int q = 0; q < (lt >> 5); ++q) rank += __popc(masks[e][q]);
        const int pre = pre_dev ? pre_dev[e] : ct.pre[e];
        const int slot = pre + tile_off[(size_t)tile * n + e] + rank;
        const bool keep = slot < ct.cap[e];
        slot_of[(size_t)t * k + r] = keep ? slot : -1;
        if (keep) {
          row = ct.base[e] + slot;
          *peer_row(token_of_slot, ptos, e, (size_t)row, 1) = (int32_t)((token_base + t) * k + r);
        }
        sexp[lt * k + r] = e;
      }
      srow[lt * k + r] = row;
    }
  }
  __syncthreads();
  // row copies: warp per token, RU tokens per warp at a time (RU > 1 for small batches,
  // whose few blocks would otherwise wait one row latency per token); KM bounds k
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int VE = Vec<T>::N;
  const int nvec = d / VE;
  for (int b0 = wid * RU; b0 < MOE_ROUTE_TILE; b0 += 8 * RU) {
    if (t0 + b0 >= Tn) break;
    T* dsts[RU][KM];  // fully unrolled (registers, no local-memory array)
    bool cp[RU];
#pragma unroll
    for (int j = 0; j < RU; ++j) {
      const int lt2 = b0 + j, tt = t0 + lt2;
      bool any = false;
#pragma unroll
      for (int r = 0; r < KM; ++r) {
        dsts[j][r] = nullptr;
        if (r < k && tt < Tn) {
          const int rw = srow[lt2 * k + r];
          if (rw >= 0) {
            any = true;
            if (xbuf) dsts[j][r] = peer_row(xbuf, px, sexp[lt2 * k + r], (size_t)rw, d);
          }
        }
      }
      if (!any && yz && tt < Tn) {  // all pairs dropped: y[t] = 0
        for (int v = lane; v < dout / VE; v += 32)
          st_v4(yz + (size_t)tt * dout + (size_t)v * VE, make_uint4(0, 0, 0, 0));
      }
      cp[j] = any && xbuf != nullptr;
    }
    for (int v0 = 0; v0 < nvec; v0 += 32 * 4) {
      uint4 buf[RU][4];
#pragma unroll
      for (int j = 0; j < RU; ++j) {
        const T* src = x + (size_t)(t0 + b0 + j) * d;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int v = v0 + u * 32 + lane;
          if (cp[j] && v < nvec) buf[j][u] = ld_nc_v4(src + (size_t)v * VE);
        }
      }
#pragma unroll
      for (int j = 0; j < RU; ++j)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int v = v0 + u * 32 + lane;
          if (cp[j] && v < nvec)
#pragma unroll
            for (int q = 0; q < KM; ++q)
              if (dsts[j][q]) st_v4(dsts[j][q] + (size_t)v * VE, buf[j][u]);
        }
    }
  }
  // (no fence here: the exchange barrier kernel that follows on this stream releases, at
  // system scope, everything this kernel wrote -- see peer.h)
}

cudaError_t launch_dispatch(int dtype, const int32_t* idx, const void* x, int T, int k,
                            int n, int d, int64_t token_base, const CapTable& ct,
                            RouteBufs b, void* xbuf, const int32_t* pad_kept, cudaStream_t s,
                            int pad_e0, const PeerBufs& px, const PeerBufs& ptos,
                            const int32_t* pre_dev, void* y_zero, int dout) {
  if (T == 0 && !(pad_kept && px.nl)) return cudaSuccess;  // peer EP: own pads still zeroed
  int ntiles = std::max(1, (T + MOE_ROUTE_TILE - 1) / MOE_ROUTE_TILE);
  // top-1 with fewer routing tiles than two per SM: four tokens per warp in flight
  const bool small = k == 1 && ntiles < 2 * 148;  // B200: 148 SMs
#define DISP(TT, RU_, KM_)                                                                   \
  launch_pdl(dispatch_kernel<TT, RU_, KM_>, ntiles, 256, 0, s, idx, (const TT*)x, T, k, n, d, \
             token_base, ct, b.tile_off, b.slot_of, b.token_of_slot, (TT*)xbuf, pad_kept,    \
             pad_e0, px, ptos, pre_dev, (TT*)y_zero, dout)
  if (dtype == 1) {
    if (small) DISP(__nv_bfloat16, 4, 1); else DISP(__nv_bfloat16, 1, MOE_MAX_K);
  } else {
    if (small) DISP(float, 4, 1); else DISP(float, 1, MOE_MAX_K);
  }
#undef DISP
  return cudaGetLastError();
}

// Zero rows [kept_e, min(roundup(kept_e, PAD), region end)) of each local expert region so
// the token-contraction (weight-gradient) GEMMs can read whole K-blocks.
template <typename T>
__global__ void zero_pad_kernel(T* __restrict__ buf, int cols, const int32_t* __restrict__ kept,
                                CapTable ct) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  const int e = blockIdx.x;
  const int kp = kept[e];
  const int r0 = ct.base[e] + kp;
  const int r1 = min(ct.base[e] + ((kp + MOE_PAD_ROWS - 1) / MOE_PAD_ROWS) * MOE_PAD_ROWS,
                     ct.base[e + 1]);
  constexpr int VE = Vec<T>::N;
  const int nvec = cols / VE;
  const size_t total = (size_t)(r1 - r0) * nvec;
  for (size_t i = threadIdx.x; i < total; i += blockDim.x)
    st_v4(buf + (size_t)r0 * cols + i * VE, make_uint4(0, 0, 0, 0));
}

cudaError_t launch_zero_pad(int dtype, void* buf, int cols, const int32_t* kept, int n,
                            const CapTable& ct, cudaStream_t s) {
  if (dtype == 1)
    launch_pdl(zero_pad_kernel<__nv_bfloat16>, n, 256, 0, s, (__nv_bfloat16*)buf, cols, kept, ct);
  else
    launch_pdl(zero_pad_kernel<float>, n, 256, 0, s, (float*)buf, cols, kept, ct);
  return cudaGetLastError();
}

// =====================================================================================
// K5: combine (Alg. 1 l.8, Aggregate P:408): y[t] = sum_r [kept] w[t,r] O[row(t,r)],
// r ascending, fp32 accumulate; warp per token, 16-byte vectors.  VPL = 16-byte vectors per
// lane per row (d_out*s/512), KM = compile-time bound on k: all of a token's row loads are
// issued before the first use (two memory round trips per token: indices, then rows).
// =====================================================================================
template <typename T, int VPL, int KM>
__global__ void __launch_bounds__(256) combine_fwd_kernel(
    const T* __restrict__ obuf, const float* __restrict__ w, const int32_t* __restrict__ idx,
    const int32_t* __restrict__ slot_of, CapTable ct, int Tn, int k, int dout,
    T* __restrict__ y, T* __restrict__ spec, uint8_t* __restrict__ valid, PeerBufs po,
    int o_pair) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= Tn) return;
  constexpr int VE = Vec<T>::N;
  const int nvec = dout / VE;
  const T* src[KM];  // O row of each kept pair (peer EP: read from the owner over NVLink)
  const T* lsrc[KM]; // the row each load reads: with o_pair known before the routing tables
  float wr[KM];
#pragma unroll
  for (int r = 0; r < KM; ++r) {
    src[r] = nullptr;
    lsrc[r] = (o_pair && r < k) ? obuf + ((size_t)t * k + r) * dout : nullptr;
    wr[r] = 0.f;
    if (r < k) {
      const int sl = slot_of[(size_t)t * k + r];
      if (sl >= 0) {
        const int e = idx[(size_t)t * k + r];
        // o_pair (O in (token, choice) order, or peer EP return rows): the GEMM stored O at
        // this (token, choice) row
        src[r] = o_pair ? obuf + ((size_t)t * k + r) * dout
                        : peer_row(obuf, po, e, (size_t)(ct.base[e] + sl), dout);
        wr[r] = w[(size_t)t * k + r];
      }
      if (!o_pair) lsrc[r] = src[r];
    }
  }
  T* yrow = y + (size_t)t * dout;
  for (int vb = 0; vb < nvec; vb += VPL * 32) {
  uint4 u[KM][VPL];
#pragma unroll
  for (int r = 0; r < KM; ++r)
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int v = vb + j * 32 + lane;
      if (lsrc[r] && v < nvec) u[r][j] = ld_nc_v4(lsrc[r] + (size_t)v * VE);
    }
  if (spec) {  // AggregateSpec (App. A): the chosen experts' rows, zeros if dropped
#pragma unroll
    for (int r = 0; r < KM; ++r) {
      if (r >= k) break;
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int v = vb + j * 32 + lane;
        if (v < nvec)
          st_v4(spec + ((size_t)t * k + r) * dout + (size_t)v * VE,
                src[r] ? u[r][j] : make_uint4(0, 0, 0, 0));
      }
    }
  }
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int v = vb + j * 32 + lane;
    if (v >= nvec) continue;
    float acc[VE];
#pragma unroll
    for (int i = 0; i < VE; ++i) acc[i] = 0.f;
#pragma unroll
    for (int r = 0; r < KM; ++r) {
      if (!src[r]) continue;
      float o[VE];
      unpack(u[r][j], o, T());
#pragma unroll
      for (int i = 0; i < VE; ++i) acc[i] = fmaf(wr[r], o[i], acc[i]);
    }
    st_v4(yrow + (size_t)v * VE, pack(acc, T()));
  }
  }
  if (valid && lane < k) {
#pragma unroll
    for (int r = 0; r < KM; ++r)
      if (r == lane) valid[(size_t)t * k + r] = src[r] ? 1 : 0;
  }
}

// generic fallback (any d_out, any k): row loop
template <typename T>
__global__ void __launch_bounds__(256) combine_fwd_generic_kernel(
    const T* __restrict__ obuf, const float* __restrict__ w, const int32_t* __restrict__ idx,
    const int32_t* __restrict__ slot_of, CapTable ct, int Tn, int k, int dout,
    T* __restrict__ y, T* __restrict__ spec, uint8_t* __restrict__ valid, PeerBufs po,
    int o_pair) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= Tn) return;
  const T* rows[MOE_MAX_K];
  float wr[MOE_MAX_K];
  int nk = 0;
  const T* rsel[MOE_MAX_K];
  for (int r = 0; r < k; ++r) {
    int sl = slot_of[(size_t)t * k + r];
    rsel[r] = nullptr;
    if (sl >= 0) {
      const int e = idx[(size_t)t * k + r];
      rows[nk] = o_pair ? obuf + ((size_t)t * k + r) * dout
                        : peer_row(obuf, po, e, (size_t)(ct.base[e] + sl), dout);
      rsel[r] = rows[nk];
      wr[nk] = w[(size_t)t * k + r];
      ++nk;
    }
  }
  constexpr int VE = Vec<T>::N;
  const int nvec = dout / VE;
  T* yrow = y + (size_t)t * dout;
  for (int v = lane; v < nvec; v += 32) {
    float acc[VE];
#pragma unroll
    for (int i = 0; i < VE; ++i) acc[i] = 0.f;
    for (int q = 0; q < nk; ++q) {
      uint4 u = ld_nc_v4(rows[q] + (size_t)v * VE);
      float o[VE];
      unpack(u, o, T());
#pragma unroll
      for (int i = 0; i < VE; ++i) acc[i] = fmaf(wr[q], o[i], acc[i]);
    }
    st_v4(yrow + (size_t)v * VE, pack(acc, T()));
    if (spec)
      for (int r = 0; r < k; ++r)
        st_v4(spec + ((size_t)t * k + r) * dout + (size_t)v * VE,
              rsel[r] ? ld_nc_v4(rsel[r] + (size_t)v * VE) : make_uint4(0, 0, 0, 0));
  }
  if (valid && lane < k) valid[(size_t)t * k + lane] = slot_of[(size_t)t * k + lane] >= 0 ? 1 : 0;
}

template <typename T>
static cudaError_t combine_fwd_t(const void* obuf, RouteBufs b, int T_, int k, int d_out,
                                 const CapTable& ct, void* y, cudaStream_t s, const PeerBufs& po) {
  T* spec = (T*)b.spec;
  uint8_t* valid = b.spec_valid;
  dim3 grid((T_ + 7) / 8);
  const int vpl = (d_out / Vec<T>::N + 31) / 32;
#define CF(V, K)                                                                            \
  launch_pdl(combine_fwd_kernel<T, V, K>, grid, 256, 0, s, (const T*)obuf, b.w, b.idx, b.slot_of, ct, \
                                                   T_, k, d_out, (T*)y, spec, valid, po, b.o_pair)
  if (k <= 2) {
    if (vpl <= 2) { if (k == 1) CF(2, 1); else CF(2, 2); }
    else if (vpl <= 4) { if (k == 1) CF(4, 1); else CF(4, 2); }
    else { if (k == 1) CF(8, 1); else CF(8, 2); }
  } else {
    launch_pdl(combine_fwd_generic_kernel<T>, grid, 256, 0, s, (const T*)obuf, b.w, b.idx, b.slot_of, ct,
                                                       T_, k, d_out, (T*)y, spec, valid, po, b.o_pair);
  }
#undef CF
  return cudaGetLastError();
}

cudaError_t launch_combine_fwd(int dtype, const void* obuf, RouteBufs b, int T, int k,
                               int d_out, const CapTable& ct, void* y, cudaStream_t s,
                               const PeerBufs& po) {
  if (T == 0) return cudaSuccess;
  if (dtype == 1) return combine_fwd_t<__nv_bfloat16>(obuf, b, T, k, d_out, ct, y, s, po);
  return combine_fwd_t<float>(obuf, b, T, k, d_out, ct, y, s, po);
}

// =====================================================================================
// K6: combine backward.  dO[row] = w dy[t]; dw[t,r] = <dy[t], O[row]> (0 if dropped);
// dl[t,:] closed form: renorm dl[i_r] = w_r (dw_r - sum w dw), 0 elsewhere;
// raw dl_j = p_j (dp_j - sum_r w_r dw_r) with dp_j = dw_r at j = i_r.  Warp per token; the
// logits, dy and O rows are all requested before the first use.
// =====================================================================================
// NL = expert pairs per lane (n <= 64 NL); FEAT bit 0 (LOSS) = the loss-variant inputs (spec
// gradients, external dw, balance term), bit 1 (PEER) = peer-EP buffers (O / dO / dl rows at
// the experts' owners, pad zeroing of the owner's regions).  Features off are compiled out:
// fewer registers and instructions, same arithmetic; without LOSS the first block of the dy
// and (token-ordered) O rows is requested before the routing tables.
template <typename T, int VPL, int KM, int NL, int FEAT>
__global__ void __launch_bounds__(256, 4) combine_bwd_kernel(
    const T* __restrict__ dy, const T* __restrict__ obuf, const float* __restrict__ w,
    const int32_t* __restrict__ idx, const int32_t* __restrict__ slot_of,
    const float* __restrict__ logits, CapTable ct, int Tn, int k, int n, int dout, int renorm,
    T* __restrict__ dobuf, float* __restrict__ dw, float* __restrict__ dl,
    __nv_bfloat16* __restrict__ dlb, int maxT, int n_pad, const float4* __restrict__ sstat,
    const T* __restrict__ dspec_,
    const float* __restrict__ dw_ext_, const float* __restrict__ bal_g_,
    int32_t* __restrict__ grow, const int32_t* __restrict__ pad_kept, int pad_e0, PeerBufs po,
    PeerBufs pdo, __nv_bfloat16* __restrict__ dlr, PeerBufs pdlr, __nv_bfloat16* __restrict__ dropb,
    int32_t* __restrict__ drop_tok, int32_t* __restrict__ drop_cnt, int o_pair, int dx_pair) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  constexpr bool LOSS = (FEAT & 1) != 0, PEER = (FEAT & 2) != 0;
  const T* dspec = LOSS ? dspec_ : nullptr;
  const float* dw_ext = LOSS ? dw_ext_ : nullptr;
  const float* bal_g = LOSS ? bal_g_ : nullptr;
  // peer EP (N1): O rows are read from, and dO rows written to, the experts' owners
  if (pad_kept)
    zero_pads_block(dobuf, dout, pad_kept, ct, (PEER && pdo.nl) ? pdo.nl : n, pad_e0, blockIdx.x,
                    gridDim.x);
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= Tn) return;
  constexpr int VE = Vec<T>::N;
  const bool need_p = !renorm || bal_g != nullptr;  // full softmax row needed
  const int nvec = dout / VE;
  const T* dyrow = dy + (size_t)t * dout;
  // Everything that does not depend on the routing tables is requested first, so the
  // slot / index loads overlap the row loads instead of preceding them: the statistics and
  // logits row, and (lean path) the first block of the dy row and -- O in (token, choice)
  // order -- of the O rows.
  uint4 g[VPL];
  uint4 u[KM][VPL];
  if (!LOSS) {
#pragma unroll
    for (int jv = 0; jv < VPL; ++jv) {
      const int v = jv * 32 + lane;
      if (v < nvec) g[jv] = ld_nc_v4(dyrow + (size_t)v * VE);
    }
    if (o_pair) {
#pragma unroll
      for (int r = 0; r < KM; ++r)
#pragma unroll
        for (int jv = 0; jv < VPL; ++jv) {
          const int v = jv * 32 + lane;
          if (r < k && v < nvec) u[r][jv] = ld_nc_v4(obuf + ((size_t)t * k + r) * dout + (size_t)v * VE);
        }
    }
  }
  float4 st4 = make_float4(0.f, 0.f, 0.f, 0.f);
  if (need_p && sstat != nullptr) st4 = sstat[t];
  // this lane's experts: pairs e = 2*lane + 64*j (+1)
  float lg[NL][2];
  const float* l = logits + (size_t)t * n;
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const int e = 2 * lane + 64 * j;
    lg[j][0] = (need_p && e < n) ? l[e] : -INFINITY;
    lg[j][1] = (need_p && e + 1 < n) ? l[e + 1] : -INFINITY;
  }
  int rows[KM], er[KM];
  float wr[KM], part[KM];
  const T* osrc[KM];
  T* odst[KM];
#pragma unroll
  for (int r = 0; r < KM; ++r) {
    rows[r] = -1; er[r] = -1; wr[r] = 0.f; part[r] = 0.f;
    osrc[r] = nullptr; odst[r] = nullptr;
    if (r < k) {
      const int sl = slot_of[(size_t)t * k + r];
      er[r] = idx[(size_t)t * k + r];
      rows[r] = sl >= 0 ? ct.base[er[r]] + sl : -1;
      wr[r] = w[(size_t)t * k + r];
      // o_pair (O in (token, choice) order: MOE_FUSE_OTOK, or peer EP return rows): the row
      // address needs no routing table, so its load is issued unconditionally, concurrently
      // with the slot / index loads (a dropped pair's row is unwritten and never used)
      if (o_pair) osrc[r] = obuf + ((size_t)t * k + r) * dout;
      if (rows[r] >= 0) {
        if (!o_pair)
          osrc[r] = PEER ? peer_row(obuf, po, er[r], (size_t)rows[r], dout)
                         : obuf + (size_t)rows[r] * dout;
        odst[r] = PEER ? peer_row(dobuf, pdo, er[r], (size_t)rows[r], dout)
                       : dobuf + (size_t)rows[r] * dout;
      }
    }
  }
  // fused dX (k = 1): a token whose pair was dropped gets a row of the compacted drop list
  // (its dl pair is the A operand of the drop-only gate-dx pass); order is immaterial
  int dpos = -1;
  if (KM == 1 && dropb != nullptr && rows[0] < 0) {
    if (lane == 0) {
      dpos = atomicAdd(drop_cnt, 1);
      drop_tok[dpos] = t;
    }
    dpos = __shfl_sync(0xffffffffu, dpos, 0);
  }
  for (int vb = 0; vb < nvec; vb += VPL * 32) {  // one pass for d_out*s <= 512*VPL bytes
  const bool early = !LOSS && vb == 0;  // the lean path's first block is already in flight
#pragma unroll
  for (int jv = 0; jv < VPL; ++jv) {
    const int v = vb + jv * 32 + lane;
    if (!early && v < nvec) g[jv] = ld_nc_v4(dyrow + (size_t)v * VE);
  }
#pragma unroll
  for (int r = 0; r < KM; ++r)
#pragma unroll
    for (int jv = 0; jv < VPL; ++jv) {
      const int v = vb + jv * 32 + lane;
      if (!(early && o_pair) && osrc[r] != nullptr && v < nvec)
        u[r][jv] = ld_nc_v4(osrc[r] + (size_t)v * VE);
    }
#pragma unroll
  for (int jv = 0; jv < VPL; ++jv) {
    const int v = vb + jv * 32 + lane;
    if (v >= nvec) continue;
    float gv[VE];
    unpack(g[jv], gv, T());
#pragma unroll
    for (int r = 0; r < KM; ++r) {
      if (rows[r] < 0) continue;
      float o[VE], dov[VE], ds[VE];
      unpack(u[r][jv], o, T());
      if (dspec) {  // specification-loss gradient of this (token, expert) row
        unpack(ld_nc_v4(dspec + ((size_t)t * k + r) * dout + (size_t)v * VE), ds, T());
      } else {
#pragma unroll
        for (int i = 0; i < VE; ++i) ds[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < VE; ++i) {
        part[r] = fmaf(gv[i], o[i], part[r]);
        dov[i] = fmaf(wr[r], gv[i], ds[i]);
      }
      st_v4(odst[r] + (size_t)v * VE, pack(dov, T()));
    }
  }
  }
  float dwr[KM];
  float c = 0.f;
#pragma unroll
  for (int r = 0; r < KM; ++r) {
    float sr = warp_sum(part[r]);
    sr = __shfl_sync(0xffffffffu, sr, 0);
    dwr[r] = rows[r] >= 0 ? sr + (dw_ext ? dw_ext[(size_t)t * k + r] : 0.f) : 0.f;
    c = fmaf(wr[r], dwr[r], c);
  }
#pragma unroll
  for (int r = 0; r < KM; ++r)
    if (r < k && lane == r) {
      dw[(size_t)t * k + r] = dwr[r];
      if (grow)  // the gate-dx kernel's gather table (peer EP: owner in the top bits; with
                 // return rows the dX row is this rank's own (token, choice) row)
        grow[(size_t)t * k + r] = rows[r] < 0 ? -1
                                  : dx_pair ? (int)((size_t)t * k + r)
                                  : (PEER && pdo.nl) ? rows[r] | ((er[r] / pdo.nl) << MOE_GROW_SHIFT)
                                           : rows[r];
    }
  float m = -INFINITY, sp = 0.f, cb = 0.f;
  float ens = 0.f;     // raw mode: exp mass of the experts NOT selected for this token
  float esel[KM];      // raw mode: exp(l - m) of each selected expert
  if (need_p && sstat != nullptr) {
    // the tcgen05 gate's statistics of this row (max, sum, mass outside the dispatch set):
    // no warp reductions here, and ens was summed without cancellation
    m = st4.x;
    sp = st4.y;
    ens = st4.z;
  } else if (need_p) {
#pragma unroll
    for (int j = 0; j < NL; ++j) m = fmaxf(m, fmaxf(lg[j][0], lg[j][1]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
#pragma unroll
    for (int j = 0; j < NL; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = 2 * lane + 64 * j + h;
        if (e >= n) continue;
        const float ex = expf(lg[j][h] - m);
        sp += ex;
        bool sel = false;
#pragma unroll
        for (int r = 0; r < KM; ++r) sel |= (r < k && er[r] == e);
        if (!sel) ens += ex;
      }
    }
    sp = __shfl_sync(0xffffffffu, warp_sum(sp), 0);
    ens = __shfl_sync(0xffffffffu, warp_sum(ens), 0);
  }
  if (need_p) {
#pragma unroll
    for (int r = 0; r < KM; ++r)
      esel[r] = (r < k && er[r] >= 0 && er[r] < n) ? expf(l[er[r]] - m) : 0.f;
    if (bal_g) {  // Eq. 3 balance term: dB/dl = p (g - <p, g>), g_i = lambda n T_i / T_g
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const int e = 2 * lane + 64 * j;
        if (e < n) cb = fmaf(expf(lg[j][0] - m) / sp, bal_g[e], cb);
        if (e + 1 < n) cb = fmaf(expf(lg[j][1] - m) / sp, bal_g[e + 1], cb);
      }
      cb = __shfl_sync(0xffffffffu, warp_sum(cb), 0);
    }
  }
  float* dlrow = dl + (size_t)t * n;
  const int ncols = dlb ? n_pad : n;
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const int e0 = 2 * lane + 64 * j;
    if (e0 >= ncols) continue;
    float v2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = e0 + h;
      float v = 0.f;
      if (e < n) {
        // The closed forms rewritten without the cancellation of dw_r against sum w dw (a
        // confident router, w_r -> 1, would otherwise lose every significant digit of dl in
        // fp32): renorm dl_r = w_r (dw_r - sum_s w_s dw_s) = w_r sum_{s != r} w_s (dw_r - dw_s)
        // since sum w = 1; raw dl_j = p_j (dp_j - sum_s p_s dw_s) with 1 - p_j expanded as the
        // exp mass of every other expert.  Same value in exact arithmetic.
        if (renorm) {
#pragma unroll
          for (int r = 0; r < KM; ++r) {
            if (r >= k || er[r] != e) continue;
            float a = 0.f;
#pragma unroll
            for (int s2 = 0; s2 < KM; ++s2)
              if (s2 < k && s2 != r) a = fmaf(wr[s2], dwr[r] - dwr[s2], a);
            v = wr[r] * a;
          }
        } else {
          const float p = expf(lg[j][h] - m) / sp;
          int rs = -1;
#pragma unroll
          for (int r = 0; r < KM; ++r)
            if (r < k && er[r] == e) rs = r;
          if (rs < 0) {
            v = -p * c;
          } else {
            float osum = ens, other = 0.f;
            float dws = 0.f;
#pragma unroll
            for (int s2 = 0; s2 < KM; ++s2) {
              if (s2 >= k) continue;
              if (s2 == rs) {
                dws = dwr[s2];
              } else {
                osum += esel[s2];
                other = fmaf(wr[s2], dwr[s2], other);
              }
            }
            v = p * (dws * (osum / sp) - other);
          }
        }
        if (bal_g) v = fmaf(expf(lg[j][h] - m) / sp, bal_g[e] - cb, v);
        dlrow[e] = v;
      }
      v2[h] = v;
    }
    if (dlb) {  // exact-ish bf16 pair for the tensor-core gate gradients: v = hi + lo
      const __nv_bfloat162 hi = __floats2bfloat162_rn(v2[0], v2[1]);
      const __nv_bfloat162 lo =
          __floats2bfloat162_rn(v2[0] - __low2float(hi), v2[1] - __high2float(hi));
      *reinterpret_cast<__nv_bfloat162*>(dlb + (size_t)t * n_pad + e0) = hi;
      *reinterpret_cast<__nv_bfloat162*>(dlb + ((size_t)maxT + t) * n_pad + e0) = lo;
      if (dlr && rows[0] >= 0) {  // k = 1 fused dispatch backward: the pair by expert row
        __nv_bfloat16* rr = PEER ? peer_row(dlr, pdlr, er[0], (size_t)rows[0], 2 * n_pad)
                                 : dlr + (size_t)rows[0] * 2 * n_pad;
        *reinterpret_cast<__nv_bfloat162*>(rr + e0) = hi;
        *reinterpret_cast<__nv_bfloat162*>(rr + n_pad + e0) = lo;
      }
      if (dpos >= 0) {  // dropped token: its pair in the compacted drop list (dlb layout)
        *reinterpret_cast<__nv_bfloat162*>(dropb + (size_t)dpos * n_pad + e0) = hi;
        *reinterpret_cast<__nv_bfloat162*>(dropb + ((size_t)maxT + dpos) * n_pad + e0) = lo;
      }
    }
  }
}

template <typename T>
static cudaError_t combine_bwd_t(const void* dy, const void* obuf, RouteBufs b, int T_, int k,
                                 int n, int d_out, int renorm, const CapTable& ct, void* dobuf,
                                 void* dlb, int maxT, int n_pad, const int32_t* pad_kept,
                                 cudaStream_t s, int pad_e0, const PeerBufs& po,
                                 const PeerBufs& pdo) {
  dim3 grid(std::max(1, (T_ + 7) / 8));
  const int vpl = (d_out / Vec<T>::N + 31) / 32;  // > 8: the kernel loops over 4 KB blocks
#define CB(V, K, NLL, F)                                                                       \
  launch_pdl(combine_bwd_kernel<T, V, K, NLL, F>, grid, 256, 0, s, (const T*)dy, (const T*)obuf, \
             b.w, b.idx, b.slot_of, b.logits, ct, T_, k, n, d_out, renorm, (T*)dobuf, b.dw,    \
             b.dl, (__nv_bfloat16*)dlb, maxT, n_pad, (const float4*)b.sstat,                   \
             (const T*)b.dspec, b.dw_ext, b.bal_g, b.grow, pad_kept, pad_e0, po, pdo, b.dlr,   \
             b.pdlr, b.dropb, b.drop_tok, b.drop_cnt, b.o_pair, b.dx_pair)
  const int km = k == 1 ? 1 : (k == 2 ? 2 : 8);
  // single-GPU product path (bf16, k <= 2, no loss variants, no peer buffers): the lean
  // instantiation, <= 4 vectors per lane per pass (the same per-lane order of the dot
  // products as one wider pass), NL = ceil(n / 64)
  const bool lean = sizeof(T) == 2 && km <= 2 && !b.dspec && !b.dw_ext && !b.bal_g;
  if (lean) {
    const int nl = n <= 64 ? 1 : (n <= 128 ? 2 : 4);
    const bool peer = po.nl || pdo.nl || b.pdlr.nl;
#define CBL(V, K)                                                            \
    {                                                                        \
      if (peer) {                                                            \
        if (nl == 1) CB(V, K, 1, 2);                                         \
        else if (nl == 2) CB(V, K, 2, 2);                                    \
        else CB(V, K, 4, 2);                                                 \
      } else {                                                               \
        if (nl == 1) CB(V, K, 1, 0);                                         \
        else if (nl == 2) CB(V, K, 2, 0);                                    \
        else CB(V, K, 4, 0);                                                 \
      }                                                                      \
    }
    if (km == 2) CBL(2, 2)  // (2 vectors per lane per pass: no spills at k = 2)
    else if (vpl <= 2) CBL(2, 1)
    else CBL(4, 1)
#undef CBL
    return cudaGetLastError();
  }
  if (vpl <= 2) { if (km == 1) CB(2, 1, 4, 3); else if (km == 2) CB(2, 2, 4, 3); else CB(2, 8, 4, 3); }
  else if (vpl <= 4) { if (km == 1) CB(4, 1, 4, 3); else if (km == 2) CB(4, 2, 4, 3); else CB(4, 8, 4, 3); }
  else { if (km == 1) CB(8, 1, 4, 3); else if (km == 2) CB(8, 2, 4, 3); else CB(8, 8, 4, 3); }
#undef CB
  return cudaGetLastError();
}

cudaError_t launch_combine_bwd(int dtype, const void* dy, const void* obuf, RouteBufs b,
                               int T, int k, int n, int d_out, int renorm,
                               const CapTable& ct, void* dobuf, void* dlb, int maxT, int n_pad,
                               const int32_t* pad_kept, cudaStream_t s, int pad_e0,
                               const PeerBufs& po, const PeerBufs& pdo) {
  if (T == 0 && !(pad_kept && pdo.nl)) return cudaSuccess;  // peer EP: own pads still zeroed
  if (dtype == 1)
    return combine_bwd_t<__nv_bfloat16>(dy, obuf, b, T, k, n, d_out, renorm, ct, dobuf, dlb,
                                        maxT, n_pad, pad_kept, s, pad_e0, po, pdo);
  return combine_bwd_t<float>(dy, obuf, b, T, k, n, d_out, renorm, ct, dobuf, dlb, maxT, n_pad,
                              pad_kept, s, pad_e0, po, pdo);
}

// Peer EP fused dispatch backward (k = 1): copy the returned dx rows of the kept tokens
// (warp per token, 16-byte vectors; + the old dx when accumulating).
__global__ void __launch_bounds__(256) dx_from_ret_kernel(
    const __nv_bfloat16* __restrict__ ret, const int32_t* __restrict__ slot_of, int Tn, int d,
    __nv_bfloat16* __restrict__ dx, int accumulate) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= Tn || slot_of[t] < 0) return;
  for (int c = lane * 8; c < d; c += 256) {
    uint4 v = ld_nc_v4(ret + (size_t)t * d + c);
    if (accumulate) {
      float a[8], o[8];
      unpack(v, a, __nv_bfloat16());
      unpack(ld_v4(dx + (size_t)t * d + c), o, __nv_bfloat16());
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] += o[j];
      v = pack(a, __nv_bfloat16());
    }
    st_v4(dx + (size_t)t * d + c, v);
  }
}

cudaError_t launch_dx_from_ret(const void* dxret, const int32_t* slot_of, int T, int d, void* dx,
                               int accumulate, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  launch_pdl(dx_from_ret_kernel, (T + 7) / 8, 256, 0, s, (const __nv_bfloat16*)dxret, slot_of, T,
             d, (__nv_bfloat16*)dx, accumulate);
  return cudaGetLastError();
}

// =====================================================================================
// K9: dispatch backward with the gate input-gradient fused in:
//   dx[t] = sum_r [kept] dX[row(t,r)] + sum_e dl[t,e] W_g[e,:]     (fp32 accumulate)
// CTA = 32 tokens x 128 columns; W_g / dl chunks staged in shared memory.
// =====================================================================================
template <typename T>
__global__ void __launch_bounds__(256) gate_dx_kernel(
    const float* __restrict__ dl, const T* __restrict__ wg, const T* __restrict__ dxbuf,
    const int32_t* __restrict__ idx, const int32_t* __restrict__ slot_of, CapTable ct, int Tn,
    int k, int n, int d, T* __restrict__ dx, int accumulate, PeerBufs pdx) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  __shared__ float dls[32][33];
  __shared__ float wgs[32][128];
  const int tid = threadIdx.x;
  const int c = tid & 31, tg = tid >> 5;
  const int t0 = blockIdx.y * 32, c0 = blockIdx.x * 128;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int e0 = 0; e0 < n; e0 += 32) {
    for (int i = tid; i < 32 * 32; i += 256) {
      int tt = i / 32, ee = i % 32;
      int t = t0 + tt, e = e0 + ee;
      dls[tt][ee] = (t < Tn && e < n) ? dl[(size_t)t * n + e] : 0.f;
    }
    for (int i = tid; i < 32 * 128; i += 256) {
      int ee = i / 128, cc = i % 128;
      int e = e0 + ee, col = c0 + cc;
      wgs[ee][cc] = (e < n && col < d) ? to_f(wg[(size_t)e * d + col]) : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int ee = 0; ee < 32; ++ee) {
      float wv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) wv[j] = wgs[ee][c + 32 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float lv = dls[tg + 8 * i][ee];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(lv, wv[j], acc[i][j]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + tg + 8 * i;
    if (t >= Tn) continue;
    float out[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) out[j] = 0.f;
    // expert-path contribution first (r order), then the gate term: fixed order
    for (int r = 0; r < k; ++r) {
      int sl = slot_of[(size_t)t * k + r];
      if (sl < 0) continue;
      const int e = idx[(size_t)t * k + r];
      const T* src = peer_row(dxbuf, pdx, e, (size_t)(ct.base[e] + sl), d);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int col = c0 + c + 32 * j;
        if (col < d) out[j] += to_f(src[col]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int col = c0 + c + 32 * j;
      if (col >= d) continue;
      float v = out[j] + acc[i][j];
      if (accumulate) v += to_f(dx[(size_t)t * d + col]);
      dx[(size_t)t * d + col] = from_f<T>(v);
    }
  }
}

cudaError_t launch_gate_dx(int dtype, const void* wg, const void* dxbuf, RouteBufs b, int T,
                           int k, int n, int d, const CapTable& ct, void* dx, int accumulate,
                           cudaStream_t s, const PeerBufs& pdx) {
  if (T == 0) return cudaSuccess;
  dim3 grid((d + 127) / 128, (T + 31) / 32);
  if (dtype == 1)
    launch_pdl(gate_dx_kernel<__nv_bfloat16>, grid, 256, 0, s, 
        b.dl, (const __nv_bfloat16*)wg, (const __nv_bfloat16*)dxbuf, b.idx, b.slot_of, ct, T, k,
        n, d, (__nv_bfloat16*)dx, accumulate, pdx);
  else
    launch_pdl(gate_dx_kernel<float>, grid, 256, 0, s, b.dl, (const float*)wg, (const float*)dxbuf,
                                               b.idx, b.slot_of, ct, T, k, n, d, (float*)dx,
                                               accumulate, pdx);
  return cudaGetLastError();
}

// =====================================================================================
// K10: gate weight gradient dW_g = dl^T x, deterministic split-K over tokens:
// partial[s][e][c] over token range s, then a fixed-order reduction over s.
// CTA = 64 columns x all n experts; thread = 1 column x n/4 experts.
// =====================================================================================
template <typename T, int NJ>
__global__ void __launch_bounds__(256) gate_dw_kernel(const float* __restrict__ dl,
                                                      const T* __restrict__ x, int Tn, int n,
                                                      int d, int chunk,
                                                      float* __restrict__ partial, int nowait) {
  pdl_enter(nowait);  // PDL (nowait: the backward tail, see launch_gate_dw_tc / moe_api)
  extern __shared__ float sm[];
  float* xs = sm;                 // [32][64]
  float* ls = sm + 32 * 64;       // [32][n]
  const int tid = threadIdx.x;
  const int col = tid & 63, eg = tid >> 6;
  const int c0 = blockIdx.x * 64;
  const int ts = blockIdx.y * chunk, te = min(Tn, ts + chunk);
  float acc[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) acc[j] = 0.f;
  for (int t0 = ts; t0 < te; t0 += 32) {
    for (int i = tid; i < 32 * 64; i += 256) {
      int tt = i / 64, cc = i % 64;
      int t = t0 + tt, cl = c0 + cc;
      xs[i] = (t < te && cl < d) ? to_f(x[(size_t)t * d + cl]) : 0.f;
    }
    for (int i = tid; i < 32 * n; i += 256) {
      int tt = i / n, e = i % n;
      int t = t0 + tt;
      ls[i] = (t < te) ? dl[(size_t)t * n + e] : 0.f;
    }
    __syncthreads();
    for (int tt = 0; tt < 32; ++tt) {
      float xv = xs[tt * 64 + col];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        int e = eg + 4 * j;
        if (e < n) acc[j] = fmaf(ls[tt * n + e], xv, acc[j]);
      }
    }
    __syncthreads();
  }
  const int cl = c0 + col;
  if (cl < d) {
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      int e = eg + 4 * j;
      if (e < n) partial[((size_t)blockIdx.y * n + e) * d + cl] = acc[j];
    }
  }
}

// out[i] = sum_q partial[q][i] (+ out[i]).  32 elements per block; warp g sums the splits
// q = g, g + 8, ... with all of its loads in flight (a serial chain of `splits` dependent
// L2 round trips was the kernel's whole cost), then warp 0 adds the 8 group sums in fixed
// order: deterministic.
template <typename T>
__global__ void __launch_bounds__(256) reduce_partials_kernel(const float* __restrict__ partial,
                                                              int splits, size_t count,
                                                              T* __restrict__ out, int accumulate) {
  pdl_enter();  // PDL: predecessor complete + visible (a no-op for a full-dependency launch)
  __shared__ float sg[8][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const size_t i = (size_t)blockIdx.x * 32 + lane;
  float s = 0.f;
  if (i < count) {
    for (int q0 = g; q0 < splits; q0 += 64) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int q = q0 + 8 * j;
        v[j] = q < splits ? __ldg(partial + (size_t)q * count + i) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[j];
    }
  }
  sg[g][lane] = s;
  __syncthreads();
  if (g != 0 || i >= count) return;
  float t = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) t += sg[q][lane];
  if (accumulate) t += to_f(out[i]);
  out[i] = from_f<T>(t);
}

cudaError_t launch_reduce_partials(int dtype, const float* partial, int splits, size_t count,
                                   void* out, int accumulate, cudaStream_t s, bool full_dep) {
  int rb = (int)((count + 31) / 32);
  if (dtype == 1) {
    auto kf = reduce_partials_kernel<__nv_bfloat16>;
    if (full_dep) launch_full(kf, rb, 256, 0, s, partial, splits, count, (__nv_bfloat16*)out, accumulate);
    else launch_pdl(kf, rb, 256, 0, s, partial, splits, count, (__nv_bfloat16*)out, accumulate);
  } else {
    auto kf = reduce_partials_kernel<float>;
    if (full_dep) launch_full(kf, rb, 256, 0, s, partial, splits, count, (float*)out, accumulate);
    else launch_pdl(kf, rb, 256, 0, s, partial, splits, count, (float*)out, accumulate);
  }
  return cudaGetLastError();
}

int gate_dw_splits(int T, int d) {
  int ctiles = (d + 63) / 64;
  int want = (2 * 148 + ctiles - 1) / ctiles;
  int maxs = (T + 63) / 64;  // >= 64 tokens per split: small T still fills the GPU
  return max(1, min(want, maxs));
}

cudaError_t launch_gate_dw(int dtype, const float* dl, const void* x, int T, int n, int d,
                           float* partial, int splits, void* dwg, int accumulate,
                           cudaStream_t s, float* f32_out, bool nowait) {
  const int nw = nowait ? 1 : 0;
  size_t count = (size_t)n * d;
  if (f32_out && T == 0) return cudaMemsetAsync(f32_out, 0, count * 4, s);
  if (T == 0) {
    if (!accumulate) return cudaMemsetAsync(dwg, 0, count * (dtype == 1 ? 2 : 4), s);
    return cudaSuccess;
  }
  int chunk = (T + splits - 1) / splits;
  chunk = ((chunk + 31) / 32) * 32;
  splits = (T + chunk - 1) / chunk;
  dim3 grid((d + 63) / 64, splits);
  size_t smem = (size_t)(32 * 64 + 32 * n) * 4;
#define GDW_CASE(NJ)                                                                        \
  if (n <= 4 * NJ) {                                                                        \
    if (dtype == 1) {                                                                       \
      auto kf = gate_dw_kernel<__nv_bfloat16, NJ>;                                          \
      cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
      launch_pdl(kf, grid, 256, smem, s, dl, (const __nv_bfloat16*)x, T, n, d, chunk, partial, nw);  \
    } else {                                                                                \
      auto kf = gate_dw_kernel<float, NJ>;                                                  \
      cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
      launch_pdl(kf, grid, 256, smem, s, dl, (const float*)x, T, n, d, chunk, partial, nw);         \
    }                                                                                       \
  } else
  GDW_CASE(2) GDW_CASE(4) GDW_CASE(8) GDW_CASE(16) GDW_CASE(32) GDW_CASE(64) {
    return cudaErrorInvalidValue;
  }
#undef GDW_CASE
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  if (f32_out) return launch_reduce_partials(0, partial, splits, count, f32_out, 0, s);
  return launch_reduce_partials(dtype, partial, splits, count, dwg, accumulate, s, nowait);
}

template <typename T>
__global__ void f32_to_kernel(const float* __restrict__ in, size_t count, T* __restrict__ out,
                              int accumulate) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  float v = in[i];
  if (accumulate) v += to_f(out[i]);
  out[i] = from_f<T>(v);
}

cudaError_t launch_f32_to(int dtype, const float* in, size_t count, void* out, int accumulate,
                          cudaStream_t s) {
  int rb = (int)((count + 255) / 256);
  if (dtype == 1)
    launch_pdl(f32_to_kernel<__nv_bfloat16>, rb, 256, 0, s, in, count, (__nv_bfloat16*)out, accumulate);
  else
    launch_pdl(f32_to_kernel<float>, rb, 256, 0, s, in, count, (float*)out, accumulate);
  return cudaGetLastError();
}

// =====================================================================================
// Bias gradients (SIMT path): db[e][j] = sum_{s < kept_e} buf[base_e + s][j], sequential
// over rows (deterministic), thread per column.
// =====================================================================================
template <typename T>
__global__ void colsum_kernel(const T* __restrict__ buf, int cols,
                              const int32_t* __restrict__ kept, CapTable ct,
                              T* __restrict__ out, int accumulate) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  const int e = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  const int m = kept[e];
  const T* p = buf + (size_t)ct.base[e] * cols + j;
  float s = 0.f;
  int r = 0;
  for (; r + 8 <= m; r += 8) {  // eight row loads in flight, added in row order
    float q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = to_f(p[(size_t)(r + i) * cols]);
#pragma unroll
    for (int i = 0; i < 8; ++i) s += q[i];
  }
  for (; r < m; ++r) s += to_f(p[(size_t)r * cols]);
  if (accumulate) s += to_f(out[(size_t)e * cols + j]);
  out[(size_t)e * cols + j] = from_f<T>(s);
}

cudaError_t launch_colsum(int dtype, const void* buf, int cols, const int32_t* kept, int n,
                          const CapTable& ct, void* out, int accumulate, cudaStream_t s) {
  dim3 grid((cols + 255) / 256, n);
  if (dtype == 1)
    launch_pdl(colsum_kernel<__nv_bfloat16>, grid, 256, 0, s, (const __nv_bfloat16*)buf, cols, kept,
                                                      ct, (__nv_bfloat16*)out, accumulate);
  else
    launch_pdl(colsum_kernel<float>, grid, 256, 0, s, (const float*)buf, cols, kept, ct, (float*)out,
                                              accumulate);
  return cudaGetLastError();
}

}  // namespace moe
