// combine_bwd_bulk.cu -- K6 combine backward (B1) with bulk-copy row staging (bf16, k <= 2).
//
//   dO[row(t,r)] = w[t,r] dy[t];   dw[t,r] = <dy[t], O[row(t,r)]> (0 if dropped);
//   dl[t,:] closed forms (renorm / raw, + Eq. 3 balance term), and the bf16 hi|lo pair of dl
//   for the tensor-core gate gradients -- the same arithmetic, in the same order, as
//   combine_bwd_kernel (route_kernels.cu), so the two are bitwise equal.
//
// OPT-IN (MOE_CB_BULK=1), not the default: measured SLOWER than the register-staged kernel.
// The idea: the warp-per-token form keeps a token's dy / O rows in registers, so the bytes in
// flight per SM are bounded by the register file and every warp idles through its metadata ->
// data -> dl phases (0.66 of HBM at c3).  Here each warp is persistent over a contiguous token
// range and runs an S-deep ring of shared-memory stages: lane 0 issues cp.async.bulk copies
// (dy row, the kept O rows, the logits row) for token i+S while the warp consumes token i
// from shared memory.  Measured at c3 (bench, CUDA events): 16 warps x 1 stage
// per SM 100 us (= the register form), 16 x 2 111 us, 12 x 3 131 us, 8 x 5 170 us, 4 x 8
// 279 us -- time scales with 1 / (warps per SM), not with the bytes in flight: the per-token
// instruction chain of a warp (dot product, dO stores, softmax / dl closed forms, several
// warp reductions; ~900 warp instructions per token, issue slots 60 % busy in ncu) bounds
// it, and fewer resident warps hide it less.  Kept as a tested, bitwise-equal alternative.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace moe {

namespace {

constexpr int CBB_MAXK = 2;

struct CbbMeta {          // one token's routing metadata (shared memory, per warp ring of 64)
  int32_t row[CBB_MAXK];  // expert-region row of each pair, -1 = dropped
  int32_t e[CBB_MAXK];
  float w[CBB_MAXK];
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct CbbParams {
  const __nv_bfloat16* dy;
  const __nv_bfloat16* obuf;
  const float* w;
  const int32_t* idx;
  const int32_t* slot_of;
  const float* logits;
  int Tn, k, n, dout, renorm;
  __nv_bfloat16* dobuf;
  float* dw;
  float* dl;
  __nv_bfloat16* dlb;
  int maxT, n_pad;
  const float* dw_ext;
  const float* bal_g;
  int32_t* grow;
  const int32_t* pad_kept;
  int pad_e0;
  PeerBufs pdo;
  __nv_bfloat16* dlr;
  PeerBufs pdlr;
  __nv_bfloat16* dropb;
  int32_t* drop_tok;
  int32_t* drop_cnt;
  int o_pair;
  int stages;            // S
  int stage_bytes;       // dy row + KM O rows + logits row, 128-byte aligned pieces
  int row_bytes;         // dout * 2
  int lg_bytes;          // n * 4 (0: logits read from global)
  int per_warp;          // tokens per warp (contiguous range)
};

template <int KM>
__global__ void __launch_bounds__(512, 1) combine_bwd_bulk_kernel(CbbParams p, CapTable ct) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  extern __shared__ __align__(128) uint8_t smem_raw[];
  if (p.pad_kept)
    zero_pads_block(p.dobuf, p.dout, p.pad_kept, ct, p.pdo.nl ? p.pdo.nl : p.n, p.pad_e0,
                    blockIdx.x, gridDim.x);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int S = p.stages;
  // per-warp carve-out: [S stages][S mbarriers][64 metadata entries]
  const size_t warp_bytes = (size_t)S * p.stage_bytes + 8 * S + 64 * sizeof(CbbMeta);
  uint8_t* base = smem_raw + (size_t)wid * ((warp_bytes + 127) & ~size_t(127));
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + (size_t)S * p.stage_bytes);
  CbbMeta* meta = reinterpret_cast<CbbMeta*>(bars + S);
  const int gw = blockIdx.x * nw + wid;
  const int t_begin = gw * p.per_warp;
  const int t_end = min(p.Tn, t_begin + p.per_warp);
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (t_begin >= t_end) return;
  const int k = p.k, n = p.n, dout = p.dout;
  const bool need_p = !p.renorm || p.bal_g != nullptr;

  // metadata batch b (tokens t_begin + 32 b + lane) -> ring slot (b & 1)
  auto load_meta = [&](int b) {
    const int t = t_begin + 32 * b + lane;
    CbbMeta m;
#pragma unroll
    for (int r = 0; r < CBB_MAXK; ++r) { m.row[r] = -1; m.e[r] = -1; m.w[r] = 0.f; }
    if (t < t_end) {
#pragma unroll
      for (int r = 0; r < KM; ++r) {
        if (r < k) {
          const int sl = p.slot_of[(size_t)t * k + r];
          m.e[r] = p.idx[(size_t)t * k + r];
          m.row[r] = sl >= 0 ? ct.base[m.e[r]] + sl : -1;
          m.w[r] = p.w[(size_t)t * k + r];
        }
      }
    }
    meta[(b & 1) * 32 + lane] = m;
  };
  auto issue = [&](int i) {  // lane 0: copies of token t_begin + i into stage i % S
    const int t = t_begin + i;
    if (t >= t_end) return;
    const CbbMeta& m = meta[(i & 63)];
    uint8_t* st = base + (size_t)(i % S) * p.stage_bytes;
    uint32_t bytes = 0;
    bool any = false;
#pragma unroll
    for (int r = 0; r < KM; ++r) any |= (r < k && m.row[r] >= 0);
    if (any) bytes += p.row_bytes;
#pragma unroll
    for (int r = 0; r < KM; ++r)
      if (r < k && m.row[r] >= 0) bytes += p.row_bytes;
    if (need_p && p.lg_bytes) bytes += p.lg_bytes;
    mbar_expect_tx(&bars[i % S], bytes);
    if (any) bulk_g2s(st, p.dy + (size_t)t * dout, p.row_bytes, &bars[i % S]);
#pragma unroll
    for (int r = 0; r < KM; ++r)
      if (r < k && m.row[r] >= 0) {
        const __nv_bfloat16* src = p.o_pair ? p.obuf + ((size_t)t * k + r) * dout
                                            : p.obuf + (size_t)m.row[r] * dout;
        bulk_g2s(st + (size_t)(1 + r) * p.row_bytes, src, p.row_bytes, &bars[i % S]);
      }
    if (need_p && p.lg_bytes)
      bulk_g2s(st + (size_t)(1 + KM) * p.row_bytes, p.logits + (size_t)t * n, p.lg_bytes,
               &bars[i % S]);
  };

  const int cnt = t_end - t_begin;
  load_meta(0);
  if (cnt > 32) load_meta(1);
  __syncwarp();
  if (lane == 0)
    for (int i = 0; i < S; ++i) issue(i);
  __syncwarp();

  constexpr int VE = 8;  // bf16 per 16-byte vector
  const int nvec = dout / VE;
  constexpr int NL = MOE_MAX_E / 64;
  for (int i = 0; i < cnt; ++i) {
    if ((i & 31) == 0 && i > 0 && i + 32 < cnt) {  // batch (i/32)+1 for the copies ahead
      load_meta((i >> 5) + 1);
      __syncwarp();
    }
    const int t = t_begin + i;
    const CbbMeta m = meta[i & 63];
    uint8_t* st = base + (size_t)(i % S) * p.stage_bytes;
    mbar_wait(&bars[i % S], (uint32_t)((i / S) & 1));
    int rows[KM], er[KM];
    float wr[KM], part[KM];
#pragma unroll
    for (int r = 0; r < KM; ++r) {
      rows[r] = r < k ? m.row[r] : -1;
      er[r] = r < k ? m.e[r] : -1;
      wr[r] = r < k ? m.w[r] : 0.f;
      part[r] = 0.f;
    }
    // fused dX (k = 1): a dropped token takes a row of the compacted drop list
    int dpos = -1;
    if (KM == 1 && p.dropb != nullptr && rows[0] < 0) {
      if (lane == 0) {
        dpos = atomicAdd(p.drop_cnt, 1);
        p.drop_tok[dpos] = t;
      }
      dpos = __shfl_sync(0xffffffffu, dpos, 0);
    }
    const uint4* sdy = reinterpret_cast<const uint4*>(st);
    for (int v = lane; v < nvec; v += 32) {
      bool any = false;
#pragma unroll
      for (int r = 0; r < KM; ++r) any |= rows[r] >= 0;
      if (!any) break;
      float gv[VE];
      unpack(sdy[v], gv, __nv_bfloat16());
#pragma unroll
      for (int r = 0; r < KM; ++r) {
        if (rows[r] < 0) continue;
        float o[VE], dov[VE];
        unpack(reinterpret_cast<const uint4*>(st + (size_t)(1 + r) * p.row_bytes)[v], o,
               __nv_bfloat16());
#pragma unroll
        for (int q = 0; q < VE; ++q) {
          part[r] = fmaf(gv[q], o[q], part[r]);
          dov[q] = fmaf(wr[r], gv[q], 0.f);
        }
        st_v4(peer_row(p.dobuf, p.pdo, er[r], (size_t)rows[r], dout) + (size_t)v * VE,
              pack(dov, __nv_bfloat16()));
      }
    }
    // logits of this token: staged row, or global
    const float* l = (need_p && p.lg_bytes)
                         ? reinterpret_cast<const float*>(st + (size_t)(1 + KM) * p.row_bytes)
                         : p.logits + (size_t)t * n;
    float lg[NL][2];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const int e = 2 * lane + 64 * j;
      lg[j][0] = (need_p && e < n) ? l[e] : -INFINITY;
      lg[j][1] = (need_p && e + 1 < n) ? l[e + 1] : -INFINITY;
    }
    float esel[KM];
#pragma unroll
    for (int r = 0; r < KM; ++r)
      esel[r] = (need_p && r < k && er[r] >= 0 && er[r] < n) ? l[er[r]] : 0.f;  // raw value
    // every lane has read the stage: it may be refilled (token i + S)
    __syncwarp();
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + S);
    }
    float dwr[KM];
    float c = 0.f;
#pragma unroll
    for (int r = 0; r < KM; ++r) {
      float sr = warp_sum(part[r]);
      sr = __shfl_sync(0xffffffffu, sr, 0);
      dwr[r] = rows[r] >= 0 ? sr + (p.dw_ext ? p.dw_ext[(size_t)t * k + r] : 0.f) : 0.f;
      c = fmaf(wr[r], dwr[r], c);
    }
#pragma unroll
    for (int r = 0; r < KM; ++r)
      if (r < k && lane == r) {
        p.dw[(size_t)t * k + r] = dwr[r];
        if (p.grow)
          p.grow[(size_t)t * k + r] = rows[r] < 0 ? -1
                                      : p.o_pair ? (int)((size_t)t * k + r)
                                      : p.pdo.nl ? rows[r] | ((er[r] / p.pdo.nl) << MOE_GROW_SHIFT)
                                                 : rows[r];
      }
    float mx = -INFINITY, sp = 0.f, cb = 0.f;
    float ens = 0.f;
    if (need_p) {
#pragma unroll
      for (int j = 0; j < NL; ++j) mx = fmaxf(mx, fmaxf(lg[j][0], lg[j][1]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
#pragma unroll
      for (int j = 0; j < NL; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = 2 * lane + 64 * j + h;
          if (e >= n) continue;
          const float ex = expf(lg[j][h] - mx);
          sp += ex;
          bool sel = false;
#pragma unroll
          for (int r = 0; r < KM; ++r) sel |= (r < k && er[r] == e);
          if (!sel) ens += ex;
        }
      }
      sp = __shfl_sync(0xffffffffu, warp_sum(sp), 0);
      ens = __shfl_sync(0xffffffffu, warp_sum(ens), 0);
#pragma unroll
      for (int r = 0; r < KM; ++r)
        esel[r] = (r < k && er[r] >= 0 && er[r] < n) ? expf(esel[r] - mx) : 0.f;
      if (p.bal_g) {
#pragma unroll
        for (int j = 0; j < NL; ++j) {
          const int e = 2 * lane + 64 * j;
          if (e < n) cb = fmaf(expf(lg[j][0] - mx) / sp, p.bal_g[e], cb);
          if (e + 1 < n) cb = fmaf(expf(lg[j][1] - mx) / sp, p.bal_g[e + 1], cb);
        }
        cb = __shfl_sync(0xffffffffu, warp_sum(cb), 0);
      }
    }
    float* dlrow = p.dl + (size_t)t * n;
    const int ncols = p.dlb ? p.n_pad : n;
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
          if (p.renorm) {  // dl_r = w_r sum_{s != r} w_s (dw_r - dw_s)  (cancellation-free)
#pragma unroll
            for (int r = 0; r < KM; ++r) {
              if (r >= k || er[r] != e) continue;
              float a = 0.f;
#pragma unroll
              for (int s2 = 0; s2 < KM; ++s2)
                if (s2 < k && s2 != r) a = fmaf(wr[s2], dwr[r] - dwr[s2], a);
              v = wr[r] * a;
            }
          } else {  // raw: dl_j = p_j (dp_j (1 - p_j) - sum_{s != j} p_s dw_s)
            const float pj = expf(lg[j][h] - mx) / sp;
            int rs = -1;
#pragma unroll
            for (int r = 0; r < KM; ++r)
              if (r < k && er[r] == e) rs = r;
            if (rs < 0) {
              v = -pj * c;
            } else {
              float osum = ens, other = 0.f, dws = 0.f;
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
              v = pj * (dws * (osum / sp) - other);
            }
          }
          if (p.bal_g) v = fmaf(expf(lg[j][h] - mx) / sp, p.bal_g[e] - cb, v);
          dlrow[e] = v;
        }
        v2[h] = v;
      }
      if (p.dlb) {
        const __nv_bfloat162 hi = __floats2bfloat162_rn(v2[0], v2[1]);
        const __nv_bfloat162 lo =
            __floats2bfloat162_rn(v2[0] - __low2float(hi), v2[1] - __high2float(hi));
        *reinterpret_cast<__nv_bfloat162*>(p.dlb + (size_t)t * p.n_pad + e0) = hi;
        *reinterpret_cast<__nv_bfloat162*>(p.dlb + ((size_t)p.maxT + t) * p.n_pad + e0) = lo;
        if (p.dlr && rows[0] >= 0) {
          __nv_bfloat16* rr = peer_row(p.dlr, p.pdlr, er[0], (size_t)rows[0], 2 * p.n_pad);
          *reinterpret_cast<__nv_bfloat162*>(rr + e0) = hi;
          *reinterpret_cast<__nv_bfloat162*>(rr + p.n_pad + e0) = lo;
        }
        if (dpos >= 0) {
          *reinterpret_cast<__nv_bfloat162*>(p.dropb + (size_t)dpos * p.n_pad + e0) = hi;
          *reinterpret_cast<__nv_bfloat162*>(p.dropb + ((size_t)p.maxT + dpos) * p.n_pad + e0) = lo;
        }
      }
    }
  }
}

}  // namespace

static int g_cbb_sms = 0;

cudaError_t launch_combine_bwd_bulk(const void* dy, const void* obuf, RouteBufs b, int T, int k,
                                    int n, int dout, int renorm, const CapTable& ct,
                                    void* dobuf, void* dlb, int maxT, int n_pad,
                                    const int32_t* pad_kept, cudaStream_t s, int pad_e0,
                                    const PeerBufs& po, const PeerBufs& pdo) {
  const char* ev = getenv("MOE_CB_BULK");  // opt-in (A/B, tests): measured slower, see header
  const int off = !(ev && ev[0] == '1');
  if (off || k > CBB_MAXK || po.nl || b.dspec || T == 0) return cudaErrorNotSupported;
  const int row_bytes = dout * 2;
  if (row_bytes % 16 || row_bytes > 16384) return cudaErrorNotSupported;
  if (!g_cbb_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_cbb_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int km = k == 1 ? 1 : 2;
  const int lg_bytes = (n % 4 == 0) ? n * 4 : 0;
  int stage_bytes = (1 + km) * row_bytes + lg_bytes;
  stage_bytes = (stage_bytes + 127) & ~127;
  // warps per block and stages per warp: ~200 KB of stages per SM, >= 2 stages per warp
  const size_t budget = 200 * 1024;
  int wpb = 8, S = 0;
  for (; wpb >= 2; wpb /= 2) {
    const size_t meta = 8 * 16 + 64 * sizeof(CbbMeta);
    S = (int)std::min<size_t>(8, (budget / wpb - meta) / stage_bytes);
    if (S >= 3) break;
  }
  if (const char* w = getenv("MOE_CB_WPB")) wpb = atoi(w);   // A/B experiments
  if (const char* w = getenv("MOE_CB_S")) S = atoi(w);
  if (S < 2) return cudaErrorNotSupported;
  const size_t warp_bytes = (((size_t)S * stage_bytes + 8 * S + 64 * sizeof(CbbMeta)) + 127) & ~size_t(127);
  const size_t smem = warp_bytes * wpb;
  const int nwarps_total = g_cbb_sms * wpb;
  const int per_warp = (T + nwarps_total - 1) / nwarps_total;
  const int grid = (T + per_warp * wpb - 1) / (per_warp * wpb);
  CbbParams p{};
  p.dy = (const __nv_bfloat16*)dy;
  p.obuf = (const __nv_bfloat16*)obuf;
  p.w = b.w; p.idx = b.idx; p.slot_of = b.slot_of; p.logits = b.logits;
  p.Tn = T; p.k = k; p.n = n; p.dout = dout; p.renorm = renorm;
  p.dobuf = (__nv_bfloat16*)dobuf; p.dw = b.dw; p.dl = b.dl; p.dlb = (__nv_bfloat16*)dlb;
  p.maxT = maxT; p.n_pad = n_pad; p.dw_ext = b.dw_ext; p.bal_g = b.bal_g; p.grow = b.grow;
  p.pad_kept = pad_kept; p.pad_e0 = pad_e0; p.pdo = pdo; p.dlr = b.dlr; p.pdlr = b.pdlr;
  p.dropb = b.dropb; p.drop_tok = b.drop_tok; p.drop_cnt = b.drop_cnt; p.o_pair = b.o_pair;
  p.stages = S; p.stage_bytes = stage_bytes; p.row_bytes = row_bytes; p.lg_bytes = lg_bytes;
  p.per_warp = per_warp;
  auto kf = km == 1 ? combine_bwd_bulk_kernel<1> : combine_bwd_bulk_kernel<2>;
  cudaError_t e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  launch_pdl(kf, std::max(1, grid), 32 * wpb, smem, s, p, ct);
  return cudaGetLastError();
}

}  // namespace moe
