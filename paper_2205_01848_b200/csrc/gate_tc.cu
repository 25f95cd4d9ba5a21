// gate_tc.cu -- the gating network's three dense contractions on tcgen05 tensor cores (bf16).
//
//  K1  gate forward (Alg. 1 l.1-3): logits = x W_g^T with the softmax / top-k /
//      normalize epilogue fused: each epilogue thread owns one token row (one TMEM lane) and
//      streams its n logits through registers -- top-k by strict '>' in ascending expert order
//      (ties -> lower index, reading 3), online softmax denominator, cached-index weights and
//      the hit test of sample-assignment caching.
//  K9  gate input gradient fused with the dispatch backward: dx = dl W_g + sum_r dX[row(t,r)].
//  K10 gate weight gradient: dW_g = dl^T x, split-K over tokens, fixed-order reduction.
//
// dl is fp32; the tensor cores take it as an exact-ish bf16 pair dl = hi + lo (hi = bf16(dl),
// lo = bf16(dl - hi); relative error <= 2^-17), i.e. two accumulating MMAs per K step.  The
// pair is written by the combine-backward kernel (dlb buffer: hi rows [0,maxT), lo rows
// [maxT, 2 maxT), n padded to a multiple of 64 with zeros).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>

#include "common.cuh"
#include "gate_tc.h"
#include "kernels.h"
#include "tc_common.cuh"

namespace moe {

constexpr int G_THREADS = 256;

struct GateFwdParams {
  int T, n, k, renorm;
  const int32_t* cached;  // [T x k] or null
  float* logits;          // [T x n]
  int32_t* idx_out;       // [T x k] fresh top-k
  float* w_out;           // [T x k]
  int32_t* hit;
  int32_t* flags;
  int32_t* idx_fix;       // fallback mode: rows of unknown samples (-1) get the fresh top-k
  int dbg;                 // timing experiments (MOE_GATE_DBG), 0 in production
  int tma_logits;          // logits written by TMA from a staged 32 x 16 box (n % 16 == 0)
  int32_t* hist;           // [T / 128 x n] per-tile expert histogram of idx_out (A3 fused into
                           // the epilogue; the 128-token M tile is the routing tile), or null
  float4* stats;           // [T] softmax statistics for the combine backward, or null:
                           // (max logit m, sum_e exp(l_e - m), sum over the experts NOT in the
                           // dispatch set of exp(l_e - m), 0)
  // Cached mode: the dispatch indices are known before the gate, so A4 rides on
  // the x stream the gate reads anyway -- warps 2-3 compute the tile's slots (token-major
  // ranks, as the dispatch kernel does) and copy each x k-block from the TMA stage to the
  // kept rows of X_buf once the stage has landed.  didx == null: off.
  const int32_t* didx;     // [T x k] dispatch indices (the cached rows)
  const int32_t* tile_off; // [ntiles x n] exclusive per-tile slot offsets (route_scan)
  int32_t* slot_of;        // [T x k]
  int32_t* token_of_slot;  // [rows]
  __nv_bfloat16* xbuf;     // X_buf rows
  const int32_t* kept;     // [n]: pad rows [kept_e, roundup(kept_e, 64)) are zeroed here
  __nv_bfloat16* yz;       // fused combine: y rows of tokens with every pair dropped -> 0
  int dout;
  CapTable ct;             // capacities, region bases
};

// logits staging of the gate epilogue: one 32-row x 16-column fp32 box (2 KB, 64-byte
// swizzle) per epilogue warp
constexpr int GF_STG_BYTES = 32 * 16 * 4;

struct GateDxParams {
  int T, n_pad, k, d;
  const int32_t* grow;    // [T x k] dX row of each (token, r) pair or -1 (from combine_bwd)
  const __nv_bfloat16* dxbuf;  // [rows x d]
  __nv_bfloat16* dx;           // [T x d]
  int accumulate;
  CapTable ct;
  PeerBufs pdx;                // peer EP (N1): dX rows read from the owners; grow encodes owner
  int drop_only;               // fused dX GEMM (k = 1): only tokens with every pair dropped
                               // (dx = dl W_g); the others were written by the dX GEMM
  const int32_t* drop_tok;     // drop_only: [count] token of each compacted dropped row
  const int32_t* drop_cnt;     // drop_only: [1] number of dropped tokens (combine_bwd)
  int nowait;                  // inputs complete before the predecessor started: no PDL wait
};

// dX row of a gather-table entry (peer EP: owner in the top bits, see MOE_GROW_SHIFT)
template <bool PEER>
__device__ __forceinline__ const __nv_bfloat16* gdx_row(const GateDxParams& p, int g) {
  if (PEER) {
    const int o = g >> MOE_GROW_SHIFT;
    const __nv_bfloat16* b = p.dxbuf;
#pragma unroll
    for (int j = 0; j < MOE_MAX_R; ++j)  // constant indices (no local copy of the table)
      if (o == j) b = reinterpret_cast<const __nv_bfloat16*>(p.pdx.p[j]);
    return b + (size_t)(g & ((1 << MOE_GROW_SHIFT) - 1)) * p.d;
  }
  return p.dxbuf + (size_t)g * p.d;
}

struct GateDwParams {
  int T, n, d, chunk, splits;
  float* partial;  // [splits x n x d]
  int nowait;      // inputs complete before the predecessor started: skip the PDL wait
};

// --------------------------------------------------------------------------------------
// common pipeline skeleton pieces
// --------------------------------------------------------------------------------------
struct Bars {
  uint64_t* full;
  uint64_t* empty;
  uint64_t* tfull;
  uint64_t* tempty;
  uint32_t* tmem;
};

template <int STAGES>
__device__ __forceinline__ Bars setup_bars(uint8_t* after_stages, int ncols, int warp, int lane,
                                           int epi_threads = 128, int empty_count = 1) {
  Bars b;
  b.full = reinterpret_cast<uint64_t*>(after_stages);
  b.empty = b.full + STAGES;
  b.tfull = b.empty + STAGES;
  b.tempty = b.tfull + 2;
  b.tmem = reinterpret_cast<uint32_t*>(b.tempty + 2);
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&b.full[s], 1);
      mbar_init(&b.empty[s], empty_count);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&b.tfull[s], 1);
      mbar_init(&b.tempty[s], epi_threads);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(b.tmem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  return b;
}

__device__ __forceinline__ void teardown(uint32_t tmem_base, int ncols, int warp) {
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(ncols));
  }
}

__device__ __forceinline__ uint8_t* align1k(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// ======================================================================================
// K1: gate forward + fused softmax / top-k / normalize epilogue
// ======================================================================================
template <int BN, int STAGES, int KM>
__global__ void __launch_bounds__(G_THREADS, 2)
    gate_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmX,
                       const __grid_constant__ CUtensorMap tmW,
                       const __grid_constant__ CUtensorMap tmL, GateFwdParams p, int K) {
  pdl_enter();  // PDL: predecessor complete + visible (common.cuh)
  constexpr int A_BYTES = TC_BM * TC_BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + BN * TC_BK * 2;
  constexpr uint32_t IDESC = make_idesc(BN, 0, 0);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmW);
  }
  // empty[s]: the MMA commit, plus one arrive per dispatch warp in fused cached mode
  Bars b = setup_bars<STAGES>(smem + STAGES * STAGE_BYTES, 2 * BN, warp, lane, 128,
                              p.didx ? 3 : 1);
  uint8_t* s_stg = smem + STAGES * STAGE_BYTES + 1024;  // [4 warps][2 KB], 1 KB aligned
  int32_t* s_hist = reinterpret_cast<int32_t*>(s_stg + 4 * GF_STG_BYTES);  // [256]
  uint32_t* s_mask = reinterpret_cast<uint32_t*>(s_hist + 256);  // fused dispatch: [n][4]
  int32_t* s_row = reinterpret_cast<int32_t*>(s_mask + 4 * p.n);   // [128 x k] X_buf row / -1
  const uint32_t tmem_base = *b.tmem;
  const int MT = (p.T + TC_BM - 1) / TC_BM;
  const int nk = K / TC_BK;

  if (warp == 0) {
    if (lane == 0) {
      if (p.tma_logits) prefetch_tmap(&tmL);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < MT; t += gridDim.x) {
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&b.empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          mbar_expect_tx(&b.full[stage], STAGE_BYTES);
          tma_load_2d(sa, &tmX, &b.full[stage], kb * TC_BK, t * TC_BM);
          tma_load_2d(sa + A_BYTES, &tmW, &b.full[stage], kb * TC_BK, 0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < MT; t += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(&b.tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&b.full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)
            tc_mma(tmem_d, umma_desc(sa + k * 32, 16, 1024), umma_desc(sa + A_BYTES + k * 32, 16, 1024),
                   IDESC, (kb | k) != 0);
          tc_commit(&b.empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&b.tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp == 2 || warp == 3) {
    if (p.didx) {
      // ============== fused cached-mode dispatch (A4, S4.2): warps 2-3, 64 threads ==============
      const int dt = threadIdx.x - 64;
      const int n = p.n, k = p.k;
      // pad rows [kept_e, roundup(kept_e, 64)) of expert regions blockIdx.x, + gridDim.x, ...
      // (the token-contraction GEMMs read whole 64-row K-blocks)
      for (int e = blockIdx.x; e < n; e += gridDim.x) {
        const int kp = p.kept[e];
        const int r0 = p.ct.base[e] + kp;
        const int r1 = p.ct.base[e] + ((kp + MOE_PAD_ROWS - 1) / MOE_PAD_ROWS) * MOE_PAD_ROWS;
        const size_t total = (size_t)max(r1 - r0, 0) * (K / 8);
        for (size_t i = dt; i < total; i += 64)
          st_v4(p.xbuf + (size_t)r0 * K + i * 8, make_uint4(0, 0, 0, 0));
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < MT; tile += gridDim.x) {
        asm volatile("bar.sync 2, 64;" ::: "memory");  // the previous tile's rows are copied
        for (int i = dt; i < 4 * n; i += 64) s_mask[i] = 0u;
        asm volatile("bar.sync 2, 64;" ::: "memory");
        // token-major ranks inside the routing tile (an expert appears at most once per token)
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int lt = dt + 64 * h2, t = tile * TC_BM + lt;
          if (t < p.T)
            for (int r = 0; r < k; ++r) {
              const int e = p.didx[(size_t)t * k + r];
              if ((unsigned)e < (unsigned)n) atomicOr(&s_mask[e * 4 + (lt >> 5)], 1u << (lt & 31));
            }
        }
        asm volatile("bar.sync 2, 64;" ::: "memory");
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int lt = dt + 64 * h2, t = tile * TC_BM + lt;
          bool any = false;
          for (int r = 0; r < k; ++r) {
            int row = -1;
            if (t < p.T) {
              const int e = p.didx[(size_t)t * k + r];
              int slot = -1;
              if ((unsigned)e < (unsigned)n) {  // invalid cached index: dropped (flag raised)
                int rank = __popc(s_mask[e * 4 + (lt >> 5)] & ((1u << (lt & 31)) - 1u));
                for (int q2 = 0; q2 < (lt >> 5); ++q2) rank += __popc(s_mask[e * 4 + q2]);
                slot = p.ct.pre[e] + p.tile_off[(size_t)tile * n + e] + rank;
                if (slot < p.ct.cap[e]) {
                  row = p.ct.base[e] + slot;
                  p.token_of_slot[row] = t * k + r;
                } else {
                  slot = -1;
                }
              }
              p.slot_of[(size_t)t * k + r] = slot;
            }
            any |= row >= 0;
            s_row[lt * k + r] = row;
          }
          if (!any && t < p.T && p.yz)  // every pair dropped: y[t] = 0
            for (int v = 0; v < p.dout / 8; ++v)
              st_v4(p.yz + (size_t)t * p.dout + v * 8, make_uint4(0, 0, 0, 0));
        }
        asm volatile("bar.sync 2, 64;" ::: "memory");
        // each k-block: 128 rows x 128 bytes in the stage (128-byte swizzle: 16-byte chunk c of
        // row r at c ^ (r & 7)).  Thread (warp w, lane l) owns chunk l % 8 of the 16 rows
        // 8 i + 4 (w - 2) + l / 8: all 16 chunks are read into registers with back-to-back
        // shared loads (a quarter warp reads one whole row: conflict-free), the stage is
        // released at once, and the registers then leave as 16-byte stores (one full 128-byte
        // line per row and destination) while the next stage lands.
        const int ch = lane & 7;
        const int rsub = (warp - 2) * 4 + (lane >> 3);
        int rowr[TC_BM / 8];
        if (KM == 1) {
#pragma unroll
          for (int i = 0; i < TC_BM / 8; ++i) {
            const int lr = i * 8 + rsub;
            rowr[i] = tile * TC_BM + lr < p.T ? s_row[lr] : -1;
          }
        }
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&b.full[stage], phase);
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          uint4 v[TC_BM / 8];
#pragma unroll
          for (int i = 0; i < TC_BM / 8; ++i) {
            const int lr = i * 8 + rsub;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v[i].x), "=r"(v[i].y), "=r"(v[i].z), "=r"(v[i].w)
                         : "r"(sa + lr * 128 + ((ch ^ (lr & 7)) << 4)));
          }
          __syncwarp();  // (orders every lane's shared loads before the release below)
          if (lane == 0) mbar_arrive(&b.empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
#pragma unroll
          for (int i = 0; i < TC_BM / 8; ++i) {
            const int lr = i * 8 + rsub;
            if (KM == 1) {
              if (rowr[i] >= 0)
                st_v4(p.xbuf + (size_t)rowr[i] * K + kb * TC_BK + ch * 8, v[i]);
            } else if (tile * TC_BM + lr < p.T) {
              for (int r = 0; r < k; ++r) {
                const int row = s_row[lr * k + r];
                if (row >= 0) st_v4(p.xbuf + (size_t)row * K + kb * TC_BK + ch * 8, v[i]);
              }
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int n = p.n, k = p.k;
    int it = 0;
    for (int tile = blockIdx.x; tile < MT; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      if (p.hist) {  // this tile's histogram starts empty (the previous one has been written)
        const int i = q * 32 + lane;
        s_hist[i] = 0;
        s_hist[i + 128] = 0;
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      mbar_wait(&b.tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const int t = tile * TC_BM + q * 32 + lane;
      const bool valid = t < p.T;
      // KM = compile-time bound on k: every per-row array below is indexed with unrolled
      // (constant) indices, so it lives in registers
      float sel_v[KM];
      int sel_e[KM];
      int cidx[KM];
      float cval[KM];
#pragma unroll
      for (int r = 0; r < KM; ++r) {
        sel_v[r] = 0.f;
        sel_e[r] = -1;
        cidx[r] = -1;
        cval[r] = 0.f;
      }
      if (valid && p.cached) {
#pragma unroll
        for (int r = 0; r < KM; ++r)
          if (r < k) cidx[r] = p.cached[(size_t)t * k + r];
      }
      float m_run = -INFINITY;
      bool nan_seen = false;
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
      float* lrow = p.logits + (size_t)t * n;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        if (c * 32 >= n) break;  // warp-uniform
        uint32_t r32[32];
        tmem_ld32(taddr + c * 32, r32);
        if (p.tma_logits) {  // warp-uniform: two 32 x 16 boxes (rows >= T clipped by TMA)
          uint8_t* stg = s_stg + q * GF_STG_BYTES;
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            if (c * 32 + h2 * 16 >= n) break;
            if (lane == 0) tma_store_wait_read<0>();
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i)  // 64-byte swizzle: chunk i of row r at i ^ ((r>>1)&3)
              *reinterpret_cast<uint4*>(stg + lane * 64 + ((i ^ ((lane >> 1) & 3)) << 4)) =
                  make_uint4(r32[h2 * 16 + 4 * i], r32[h2 * 16 + 4 * i + 1],
                             r32[h2 * 16 + 4 * i + 2], r32[h2 * 16 + 4 * i + 3]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) tma_store_2d(&tmL, stg, c * 32 + h2 * 16, tile * TC_BM + q * 32);
          }
        }
        if (!valid || p.dbg) continue;
        if (p.tma_logits) {
        } else if ((n & 3) == 0 && c * 32 + 32 <= n) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<uint4*>(lrow + c * 32 + j) = make_uint4(r32[j], r32[j + 1], r32[j + 2], r32[j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c * 32 + j < n) lrow[c * 32 + j] = __uint_as_float(r32[j]);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int e = c * 32 + j;
          if (e < n) {
          const float v = __uint_as_float(r32[j]);
          nan_seen |= (v != v);
          // streaming top-k in ascending expert order: a strictly larger value displaces and
          // the displaced entry bubbles down, so equal values keep the lower index first
          // (once inserted, every later entry shifts down by one: the displaced entry ranks
          // above all entries after it, ties included)
          float cv = v;
          int ce = e;
          bool ins = false;
#pragma unroll
          for (int pos = 0; pos < KM; ++pos) {
            if (pos < k && (ins || sel_e[pos] < 0 || cv > sel_v[pos])) {
              ins = true;
              const float tv = sel_v[pos];
              const int te = sel_e[pos];
              sel_v[pos] = cv;
              sel_e[pos] = ce;
              cv = tv;
              ce = te;
            }
          }
#pragma unroll
          for (int r = 0; r < KM; ++r)
            if (cidx[r] == e) cval[r] = v;
          }
        }
        // row max from registers
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c * 32 + j < n) m_run = fmaxf(m_run, __uint_as_float(r32[j]));
      }
      // the dispatch set: the cached indices when valid, else the fresh top-k
      float lv[KM];
      int use[KM];
      bool ok = true, unknown = false;
      if (p.cached) {
#pragma unroll
        for (int r = 0; r < KM; ++r) {
          if (r >= k) break;
          ok &= (cidx[r] >= 0 && cidx[r] < n);
          unknown |= cidx[r] == -1;
#pragma unroll
          for (int q2 = 0; q2 < r; ++q2) ok &= (cidx[q2] != cidx[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < KM; ++r) {
        use[r] = (p.cached && ok) ? cidx[r] : sel_e[r];
        lv[r] = (p.cached && ok) ? cval[r] : sel_v[r];
      }
      // Softmax denominator (raw mode) and the backward's statistics: a second pass over the
      // accumulator (warp-collective TMEM loads, every lane) splits sum_e exp(l_e - m) into the
      // experts outside the dispatch set (ens, ascending e) and the selected ones (esel), so the
      // combine backward gets 1 - p_sel = ens / s without cancellation.
      float ens = 0.f, s_run = 0.f;
      float esel[KM];
#pragma unroll
      for (int r = 0; r < KM; ++r) esel[r] = (r < k) ? expf(lv[r] - m_run) : 0.f;
      if (!p.renorm || p.stats) {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          if (c * 32 >= n) break;  // warp-uniform
          uint32_t r32[32];
          tmem_ld32(taddr + c * 32, r32);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int e = c * 32 + j;
            bool sel = false;
#pragma unroll
            for (int r = 0; r < KM; ++r) sel |= (r < k && use[r] == e);
            if (e < n && !sel) ens += expf(__uint_as_float(r32[j]) - m_run);
          }
        }
        s_run = ens;
#pragma unroll
        for (int r = 0; r < KM; ++r) s_run += esel[r];
      }
      tc_fence_before();
      mbar_arrive(&b.tempty[acc]);
      if (valid) {
        if (nan_seen) atomicOr(p.flags, 1);
        if (p.stats) p.stats[t] = make_float4(m_run, s_run, ens, 0.f);
        if (p.cached) {
          // an unknown sample (fallback mode) is routed by its fresh top-k, a miss
          if (!ok && !(unknown && p.idx_fix)) atomicOr(p.flags, 2);
          if (!ok && p.idx_fix) {
#pragma unroll
            for (int r = 0; r < KM; ++r)
              if (r < k) p.idx_fix[(size_t)t * k + r] = sel_e[r];
          }
          bool same = true;
#pragma unroll
          for (int r = 0; r < KM; ++r) {
            if (r >= k) break;
            bool found = false;
#pragma unroll
            for (int q2 = 0; q2 < KM; ++q2) found |= (q2 < k && cidx[r] == sel_e[q2]);
            same &= found;
          }
          if (same && ok) atomicAdd(p.hit, 1);
        }
        int32_t* orow = p.idx_out + (size_t)t * k;
        float* wrow = p.w_out + (size_t)t * k;
        // raw mode: p_i = exp(l_i - max) / sum_e exp(l_e - max), the row re-read from L1/L2
        if (p.renorm) {
          float m = lv[0];
#pragma unroll
          for (int r = 1; r < KM; ++r)
            if (r < k) m = fmaxf(m, lv[r]);
          float ev[KM], ssum = 0.f;
#pragma unroll
          for (int r = 0; r < KM; ++r)
            if (r < k) { ev[r] = expf(lv[r] - m); ssum += ev[r]; }
#pragma unroll
          for (int r = 0; r < KM; ++r)
            if (r < k) { wrow[r] = ev[r] / ssum; orow[r] = sel_e[r]; }
        } else {
#pragma unroll
          for (int r = 0; r < KM; ++r)
            if (r < k) { wrow[r] = esel[r] / s_run; orow[r] = sel_e[r]; }
        }
        if (p.hist) {
#pragma unroll
          for (int r = 0; r < KM; ++r)
            if (r < k) atomicAdd(&s_hist[sel_e[r]], 1);
        }
      }
      if (p.hist) {  // A3 histogram of this routing tile (integer counts: order-free)
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int i = q * 32 + lane;
        int32_t* hrow = p.hist + (size_t)tile * n;
        if (i < n) hrow[i] = s_hist[i];
        if (i + 128 < n) hrow[i + 128] = s_hist[i + 128];
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
  }
  if (warp >= 4 && lane == 0 && p.tma_logits) tma_store_wait_all();
  teardown(tmem_base, 2 * BN, warp);
}

// ======================================================================================
// K9: dx = [hi | lo](dl) . [W_g ; W_g] + gather(dX)
// ======================================================================================
constexpr int GX_THREADS = 384;  // 4 control warps + 8 epilogue warps (gather-heavy epilogue)

template <int BN, int STAGES, bool PEER>
__global__ void __launch_bounds__(GX_THREADS, 1)
    gate_dx_tc_kernel(const __grid_constant__ CUtensorMap tmHi,
                      const __grid_constant__ CUtensorMap tmLo,
                      const __grid_constant__ CUtensorMap tmW, GateDxParams p) {
  pdl_enter(p.nowait);  // PDL: predecessor complete + visible (common.cuh)
  constexpr int A_BYTES = TC_BM * TC_BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + BN * TC_BK * 2;
  constexpr uint32_t IDESC = make_idesc(BN, 0, 1);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmHi);
    prefetch_tmap(&tmLo);
    prefetch_tmap(&tmW);
  }
  Bars b = setup_bars<STAGES>(smem + STAGES * STAGE_BYTES, 2 * BN, warp, lane, 256);
  const uint32_t tmem_base = *b.tmem;
  int MT = (p.T + TC_BM - 1) / TC_BM;
  const int NT = p.d / BN;
  const int nb = p.n_pad / TC_BK;
  const int nk = 2 * nb;
  // drop_only: the rows are the dropped tokens compacted by the combine backward (A = their
  // [hi|lo](dl) rows, token of row i = drop_tok[i]); the same count in every role
  __shared__ int32_t s_cnt;
  int rows_valid = p.T;
  if (p.drop_only) {
    if (threadIdx.x == 0) s_cnt = *reinterpret_cast<const volatile int32_t*>(p.drop_cnt);
    __syncthreads();
    rows_valid = s_cnt;
    MT = (rows_valid + TC_BM - 1) / TC_BM;
  }
  auto mtile = [&](int t) { return t % MT; };
  // token of compacted row i (identity unless drop_only), -1 past the end
  auto tok_of = [&](int i) { return i < rows_valid ? (p.drop_only ? p.drop_tok[i] : i) : -1; };
  const int total = MT * NT;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int mt = mtile(t), nt = t / MT;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&b.empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx(&b.full[stage], STAGE_BYTES);
          const int kk = (kb % nb) * TC_BK;
          tma_load_2d(sa, kb < nb ? &tmHi : &tmLo, &b.full[stage], kk, mt * TC_BM);
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)
            tma_load_2d(sb + j * 8192, &tmW, &b.full[stage], nt * BN + j * 64, kk);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(&b.tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&b.full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)
            tc_mma(tmem_d, umma_desc(sa + k * 32, 16, 1024), umma_desc(sb + k * 2048, 8192, 1024),
                   IDESC, (kb | k) != 0);
          tc_commit(&b.empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&b.tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // Epilogue, software-pipelined over this CTA's tiles.  Warp (q, half) owns token rows
    // 32q..32q+31 (its TMEM lanes) x HC columns.  The dX rows gathered for the NEXT tile are
    // fetched with cp.async into a second shared-memory staging buffer while the current
    // tile is combined, and dx leaves through the staging buffer with coalesced stores, so a
    // tile costs about one memory round trip instead of three dependent ones.
    const int q = warp & 3, half = (warp - 4) >> 2;
    constexpr int HC = BN / 2;    // columns per warp
    constexpr int RB = HC * 2;    // bytes of one row segment
    constexpr int RS = RB + 16;   // padded staging stride (conflict-free 16-B row reads)
    constexpr int LPR = RB / 16;  // lanes per row segment
    constexpr int RPI = 32 / LPR; // rows per cooperative instruction
    constexpr int KS = 2;         // rows per token staged asynchronously (k > 2: direct loads)
    uint8_t* stg_w = smem + STAGES * STAGE_BYTES + 256 + (warp - 4) * (2 * KS * 32 * RS);
    const int sub = lane / LPR, seg = lane % LPR;
    const int kk = p.k;
    auto stg = [&](int par, int r) { return stg_w + (par * KS + r) * 32 * RS; };
    auto load_rows = [&](int tile, int* rows) {
      const int t = (tile < total ? mtile(tile) : 0) * TC_BM + q * 32 + lane;
#pragma unroll
      for (int r = 0; r < MOE_MAX_K; ++r)
        rows[r] = (tile < total && !p.drop_only && t < p.T && r < kk) ? p.grow[(size_t)t * kk + r] : -1;
    };
    auto issue_gather = [&](int tile, int par, const int* rows) {
      if (tile < total) {
        const int col_base = (tile / MT) * BN + half * HC;
#pragma unroll
        for (int r = 0; r < KS; ++r) {
          if (r >= kk) break;
#pragma unroll
          for (int i = 0; i < 32; i += RPI) {
            const int rowid = __shfl_sync(0xffffffffu, rows[r], i + sub);
            if (rowid >= 0 && !p.drop_only)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                               smem_u32(stg(par, r) + (i + sub) * RS + seg * 16)),
                           "l"(gdx_row<PEER>(p, rowid) + col_base + seg * 8)
                           : "memory");
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int rows_cur[MOE_MAX_K], rows_nxt[MOE_MAX_K];
    int tile = blockIdx.x;
    load_rows(tile, rows_cur);
    issue_gather(tile, 0, rows_cur);
    for (int it = 0; tile < total; tile += gridDim.x, ++it) {
      const int acc = it & 1, par = it & 1;
      const int mt = mtile(tile), nt = tile / MT;
      const int t0w = mt * TC_BM + q * 32;
      const int t = tok_of(t0w + lane);   // this lane's token (drop_only: compacted row)
      const bool valid = t >= 0;
      const int col_base = nt * BN + half * HC;
      load_rows(tile + gridDim.x, rows_nxt);
      issue_gather(tile + gridDim.x, par ^ 1, rows_nxt);
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // this tile's gather landed
      __syncwarp();
      float v[HC];
#pragma unroll
      for (int i = 0; i < HC; ++i) v[i] = 0.f;
#pragma unroll
      for (int r = 0; r < MOE_MAX_K; ++r) {  // expert path first, r order (as the SIMT form)
        if (r >= kk) break;
        if (rows_cur[r] < 0 || p.drop_only) continue;
        if (r < KS) {
#pragma unroll
          for (int c = 0; c < HC / 8; ++c) {
            float xv[8];
            unpack(*reinterpret_cast<const uint4*>(stg(par, r) + lane * RS + c * 16), xv, __nv_bfloat16());
#pragma unroll
            for (int j = 0; j < 8; ++j) v[8 * c + j] += xv[j];
          }
        } else {
#pragma unroll
          for (int c = 0; c < HC / 8; ++c) {
            float xv[8];
            unpack(ld_nc_v4(gdx_row<PEER>(p, rows_cur[r]) + col_base + 8 * c), xv, __nv_bfloat16());
#pragma unroll
            for (int j = 0; j < 8; ++j) v[8 * c + j] += xv[j];
          }
        }
      }
      mbar_wait(&b.tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
#pragma unroll
      for (int c = 0; c < HC / 32; ++c) {
        uint32_t r32[32];
        tmem_ld32(taddr + half * HC + c * 32, r32);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[32 * c + i] += __uint_as_float(r32[i]);
      }
      tc_fence_before();
      mbar_arrive(&b.tempty[acc]);  // TMEM drained: the next tile's MMAs may start
      __nv_bfloat16* drow = p.dx + (size_t)t * p.d + col_base;
      if (valid && p.accumulate) {
#pragma unroll
        for (int c = 0; c < HC / 8; ++c) {
          float o[8];
          unpack(ld_v4(drow + 8 * c), o, __nv_bfloat16());
#pragma unroll
          for (int j = 0; j < 8; ++j) v[8 * c + j] += o[j];
        }
      }
      __syncwarp();  // every lane finished reading stg(par, 0) before it is reused for dx
#pragma unroll
      for (int c = 0; c < HC / 8; ++c)
        *reinterpret_cast<uint4*>(stg(par, 0) + lane * RS + c * 16) = pack(v + 8 * c, __nv_bfloat16());
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 32; i += RPI) {
        const int tok = __shfl_sync(0xffffffffu, t, i + sub);
        if (tok >= 0)
          st_v4(p.dx + (size_t)tok * p.d + col_base + seg * 8,
                *reinterpret_cast<const uint4*>(stg(par, 0) + (i + sub) * RS + seg * 16));
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < MOE_MAX_K; ++r) rows_cur[r] = rows_nxt[r];
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  teardown(tmem_base, 2 * BN, warp);
}

// ======================================================================================
// K10: dW_g partials = [hi ; lo](dl)^T x over a token chunk per split
// ======================================================================================
template <int BN, int STAGES>
__global__ void __launch_bounds__(G_THREADS, 1)
    gate_dw_tc_kernel(const __grid_constant__ CUtensorMap tmHi,
                      const __grid_constant__ CUtensorMap tmLo,
                      const __grid_constant__ CUtensorMap tmX, GateDwParams p) {
  pdl_enter(p.nowait);  // PDL: predecessor complete + visible (common.cuh)
  constexpr int A_BYTES = TC_BM * TC_BK * 2;  // one of hi / lo
  constexpr int STAGE_BYTES = 2 * A_BYTES + BN * TC_BK * 2;
  constexpr uint32_t IDESC = make_idesc(BN, 1, 1);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmHi);
    prefetch_tmap(&tmLo);
    prefetch_tmap(&tmX);
  }
  Bars b = setup_bars<STAGES>(smem + STAGES * STAGE_BYTES, 2 * BN, warp, lane);
  const uint32_t tmem_base = *b.tmem;
  const int MT = (p.n + TC_BM - 1) / TC_BM;
  const int NT = p.d / BN;
  const int total = p.splits * MT * NT;

  auto decode = [&](int t, int& s, int& mt, int& nt) {
    nt = t % NT;
    int r = t / NT;
    mt = r % MT;
    s = r / MT;
  };
  auto krange = [&](int s, int& k0, int& nkb) {
    k0 = s * p.chunk;
    int k1 = min(p.T, k0 + p.chunk);
    nkb = k1 > k0 ? (k1 - k0 + TC_BK - 1) / TC_BK : 0;
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int s, mt, nt, k0, nkb;
        decode(t, s, mt, nt);
        krange(s, k0, nkb);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&b.empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          mbar_expect_tx(&b.full[stage], STAGE_BYTES);
          const int tk = k0 + kb * TC_BK;
          tma_load_2d(sa, &tmHi, &b.full[stage], mt * TC_BM, tk);
          tma_load_2d(sa + 8192, &tmHi, &b.full[stage], mt * TC_BM + 64, tk);
          tma_load_2d(sa + A_BYTES, &tmLo, &b.full[stage], mt * TC_BM, tk);
          tma_load_2d(sa + A_BYTES + 8192, &tmLo, &b.full[stage], mt * TC_BM + 64, tk);
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)
            tma_load_2d(sa + 2 * A_BYTES + j * 8192, &tmX, &b.full[stage], nt * BN + j * 64, tk);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
        int s, mt, nt, k0, nkb;
        decode(t, s, mt, nt);
        krange(s, k0, nkb);
        const int acc = it & 1;
        mbar_wait(&b.tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&b.full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + 2 * A_BYTES;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            const uint64_t dbx = umma_desc(sb + k * 2048, 8192, 1024);
            tc_mma(tmem_d, umma_desc(sa + k * 2048, 8192, 1024), dbx, IDESC, (kb | k) != 0);
            tc_mma(tmem_d, umma_desc(sa + A_BYTES + k * 2048, 8192, 1024), dbx, IDESC, 1);
          }
          tc_commit(&b.empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&b.tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;
    int it = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
      int s, mt, nt, k0, nkb;
      decode(tile, s, mt, nt);
      krange(s, k0, nkb);
      const int acc = it & 1;
      mbar_wait(&b.tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const int m = mt * TC_BM + q * 32 + lane;  // expert row
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
      float* prow = p.partial + ((size_t)s * p.n + m) * p.d;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r32[32];
        if (nkb > 0) {
          tmem_ld32(taddr + c * 32, r32);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) r32[i] = 0u;
        }
        if (m >= p.n) continue;
        const int col0 = nt * BN + c * 32;
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          st_v4(prow + col0 + i, make_uint4(r32[i], r32[i + 1], r32[i + 2], r32[i + 3]));
      }
      tc_fence_before();
      mbar_arrive(&b.tempty[acc]);
    }
  }
  teardown(tmem_base, 2 * BN, warp);
}

// ------------------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_enc = nullptr;
static int g_sms = 148;

static bool enc_init() {
  if (g_enc) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return false;
  g_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  return true;
}

static bool map2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                  uint32_t box_inner, uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return g_enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
               es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename KF>
static cudaError_t set_smem(KF kf, size_t smem) {
  return cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

static size_t smem_for(int stage_bytes, int stages) {
  return (size_t)stage_bytes * stages + 1024 + 256;
}

cudaError_t launch_gate_fwd_tc(const void* x, const void* wg, int T, int n, int d, int k,
                               int renorm, const int32_t* cached, RouteBufs b, cudaStream_t s,
                               const GateDispatch* gd) {
  if (T == 0) return cudaSuccess;
  if (!enc_init()) return cudaErrorNotSupported;
  CUtensorMap mx, mw;
  const int bn = n <= 64 ? 64 : (n <= 128 ? 128 : 256);
  if (!map2d(&mx, x, d, T, 64, 128) || !map2d(&mw, wg, d, n, 64, bn)) return cudaErrorInvalidValue;
  CUtensorMap ml{};
  int tma_logits = 0;
  if (n % 16 == 0) {  // fp32 logits [T x n], 16 x 32 boxes, 64-byte swizzle
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)T};
    cuuint64_t strides[1] = {(cuuint64_t)n * 4};
    cuuint32_t box[2] = {16, 32};
    cuuint32_t es[2] = {1, 1};
    tma_logits = g_enc(&ml, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, b.logits, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  GateFwdParams p{T, n, k, renorm, cached, b.logits, cached ? b.fresh_idx : b.idx, b.w,
                  b.hit_count, b.flags, cached ? b.idx_fix : nullptr,
                  getenv("MOE_GATE_DBG") ? atoi(getenv("MOE_GATE_DBG")) : 0, tma_logits,
                  (!cached && b.gate_hist) ? b.tile_hist : nullptr, (float4*)b.sstat};
  size_t extra = 0;  // fused dispatch: tile masks [n][4] + destination rows [128 x k]
  if (gd) {
    if (!cached || d % 64 != 0) return cudaErrorInvalidValue;
    p.didx = b.idx;
    p.tile_off = b.tile_off;
    p.slot_of = b.slot_of;
    p.token_of_slot = b.token_of_slot;
    p.xbuf = (__nv_bfloat16*)gd->xbuf;
    p.kept = b.kept;
    p.yz = (__nv_bfloat16*)gd->y_zero;
    p.dout = gd->dout;
    p.ct = *gd->ct;
    extra = (size_t)n * 16 + (size_t)128 * k * 4;
  }
  const int MT = (T + 127) / 128;
  // two CTAs per SM (4-stage rings): twice the epilogue warps, which bound this kernel
  // as many tiles on every CTA: the fewest CTAs (up to two per SM) that keep the per-CTA tile
  // count (c3: 512 tiles on 256 CTAs x 2 rather than 296 CTAs with 1 or 2; measured 1.5 us)
  int grid = MT < 2 * g_sms ? MT : 2 * g_sms;
  const int per_cta = (MT + grid - 1) / grid;
  grid = (MT + per_cta - 1) / per_cta;
#define GF(BN, ST)                                                                       \
  {                                                                                      \
    auto kf = k == 1 ? gate_fwd_tc_kernel<BN, ST, 1>                                     \
                     : (k == 2 ? gate_fwd_tc_kernel<BN, ST, 2>                           \
                               : (k <= 4 ? gate_fwd_tc_kernel<BN, ST, 4>                 \
                                         : gate_fwd_tc_kernel<BN, ST, 8>));              \
    size_t sm = smem_for((128 + BN) * 64 * 2, ST) + 1024 + 4 * GF_STG_BYTES + 1024 + extra; \
    cudaError_t e = set_smem(kf, sm);                                                    \
    if (e != cudaSuccess) return e;                                                      \
    launch_pdl(kf, grid, G_THREADS, sm, s, mx, mw, ml, p, d);                                    \
  }
  if (bn == 64) GF(64, 4) else if (bn == 128) GF(128, 3) else GF(256, 2)
#undef GF
  return cudaGetLastError();
}

cudaError_t launch_gate_dx_tc(const void* wg, const void* dxbuf, const void* dlb, int maxT,
                              int n_pad, RouteBufs b, int T, int k, int n, int d,
                              const CapTable& ct, void* dx, int accumulate, cudaStream_t s,
                              const PeerBufs& pdx, int drop_only, bool nowait) {
  if (T == 0) return cudaSuccess;
  if (!enc_init()) return cudaErrorNotSupported;
  CUtensorMap mhi, mlo, mw;
  const __nv_bfloat16* hi = (const __nv_bfloat16*)dlb;
  const __nv_bfloat16* lo = hi + (size_t)maxT * n_pad;
  if (!map2d(&mhi, hi, n_pad, T, 64, 128) || !map2d(&mlo, lo, n_pad, T, 64, 128) ||
      !map2d(&mw, wg, d, n, 64, 64))
    return cudaErrorInvalidValue;
  GateDxParams p{};
  p.T = T; p.n_pad = n_pad; p.k = k; p.d = d; p.grow = b.grow;
  p.dxbuf = (const __nv_bfloat16*)dxbuf; p.dx = (__nv_bfloat16*)dx; p.accumulate = accumulate;
  p.ct = ct;
  p.pdx = pdx;
  p.drop_only = drop_only;
  p.drop_tok = b.drop_tok;
  p.drop_cnt = b.drop_cnt;
  p.nowait = (nowait && drop_only) ? 1 : 0;  // the drop-only pass reads nothing of the dX GEMM
  const int bn = d % 128 == 0 ? 128 : 64;
  const int total = ((T + 127) / 128) * (d / bn);
  const int grid = total < g_sms ? total : g_sms;
  (void)n;
#define GX(BN, ST)                                                                       \
  {                                                                                      \
    auto kf = pdx.nl ? gate_dx_tc_kernel<BN, ST, true> : gate_dx_tc_kernel<BN, ST, false>; \
    size_t sm = smem_for((128 + BN) * 64 * 2, ST) + 8 * 2 * 2 * 32 * (BN + 16);          \
    cudaError_t e = set_smem(kf, sm);                                                    \
    if (e != cudaSuccess) return e;                                                      \
    launch_pdl(kf, grid, GX_THREADS, sm, s, mhi, mlo, mw, p);                                     \
  }
  if (bn == 128) GX(128, 2) else GX(64, 4)
#undef GX
  return cudaGetLastError();
}

int gate_dw_tc_splits(int T, int n, int d) {
  const int bn = d % 256 == 0 ? 256 : (d % 128 == 0 ? 128 : 64);
  const int tiles = ((n + 127) / 128) * (d / bn);
  int want = (g_sms + tiles - 1) / tiles;
  int maxs = (T + 255) / 256;
  if (want > maxs) want = maxs;
  return want < 1 ? 1 : want;
}

cudaError_t launch_gate_dw_tc(const void* dlb, int maxT, int n_pad, const void* x, int T, int n,
                              int d, float* partial, void* dwg, int accumulate, cudaStream_t s,
                              float* f32_out, bool nowait) {
  const size_t count = (size_t)n * d;
  if (f32_out && T == 0) return cudaMemsetAsync(f32_out, 0, count * 4, s);
  if (T == 0) {
    if (!accumulate) return cudaMemsetAsync(dwg, 0, count * 2, s);
    return cudaSuccess;
  }
  if (!enc_init()) return cudaErrorNotSupported;
  int splits = gate_dw_tc_splits(T, n, d);
  int chunk = (T + splits - 1) / splits;
  chunk = (chunk + 63) / 64 * 64;
  splits = (T + chunk - 1) / chunk;
  CUtensorMap mhi, mlo, mx;
  const __nv_bfloat16* hi = (const __nv_bfloat16*)dlb;
  const __nv_bfloat16* lo = hi + (size_t)maxT * n_pad;
  if (!map2d(&mhi, hi, n_pad, T, 64, 64) || !map2d(&mlo, lo, n_pad, T, 64, 64) ||
      !map2d(&mx, x, d, T, 64, 64))
    return cudaErrorInvalidValue;
  GateDwParams p{T, n, d, chunk, splits, partial, nowait ? 1 : 0};
  const int bn = d % 256 == 0 ? 256 : (d % 128 == 0 ? 128 : 64);
  const int total = splits * ((n + 127) / 128) * (d / bn);
  const int grid = total < g_sms ? total : g_sms;
#define GW(BN, ST)                                                                       \
  {                                                                                      \
    auto kf = gate_dw_tc_kernel<BN, ST>;                                                 \
    size_t sm = smem_for((2 * 128 + BN) * 64 * 2, ST);                                   \
    cudaError_t e = set_smem(kf, sm);                                                    \
    if (e != cudaSuccess) return e;                                                      \
    launch_pdl(kf, grid, G_THREADS, sm, s, mhi, mlo, mx, p);                                     \
  }
  if (bn == 256) GW(256, 3) else if (bn == 128) GW(128, 4) else GW(64, 5)
#undef GW
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (f32_out) return launch_reduce_partials(0, partial, splits, count, f32_out, 0, s);
  // nowait: the reduction closes the backward with a full-dependency launch (it also waits for
  // every kernel that skipped its PDL wait)
  return launch_reduce_partials(1, partial, splits, count, dwg, accumulate, s, nowait);
}

}  // namespace moe
