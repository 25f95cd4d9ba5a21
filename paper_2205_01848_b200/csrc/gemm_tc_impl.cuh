// gemm_tc_impl.cuh -- definitions shared by the 1-CTA and 2-CTA tcgen05 grouped GEMMs.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include "common.cuh"
#include "tc_common.cuh"

namespace moe {

enum TcKind { TC_FWD1 = 0, TC_FWD2 = 1, TC_DGRAD_A = 2, TC_DGRAD_X = 3, TC_WGRAD = 4 };

constexpr int TC_THREADS = 384;     // 4 control warps + 8 epilogue warps
constexpr int TC_EPI_THREADS = 256;

struct TcParams {
  const int32_t* kept;          // [n_local] M_e (M-grouped) or K_e (WGRAD)
  const int32_t* mtile_prefix;  // [n_local+1] prefix of ceil(kept/128) (M-grouped)
  int n_local;
  int M, N, K;                  // WGRAD: M, N output dims; M-grouped: N cols, K depth
  const __nv_bfloat16* bias;    // FWD1/FWD2 bias [n_local, N]
  __nv_bfloat16* bias_out;      // WGRAD: fused bias gradient db[e][m] = sum_t A[t, m] (or null)
  __nv_bfloat16* C;             // output base (buffer or weight-gradient tensor)
  int ldc;                      // leading dim of C (M-grouped buffers)
  int accumulate;               // WGRAD
  float* bias_part;             // 2-CTA DGRAD_A: per-(256-row m-tile, CTA) column sums of dA,
                                // [sum_e ceil(kept_e/256) * 2][N] fp32 (db1 partials)
  uint32_t* mask;               // FWD1 writes / DGRAD_A reads: bit j of word [row][c] = (H > 0)
                                // for column 32c + j (relu' mask, 16x fewer bytes than H)
  int pf_kb;                    // 2-CTA: k-blocks of the next wave's B tile to prefetch to L2
  int sched;                    // 2-CTA tile schedule: 0 round-robin (m fastest),
                                // 1 contiguous chunk per CTA pair (n fastest), 2 chunk (m fastest)
  int dbg;                      // timing experiments (MOE_TC_DBG), 0 in production
  // N2 gather fusion (2-CTA only).  gtos != null: the x rows of expert slot (base_e + s) are
  // loaded by TMA tile::gather4 straight from x (row token_of_slot / gk) instead of from a
  // dispatched X buffer -- FWD1: the A operand, WGRAD: the B operand (token rows).  Slots
  // s >= kept_e use row grows (= T, out of bounds: TMA fills zeros).
  const int32_t* gtos;
  int gk;
  int grows;
  // N2 combine fusion (FWD2, k = 1): y[t] = w[t] * O[row] written by the epilogue next to O.
  __nv_bfloat16* y;
  const float* wt;
  // k = 2 (comb2, with O in (token, choice) order in pret.p[0]): per (token, column block) the
  // epilogue that finishes second reads both stored O rows and writes y (counters ycnt, ycb
  // blocks per token, self-resetting; slot2 = slot_of [T x 2] to see dropped pairs)
  int comb2;
  const int32_t* slot2;
  uint32_t* ycnt;
  int ycb;
  // N2 dispatch-backward fusion (DGRAD_X, k = 1): nkx extra k-blocks accumulate the gate term
  // dl[t] W_g (A2 = [hi | lo](dl) rows in expert-row order, B2 = W_g, nbx = n_pad / 64), and
  // the epilogue writes dx[t] (token order, via gtos) instead of the dX buffer.
  __nv_bfloat16* dxo;
  int nkx, nbx;
  // N1 return rows (peer EP, FWD2 / DGRAD_X): pret.p[j] = rank j's return buffer; output row
  // of global pair gp = t_g k + r goes to rank gp / (k tpr) at pair gp mod (k tpr); nl != 0 = on
  PeerBufs pret;
  int tpr;
  CapTable ct;                  // base rows of each local expert region
  int nowait;                   // inputs complete once the predecessor started: no PDL wait
  int half_tiles;               // 2-CTA M-grouped: remainder m-tiles of <= 128 rows run as M = 128
  int no_ktrim;                 // 2-CTA WGRAD: 1 = the last k-block issues all four 16-deep MMAs
                                // (A/B switch MOE_NO_KTRIM=1; default: only those holding tokens)
  const void* hsrc;             // fp32 DGRAD_A: H for the ReLU' test when dA is not written
                                // over it (null = C itself holds H)
};

template <int KIND>
struct KindTraits {
  static constexpr bool kgroup = (KIND == TC_WGRAD);
  static constexpr int a_mn = (KIND == TC_WGRAD) ? 1 : 0;
  static constexpr int b_mn = (KIND == TC_DGRAD_A || KIND == TC_DGRAD_X || KIND == TC_WGRAD) ? 1 : 0;
};

// Decode a linear tile index into (expert, m0, n0).
// total number of tiles (M-grouped: prefix of m-tiles x NT; K-grouped: n_local x MT x NT)
template <bool KG>
__device__ __forceinline__ int total_tiles(const int32_t* s_prefix, int n_local, int MT, int NT) {
  return KG ? n_local * MT * NT : s_prefix[n_local] * NT;
}

// Like decode_tile, with the order inside an expert selectable: nfast = n-tile fastest (the
// A m-tile is reused by consecutive tiles of one CTA pair) or m-tile fastest.
template <bool KG>
__device__ __forceinline__ bool decode_tile_ord(int t, const int32_t* s_prefix, int n_local,
                                                int MT, int NT, bool nfast, int& e, int& mt,
                                                int& nt) {
  int r, mte;
  if (KG) {
    const int per = MT * NT;
    e = t / per;
    if (e >= n_local) return false;
    r = t - e * per;
    mte = MT;
  } else {
    if (t >= s_prefix[n_local] * NT) return false;
    int lo = 0, hi = n_local - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (s_prefix[mid] * NT <= t) lo = mid; else hi = mid - 1;
    }
    e = lo;
    r = t - s_prefix[e] * NT;
    mte = s_prefix[e + 1] - s_prefix[e];
  }
  if (nfast) {
    mt = r / NT;
    nt = r - mt * NT;
  } else {
    nt = r / mte;
    mt = r - nt * mte;
  }
  return true;
}

template <bool KG>
__device__ __forceinline__ bool decode_tile(int t, const int32_t* s_prefix, int n_local, int MT,
                                            int NT, int& e, int& mt, int& nt) {
  if (KG) {
    int per = MT * NT;
    e = t / per;
    if (e >= n_local) return false;
    int r = t - e * per;
    nt = r / MT;
    mt = r - nt * MT;
    return true;
  } else {
    // s_prefix[j] = sum_{e<j} mtiles(e); tiles of expert e: [prefix[e]*NT, prefix[e+1]*NT)
    int total = s_prefix[n_local] * NT;
    if (t >= total) return false;
    int lo = 0, hi = n_local - 1;
    while (lo < hi) {  // largest e with prefix[e]*NT <= t
      int mid = (lo + hi + 1) >> 1;
      if (s_prefix[mid] * NT <= t) lo = mid; else hi = mid - 1;
    }
    e = lo;
    int r = t - s_prefix[e] * NT;
    int mte = s_prefix[e + 1] - s_prefix[e];
    nt = r / mte;
    mt = r - nt * mte;
    return true;
  }
}


}  // namespace moe
