// kernels.h -- host-side launchers of the hot-path kernels (internal; not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "common.cuh"

namespace moe {

// Device scratch shared by the launchers (all pointers into the caller's workspace).
struct RouteBufs {
  float* logits;          // [T x n]
  int32_t* idx;           // [T x k] dispatch indices
  int32_t* fresh_idx;     // [T x k] fresh top-k (cached mode; == idx otherwise)
  float* w;               // [T x k]
  int32_t* slot_of;       // [T x k]
  int32_t* token_of_slot; // [rows]
  int32_t* tile_hist;     // [ntiles x n]
  int32_t* tile_off;      // [ntiles x n]
  int32_t* counts;        // [n]
  int32_t* kept;          // [n]
  int32_t* mtile_prefix;  // [n+1] prefix of ceil(kept_e / 128) (GEMM tile scheduler)
  int64_t* drops;         // [1]
  int32_t* hit_count;     // [1]
  int32_t* flags;         // [1] device error flags
  uint32_t* ticket;       // [1] last-block ticket of route_scan (self-resetting)
  float* dw;              // [T x k]
  float* dl;              // [T x n]
  // optional loss variants (N3); null = off
  void* spec;             // [T*k x d_out] AggregateSpec rows (forward output)
  uint8_t* spec_valid;    // [T*k]
  const void* dspec;      // [T*k x d_out] gradient w.r.t. the spec rows (backward input)
  const float* dw_ext;    // [T x k] extra gradient w.r.t. the gate weights (backward input)
  const float* bal_g;     // [n] balance-term coefficients lambda*n*T_i/T_g (backward)
  int32_t* grow;          // [T x k] token-side dO/dX row of each pair or -1 (combine_bwd)
  __nv_bfloat16* dlr;     // [rows x 2 n_pad] hi | lo of dl by expert row (fused dX, k = 1)
  PeerBufs pdlr;          // peer EP: the owners' dlr regions (nl == 0: dlr is local)
  __nv_bfloat16* dropb;   // fused dX (k = 1): [2 maxT x n_pad] dl pairs of dropped tokens,
                          // compacted (dlb layout); null = off
  int32_t* drop_tok;      // [maxT] token of each compacted row
  int32_t* drop_cnt;      // [1] rows in the list (reset by route_scan, counted by combine_bwd)
  int gate_hist;          // the tcgen05 gate also writes tile_hist (route_hist skipped)
  int o_pair;             // O of pair (t, r) at row t k + r: peer EP return rows (stored by the
                          // owners' GEMM epilogues) or the single-GPU token-ordered O (OTOK)
  int dx_pair;            // peer EP return rows: dX of pair (t, r) at row t k + r as well
  int32_t* idx_fix;       // cache fallback mode: the gate writes the fresh top-k of unknown
                          // samples (cached row with -1) into these dispatch-index rows
  float* sstat;           // [T x 4] softmax statistics (m, sum exp, exp mass outside the dispatch
                          // set, 0) written by the tcgen05 gate for the combine backward, or null
};

// Per-sample assignment cache (N4; SPEC cache_step / cached_route): idx[t] = table[ids[t]]
// (flag 4 and a -1 row for an out-of-range id) / table[ids[t]] = fresh[t].
cudaError_t launch_cache_gather(const int32_t* table, int64_t num, int k, const int64_t* ids,
                                int T, int32_t* idx, int32_t* flags, cudaStream_t s);
cudaError_t launch_cache_observe(int32_t* table, int64_t num, int k, const int64_t* ids, int T,
                                 const int32_t* fresh, int32_t* hit, int32_t* flags,
                                 cudaStream_t s);
cudaError_t launch_cache_update(int32_t* table, int64_t num, int k, const int64_t* ids, int T,
                                const int32_t* fresh, cudaStream_t s);

// dtype: 0 = fp32, 1 = bf16 for every templated launcher below.
cudaError_t launch_gate_topk(int dtype, const void* x, const void* wg, int T, int n, int d,
                             int k, int renorm, const int32_t* cached, RouteBufs b,
                             cudaStream_t s);
cudaError_t launch_route_hist(int32_t* idx, int T, int k, int n, int32_t* hist,
                              cudaStream_t s, const int32_t* src = nullptr);
cudaError_t launch_route_scan(const int32_t* hist, int ntiles, int n, const CapTable& ct,
                              RouteBufs b, cudaStream_t s);
cudaError_t launch_dispatch(int dtype, const int32_t* idx, const void* x, int T, int k,
                            int n, int d, int64_t token_base, const CapTable& ct,
                            RouteBufs b, void* xbuf, const int32_t* pad_kept, cudaStream_t s,
                            int pad_e0 = 0, const PeerBufs& px = PeerBufs{},
                            const PeerBufs& ptos = PeerBufs{}, const int32_t* pre_dev = nullptr,
                            void* y_zero = nullptr, int dout = 0);
// fused dispatch backward in peer EP (k = 1): dx[t] = the (t, 0) row the owner's dX GEMM
// returned (dX + dl W_g), for kept tokens (dropped ones come from the drop-only gate-dx pass)
cudaError_t launch_dx_from_ret(const void* dxret, const int32_t* slot_of, int T, int d, void* dx,
                               int accumulate, cudaStream_t s);
cudaError_t launch_zero_pad(int dtype, void* buf, int cols, const int32_t* kept, int n,
                            const CapTable& ct, cudaStream_t s);
cudaError_t launch_combine_fwd(int dtype, const void* obuf, RouteBufs b, int T, int k,
                               int d_out, const CapTable& ct, void* y, cudaStream_t s,
                               const PeerBufs& po = PeerBufs{});
cudaError_t launch_combine_bwd(int dtype, const void* dy, const void* obuf, RouteBufs b,
                               int T, int k, int n, int d_out, int renorm,
                               const CapTable& ct, void* dobuf, void* dlb, int maxT, int n_pad,
                               const int32_t* pad_kept, cudaStream_t s, int pad_e0 = 0,
                               const PeerBufs& po = PeerBufs{}, const PeerBufs& pdo = PeerBufs{});
cudaError_t launch_gate_dx(int dtype, const void* wg, const void* dxbuf, RouteBufs b, int T,
                           int k, int n, int d, const CapTable& ct, void* dx, int accumulate,
                           cudaStream_t s, const PeerBufs& pdx = PeerBufs{});
// f32_out != null: write the fp32 sum there instead (EP: all-reduced before rounding)
cudaError_t launch_gate_dw(int dtype, const float* dl, const void* x, int T, int n, int d,
                           float* partial, int splits, void* dwg, int accumulate,
                           cudaStream_t s, float* f32_out = nullptr, bool nowait = false);
// (nowait: no PDL wait in the partial kernel, full-dependency reduction -- the backward tail)
cudaError_t launch_f32_to(int dtype, const float* in, size_t count, void* out, int accumulate,
                          cudaStream_t s);
int gate_dw_splits(int T, int d);
cudaError_t launch_reduce_partials(int dtype, const float* partial, int splits, size_t count,
                                   void* out, int accumulate, cudaStream_t s,
                                   bool full_dep = false);
cudaError_t launch_colsum(int dtype, const void* buf, int cols, const int32_t* kept, int n,
                          const CapTable& ct, void* out, int accumulate, cudaStream_t s);

// Eq. 3 balance term (aux_kernels.cu)
cudaError_t launch_balance_partial(const float* logits, int T, int n, float* partial,
                                   float* gsum, cudaStream_t s);
cudaError_t launch_balance_final(const float* gsum, const int32_t* counts, int n, int k,
                                 int64_t Tg, float lam, float* g_out, float* aux_out,
                                 cudaStream_t s);

// Grouped GEMMs of the expert FFN (SIMT fp32/bf16 path, gemm_simt.cu).
enum EpiKind { EPI_BIAS_RELU = 0, EPI_BIAS = 1, EPI_RELU_MASK = 2, EPI_NONE = 3 };
// M-grouped: for each local expert e with M_e = kept[e] rows:
//   C[base_e + m, :] = epi( A[base_e + m, :K] . B_e )
//   b_kmajor = 1: B_e stored [N x K] (row-major, torch Linear weight), 0: stored [K x N].
cudaError_t launch_gemm_simt_mgroup(int dtype, const void* A, int lda, const void* B,
                                    int b_kmajor, int64_t b_estride, const void* bias,
                                    void* C, int ldc, int N, int K, const int32_t* kept,
                                    int n_local, const CapTable& ct, int max_rows, int epi,
                                    cudaStream_t s);
// K-grouped (weight gradients): for each local expert e, Out_e[M x N] (+)= A_e^T . B_e with
// A_e = Abuf[base_e : base_e + kept_e, :M], B_e = Bbuf[base_e : base_e + kept_e, :N].
cudaError_t launch_gemm_simt_kgroup(int dtype, const void* Abuf, int lda, const void* Bbuf,
                                    int ldb, void* Out, int M, int N, const int32_t* kept,
                                    int n_local, const CapTable& ct, int accumulate,
                                    cudaStream_t s);

}  // namespace moe
