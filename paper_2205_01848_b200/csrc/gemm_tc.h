// gemm_tc.h -- tcgen05/TMEM/TMA grouped GEMMs of the expert FFN (bf16, sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/moe.h"
#include "common.cuh"
#include "prof.h"

namespace moe {

// Host-side cache of TMA descriptors keyed by the buffer pointers they were encoded for.
struct TcPlan {
  void* dev_maps = nullptr;   // device copy of tensor maps (unused when passed as params)
  int ready = 0;
};
void tc_plan_free(TcPlan* p);

// N2 fusions of the single-GPU path: the expert GEMMs read the x rows of each
// expert slot straight from x (TMA gather4 by token_of_slot) instead of a dispatched X buffer,
// and (k = 1) the second forward GEMM writes y = w * O next to O instead of a combine pass.
struct TcFusion {
  const void* x = nullptr;        // x [T, d]; null = no gather (X buffer is used)
  int T = 0;
  const int32_t* tos = nullptr;   // token_of_slot by expert-region row (t * k + r)
  int k = 1;
  void* y = nullptr;              // y [T, d_out]; null = separate combine kernel
  const float* w = nullptr;       // gate weights [T] (k = 1)
  // dispatch backward in the dX GEMM (k = 1): dx[t] = dA[row] W1 + [hi|lo](dl)[row] [W_g;W_g]
  bool dx_fused = false;          // dispatch backward inside the dX GEMM (extra k-blocks)
  void* dx = nullptr;             // dx [T, d] written by the epilogue (single GPU), or null
                                  // (peer EP: the rows go to the token owners' dxret)
  const void* dlr = nullptr;      // [rows, 2 n_pad] bf16 hi | lo of dl in expert-row order
  const void* wg = nullptr;       // W_g [n, d]
  int n = 0, n_pad = 64, accumulate = 0;
  // peer EP return rows (N1): O (FWD2) / dX (DGRAD_X) rows stored by the epilogue into the
  // token owners' windows in (token, choice) order; nl == 0 = off
  PeerBufs pret_o{}, pret_dx{};
  int tpr = 0;
  // k = 2 combine in FWD2's epilogue (needs O in (token, choice) order, pret_o.p[0] local):
  // slot_of [T x 2] and the per-(token, column block) counters, zero before the first forward
  int comb2 = 0;
  const int32_t* slot = nullptr;
  uint32_t* ycnt = nullptr;
};
bool tc_gather_supported(int d, int f);     // 2-CTA kernels for FWD1 (N = f) and WGRAD_W1 (N = d)
bool tc_combine_supported(int dout);        // 2-CTA kernel for FWD2 (N = d_out)
bool tc_dx_fusion_supported(int d);         // 2-CTA kernel for DGRAD_X (N = d)
bool tc_peer_return_supported(int d, int dout);  // N1 return rows from FWD2 / DGRAD_X

// Forward: H = relu(X W1_e^T + b1_e), O = H W2_e^T + b2_e over kept_e rows per local expert.
moe_status_t tc_ffn_forward(TcPlan* p, void* X, const void* w1, const void* b1,
                            const void* w2, const void* b2, void* H, void* O, int64_t rows,
                            int d, int f, int dout, const int32_t* kept,
                            const int32_t* mtile_prefix, int n_local, const CapTable& ct,
                            int max_cap, cudaStream_t s, int64_t* nlaunch, Prof* prof,
                            uint32_t* mask, const TcFusion* fz = nullptr,
                            cudaError_t (*between)(void*) = nullptr, void* between_ctx = nullptr);
// (between: enqueued after the FWD1 launch and before FWD2, e.g. the cached-mode join with the
//  gate stream so FWD2's fused combine sees the gate weights)
// Backward: dW2 = dO^T H, db2 = sum dO; dA = (dO W2) * 1[H>0] (into H);
// dW1 = dA^T X, db1 = sum dA; dX = dA W1.
moe_status_t tc_ffn_backward(TcPlan* p, void* X, void* H, void* dO, void* dX, const void* w1,
                             const void* w2, void* dw1, void* db1, void* dw2, void* db2,
                             int accumulate, int64_t rows, int d, int f, int dout,
                             const int32_t* kept, const int32_t* mtile_prefix, int n_local,
                             const CapTable& ct, int max_cap, cudaStream_t s,
                             int64_t* nlaunch, Prof* prof, uint32_t* mask, float* bias_part,
                             const TcFusion* fz = nullptr, int tail_nowait = 0,
                             void* dA_sep = nullptr);
// tail_nowait: the db1 reduction runs after the dX GEMM without a PDL wait (single GPU; the
// caller closes the backward with a full-dependency launch).  dA_sep: [rows x f] buffer for dA
// (else dA is written over H); with it, DGRAD_A also skips its wait in the tail mode.

// fp32 path (c1 / c2): the same expert GEMMs on tcgen05 kind::tf32 with each fp32 operand
// split into two tf32 terms (gemm_tf32.cu): fp32 buffers, bias / db fused as in the bf16
// 1-CTA kernels.
bool tf32_supported(int d, int f, int dout);   // d, f, d_out multiples of 32
moe_status_t tf32_ffn_forward(void* X, const void* w1, const void* b1, const void* w2,
                              const void* b2, void* H, void* O, int64_t rows, int d, int f,
                              int dout, const int32_t* kept, const int32_t* mtile_prefix,
                              int n_local, const CapTable& ct, cudaStream_t s, int64_t* nlaunch,
                              Prof* prof);
moe_status_t tf32_ffn_backward(void* X, void* H, void* dO, void* dX, const void* w1,
                               const void* w2, void* dw1, void* db1, void* dw2, void* db2,
                               int accumulate, int64_t rows, int d, int f, int dout,
                               const int32_t* kept, const int32_t* mtile_prefix, int n_local,
                               const CapTable& ct, cudaStream_t s, int64_t* nlaunch, Prof* prof,
                               int tail_nowait = 0, void* dA_sep = nullptr);

}  // namespace moe
