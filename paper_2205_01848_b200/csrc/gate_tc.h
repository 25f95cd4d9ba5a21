// gate_tc.h -- launchers of the tcgen05 gate kernels (bf16 layers), see gate_tc.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "common.cuh"
#include "kernels.h"

namespace moe {
// Cached mode with the dispatch fused into the gate (single GPU, bf16): the gate kernel also
// writes slot_of / token_of_slot from the cached rows and copies the kept x rows into X_buf
// from its TMA stages (x read once for both), zeroes X_buf's pad rows and, with the fused
// combine, the y rows of tokens with every pair dropped.  Needs route_scan's tile offsets.
struct GateDispatch {
  const CapTable* ct;
  void* xbuf;
  void* y_zero;  // or null
  int dout;
};
cudaError_t launch_gate_fwd_tc(const void* x, const void* wg, int T, int n, int d, int k,
                               int renorm, const int32_t* cached, RouteBufs b, cudaStream_t s,
                               const GateDispatch* gd = nullptr);
cudaError_t launch_gate_dx_tc(const void* wg, const void* dxbuf, const void* dlb, int maxT,
                              int n_pad, RouteBufs b, int T, int k, int n, int d,
                              const CapTable& ct, void* dx, int accumulate, cudaStream_t s,
                              const PeerBufs& pdx = PeerBufs{}, int drop_only = 0,
                              bool nowait = false);
cudaError_t launch_gate_dw_tc(const void* dlb, int maxT, int n_pad, const void* x, int T, int n,
                              int d, float* partial, void* dwg, int accumulate, cudaStream_t s,
                              float* f32_out = nullptr, bool nowait = false);
// nowait (single GPU, backward tail): the drop-only gate-dx pass and the gate-weight
// gradient skip their PDL wait (their inputs are complete before their predecessor started)
// and run beside the dX GEMM's tail; the gate-weight reduction then closes the backward with
// a full-dependency launch.
int gate_dw_tc_splits(int T, int n, int d);
}  // namespace moe
