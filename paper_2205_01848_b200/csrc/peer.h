// peer.h -- expert parallelism through peer memory.
//
// Every rank owns one library-allocated "window" (cudaMalloc, so it can be exported as a CUDA
// IPC handle) holding the buffers other ranks read or write directly over NVLink / NVSwitch:
// the expert-major X / O / dO / dX rows of its LOCAL experts, token_of_slot, the all-gathered
// counts, fp32 reduction slots and the phase flags.  All windows have the same layout, so a
// rank addresses a peer's buffer as  win[peer] + offset.
//
// The exchange is device-initiated -- no host sync, no send buffers, no separate all-to-all:
//  * the plan kernel pushes this rank's pre-drop counts into every peer's count table, waits
//    for all peers (flags), and derives on the device what the NCCL path computes on the host
//    (global counts, this rank's global slot offsets pre[e], the local experts' kept counts,
//    the GEMM m-tile prefix, drops) -- reading 12's global capacity and token-major order;
//  * dispatch stores each kept token row straight into its owner's X buffer at the global
//    slot; combine (and its backward) read O rows from the owners and store dO rows into
//    them; the gate-input gradient reads dX rows from the owners;
//  * between producer and consumer kernels a one-block barrier kernel publishes an epoch
//    value into every peer's flag slot (fence.sc.sys; st.release.sys) and spins until all
//    peers published theirs (ld.acquire.sys).  The producer kernels themselves carry no
//    fences: their (remote) stores precede the barrier kernel in stream order, and the
//    barrier's system-scope release is cumulative over them (the pattern of a separate
//    signal kernel after a peer-writing kernel, as symmetric-memory barriers use).  The plan
//    kernel's barrier also orders iteration i+1's writes into a peer after everything that
//    peer did with its buffers in iteration i.
//  * dW_g and the balance term's column sums are reduced by pulling every rank's fp32 slot
//    and summing in rank order (deterministic, identical on every rank).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace moe {

enum PeerPhase { PH_CNT = 0, PH_X = 1, PH_O = 2, PH_BAL = 3, PH_DO = 4, PH_DX = 5, PH_DW = 6,
                 PH_NUM = 8 };

struct PeerLayout {
  size_t epoch = 0, flags = 256, cnt = 512, bal = 0, dwg = 0, tos = 0, x = 0, o = 0, dob = 0,
         dxb = 0, oret = 0, dxret = 0, dlr = 0, total = 0;
  int64_t rows = 0;  // rows of each expert buffer
};

// Byte layout of a window with `rows` expert-buffer rows.
// oret / dxret: [pair_rows x d_out] / [pair_rows x d] expert outputs and input gradients of
// THIS rank's tokens in (token, choice) order, stored there by the owners' GEMM epilogues.
void peer_layout(PeerLayout& L, int64_t rows, int n, int d, int dout, size_t elem,
                 int64_t pair_rows);

// Plan (one block): publish local counts, barrier, derive the global plan into b.counts
// (global pre-drop counts), b.kept / b.mtile_prefix (local experts), b.drops and pre_out[n].
cudaError_t launch_peer_plan(const PeerBufs& win, int R, int rank, int n, int n_local,
                             const int32_t* local_counts, const CapTable& ct, RouteBufs b,
                             int32_t* pre_out, cudaStream_t s);
// Exchange barrier of `phase` at the current epoch (one block of 32 threads).
cudaError_t launch_peer_barrier(const PeerBufs& win, int R, int rank, int phase, cudaStream_t s,
                                uint32_t* err_flags);
// bounded wait of the barrier kernels (a peer that never arrives raises device flag 8)
#ifndef MOE_PEER_TIMEOUT_NS
#define MOE_PEER_TIMEOUT_NS 20000000000ull
#endif
#define MOE_FLAG_PEER_TIMEOUT 8u
// out[i] (dtype; accumulate) = sum over ranks j = 0..R-1 of ((float*)(win[j] + off))[i].
// dtype 2 = fp32 output.
cudaError_t launch_peer_sum(const PeerBufs& win, size_t off, int R, size_t count, int dtype,
                            void* out, int accumulate, cudaStream_t s);

}  // namespace moe
