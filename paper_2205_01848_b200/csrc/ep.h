// ep.h -- expert parallelism over NCCL: experts are partitioned contiguously
// over R ranks (rank r owns [r n/R, (r+1) n/R)), tokens are data-parallel, capacity is GLOBAL
// (reading 12) so routing equals the single-GPU routing over the concatenated batch.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/moe.h"
#include "common.cuh"

namespace moe {

// Host-side exchange plan computed identically on every rank from the all-gathered
// per-(rank, expert) pre-drop counts (one host sync per forward; reused by the backward).
struct EpPlan {
  int R = 1, rank = 0, n = 0, n_local = 0, e_lo = 0;
  std::vector<int32_t> cnt;       // [R*n] all-gathered local counts
  std::vector<int32_t> pre;       // [R*n] pairs of lower ranks routed to e (global slot offset)
  std::vector<int32_t> kl;        // [R*n] kept pairs of rank r for expert e
  std::vector<int32_t> send_off;  // [n] this rank's send-buffer row offset per expert
  std::vector<int32_t> counts;    // [n] global pre-drop counts
  std::vector<int32_t> kept_local;   // [n_local] global kept for local experts
  std::vector<int32_t> mtile_prefix; // [n_local+1] prefix of ceil(kept_local/128)
  int64_t drops = 0;
  int64_t send_rows = 0;
};

// Pure host planning (exported through moe_ep_plan for tests).
void ep_make_plan(EpPlan& P, int R, int rank, int n, const int32_t* cnt_all, const int32_t* cap);

struct EpState;
moe_status_t ep_create(EpState** out, void* nccl_comm, int R, int rank, std::string* err);
void ep_destroy(EpState* s);

// C1: all-gather the local counts [n] -> dev_all [R*n] and copy them to the host (synchronises
// the calling thread with `st`).  Fills the plan.
moe_status_t ep_exchange_counts(EpState* s, const int32_t* dev_counts, int32_t* dev_all, int n,
                                const int32_t* cap, cudaStream_t st, EpPlan& plan,
                                std::string* err);
// C2/C4: token rows src(send layout) -> owners' expert regions (dst = X_buf / dO_buf).
moe_status_t ep_to_experts(EpState* s, const EpPlan& P, const void* sendbuf, void* dst,
                           const CapTable& ct_local, int cols, int elem_bytes, cudaStream_t st,
                           std::string* err);
// C3/C5: expert rows (src = O_buf / dX_buf) -> back to the token owners' send layout.
moe_status_t ep_from_experts(EpState* s, const EpPlan& P, const void* src, void* recvbuf,
                             const CapTable& ct_local, int cols, int elem_bytes,
                             cudaStream_t st, std::string* err);
// C6: in-place sum all-reduce of fp32 data.
moe_status_t ep_allreduce_f32(EpState* s, float* buf, size_t count, cudaStream_t st,
                              std::string* err);

// Virtual communicator (R ranks as threads of one process on one GPU; test transport).
moe_status_t vcomm_create(int R, void** out);
moe_status_t vcomm_destroy(void* p);

}  // namespace moe
