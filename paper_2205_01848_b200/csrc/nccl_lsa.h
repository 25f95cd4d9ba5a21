// nccl_lsa.h -- peer windows allocated and mapped through NCCL symmetric memory (see .cu).
#pragma once
#include <stddef.h>
#include <string>

#include "../../include/moe.h"

namespace moe {

struct LsaWindow {
  void* comm = nullptr;  // ncclComm_t the window is registered on
  void* win = nullptr;   // ncclWindow_t
  void* buf = nullptr;   // this rank's window (ncclMemAlloc)
  size_t bytes = 0;
};

// Collective over `comm` (every rank of the layer's expert-parallel group, in rank order of
// the communicator): allocate `bytes` of symmetric memory, zero it, register it as a window
// and return every world rank's mapping of it in ptrs_out[R] (ptrs_out[rank] = w->buf, the
// peers' entries are their windows' addresses in this process's LSA flat mapping).
moe_status_t lsa_window_create(void* comm, int R, int rank, size_t bytes, LsaWindow* w,
                               void** ptrs_out, std::string* err);
// Deregister (collective on the communicator) and free.
void lsa_window_destroy(LsaWindow* w);

}  // namespace moe
