// nccl_lsa.cu -- peer windows as NCCL symmetric memory (NCCL >= 2.28 device API, LSA team).
//
// The peer transport (peer.h, N1) needs every rank's window mapped in every rank's address
// space.  moe_peer_import does it with CUDA IPC handles all-gathered over a host channel;
// this file does it on the caller's NCCL communicator instead (torch's ProcessGroupNCCL
// communicator in practice), so the exchange rides the same communicator as everything else:
//   ncclMemAlloc (cuMem, NVLink-mappable) -> zero -> ncclCommWindowRegister(..., SYMMETRIC)
//   (collective) -> one device thread asks ncclGetPeerPointer(window, 0, r) for every world
//   rank r of the load/store-accessible (LSA) team -> the same PeerBufs the kernels use.
// The LSA team must span all R ranks (one NVLink / NVSwitch domain, e.g. the 8 GPUs of a
// B200 box); otherwise MOE_ERR_NCCL and the caller keeps the IPC path.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstring>
#include <string>

#include "nccl_lsa.h"

namespace moe {

namespace {

struct NcclSyms {
  void* lib = nullptr;
  ncclResult_t (*memAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*memFree)(void*) = nullptr;
  ncclResult_t (*winRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
  ncclResult_t (*winDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
  ncclTeam_t (*teamLsa)(ncclComm_t) = nullptr;
  ncclResult_t (*commCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*commUserRank)(const ncclComm_t, int*) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
};

template <typename F>
bool sym(void* lib, const char* name, F& fn) {
  fn = reinterpret_cast<F>(dlsym(lib, name));
  return fn != nullptr;
}

NcclSyms* syms(std::string* err) {
  static NcclSyms s;
  static bool tried = false, ok = false;
  if (tried) {
    if (!ok) *err = "libnccl.so.2 without the symmetric-memory / device API (NCCL >= 2.28)";
    return ok ? &s : nullptr;
  }
  tried = true;
  s.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's, already loaded
  if (!s.lib) s.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  ok = s.lib && sym(s.lib, "ncclMemAlloc", s.memAlloc) && sym(s.lib, "ncclMemFree", s.memFree) &&
       sym(s.lib, "ncclCommWindowRegister", s.winRegister) &&
       sym(s.lib, "ncclCommWindowDeregister", s.winDeregister) &&
       sym(s.lib, "ncclTeamLsa", s.teamLsa) && sym(s.lib, "ncclCommCount", s.commCount) &&
       sym(s.lib, "ncclCommUserRank", s.commUserRank) &&
       sym(s.lib, "ncclGetErrorString", s.errStr);
  if (!ok) *err = "libnccl.so.2 without the symmetric-memory / device API (NCCL >= 2.28)";
  return ok ? &s : nullptr;
}

// world rank r's mapping of the window (LSA team = all ranks, checked on the host)
__global__ void lsa_pointers_kernel(ncclWindow_t win, int R, void** out) {
  if (threadIdx.x == 0)
    for (int r = 0; r < R; ++r) out[r] = ncclGetPeerPointer(win, 0, r);
}

}  // namespace

moe_status_t lsa_window_create(void* comm_v, int R, int rank, size_t bytes, LsaWindow* w,
                               void** ptrs_out, std::string* err) {
  NcclSyms* s = syms(err);
  if (!s) return MOE_ERR_NCCL;
  ncclComm_t comm = (ncclComm_t)comm_v;
  int nr = 0, me = -1;
  if (s->commCount(comm, &nr) != ncclSuccess || s->commUserRank(comm, &me) != ncclSuccess ||
      nr != R || me != rank) {
    *err = "NCCL communicator size / rank differ from the layer's world_size / rank";
    return MOE_ERR_INVALID_ARG;
  }
  const ncclTeam_t team = s->teamLsa(comm);
  if (team.nRanks != R) {
    *err = "not every rank is load/store-accessible over NVLink (LSA team " +
           std::to_string(team.nRanks) + " of " + std::to_string(R) + ")";
    return MOE_ERR_NCCL;
  }
  const size_t sz = (bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) /
                    NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
  void* buf = nullptr;
  ncclResult_t nr_ = s->memAlloc(&buf, sz);
  if (nr_ != ncclSuccess) {
    *err = std::string("ncclMemAlloc: ") + s->errStr(nr_);
    return MOE_ERR_NCCL;
  }
  // zeroed and complete before any peer can see it (epoch / flag words start at 0)
  if (cudaMemset(buf, 0, sz) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    s->memFree(buf);
    *err = "zeroing the NCCL window failed";
    return MOE_ERR_CUDA;
  }
  ncclWindow_t win = nullptr;
  nr_ = s->winRegister(comm, buf, sz, &win, NCCL_WIN_COLL_SYMMETRIC);  // collective
  if (nr_ != ncclSuccess) {
    s->memFree(buf);
    *err = std::string("ncclCommWindowRegister: ") + s->errStr(nr_);
    return MOE_ERR_NCCL;
  }
  void** dptrs = nullptr;
  if (cudaMalloc(&dptrs, sizeof(void*) * R) != cudaSuccess) {
    s->winDeregister(comm, win);
    s->memFree(buf);
    return MOE_ERR_CUDA;
  }
  lsa_pointers_kernel<<<1, 32>>>(win, R, dptrs);
  cudaError_t ce = cudaMemcpy(ptrs_out, dptrs, sizeof(void*) * R, cudaMemcpyDeviceToHost);
  cudaFree(dptrs);
  if (ce != cudaSuccess || !ptrs_out[rank]) {
    s->winDeregister(comm, win);
    s->memFree(buf);
    *err = "reading the LSA pointers failed";
    return MOE_ERR_CUDA;
  }
  // own window through the allocation's own address (the LSA flat mapping of it is another
  // virtual address of the same memory)
  ptrs_out[rank] = buf;
  w->comm = comm_v;
  w->win = win;
  w->buf = buf;
  w->bytes = sz;
  return MOE_OK;
}

void lsa_window_destroy(LsaWindow* w) {
  if (!w || !w->buf) return;
  std::string err;
  NcclSyms* s = syms(&err);
  if (s) {
    cudaDeviceSynchronize();
    s->winDeregister((ncclComm_t)w->comm, (ncclWindow_t)w->win);
    s->memFree(w->buf);
  }
  *w = LsaWindow{};
}

}  // namespace moe
