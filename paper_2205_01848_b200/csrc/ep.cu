// ep.cu -- NCCL plumbing of the expert-parallel MoE layer (C1-C6 of SURVEY §2c).
//
// NCCL is resolved at run time from the libnccl.so.2 already loaded by torch (dlopen with
// RTLD_NOLOAD first), so the library shares torch's NCCL instance and communicator
// (ProcessGroupNCCL._comm_ptr()).  All collectives are enqueued on the layer's stream.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>

#include "ep.h"

namespace moe {

typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
enum { NCCL_INT32 = 2, NCCL_FLOAT32 = 7, NCCL_BF16 = 9, NCCL_UINT8 = 1 };
enum { NCCL_SUM = 0 };

struct EpState {
  void* lib = nullptr;
  ncclComm_t comm = nullptr;
  int R = 1, rank = 0;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  int32_t* host_all = nullptr;  // pinned [R * 256]
  cudaEvent_t ev = nullptr;
};

void ep_make_plan(EpPlan& P, int R, int rank, int n, const int32_t* cnt_all, const int32_t* cap) {
  P.R = R; P.rank = rank; P.n = n; P.n_local = n / R; P.e_lo = rank * P.n_local;
  P.cnt.assign(cnt_all, cnt_all + (size_t)R * n);
  P.pre.assign((size_t)R * n, 0);
  P.kl.assign((size_t)R * n, 0);
  P.counts.assign(n, 0);
  for (int e = 0; e < n; ++e) {
    int64_t run = 0;
    for (int r = 0; r < R; ++r) {
      const int c = cnt_all[(size_t)r * n + e];
      P.pre[(size_t)r * n + e] = (int32_t)run;
      // kept pairs of rank r for expert e: global slots [run, run + c) below the capacity
      const int64_t room = std::max<int64_t>(0, (int64_t)cap[e] - run);
      P.kl[(size_t)r * n + e] = (int32_t)std::min<int64_t>(room, c);
      run += c;
    }
    P.counts[e] = (int32_t)run;
  }
  P.drops = 0;
  for (int e = 0; e < n; ++e) P.drops += P.counts[e] - std::min<int64_t>(P.counts[e], cap[e]);
  P.send_off.assign(n, 0);
  int64_t off = 0;
  for (int e = 0; e < n; ++e) {
    P.send_off[e] = (int32_t)off;
    off += P.kl[(size_t)rank * n + e];
  }
  P.send_rows = off;
  P.kept_local.assign(P.n_local, 0);
  P.mtile_prefix.assign(P.n_local + 1, 0);
  int pre = 0;
  for (int j = 0; j < P.n_local; ++j) {
    const int e = P.e_lo + j;
    P.kept_local[j] = std::min(P.counts[e], cap[e]);
    P.mtile_prefix[j] = pre;
    pre += (P.kept_local[j] + 127) / 128;
  }
  P.mtile_prefix[P.n_local] = pre;
}

template <typename F>
static bool sym(void* lib, const char* name, F& fn) {
  fn = reinterpret_cast<F>(dlsym(lib, name));
  return fn != nullptr;
}

moe_status_t ep_create(EpState** out, void* nccl_comm, int R, int rank, std::string* err) {
  EpState* s = new EpState();
  s->comm = (ncclComm_t)nccl_comm;
  s->R = R;
  s->rank = rank;
  s->lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!s->lib) s->lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!s->lib) {
    *err = std::string("cannot load libnccl.so.2: ") + dlerror();
    delete s;
    return MOE_ERR_NCCL;
  }
  bool ok = sym(s->lib, "ncclGroupStart", s->groupStart) && sym(s->lib, "ncclGroupEnd", s->groupEnd) &&
            sym(s->lib, "ncclSend", s->send) && sym(s->lib, "ncclRecv", s->recv) &&
            sym(s->lib, "ncclAllGather", s->allGather) && sym(s->lib, "ncclAllReduce", s->allReduce) &&
            sym(s->lib, "ncclGetErrorString", s->errStr);
  if (!ok) {
    *err = "libnccl.so.2 lacks a required symbol";
    delete s;
    return MOE_ERR_NCCL;
  }
  if (cudaMallocHost(&s->host_all, sizeof(int32_t) * (size_t)R * MOE_MAX_E) != cudaSuccess ||
      cudaEventCreateWithFlags(&s->ev, cudaEventDisableTiming) != cudaSuccess) {
    *err = "cudaMallocHost/cudaEventCreate failed";
    delete s;
    return MOE_ERR_CUDA;
  }
  *out = s;
  return MOE_OK;
}

void ep_destroy(EpState* s) {
  if (!s) return;
  if (s->host_all) cudaFreeHost(s->host_all);
  if (s->ev) cudaEventDestroy(s->ev);
  delete s;
}

#define NCCL_TRY(s, expr)                                                  \
  do {                                                                     \
    ncclResult_t _r = (expr);                                              \
    if (_r != 0) {                                                         \
      *err = std::string(#expr) + ": " + (s)->errStr(_r);                  \
      return MOE_ERR_NCCL;                                                 \
    }                                                                      \
  } while (0)

moe_status_t ep_exchange_counts(EpState* s, const int32_t* dev_counts, int32_t* dev_all, int n,
                                const int32_t* cap, cudaStream_t st, EpPlan& plan,
                                std::string* err) {
  NCCL_TRY(s, s->allGather(dev_counts, dev_all, (size_t)n, NCCL_INT32, s->comm, st));
  if (cudaMemcpyAsync(s->host_all, dev_all, sizeof(int32_t) * (size_t)s->R * n,
                      cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaEventRecord(s->ev, st) != cudaSuccess || cudaEventSynchronize(s->ev) != cudaSuccess) {
    *err = "count exchange D2H failed";
    return MOE_ERR_CUDA;
  }
  ep_make_plan(plan, s->R, s->rank, n, s->host_all, cap);
  return MOE_OK;
}

moe_status_t ep_to_experts(EpState* s, const EpPlan& P, const void* sendbuf, void* dst,
                           const CapTable& ct_local, int cols, int elem_bytes, cudaStream_t st,
                           std::string* err) {
  const size_t row_bytes = (size_t)cols * elem_bytes;
  const int dt = elem_bytes == 2 ? NCCL_BF16 : NCCL_FLOAT32;
  NCCL_TRY(s, s->groupStart());
  // sends: this rank's kept pairs of expert e (ascending e) to owner(e)
  for (int e = 0; e < P.n; ++e) {
    const int rows = P.kl[(size_t)P.rank * P.n + e];
    if (rows <= 0) continue;
    const char* src = (const char*)sendbuf + (size_t)P.send_off[e] * row_bytes;
    NCCL_TRY(s, s->send(src, (size_t)rows * cols, dt, e / P.n_local, s->comm, st));
  }
  // receives: for every local expert (ascending), every source rank's kept pairs land at
  // their global slots (src-major within the expert region, so no second permutation)
  for (int j = 0; j < P.n_local; ++j) {
    const int e = P.e_lo + j;
    for (int r = 0; r < P.R; ++r) {
      const int rows = P.kl[(size_t)r * P.n + e];
      if (rows <= 0) continue;
      char* d = (char*)dst + (size_t)(ct_local.base[j] + P.pre[(size_t)r * P.n + e]) * row_bytes;
      NCCL_TRY(s, s->recv(d, (size_t)rows * cols, dt, r, s->comm, st));
    }
  }
  NCCL_TRY(s, s->groupEnd());
  return MOE_OK;
}

moe_status_t ep_from_experts(EpState* s, const EpPlan& P, const void* src, void* recvbuf,
                             const CapTable& ct_local, int cols, int elem_bytes,
                             cudaStream_t st, std::string* err) {
  const size_t row_bytes = (size_t)cols * elem_bytes;
  const int dt = elem_bytes == 2 ? NCCL_BF16 : NCCL_FLOAT32;
  NCCL_TRY(s, s->groupStart());
  for (int j = 0; j < P.n_local; ++j) {
    const int e = P.e_lo + j;
    for (int r = 0; r < P.R; ++r) {
      const int rows = P.kl[(size_t)r * P.n + e];
      if (rows <= 0) continue;
      const char* sp = (const char*)src + (size_t)(ct_local.base[j] + P.pre[(size_t)r * P.n + e]) * row_bytes;
      NCCL_TRY(s, s->send(sp, (size_t)rows * cols, dt, r, s->comm, st));
    }
  }
  for (int e = 0; e < P.n; ++e) {
    const int rows = P.kl[(size_t)P.rank * P.n + e];
    if (rows <= 0) continue;
    char* d = (char*)recvbuf + (size_t)P.send_off[e] * row_bytes;
    NCCL_TRY(s, s->recv(d, (size_t)rows * cols, dt, e / P.n_local, s->comm, st));
  }
  NCCL_TRY(s, s->groupEnd());
  return MOE_OK;
}

moe_status_t ep_allreduce_f32(EpState* s, float* buf, size_t count, cudaStream_t st,
                              std::string* err) {
  NCCL_TRY(s, s->allReduce(buf, buf, count, NCCL_FLOAT32, NCCL_SUM, s->comm, st));
  return MOE_OK;
}

}  // namespace moe
