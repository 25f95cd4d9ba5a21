// ep.cu -- NCCL plumbing of the expert-parallel MoE layer (C1-C6 of SURVEY §2c).
//
// NCCL is resolved at run time from the libnccl.so.2 already loaded by torch (dlopen with
// RTLD_NOLOAD first), so the library shares torch's NCCL instance and communicator
// (ProcessGroupNCCL._comm_ptr()).  All collectives are enqueued on the layer's stream.
#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <set>

#include "ep.h"

namespace moe {

// ------------------------------------------------------------------------------------------
// Virtual communicator: R ranks as threads of ONE process on ONE GPU, exchanging through
// cudaMemcpyAsync with event rendezvous.  A test transport (NCCL refuses two ranks on one
// device) that runs the complete multi-rank EP code path -- plan, tables, grouped
// send/recv matching, all-gather, fixed-order all-reduce -- on a single B200.
// ------------------------------------------------------------------------------------------
struct VOp {
  bool send;
  const void* sbuf;
  void* rbuf;
  size_t bytes;
  int peer;
};

struct VComm {
  int R = 1;
  std::mutex mu;
  std::condition_variable cv;
  int count = 0;
  uint64_t gen = 0;
  std::vector<std::vector<VOp>> ops;
  std::vector<cudaEvent_t> ready, done;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++count == R) {
      count = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

static std::mutex g_vc_mu;
static std::set<void*> g_vcomms;

static bool is_vcomm(void* p) {
  std::lock_guard<std::mutex> lk(g_vc_mu);
  return g_vcomms.count(p) != 0;
}

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
  // virtual transport state
  VComm* vc = nullptr;
  std::vector<VOp> pending;
  float* scratch = nullptr;
  size_t scratch_bytes = 0;
};

__global__ void vsum_kernel(const float* __restrict__ parts, int R, size_t count,
                            float* __restrict__ out) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  float v = 0.f;
  for (int r = 0; r < R; ++r) v += parts[(size_t)r * count + i];  // fixed rank order
  out[i] = v;
}

// Transport primitives (NCCL or virtual); every rank issues them in the same order.
static moe_status_t tr_group_start(EpState* s, std::string* err) {
  if (s->vc) {
    s->pending.clear();
    return MOE_OK;
  }
  if (s->groupStart() != 0) { *err = "ncclGroupStart failed"; return MOE_ERR_NCCL; }
  return MOE_OK;
}
static moe_status_t tr_send(EpState* s, const void* buf, size_t count, int dt, int esz, int peer,
                            cudaStream_t st, std::string* err) {
  if (s->vc) {
    s->pending.push_back({true, buf, nullptr, count * esz, peer});
    return MOE_OK;
  }
  int r = s->send(buf, count, dt, peer, s->comm, st);
  if (r != 0) { *err = std::string("ncclSend: ") + s->errStr(r); return MOE_ERR_NCCL; }
  return MOE_OK;
}
static moe_status_t tr_recv(EpState* s, void* buf, size_t count, int dt, int esz, int peer,
                            cudaStream_t st, std::string* err) {
  if (s->vc) {
    s->pending.push_back({false, nullptr, buf, count * esz, peer});
    return MOE_OK;
  }
  int r = s->recv(buf, count, dt, peer, s->comm, st);
  if (r != 0) { *err = std::string("ncclRecv: ") + s->errStr(r); return MOE_ERR_NCCL; }
  return MOE_OK;
}
static moe_status_t tr_group_end(EpState* s, cudaStream_t st, std::string* err) {
  if (!s->vc) {
    if (s->groupEnd() != 0) { *err = "ncclGroupEnd failed"; return MOE_ERR_NCCL; }
    return MOE_OK;
  }
  VComm* vc = s->vc;
  const int me = s->rank;
  if (cudaEventRecord(vc->ready[me], st) != cudaSuccess) { *err = "event"; return MOE_ERR_CUDA; }
  vc->ops[me] = s->pending;
  vc->barrier();  // every rank posted its ops and recorded its ready event
  std::vector<int> seen(vc->R, 0);
  moe_status_t status = MOE_OK;
  for (const VOp& op : s->pending) {
    if (op.send) continue;
    const int src = op.peer;
    int want = seen[src]++, j = -1;
    for (const VOp& so : vc->ops[src]) {  // the want-th send from src to me
      if (so.send && so.peer == me && want-- == 0) {
        if (so.bytes != op.bytes) status = MOE_ERR_NCCL;
        cudaStreamWaitEvent(st, vc->ready[src], 0);
        cudaMemcpyAsync(op.rbuf, so.sbuf, op.bytes, cudaMemcpyDeviceToDevice, st);
        j = 0;
        break;
      }
    }
    if (j < 0) status = MOE_ERR_NCCL;  // unmatched receive: NCCL would hang here
  }
  cudaEventRecord(vc->done[me], st);
  vc->barrier();  // every receiver enqueued its copies
  for (int p = 0; p < vc->R; ++p) cudaStreamWaitEvent(st, vc->done[p], 0);  // then reuse
  vc->barrier();
  s->pending.clear();
  if (status != MOE_OK) *err = "virtual transport: send/recv mismatch";
  return status;
}

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
  if (is_vcomm(nccl_comm)) {
    s->vc = (VComm*)nccl_comm;
    if (s->vc->R != R) {
      *err = "virtual communicator size != world_size";
      delete s;
      return MOE_ERR_INVALID_ARG;
    }
    if (cudaMallocHost(&s->host_all, sizeof(int32_t) * (size_t)R * MOE_MAX_E) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ev, cudaEventDisableTiming) != cudaSuccess) {
      delete s;
      return MOE_ERR_CUDA;
    }
    *out = s;
    return MOE_OK;
  }
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
  if (s->scratch) cudaFree(s->scratch);
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
  if (s->vc) {
    moe_status_t q = tr_group_start(s, err);
    for (int r = 0; r < s->R && q == MOE_OK; ++r) q = tr_send(s, dev_counts, (size_t)n, NCCL_INT32, 4, r, st, err);
    for (int r = 0; r < s->R && q == MOE_OK; ++r) q = tr_recv(s, dev_all + (size_t)r * n, (size_t)n, NCCL_INT32, 4, r, st, err);
    if (q == MOE_OK) q = tr_group_end(s, st, err);
    if (q != MOE_OK) return q;
  } else {
    NCCL_TRY(s, s->allGather(dev_counts, dev_all, (size_t)n, NCCL_INT32, s->comm, st));
  }
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
  moe_status_t q = tr_group_start(s, err);
  if (q != MOE_OK) return q;
  // sends: this rank's kept pairs of expert e (ascending e) to owner(e)
  for (int e = 0; e < P.n; ++e) {
    const int rows = P.kl[(size_t)P.rank * P.n + e];
    if (rows <= 0) continue;
    const char* src = (const char*)sendbuf + (size_t)P.send_off[e] * row_bytes;
    q = tr_send(s, src, (size_t)rows * cols, dt, elem_bytes, e / P.n_local, st, err);
    if (q != MOE_OK) return q;
  }
  // receives: for every local expert (ascending), every source rank's kept pairs land at
  // their global slots (src-major within the expert region, so no second permutation)
  for (int j = 0; j < P.n_local; ++j) {
    const int e = P.e_lo + j;
    for (int r = 0; r < P.R; ++r) {
      const int rows = P.kl[(size_t)r * P.n + e];
      if (rows <= 0) continue;
      char* d = (char*)dst + (size_t)(ct_local.base[j] + P.pre[(size_t)r * P.n + e]) * row_bytes;
      q = tr_recv(s, d, (size_t)rows * cols, dt, elem_bytes, r, st, err);
      if (q != MOE_OK) return q;
    }
  }
  return tr_group_end(s, st, err);
}

moe_status_t ep_from_experts(EpState* s, const EpPlan& P, const void* src, void* recvbuf,
                             const CapTable& ct_local, int cols, int elem_bytes,
                             cudaStream_t st, std::string* err) {
  const size_t row_bytes = (size_t)cols * elem_bytes;
  const int dt = elem_bytes == 2 ? NCCL_BF16 : NCCL_FLOAT32;
  moe_status_t q = tr_group_start(s, err);
  if (q != MOE_OK) return q;
  for (int j = 0; j < P.n_local; ++j) {
    const int e = P.e_lo + j;
    for (int r = 0; r < P.R; ++r) {
      const int rows = P.kl[(size_t)r * P.n + e];
      if (rows <= 0) continue;
      const char* sp = (const char*)src + (size_t)(ct_local.base[j] + P.pre[(size_t)r * P.n + e]) * row_bytes;
      q = tr_send(s, sp, (size_t)rows * cols, dt, elem_bytes, r, st, err);
      if (q != MOE_OK) return q;
    }
  }
  for (int e = 0; e < P.n; ++e) {
    const int rows = P.kl[(size_t)P.rank * P.n + e];
    if (rows <= 0) continue;
    char* d = (char*)recvbuf + (size_t)P.send_off[e] * row_bytes;
    q = tr_recv(s, d, (size_t)rows * cols, dt, elem_bytes, e / P.n_local, st, err);
    if (q != MOE_OK) return q;
  }
  return tr_group_end(s, st, err);
}

moe_status_t ep_allreduce_f32(EpState* s, float* buf, size_t count, cudaStream_t st,
                              std::string* err) {
  if (!s->vc) {
    NCCL_TRY(s, s->allReduce(buf, buf, count, NCCL_FLOAT32, NCCL_SUM, s->comm, st));
    return MOE_OK;
  }
  const size_t need = count * 4 * s->R;
  if (s->scratch_bytes < need) {
    if (s->scratch) cudaFree(s->scratch);
    if (cudaMalloc(&s->scratch, need) != cudaSuccess) { *err = "scratch alloc"; return MOE_ERR_CUDA; }
    s->scratch_bytes = need;
  }
  moe_status_t q = tr_group_start(s, err);
  for (int r = 0; r < s->R && q == MOE_OK; ++r) q = tr_send(s, buf, count, NCCL_FLOAT32, 4, r, st, err);
  for (int r = 0; r < s->R && q == MOE_OK; ++r) q = tr_recv(s, s->scratch + (size_t)r * count, count, NCCL_FLOAT32, 4, r, st, err);
  if (q == MOE_OK) q = tr_group_end(s, st, err);
  if (q != MOE_OK) return q;
  vsum_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(s->scratch, s->R, count, buf);
  return cudaGetLastError() == cudaSuccess ? MOE_OK : MOE_ERR_CUDA;
}

moe_status_t vcomm_create(int R, void** out) {
  if (R < 1 || !out) return MOE_ERR_INVALID_ARG;
  VComm* vc = new VComm();
  vc->R = R;
  vc->ops.resize(R);
  vc->ready.resize(R);
  vc->done.resize(R);
  for (int r = 0; r < R; ++r)
    if (cudaEventCreateWithFlags(&vc->ready[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&vc->done[r], cudaEventDisableTiming) != cudaSuccess)
      return MOE_ERR_CUDA;
  std::lock_guard<std::mutex> lk(g_vc_mu);
  g_vcomms.insert(vc);
  *out = vc;
  return MOE_OK;
}

moe_status_t vcomm_destroy(void* p) {
  std::lock_guard<std::mutex> lk(g_vc_mu);
  if (!g_vcomms.count(p)) return MOE_ERR_INVALID_ARG;
  g_vcomms.erase(p);
  VComm* vc = (VComm*)p;
  for (auto e : vc->ready) cudaEventDestroy(e);
  for (auto e : vc->done) cudaEventDestroy(e);
  delete vc;
  return MOE_OK;
}

}  // namespace moe
