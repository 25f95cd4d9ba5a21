// moe_api.cu -- the C-ABI runtime (moe_ctx): configuration, capacity table and workspace
// layout, stream-ordered forward/backward orchestration, cached-assignment fork/join,
// statistics, and the dynamic-capacity policy helper.  See include/moe.h for the contract.
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <string>
#include <vector>

#include "../../include/moe.h"
#include "common.cuh"
#include "kernels.h"
#include "gemm_tc.h"
#include "gate_tc.h"
#include "prof.h"
#include "ep.h"
#include "peer.h"
#include "nccl_lsa.h"
#include <map>

using namespace moe;

static bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && v[0] == '1';
}

int moe::pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MOE_PDL");
    v = e ? (atoi(e) != 0) : 1;
  }
  return v;
}

struct Layout {
  size_t logits, idx, fresh_idx, slot_of, w, dw, dl, tile_hist, tile_off, meta, token_of_slot,
      xbuf, hbuf, obuf, dobuf, dxbuf, partial, dlb, mask, bpart, bal, grow, ep_all, sendbuf, oret, dwg32,
      pre_dev, dlr, dropb, droptok, sstat, ycnt, dabuf, total;
};

struct moe_ctx {
  moe_config_t cfg{};
  int n = 0, k = 0, d = 0, f = 0, dout = 0, maxT = 0, dtype = 0, renorm = 1, R = 1, rank = 0;
  int n_local = 0, e_lo = 0, n_pad = 64;
  size_t s = 4;  // bytes per element
  cudaStream_t stream = nullptr, side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_gate = nullptr;
  std::vector<int32_t> cap;   // global capacities C_e (all n)
  CapTable ct{};              // GEMM side: cap (all n) + base of LOCAL expert regions
  CapTable cts{};             // token side (dispatch/combine/gate_dx): base/pre per global e
  int64_t rows = 0;           // total local buffer rows
  int max_cap_local = 0;
  Layout L{};
  uint8_t* ws = nullptr;
  size_t ws_bytes = 0;
  RouteBufs rb{};
  const int32_t* cached = nullptr;
  // per-sample assignment cache (N4): caller-owned table [ctab_num x k], sample ids [T]
  int32_t* ctab = nullptr;
  int64_t ctab_num = 0;
  const int64_t* cids = nullptr;
  int ctab_mode = 0;
  int last_cached = 0;        // the last forward dispatched from cached indices
  // saved forward state for backward
  int have_fwd = 0, T_last = 0;
  moe_fwd_args_t fa{};
  int64_t launches = 0;
  int use_tc = 0;             // tcgen05 path for bf16 (env MOE_FORCE_SIMT=1 disables)
  int use_tf32 = 0;           // fp32: expert GEMMs on tcgen05 kind::tf32 (split operands), else SIMT
  int fusion = MOE_FUSE_COMBINE | MOE_FUSE_DX | MOE_FUSE_OTOK;  // N2 (moe_set_fusion; GATHER, COMBINE2, CDISP opt-in)
  int fused_gather = 0;       // the last forward gathered x rows in the GEMMs (no X buffer)
  int peer_ret = 0;           // peer EP: O / dX rows returned by the GEMM epilogues (N1)
  int otok = 0;               // the last forward stored O in (token, choice) order (MOE_FUSE_OTOK)
  TcPlan tc{};
  Prof prof;
  float balance_lambda = 0.f; // Eq. 3 balance term weight (0 = off)
  void* spec = nullptr;       // AggregateSpec outputs of the next forward (N3)
  uint8_t* spec_valid = nullptr;
  const void* dspec = nullptr;   // extra gradients for the next backward (N3)
  const float* dw_ext = nullptr;
  // model-metric future queue (App. B)
  struct MetricSlot {
    moe_metrics_t* host = nullptr;  // pinned
    cudaEvent_t ev = nullptr;
  };
  std::vector<MetricSlot> mq;
  int mq_head = 0, mq_count = 0;
  int64_t mq_iter = 0;
  int use_ep = 0;             // expert-parallel path (nccl_comm given; R may be 1 = loopback)
  EpState* ep = nullptr;
  EpPlan plan;
  // peer-memory transport (N1)
  int use_peer = 0, peer_attached = 0;
  PeerLayout PL{};
  char* pwin = nullptr;              // own window (cudaMalloc, or NCCL symmetric memory)
  LsaWindow lsa{};                   // set when the window is an NCCL symmetric window
  PeerBufs wins{};                   // all ranks' windows in this process
  bool opened[MOE_MAX_R] = {};       // windows opened from IPC handles (closed at destroy)
  std::string err;
};

namespace {

moe_status_t fail(moe_ctx* h, moe_status_t st, const std::string& msg) {
  if (h) h->err = msg;
  return st;
}

#define CUDA_TRY(h, expr)                                                              \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      return fail(h, MOE_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// count (and optionally time) our kernel launches: nk kernels per launcher call
#define KL(h, nk, name, st, expr)                  \
  do {                                             \
    ProfScope _ps(&(h)->prof, name, st);           \
    CUDA_TRY(h, expr);                             \
    (h)->launches += (nk);                         \
  } while (0)

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

void compute_layout(moe_ctx* h) {
  const size_t T = h->maxT, n = h->n, k = h->k;
  const size_t ntiles = (T + MOE_ROUTE_TILE - 1) / MOE_ROUTE_TILE + 1;
  Layout& L = h->L;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += al(bytes); return r; };
  L.logits = take(T * n * 4);
  L.idx = take(T * k * 4);
  L.fresh_idx = take(T * k * 4);
  L.slot_of = take(T * k * 4);
  L.w = take(T * k * 4);
  L.dw = take(T * k * 4);
  L.dl = take(T * n * 4);
  L.tile_hist = take(ntiles * n * 4);
  L.tile_off = take(ntiles * n * 4);
  L.meta = take(4096);
  // peer transport: X/O/dO/dX and token_of_slot live in the peer window instead
  const size_t prow = h->use_peer ? 0 : (size_t)h->rows;
  L.token_of_slot = take(h->use_peer ? 0 : std::max<size_t>((size_t)h->rows, T * k) * 4);
  L.xbuf = take(prow * h->d * h->s);
  L.hbuf = take((size_t)h->rows * h->f * h->s);
  // single GPU, tcgen05: O may be stored in (token, choice) order instead (MOE_FUSE_OTOK)
  const size_t orow = (!h->use_ep && h->use_tc) ? std::max(prow, T * k) : prow;
  L.obuf = take(orow * h->dout * h->s);
  L.dobuf = take(prow * h->dout * h->s);
  L.dxbuf = take(prow * h->d * h->s);
  const size_t splits = std::max(gate_dw_splits(h->maxT, h->d), gate_dw_tc_splits(h->maxT, h->n, h->d));
  L.partial = take(splits * n * h->d * 4 + 4096);
  L.dlb = take(h->dtype == MOE_BF16 ? 2 * T * (size_t)h->n_pad * 2 : 0);
  L.mask = take(h->dtype == MOE_BF16 ? (size_t)h->rows * (h->f / 32) * 4 : 0);
  // db1 partials: sum_e ceil(kept_e/256) <= rows/256 + n_local tiles x 8 rows x f
  // balance term: partial column sums [ceil(T/64) x n], gsum [n], g [n], aux [1]
  L.bal = take(((T + 63) / 64 + 3) * n * 4 + 256);
  L.grow = take(T * k * 4);
  L.bpart = take(h->dtype == MOE_BF16 ? ((size_t)h->rows / 256 + h->n_local) * 2 * h->f * 4 : 0);
  // fused dispatch backward (k = 1, one GPU): [hi | lo](dl) by expert row
  L.dropb = take(h->dtype == MOE_BF16 && k == 1 && (!h->use_ep || h->use_peer)
                     ? 2 * T * (size_t)h->n_pad * 2 : 0);
  L.droptok = take(k == 1 ? T * 4 : 0);
  L.dlr = take(h->dtype == MOE_BF16 && k == 1 && !h->use_ep ? (size_t)h->rows * 2 * h->n_pad * 2 : 0);
  const bool ep = h->use_ep && !h->use_peer;  // NCCL transport buffers
  L.pre_dev = take(n * 4);
  L.ep_all = take(ep ? (size_t)h->R * n * 4 : 0);
  L.sendbuf = take(ep ? T * k * (size_t)std::max(h->d, h->dout) * h->s : 0);
  L.oret = take(ep ? T * k * (size_t)h->dout * h->s : 0);
  L.dwg32 = take(ep ? n * (size_t)h->d * 4 : 0);
  L.sstat = take(h->use_tc ? T * 16 : 0);
  // k = 2 combine in FWD2: one counter per (token, column block of <= 64 columns)
  L.ycnt = take(h->use_tc && k == 2 && !h->use_ep ? T * (size_t)(h->dout / 64) * 4 : 0);
  // single GPU: dA in its own buffer (H stays intact; lets DGRAD_A overlap the dW2 GEMM)
  L.dabuf = take((h->use_tc || h->use_tf32) && !h->use_ep ? (size_t)h->rows * h->f * h->s : 0);
  L.total = o;
}

void bind_buffers(moe_ctx* h) {
  uint8_t* b = h->ws;
  const Layout& L = h->L;
  RouteBufs& r = h->rb;
  r.logits = (float*)(b + L.logits);
  r.idx = (int32_t*)(b + L.idx);
  r.fresh_idx = (int32_t*)(b + L.fresh_idx);
  r.slot_of = (int32_t*)(b + L.slot_of);
  r.w = (float*)(b + L.w);
  r.dw = (float*)(b + L.dw);
  r.dl = (float*)(b + L.dl);
  r.tile_hist = (int32_t*)(b + L.tile_hist);
  r.tile_off = (int32_t*)(b + L.tile_off);
  int32_t* meta = (int32_t*)(b + L.meta);
  r.counts = meta;                           // [256]
  r.kept = meta + 256;                       // [256]
  r.mtile_prefix = meta + 512;               // [257]
  r.drops = (int64_t*)(meta + 776);          // 8-byte aligned
  r.hit_count = meta + 780;
  r.flags = meta + 781;
  r.ticket = (uint32_t*)(meta + 782);
  r.token_of_slot = h->use_peer ? (int32_t*)(h->pwin + h->PL.tos) : (int32_t*)(b + L.token_of_slot);
  r.grow = (int32_t*)(b + L.grow);
  r.dropb = nullptr;  // set per backward (fused dX only)
  r.dlr = nullptr;
  r.pdlr = PeerBufs{};
  r.o_pair = 0;
  r.dx_pair = 0;
  r.gate_hist = 0;
  r.drop_tok = (int32_t*)(b + L.droptok);
  r.sstat = nullptr;  // set per forward (tcgen05 gate, when the backward needs p)
  r.drop_cnt = meta + 783;
}

void relayout(moe_ctx* h) {
  int64_t base = 0;
  h->max_cap_local = 0;
  for (int e = 0; e < MOE_MAX_E; ++e) h->ct.cap[e] = 0;
  for (int e = 0; e < h->n; ++e) h->ct.cap[e] = h->cap[e];
  for (int j = 0; j < h->n_local; ++j) {
    h->ct.base[j] = (int32_t)base;
    int c = h->cap[h->e_lo + j];
    h->max_cap_local = std::max(h->max_cap_local, c);
    base += ((int64_t)c + MOE_ROW_ALIGN - 1) / MOE_ROW_ALIGN * MOE_ROW_ALIGN;
  }
  h->ct.base[h->n_local] = (int32_t)base;
  h->rows = base;
  h->cts = h->ct;  // single GPU: token side indexes the same regions, pre = 0
  for (int e = 0; e < MOE_MAX_E; ++e) h->cts.pre[e] = 0;
  if (h->use_peer) {  // token side: every global expert's region base inside its owner's window
    for (int o = 0; o < h->R; ++o) {
      int64_t b = 0;
      for (int j = 0; j < h->n_local; ++j) {
        const int e = o * h->n_local + j;
        h->cts.base[e] = (int32_t)b;
        b += ((int64_t)h->cap[e] + MOE_ROW_ALIGN - 1) / MOE_ROW_ALIGN * MOE_ROW_ALIGN;
      }
    }
  }
  compute_layout(h);
}

// The expert-major buffers: in the peer window (N1) or in the workspace.
void* buf_x(moe_ctx* h) { return h->use_peer ? (void*)(h->pwin + h->PL.x) : (void*)(h->ws + h->L.xbuf); }
void* buf_o(moe_ctx* h) { return h->use_peer ? (void*)(h->pwin + h->PL.o) : (void*)(h->ws + h->L.obuf); }
void* buf_do(moe_ctx* h) { return h->use_peer ? (void*)(h->pwin + h->PL.dob) : (void*)(h->ws + h->L.dobuf); }
void* buf_dx(moe_ctx* h) { return h->use_peer ? (void*)(h->pwin + h->PL.dxb) : (void*)(h->ws + h->L.dxbuf); }
// per-owner pointers of one window buffer
PeerBufs peer_bufs(const moe_ctx* h, size_t off) {
  PeerBufs p{};
  for (int j = 0; j < h->R; ++j) p.p[j] = h->wins.p[j] + off;
  p.nl = h->n_local;
  return p;
}
// Sum over the local experts of roundup(C_e, 128) for every owner (the rows a window needs).
int64_t max_owner_rows(const moe_ctx* h, const std::vector<int32_t>& cap) {
  int64_t m = 0;
  for (int o = 0; o < h->R; ++o) {
    int64_t b = 0;
    for (int j = 0; j < h->n_local; ++j)
      b += ((int64_t)cap[o * h->n_local + j] + MOE_ROW_ALIGN - 1) / MOE_ROW_ALIGN * MOE_ROW_ALIGN;
    m = std::max(m, b);
  }
  return m;
}

int64_t tokens_global(const moe_ctx* h) { return (int64_t)h->maxT * h->R; }

}  // namespace

extern "C" {

// why the last moe_init on this thread failed (moe_last_error(NULL))
static thread_local std::string g_init_err;

const char* moe_last_error(moe_handle_t h) {
  if (h) return h->err.c_str();
  return g_init_err.empty() ? "null handle" : g_init_err.c_str();
}

moe_status_t moe_capacity_from_factors(int32_t n, int64_t tokens_global, int32_t k,
                                       const double* alpha, int32_t* cap_out) {
  if (n <= 0 || k <= 0 || tokens_global < 0 || !alpha || !cap_out) return MOE_ERR_INVALID_ARG;
  for (int e = 0; e < n; ++e) {
    if (!(alpha[e] >= 0.0) || !std::isfinite(alpha[e])) return MOE_ERR_INVALID_ARG;
    double c = std::ceil(alpha[e] * (double)tokens_global * (double)k / (double)n);  // Eq. 4
    if (c > 2147483647.0) return MOE_ERR_INVALID_ARG;
    cap_out[e] = std::max(1, (int)c);
  }
  return MOE_OK;
}

moe_status_t moe_init(const moe_config_t* cfg, moe_handle_t* out) {
  if (!cfg || !out) return MOE_ERR_INVALID_ARG;
  *out = nullptr;
  const moe_config_t& c = *cfg;
  int dout = c.d_out ? c.d_out : c.d_model;
  if (c.n_experts < 1 || c.n_experts > MOE_MAX_E) return MOE_ERR_CONFIG;
  if (c.top_k < 1 || c.top_k > c.n_experts || c.top_k > MOE_MAX_K) return MOE_ERR_CONFIG;
  if (c.dtype != MOE_F32 && c.dtype != MOE_BF16) return MOE_ERR_CONFIG;
  const int mult = c.dtype == MOE_BF16 ? 64 : 4;
  if (c.d_model <= 0 || c.d_ff <= 0 || dout <= 0 || c.d_model % mult || c.d_ff % mult ||
      dout % mult)
    return MOE_ERR_CONFIG;
  if (c.max_tokens < 0) return MOE_ERR_INVALID_ARG;
  if (c.world_size < 1 || c.rank < 0 || c.rank >= c.world_size) return MOE_ERR_INVALID_ARG;
  if (c.n_experts % c.world_size) return MOE_ERR_CONFIG;
  if (c.transport != MOE_TRANSPORT_NCCL && c.transport != MOE_TRANSPORT_PEER) return MOE_ERR_CONFIG;
  if (c.reserved0 != 0 || c.window_rows < 0) return MOE_ERR_INVALID_ARG;
  if (c.transport == MOE_TRANSPORT_NCCL && c.world_size > 1 && !c.nccl_comm) return MOE_ERR_INVALID_ARG;
  if (c.transport == MOE_TRANSPORT_PEER && c.world_size > MOE_MAX_R) return MOE_ERR_CONFIG;
  if (c.n_experts / c.world_size > MOE_MAX_E) return MOE_ERR_CONFIG;
  moe_ctx* h = new moe_ctx();
  h->cfg = c;
  h->n = c.n_experts; h->k = c.top_k; h->d = c.d_model; h->f = c.d_ff; h->dout = dout;
  h->maxT = c.max_tokens; h->dtype = c.dtype; h->renorm = c.renormalize ? 1 : 0;
  h->R = c.world_size; h->rank = c.rank;
  h->n_local = h->n / h->R; h->e_lo = h->rank * h->n_local;
  h->n_pad = (h->n + 63) / 64 * 64;
  h->s = c.dtype == MOE_BF16 ? 2 : 4;
  h->stream = (cudaStream_t)c.stream;
  const char* fs = getenv("MOE_FORCE_SIMT");
  h->use_tc = (c.dtype == MOE_BF16) && !(fs && fs[0] == '1');
  h->use_tf32 = (c.dtype == MOE_F32) && !(fs && fs[0] == '1') && tf32_supported(h->d, h->f, dout);

  g_init_err.clear();
  if (cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_gate, cudaEventDisableTiming) != cudaSuccess) {
    g_init_err = std::string("moe_init: stream / event creation: ") +
                 cudaGetErrorString(cudaGetLastError());
    delete h;
    return MOE_ERR_CUDA;
  }
  h->use_peer = c.transport == MOE_TRANSPORT_PEER ? 1 : 0;
  {
    const char* pr = getenv("MOE_PEER_RET");  // 0: combine / gate-dx read the owners' rows
    h->peer_ret = h->use_peer && h->use_tc && tc_peer_return_supported(h->d, h->dout) &&
                  !(pr && pr[0] == '0');
  }
  h->use_ep = (c.nccl_comm || h->use_peer) ? 1 : 0;
  if (h->use_peer) {  // the peer window, sized for the largest capacities allowed later
    int64_t wrows = c.window_rows;
    if (wrows == 0) {
      std::vector<int32_t> c8(h->n);
      std::vector<double> a8(h->n, 8.0);
      moe_capacity_from_factors(h->n, tokens_global(h), h->k, a8.data(), c8.data());
      for (auto& v : c8) v = (int32_t)std::min<int64_t>(v, std::max<int64_t>(1, tokens_global(h)));
      wrows = max_owner_rows(h, c8);
    }
    wrows = (wrows + MOE_ROW_ALIGN - 1) / MOE_ROW_ALIGN * MOE_ROW_ALIGN;
    peer_layout(h->PL, wrows, h->n, h->d, h->dout, h->s, (int64_t)h->maxT * h->k);
    // zeroed and COMPLETE before any rank can see the window: the epoch / flag words start at
    // 0, and a memset still in flight (legacy stream) could race with a peer's first count
    // push or with kernels on non-blocking streams
    cudaError_t ce = cudaMalloc((void**)&h->pwin, h->PL.total);
    if (ce == cudaSuccess) ce = cudaMemset(h->pwin, 0, h->PL.total);
    if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
    if (ce != cudaSuccess) {
      g_init_err = "moe_init: peer window of " + std::to_string(h->PL.total >> 20) +
                   " MiB (window_rows " + std::to_string(wrows) + "): " + cudaGetErrorString(ce);
      if (h->pwin) cudaFree(h->pwin);
      cudaEventDestroy(h->ev_fork);
      cudaEventDestroy(h->ev_join);
      cudaEventDestroy(h->ev_gate);
      cudaStreamDestroy(h->side);
      delete h;
      return MOE_ERR_CUDA;
    }
  }
  // default capacities: Eq. 4 with alpha = 1 over the global token count
  h->cap.assign(h->n, 1);
  std::vector<double> a(h->n, 1.0);
  moe_capacity_from_factors(h->n, tokens_global(h), h->k, a.data(), h->cap.data());
  for (auto& v : h->cap) v = (int32_t)std::min<int64_t>(v, std::max<int64_t>(1, tokens_global(h)));
  if (h->use_peer && max_owner_rows(h, h->cap) > h->PL.rows) {
    cudaFree(h->pwin);
    delete h;
    return MOE_ERR_CONFIG;
  }
  relayout(h);
  if (c.nccl_comm && !h->use_peer) {
    h->use_ep = 1;
    moe_status_t st = ep_create(&h->ep, c.nccl_comm, h->R, h->rank, &h->err);
    if (st != MOE_OK) {
      delete h;
      return st;
    }
  }
  *out = h;
  return MOE_OK;
}

moe_status_t moe_destroy(moe_handle_t h) {
  if (!h) return MOE_ERR_INVALID_ARG;
  if (h->side) cudaStreamSynchronize(h->side);
  if (h->ep) ep_destroy(h->ep);
  for (int j = 0; j < MOE_MAX_R; ++j)
    if (h->opened[j]) cudaIpcCloseMemHandle(h->wins.p[j]);
  if (h->lsa.buf) {
    lsa_window_destroy(&h->lsa);  // (synchronises the device first)
  } else if (h->pwin) {
    cudaDeviceSynchronize();
    cudaFree(h->pwin);
  }
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->ev_gate) cudaEventDestroy(h->ev_gate);
  if (h->side) cudaStreamDestroy(h->side);
  tc_plan_free(&h->tc);
  h->prof.destroy();
  for (auto& sl : h->mq) {
    if (sl.host) cudaFreeHost(sl.host);
    if (sl.ev) cudaEventDestroy(sl.ev);
  }
  delete h;
  return MOE_OK;
}

moe_status_t moe_set_stream(moe_handle_t h, void* stream) {
  if (!h) return MOE_ERR_INVALID_ARG;
  h->stream = (cudaStream_t)stream;
  return MOE_OK;
}

moe_status_t moe_set_capacities(moe_handle_t h, const int32_t* cap) {
  if (!h || !cap) return MOE_ERR_INVALID_ARG;
  for (int e = 0; e < h->n; ++e)
    if (cap[e] < 1) return fail(h, MOE_ERR_INVALID_ARG, "capacity < 1");
  const int64_t tg = std::max<int64_t>(1, tokens_global(h));
  std::vector<int32_t> nc(h->n);
  for (int e = 0; e < h->n; ++e) nc[e] = (int32_t)std::min<int64_t>(cap[e], tg);
  if (h->use_peer && max_owner_rows(h, nc) > h->PL.rows)
    return fail(h, MOE_ERR_CONFIG, "peer window too small for these capacities "
                                   "(raise cfg.window_rows); capacities unchanged");
  h->cap = nc;
  relayout(h);
  h->have_fwd = 0;  // saved activations no longer match the layout
  if (h->ws && h->ws_bytes < h->L.total) {
    h->ws = nullptr;
    h->ws_bytes = 0;
    return fail(h, MOE_ERR_WORKSPACE_TOO_SMALL, "workspace too small for new capacities");
  }
  if (h->ws) bind_buffers(h);
  return MOE_OK;
}

moe_status_t moe_get_capacities(moe_handle_t h, int32_t* cap_out) {
  if (!h || !cap_out) return MOE_ERR_INVALID_ARG;
  std::memcpy(cap_out, h->cap.data(), sizeof(int32_t) * h->n);
  return MOE_OK;
}

moe_status_t moe_workspace_size(moe_handle_t h, size_t* bytes) {
  if (!h || !bytes) return MOE_ERR_INVALID_ARG;
  *bytes = h->L.total;
  return MOE_OK;
}

moe_status_t moe_set_workspace(moe_handle_t h, void* dptr, size_t bytes) {
  if (!h || !dptr) return MOE_ERR_INVALID_ARG;
  if ((uintptr_t)dptr % 256) return fail(h, MOE_ERR_INVALID_ARG, "workspace must be 256-B aligned");
  if (bytes < h->L.total) return fail(h, MOE_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
  bool was_set = h->ws != nullptr;
  h->ws = (uint8_t*)dptr;
  h->ws_bytes = bytes;
  bind_buffers(h);
  (void)was_set;
  CUDA_TRY(h, cudaMemsetAsync(h->ws + h->L.meta, 0, 4096, h->stream));
  // the k = 2 combine counters reset themselves after each use: zero once per workspace
  if (h->use_tc && h->k == 2 && !h->use_ep && h->maxT > 0)
    CUDA_TRY(h, cudaMemsetAsync(h->ws + h->L.ycnt, 0, (size_t)h->maxT * (h->dout / 64) * 4,
                                h->stream));
  h->have_fwd = 0;
  return MOE_OK;
}

moe_status_t moe_set_cached_assignment(moe_handle_t h, const int32_t* d_idx) {
  if (!h) return MOE_ERR_INVALID_ARG;
  if (d_idx && h->ctab_mode)
    return fail(h, MOE_ERR_STATE, "an assignment cache table is active (mode != 0)");
  h->cached = d_idx;
  return MOE_OK;
}

moe_status_t moe_set_assignment_cache(moe_handle_t h, int32_t* d_table, int64_t num_samples,
                                      const int64_t* d_sample_ids, int32_t mode) {
  if (!h) return MOE_ERR_INVALID_ARG;
  if (mode < 0 || mode > 3) return fail(h, MOE_ERR_INVALID_ARG, "mode must be 0..3");
  if (mode && (!d_table || num_samples <= 0 || !d_sample_ids))
    return fail(h, MOE_ERR_INVALID_ARG, "null table / sample ids");
  if (mode && h->cached)
    return fail(h, MOE_ERR_STATE, "raw cached indices are set (moe_set_cached_assignment)");
  h->ctab = mode ? d_table : nullptr;
  h->ctab_num = mode ? num_samples : 0;
  h->cids = mode ? d_sample_ids : nullptr;
  h->ctab_mode = mode;
  return MOE_OK;
}

moe_status_t moe_forward(moe_handle_t h, const moe_fwd_args_t* a) {
  if (!h || !a) return MOE_ERR_INVALID_ARG;
  if (!h->ws) return fail(h, MOE_ERR_STATE, "workspace not set");
  if (a->T < 0 || a->T > h->maxT) return fail(h, MOE_ERR_INVALID_ARG, "T out of range");
  if (a->T > 0 && (!a->x || !a->w_gate || !a->w1 || !a->b1 || !a->w2 || !a->b2 || !a->y))
    return fail(h, MOE_ERR_INVALID_ARG, "null tensor");
  if (!h->mq.empty() && h->mq_count == (int)h->mq.size())
    return fail(h, MOE_ERR_STATE, "metrics queue full: pop before launching more iterations");
  if (h->use_peer && !h->peer_attached)
    return fail(h, MOE_ERR_STATE, "peer transport: call moe_peer_attach / moe_peer_import first");
  const int T = a->T, n = h->n, k = h->k, d = h->d, f = h->f, dout = h->dout, dt = h->dtype;
  cudaStream_t s0 = h->stream;
  RouteBufs& rb = h->rb;
  uint8_t* ws = h->ws;
  void* X = buf_x(h);
  void* H = ws + h->L.hbuf;
  void* O = buf_o(h);
  const int ntiles = (T + MOE_ROUTE_TILE - 1) / MOE_ROUTE_TILE;
  // dispatch-index sources: raw cached indices, or the per-sample table (mode 1: every
  // sample known -> the same side-stream overlap; mode 2: unknown samples fall back to the
  // gate, so routing waits for it), else the gate's top-k
  const bool observe = h->ctab_mode == 3;   // metric + remember only, fresh routing
  const bool tab = h->ctab_mode != 0 && !observe;
  const bool fallback = h->ctab_mode == 2;
  const bool cached = h->cached != nullptr || (tab && !fallback);
  const int32_t* cidx = tab ? rb.idx : h->cached;   // what the gate compares/weights against
  h->last_cached = cached || fallback;
  // N2 (single GPU, tcgen05 path).  GATHER: the expert GEMMs gather x rows by
  // token_of_slot (no X buffer; the dispatch writes only the routing tables).  COMBINE: with
  // k = 1, FWD2's epilogue also writes y (no combine pass re-reading O); in cached mode FWD2
  // then waits for the gate (which ran concurrently with the routing, dispatch and FWD1).
  const bool tc1 = h->use_tc && !h->use_ep && T > 0;
  const bool gather = tc1 && (h->fusion & MOE_FUSE_GATHER) && ((uintptr_t)a->x % 16) == 0 &&
                      tc_gather_supported(d, f);
  const bool fcomb = tc1 && (h->fusion & MOE_FUSE_COMBINE) && k == 1 &&
                     h->spec == nullptr && ((uintptr_t)a->y % 16) == 0 &&
                     tc_combine_supported(dout);
  // O rows in (token, choice) order: FWD2's epilogue stores row t k + r (the peer EP return-row
  // store with this rank as the only owner), so the combine and its backward read O by token
  // with no routing-table lookup in front of the row loads
  const bool otok = tc1 && (h->fusion & MOE_FUSE_OTOK) && tc_combine_supported(dout);
  // k = 2: the combine in FWD2's epilogue (second epilogue of a token writes y), on top of the
  // token-ordered O
  const bool fcomb2 = otok && (h->fusion & MOE_FUSE_COMBINE2) && k == 2 && h->spec == nullptr &&
                      ((uintptr_t)a->y % 16) == 0;
  // Cached mode, one GPU, tcgen05 gate: the dispatch (A4) rides inside the gate kernel (x read
  // once for the gate GEMM and the row copies), so the chain stays on s0 with no fork / join
  const bool cdisp = cached && tc1 && !gather && (h->fusion & MOE_FUSE_CDISP) && d % 64 == 0;
  h->fused_gather = gather;
  h->otok = otok;
  TcFusion fz;
  fz.T = T;
  fz.tos = rb.token_of_slot;
  fz.k = k;
  if (gather) fz.x = a->x;
  if (fcomb) {
    fz.y = a->y;
    fz.w = rb.w;
  }
  if (h->peer_ret) {  // N1: FWD2's epilogue stores O rows into the token owners' windows
    fz.pret_o = peer_bufs(h, h->PL.oret);
    fz.tpr = T;
  } else if (otok) {
    fz.pret_o.p[0] = (char*)O;
    fz.pret_o.nl = 1;
    fz.tpr = T;
  }
  if (fcomb2) {
    fz.y = a->y;
    fz.w = rb.w;
    fz.comb2 = 1;
    fz.slot = rb.slot_of;
    fz.ycnt = (uint32_t*)(ws + h->L.ycnt);
  }
  CUDA_TRY(h, cudaMemsetAsync(rb.hit_count, 0, 4, s0));
  // softmax statistics from the tcgen05 gate for the combine backward (raw weights or the
  // Eq. 3 balance term need the full p); kept with the forward's state
  rb.sstat = (h->use_tc && (!h->renorm || h->balance_lambda != 0.f))
                 ? (float*)(ws + h->L.sstat) : nullptr;
  if (tab)  // idx[t] = table[sample_ids[t]] (before the fork: the side stream reads it)
    KL(h, T > 0, "cache_gather", s0, launch_cache_gather(h->ctab, h->ctab_num, k, h->cids, T,
                                                         rb.idx, rb.flags, s0));

  // Everything from the routing tables up to the expert outputs depends only on the
  // dispatch indices.  Uncached: they are the gate's top-k, so it all follows the gate on
  // s0.  Cached (S4.2): they are known before the gate, so this chain runs on a
  // side stream concurrently with the gate; the join is before the combine, the first step
  // that needs the gate weights.
  cudaStream_t sd = s0;
  if (cdisp) {
    // (raw cached indices are copied into idx by the histogram kernel; the gate follows the
    // routing scan on s0 and performs the dispatch)
  } else if (cached) {
    CUDA_TRY(h, cudaEventRecord(h->ev_fork, s0));
    CUDA_TRY(h, cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    sd = h->side;
    // (raw cached indices are copied into idx by the histogram kernel itself, below)
  } else {
    // fallback mode: the gate rewrites the rows of unknown samples with their fresh top-k
    rb.idx_fix = fallback ? rb.idx : nullptr;
    const int32_t* gc = fallback ? rb.idx : nullptr;
    // A3 histogram inside the tcgen05 gate's epilogue when its top-k is the dispatch index
    rb.gate_hist = h->use_tc && !fallback && !getenv_flag("MOE_NO_GATE_HIST");
    if (h->use_tc)
      KL(h, T > 0, "gate_topk", s0, launch_gate_fwd_tc(a->x, a->w_gate, T, n, d, k, h->renorm, gc, rb, s0));
    else
      KL(h, T > 0, "gate_topk", s0, launch_gate_topk(dt, a->x, a->w_gate, T, n, d, k, h->renorm, gc, rb, s0));
    rb.idx_fix = nullptr;
    if (tab)  // cache_step: remember this batch's fresh decisions
      KL(h, T > 0, "cache_update", s0, launch_cache_update(h->ctab, h->ctab_num, k, h->cids, T,
                                                           fallback ? rb.fresh_idx : rb.idx, s0));
    if (observe)  // hit metric against the remembered rows, then remember
      KL(h, T > 0, "cache_update", s0, launch_cache_observe(h->ctab, h->ctab_num, k, h->cids, T,
                                                            rb.idx, rb.hit_count, rb.flags, s0));
  }
  if (!rb.gate_hist)
    KL(h, T > 0, "route_hist", sd, launch_route_hist(rb.idx, T, k, n, rb.tile_hist, sd,
                                                     (cached && !tab) ? h->cached : nullptr));
  rb.gate_hist = 0;
  KL(h, 1, "route_scan", sd, launch_route_scan(rb.tile_hist, ntiles, n, h->ct, rb, sd));
  if (cdisp) {
    GateDispatch gd{&h->cts, X, (fcomb || fcomb2) ? a->y : nullptr, dout};
    KL(h, T > 0, "gate_topk", s0, launch_gate_fwd_tc(a->x, a->w_gate, T, n, d, k, h->renorm, cidx,
                                                     rb, s0, &gd));
    if (tab)  // cache_step
      KL(h, T > 0, "cache_update", s0, launch_cache_update(h->ctab, h->ctab_num, k, h->cids, T,
                                                           rb.fresh_idx, s0));
  } else if (!h->use_ep) {
    KL(h, T > 0, "dispatch", sd, launch_dispatch(dt, rb.idx, a->x, T, k, n, d, 0, h->cts, rb,
                                                 gather ? nullptr : X, gather ? nullptr : rb.kept,
                                                 sd, 0, PeerBufs{}, PeerBufs{}, nullptr,
                                                 (fcomb || fcomb2) ? a->y : nullptr, dout));
  } else if (h->use_peer) {
    // N1: counts exchange + global plan on the device, then the dispatch stores every kept
    // row straight into its owner's X buffer; the barrier publishes "X rows landed".
    int32_t* pre_dev = (int32_t*)(ws + h->L.pre_dev);
    KL(h, 1, "peer_plan", sd, launch_peer_plan(h->wins, h->R, h->rank, n, h->n_local, rb.counts,
                                               h->ct, rb, pre_dev, sd));
    KL(h, 1, "dispatch", sd, launch_dispatch(dt, rb.idx, a->x, T, k, n, d, (int64_t)h->rank * T,
                                             h->cts, rb, X, rb.kept, sd, h->e_lo,
                                             peer_bufs(h, h->PL.x), peer_bufs(h, h->PL.tos),
                                             pre_dev));
    KL(h, 1, "peer_barrier", sd, launch_peer_barrier(h->wins, h->R, h->rank, PH_X, sd, (uint32_t*)rb.flags));
  } else {
    // C1 + the single host sync of EP v1: all-gather the per-rank pre-drop counts, then every
    // rank derives the same global slot offsets, kept counts and message sizes (reading 12).
    std::string err;
    moe_status_t st = ep_exchange_counts(h->ep, rb.counts, (int32_t*)(ws + h->L.ep_all), n,
                                         h->cap.data(), sd, h->plan, &err);
    if (st != MOE_OK) return fail(h, st, err);
    const EpPlan& P = h->plan;
    for (int e = 0; e < n; ++e) {
      h->cts.pre[e] = P.pre[(size_t)h->rank * n + e];
      h->cts.base[e] = P.send_off[e] - h->cts.pre[e];
    }
    // device copies of the global routing statistics and local GEMM tile tables
    int64_t drops = P.drops;
    CUDA_TRY(h, cudaMemcpyAsync(rb.counts, P.counts.data(), 4 * n, cudaMemcpyHostToDevice, sd));
    CUDA_TRY(h, cudaMemcpyAsync(rb.kept, P.kept_local.data(), 4 * h->n_local, cudaMemcpyHostToDevice, sd));
    CUDA_TRY(h, cudaMemcpyAsync(rb.mtile_prefix, P.mtile_prefix.data(), 4 * (h->n_local + 1),
                                cudaMemcpyHostToDevice, sd));
    CUDA_TRY(h, cudaMemcpyAsync(rb.drops, &drops, 8, cudaMemcpyHostToDevice, sd));
    void* sendbuf = ws + h->L.sendbuf;
    KL(h, T > 0, "dispatch", sd, launch_dispatch(dt, rb.idx, a->x, T, k, n, d, (int64_t)h->rank * T,
                                                 h->cts, rb, sendbuf, nullptr, sd));
    st = ep_to_experts(h->ep, P, sendbuf, X, h->ct, d, (int)h->s, sd, &err);   // C2
    if (st != MOE_OK) return fail(h, st, err);
    // pad rows of the received regions (single GPU: fused into the dispatch kernel)
    KL(h, 1, "zero_pad", sd, launch_zero_pad(dt, X, d, rb.kept, h->n_local, h->ct, sd));
  }
  // Cached (S4.2): the gate is enqueued now -- after the routing / dispatch chain on the side
  // stream, before the expert GEMMs -- so it runs concurrently with the routing and dispatch
  // (enqueued after FWD1 it could only start once the persistent GEMM frees the SMs).
  if (cached && !cdisp) {
    if (h->use_tc)
      KL(h, T > 0, "gate_topk", s0, launch_gate_fwd_tc(a->x, a->w_gate, T, n, d, k, h->renorm, cidx, rb, s0));
    else
      KL(h, T > 0, "gate_topk", s0, launch_gate_topk(dt, a->x, a->w_gate, T, n, d, k, h->renorm, cidx, rb, s0));
    if (tab)  // cache_step; the side stream only reads idx, never the table
      KL(h, T > 0, "cache_update", s0, launch_cache_update(h->ctab, h->ctab_num, k, h->cids, T,
                                                           rb.fresh_idx, s0));
    CUDA_TRY(h, cudaEventRecord(h->ev_gate, s0));
  }
  // expert FFN: H = relu(X W1^T + b1); O = H W2^T + b2 over kept_e rows per local expert
  const int nl = h->n_local;
  const char* w1 = (const char*)a->w1 + (size_t)h->e_lo * f * d * h->s;
  const char* b1 = (const char*)a->b1 + (size_t)h->e_lo * f * h->s;
  const char* w2 = (const char*)a->w2 + (size_t)h->e_lo * dout * f * h->s;
  const char* b2 = (const char*)a->b2 + (size_t)h->e_lo * dout * h->s;
  const int32_t* kept_local = rb.kept;
  if (h->use_tc) {
    int64_t nk = 0;
    // cached + fused combine: FWD2's epilogue reads the gate weights -> join with the gate
    struct Join { cudaStream_t sd; cudaEvent_t ev; } join{sd, h->ev_gate};
    auto wait_gate = [](void* c) -> cudaError_t {
      Join* j = static_cast<Join*>(c);
      return cudaStreamWaitEvent(j->sd, j->ev, 0);
    };
    moe_status_t st = tc_ffn_forward(&h->tc, X, w1, b1, w2, b2, H, O, h->rows, d, f, dout,
                                     kept_local, rb.mtile_prefix, nl, h->ct, h->max_cap_local,
                                     sd, &nk, &h->prof, (uint32_t*)(ws + h->L.mask),
                                     (gather || fcomb || h->peer_ret || otok) ? &fz : nullptr,
                                     (cached && !cdisp && (fcomb || fcomb2)) ? +wait_gate : nullptr,
                                     &join);
    h->launches += nk;
    if (st != MOE_OK) return fail(h, st, "tcgen05 forward failed");
  } else if (h->use_tf32) {
    int64_t nk = 0;
    moe_status_t st = tf32_ffn_forward(X, w1, b1, w2, b2, H, O, h->rows, d, f, dout, kept_local,
                                       rb.mtile_prefix, nl, h->ct, sd, &nk, &h->prof);
    h->launches += nk;
    if (st != MOE_OK) return fail(h, st, "tcgen05 tf32 forward failed");
  } else {
    KL(h, 1, "ffn_gemm1", sd, launch_gemm_simt_mgroup(dt, X, d, w1, 1, (int64_t)f * d, b1, H, f, f, d, kept_local,
                                     nl, h->ct, h->max_cap_local, EPI_BIAS_RELU, sd));
    KL(h, 1, "ffn_gemm2", sd, launch_gemm_simt_mgroup(dt, H, f, w2, 1, (int64_t)dout * f, b2, O, dout, dout, f,
                                     kept_local, nl, h->ct, h->max_cap_local, EPI_BIAS, sd));
  }
  void* O_tok = O;  // expert outputs as the token side indexes them
  PeerBufs po{};    // peer EP: combine reads O rows from the owners
  if (h->use_peer) {
    KL(h, 1, "peer_barrier", sd, launch_peer_barrier(h->wins, h->R, h->rank, PH_O, sd, (uint32_t*)rb.flags));
    if (h->peer_ret)
      O_tok = h->pwin + h->PL.oret;  // this rank's (token, choice) rows, stored by the owners
    else
      po = peer_bufs(h, h->PL.o);
  } else if (h->use_ep) {
    std::string err;
    O_tok = ws + h->L.oret;
    moe_status_t st = ep_from_experts(h->ep, h->plan, O, O_tok, h->ct, dout, (int)h->s, sd, &err);  // C3
    if (st != MOE_OK) return fail(h, st, err);
  }
  if (cached && !cdisp) {  // join: everything after needs both the gate and the expert outputs
    CUDA_TRY(h, cudaEventRecord(h->ev_join, sd));
    CUDA_TRY(h, cudaStreamWaitEvent(s0, h->ev_join, 0));
  }
  if (h->balance_lambda != 0.f) {  // Eq. 3 balance term (N3)
    float* bal = (float*)(ws + h->L.bal);
    float* gsum = bal + (size_t)((h->maxT + 63) / 64) * n;
    if (h->use_peer) {  // column sums through the windows, summed in rank order
      KL(h, T > 0 ? 2 : 1, "balance", s0, launch_balance_partial(rb.logits, T, n, bal,
                                                                 (float*)(h->pwin + h->PL.bal), s0));
      KL(h, 1, "peer_barrier", s0, launch_peer_barrier(h->wins, h->R, h->rank, PH_BAL, s0, (uint32_t*)rb.flags));
      KL(h, 1, "peer_sum", s0, launch_peer_sum(h->wins, h->PL.bal, h->R, (size_t)n, 2, gsum, 0, s0));
    } else {
      KL(h, T > 0 ? 2 : 1, "balance", s0, launch_balance_partial(rb.logits, T, n, bal, gsum, s0));
    }
    if (h->use_ep && !h->use_peer) {
      std::string err;
      moe_status_t st = ep_allreduce_f32(h->ep, gsum, (size_t)n, s0, &err);
      if (st != MOE_OK) return fail(h, st, err);
    }
    KL(h, 1, "balance", s0, launch_balance_final(gsum, rb.counts, n, k, (int64_t)T * h->R,
                                                 h->balance_lambda, gsum + n, gsum + 2 * n, s0));
  }
  rb.spec = h->spec;
  rb.spec_valid = h->spec_valid;
  rb.o_pair = h->peer_ret || otok;
  if (!fcomb && !fcomb2)
    KL(h, T > 0, "combine_fwd", s0, launch_combine_fwd(dt, O_tok, rb, T, k, dout, h->cts, a->y, s0, po));
  rb.spec = nullptr;
  rb.spec_valid = nullptr;
  rb.o_pair = 0;
  if (!h->mq.empty()) {  // push this iteration's metric futures (App. B)
    auto& sl = h->mq[(h->mq_head + h->mq_count) % h->mq.size()];
    sl.host->iteration = h->mq_iter;
    sl.host->T = T;
    CUDA_TRY(h, cudaMemcpyAsync(sl.host->counts, rb.counts, 4 * n, cudaMemcpyDeviceToHost, s0));
    CUDA_TRY(h, cudaMemcpyAsync(&sl.host->drops, rb.drops, 8, cudaMemcpyDeviceToHost, s0));
    CUDA_TRY(h, cudaMemcpyAsync(&sl.host->hit_count, rb.hit_count, 4, cudaMemcpyDeviceToHost, s0));
    if (h->balance_lambda != 0.f) {
      const float* aux = (const float*)(ws + h->L.bal) + (size_t)((h->maxT + 63) / 64) * n + 2 * n;
      CUDA_TRY(h, cudaMemcpyAsync(&sl.host->aux_loss, aux, 4, cudaMemcpyDeviceToHost, s0));
    } else {
      sl.host->aux_loss = 0.f;
    }
    CUDA_TRY(h, cudaEventRecord(sl.ev, s0));
    ++h->mq_count;
  }
  ++h->mq_iter;
  h->fa = *a;
  h->T_last = T;
  h->have_fwd = 1;
  return MOE_OK;
}

moe_status_t moe_backward(moe_handle_t h, const moe_bwd_args_t* a) {
  if (!h || !a) return MOE_ERR_INVALID_ARG;
  if (!h->have_fwd) return fail(h, MOE_ERR_STATE, "backward without a matching forward");
  const int T = h->T_last, n = h->n, k = h->k, d = h->d, f = h->f, dout = h->dout,
            dt = h->dtype;
  if (T > 0 && !a->dy) return fail(h, MOE_ERR_INVALID_ARG, "null dy");
  cudaStream_t s0 = h->stream;
  RouteBufs& rb = h->rb;
  uint8_t* ws = h->ws;
  void* X = buf_x(h);
  void* H = ws + h->L.hbuf;   // holds H; overwritten by dA below
  void* O = buf_o(h);
  void* dO = buf_do(h);
  void* dXb = buf_dx(h);
  const bool peer = h->use_peer != 0;
  const bool nccl_ep = h->use_ep && !peer;
  const moe_fwd_args_t& fa = h->fa;
  const int nl = h->n_local;
  const int acc = a->accumulate ? 1 : 0;
  const int32_t* kept_local = rb.kept;

  // K6 combine backward -> dO rows (local or, in EP, returned to the expert owners), dw, dl
  void* dlb = h->use_tc ? (void*)(ws + h->L.dlb) : nullptr;
  void* O_tok = nccl_ep ? (void*)(ws + h->L.oret)
                : (peer && h->peer_ret) ? (void*)(h->pwin + h->PL.oret) : O;
  void* dO_tok = nccl_ep ? (void*)(ws + h->L.sendbuf) : dO;
  std::string err;
  rb.dspec = h->dspec;
  rb.dw_ext = h->dw_ext;
  rb.bal_g = h->balance_lambda != 0.f
                 ? (const float*)(ws + h->L.bal) + (size_t)((h->maxT + 63) / 64) * n + n
                 : nullptr;
  // N2 dispatch backward fused into the dX GEMM (k = 1, one GPU, tcgen05): the combine
  // backward also writes [hi|lo](dl) by expert row, the GEMM adds dl W_g and writes dx rows
  const bool fdx_ok = h->use_tc && k == 1 && (h->fusion & MOE_FUSE_DX) && T > 0 &&
                      a->dx != nullptr && ((uintptr_t)a->dx % 16) == 0 && tc_dx_fusion_supported(d);
  const bool fdx = fdx_ok && !h->use_ep;
  // peer EP (N1 return rows): the owners' dX GEMMs add dl W_g and return dx rows
  const bool fdx_ep = fdx_ok && h->use_peer && h->peer_ret;
  rb.dlr = fdx ? (__nv_bfloat16*)(ws + h->L.dlr)
         : fdx_ep ? (__nv_bfloat16*)(h->pwin + h->PL.dlr) : nullptr;
  rb.pdlr = fdx_ep ? peer_bufs(h, h->PL.dlr) : PeerBufs{};
  rb.dropb = (fdx || fdx_ep) ? (__nv_bfloat16*)(ws + h->L.dropb) : nullptr;

  rb.o_pair = (peer && h->peer_ret) || h->otok;
  rb.dx_pair = peer && h->peer_ret;
  KL(h, T > 0, "combine_bwd", s0, launch_combine_bwd(dt, a->dy, O_tok, rb, T, k, n, dout, h->renorm, h->cts,
                                                     dO_tok, dlb, h->maxT, h->n_pad,
                                                     nccl_ep ? nullptr : rb.kept, s0,
                                                     peer ? h->e_lo : 0,
                                                     peer && !h->peer_ret ? peer_bufs(h, h->PL.o) : PeerBufs{},
                                                     peer ? peer_bufs(h, h->PL.dob) : PeerBufs{}));
  rb.o_pair = 0;
  rb.dx_pair = 0;
  rb.dspec = nullptr;
  rb.dw_ext = nullptr;
  rb.bal_g = nullptr;
  rb.dlr = nullptr;
  rb.pdlr = PeerBufs{};
  rb.dropb = nullptr;
  if (peer) {  // N1: dO rows were stored into the owners by the combine backward
    KL(h, 1, "peer_barrier", s0, launch_peer_barrier(h->wins, h->R, h->rank, PH_DO, s0, (uint32_t*)rb.flags));
  } else if (h->use_ep) {  // C4: dO rows to the expert owners
    moe_status_t st = ep_to_experts(h->ep, h->plan, dO_tok, dO, h->ct, dout, (int)h->s, s0, &err);
    if (st != MOE_OK) return fail(h, st, err);
    KL(h, 1, "zero_pad", s0, launch_zero_pad(dt, dO, dout, kept_local, nl, h->ct, s0));
  }
  const char* w1 = (const char*)fa.w1 + (size_t)h->e_lo * f * d * h->s;
  const char* w2 = (const char*)fa.w2 + (size_t)h->e_lo * dout * f * h->s;
  char* dw1 = a->dw1 ? (char*)a->dw1 + (size_t)h->e_lo * f * d * h->s : nullptr;
  char* db1 = a->db1 ? (char*)a->db1 + (size_t)h->e_lo * f * h->s : nullptr;
  char* dw2 = a->dw2 ? (char*)a->dw2 + (size_t)h->e_lo * dout * f * h->s : nullptr;
  char* db2 = a->db2 ? (char*)a->db2 + (size_t)h->e_lo * dout * h->s : nullptr;
  if (h->R > 1 && !acc) {  // EP: the other ranks' expert slices of the full tensors read zero
    const size_t per[4] = {(size_t)f * d * h->s, (size_t)f * h->s, (size_t)dout * f * h->s,
                           (size_t)dout * h->s};
    void* full[4] = {a->dw1, a->db1, a->dw2, a->db2};
    for (int q = 0; q < 4; ++q) {
      if (!full[q]) continue;
      char* base = (char*)full[q];
      if (h->e_lo > 0) CUDA_TRY(h, cudaMemsetAsync(base, 0, per[q] * h->e_lo, s0));
      const size_t hi = (size_t)(h->e_lo + nl);
      if (hi < (size_t)n) CUDA_TRY(h, cudaMemsetAsync(base + per[q] * hi, 0, per[q] * (n - hi), s0));
    }
  }
  // Backward tail (single GPU, fused dispatch backward, dW_g requested): the db1 reduction, the
  // drop-only gate-dx pass and the gate-weight gradient read only data of kernels that are
  // complete once the dX GEMM has started, so they skip their PDL wait and run beside that
  // GEMM's tail and each other; the gate-weight reduction closes the backward with a
  // full-dependency launch (every later kernel again sees all of this step complete).
  const char* tail_e = getenv("MOE_TAIL");  // (read per call: the tests toggle it)
  const bool tail_env = !(tail_e && tail_e[0] == '0');
  const bool tail = tail_env && !h->use_ep && h->use_tc && T > 0 && a->dw_gate != nullptr &&
                    (fdx || a->dx == nullptr);
  // fp32 (split-tf32 GEMMs): dA / dX GEMMs and the gate-weight partials skip their waits the
  // same way; the gate-dx pass (it reads dX) keeps its wait on the dX GEMM
  const bool tail32 = tail_env && !h->use_ep && h->use_tf32 && T > 0 && a->dw_gate != nullptr;
  if (h->use_tc) {
    int64_t nk = 0;
    TcFusion fz;  // N2: dW1 = dA^T X gathers the x rows like the forward did
    fz.T = T;
    fz.tos = rb.token_of_slot;
    fz.k = k;
    if (h->fused_gather) fz.x = fa.x;
    if (peer && h->peer_ret) {  // N1: DGRAD_X's epilogue returns dX rows to the token owners
      fz.pret_dx = peer_bufs(h, h->PL.dxret);
      fz.tpr = T;
    }
    if (fdx || fdx_ep) {
      fz.dx_fused = true;
      fz.dx = fdx ? a->dx : nullptr;
      fz.dlr = fdx ? (void*)(ws + h->L.dlr) : (void*)(h->pwin + h->PL.dlr);
      fz.wg = fa.w_gate;
      fz.n = n;
      fz.n_pad = h->n_pad;
      fz.accumulate = acc;
    }
    moe_status_t st = tc_ffn_backward(&h->tc, X, H, dO, dXb, w1, w2, dw1, db1, dw2, db2, acc,
                                      h->rows, d, f, dout, kept_local, rb.mtile_prefix, nl,
                                      h->ct, h->max_cap_local, s0, &nk, &h->prof,
                                      (uint32_t*)(ws + h->L.mask), (float*)(ws + h->L.bpart),
                                      (h->fused_gather || fdx || fdx_ep || (peer && h->peer_ret)) ? &fz : nullptr,
                                      tail ? 1 : 0, tail ? (void*)(ws + h->L.dabuf) : nullptr);
    h->launches += nk;
    if (st != MOE_OK) return fail(h, st, "tcgen05 backward failed");
  } else if (h->use_tf32) {
    int64_t nk = 0;
    moe_status_t st = tf32_ffn_backward(X, H, dO, dXb, w1, w2, dw1, db1, dw2, db2, acc, h->rows,
                                        d, f, dout, kept_local, rb.mtile_prefix, nl, h->ct, s0,
                                        &nk, &h->prof, tail32 ? 1 : 0,
                                        tail32 ? (void*)(ws + h->L.dabuf) : nullptr);
    h->launches += nk;
    if (st != MOE_OK) return fail(h, st, "tcgen05 tf32 backward failed");
  } else {
    // B3a: dW2_e = dO_e^T H_e ; db2 = sum dO   (before H is overwritten by dA)
    if (dw2) KL(h, 1, "wgrad_w2", s0, launch_gemm_simt_kgroup(dt, dO, dout, H, f, dw2, dout, f, kept_local, nl, h->ct, acc, s0));
    if (db2) KL(h, 1, "bias_grad", s0, launch_colsum(dt, dO, dout, kept_local, nl, h->ct, db2, acc, s0));
    // B2a: dA = (dO W2_e) * 1[H > 0]   (in place over H)
    KL(h, 1, "dgrad_dA", s0, launch_gemm_simt_mgroup(dt, dO, dout, w2, 0, (int64_t)dout * f, nullptr, H, f, f,
                                     dout, kept_local, nl, h->ct, h->max_cap_local, EPI_RELU_MASK, s0));
    // B3b: dW1_e = dA_e^T X_e ; db1 = sum dA
    if (dw1) KL(h, 1, "wgrad_w1", s0, launch_gemm_simt_kgroup(dt, H, f, X, d, dw1, f, d, kept_local, nl, h->ct, acc, s0));
    if (db1) KL(h, 1, "bias_grad", s0, launch_colsum(dt, H, f, kept_local, nl, h->ct, db1, acc, s0));
    // B2b: dX_e = dA_e W1_e
    KL(h, 1, "dgrad_dX", s0, launch_gemm_simt_mgroup(dt, H, f, w1, 0, (int64_t)f * d, nullptr, dXb, d, d, f,
                                     kept_local, nl, h->ct, h->max_cap_local, EPI_NONE, s0));
  }
  // B4: dx = gather(dX) + dl W_g ;  B5: dW_g = dl^T x
  void* dX_tok = dXb;
  PeerBufs pdx{};
  // peer EP: the gate-weight gradient partial needs only local data (dl, x); computed before
  // the exchange barrier, one barrier then covers the returned dX rows and every rank's
  // dW_g partial
  float* dwg_f32 = peer ? (float*)(h->pwin + h->PL.dwg) : nccl_ep ? (float*)(ws + h->L.dwg32) : nullptr;
  auto gate_dw_partial = [&]() -> moe_status_t {
    if (h->use_tc) {
      KL(h, T > 0 ? 2 : 0, "gate_dw", s0, launch_gate_dw_tc(dlb, h->maxT, h->n_pad, fa.x, T, n, d,
                                                            (float*)(ws + h->L.partial), a->dw_gate, acc, s0,
                                                            dwg_f32, tail));
    } else {
      int splits = gate_dw_splits(h->maxT, d);
      KL(h, T > 0 ? 2 : 0, "gate_dw", s0, launch_gate_dw(dt, rb.dl, fa.x, T, n, d, (float*)(ws + h->L.partial),
                                          splits, a->dw_gate, acc, s0, dwg_f32, tail32));
    }
    if (T == 0 && dwg_f32) CUDA_TRY(h, cudaMemsetAsync(dwg_f32, 0, (size_t)n * d * 4, s0));  // no tokens
    return MOE_OK;
  };
  if (peer && a->dw_gate) {
    moe_status_t st = gate_dw_partial();
    if (st != MOE_OK) return st;
  }
  if (peer) {  // N1: the gate-input gradient reads dX rows from the owners (or, with return
               // rows, this rank's own (token, choice) rows the owners stored)
    KL(h, 1, "peer_barrier", s0, launch_peer_barrier(h->wins, h->R, h->rank, PH_DX, s0, (uint32_t*)rb.flags));
    if (h->peer_ret)
      dX_tok = h->pwin + h->PL.dxret;
    else
      pdx = peer_bufs(h, h->PL.dxb);
  } else if (h->use_ep) {  // C5: dX rows back to the token owners (send layout, reuses the send buffer)
    dX_tok = ws + h->L.sendbuf;
    moe_status_t st = ep_from_experts(h->ep, h->plan, dXb, dX_tok, h->ct, d, (int)h->s, s0, &err);
    if (st != MOE_OK) return fail(h, st, err);
  }
  if (a->dx) {  // fused dX GEMM: it wrote the kept tokens, this pass only the dropped ones
    if (fdx_ep)  // peer EP: the kept tokens' dx rows came back from the owners' dX GEMMs
      KL(h, T > 0, "dx_from_ret", s0, launch_dx_from_ret(h->pwin + h->PL.dxret, rb.slot_of, T, d,
                                                         a->dx, acc, s0));
    const bool drop_only = fdx || fdx_ep;
    if (h->use_tc)
      KL(h, T > 0, "gate_dx", s0, launch_gate_dx_tc(fa.w_gate, dX_tok,
                                                    drop_only ? (void*)(ws + h->L.dropb) : dlb,
                                                    h->maxT, h->n_pad, rb, T, k, n, d, h->cts,
                                                    a->dx, acc, s0, pdx, drop_only ? 1 : 0, tail));
    else
      KL(h, T > 0, "gate_dx", s0, launch_gate_dx(dt, fa.w_gate, dX_tok, rb, T, k, n, d, h->cts, a->dx, acc, s0,
                                                 pdx));
  }
  if (a->dw_gate) {
    if (!peer) {
      moe_status_t st = gate_dw_partial();
      if (st != MOE_OK) return st;
    }
    if (peer) {  // N1: sum of every rank's fp32 partial in rank order (after the PH_DX barrier)
      KL(h, 1, "gate_dw", s0, launch_peer_sum(h->wins, h->PL.dwg, h->R, (size_t)n * d, dt,
                                              a->dw_gate, acc, s0));
    } else if (h->use_ep) {  // C6
      moe_status_t st = ep_allreduce_f32(h->ep, dwg_f32, (size_t)n * d, s0, &err);
      if (st != MOE_OK) return fail(h, st, err);
      KL(h, 1, "gate_dw", s0, launch_f32_to(dt, dwg_f32, (size_t)n * d, a->dw_gate, acc, s0));
    }
  }
  h->have_fwd = 0;  // H has been consumed
  return MOE_OK;
}

moe_status_t moe_peer_window(moe_handle_t h, void** window, size_t* bytes) {
  if (!h || !window) return MOE_ERR_INVALID_ARG;
  if (!h->use_peer) return fail(h, MOE_ERR_STATE, "not a peer-transport handle");
  *window = h->pwin;
  if (bytes) *bytes = h->PL.total;
  return MOE_OK;
}

moe_status_t moe_peer_export(moe_handle_t h, void* ipc_handle) {
  if (!h || !ipc_handle) return MOE_ERR_INVALID_ARG;
  if (!h->use_peer) return fail(h, MOE_ERR_STATE, "not a peer-transport handle");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t hd;
  CUDA_TRY(h, cudaIpcGetMemHandle(&hd, h->pwin));
  std::memcpy(ipc_handle, &hd, 64);
  return MOE_OK;
}

moe_status_t moe_peer_attach(moe_handle_t h, void* const* windows) {
  if (!h || !windows) return MOE_ERR_INVALID_ARG;
  if (!h->use_peer) return fail(h, MOE_ERR_STATE, "not a peer-transport handle");
  if (windows[h->rank] != h->pwin)
    return fail(h, MOE_ERR_INVALID_ARG, "windows[rank] must be this handle's own window");
  for (int j = 0; j < h->R; ++j)
    if (!windows[j]) return fail(h, MOE_ERR_INVALID_ARG, "null peer window");
  for (int j = 0; j < MOE_MAX_R; ++j) h->wins.p[j] = j < h->R ? (char*)windows[j] : nullptr;
  h->wins.nl = h->n_local;
  h->peer_attached = 1;
  return MOE_OK;
}

moe_status_t moe_peer_connect_nccl(moe_handle_t h, void* nccl_comm) {
  if (!h || !nccl_comm) return MOE_ERR_INVALID_ARG;
  if (!h->use_peer) return fail(h, MOE_ERR_STATE, "not a peer-transport handle");
  if (h->peer_attached || h->lsa.buf)
    return fail(h, MOE_ERR_STATE, "peer windows already attached");
  void* ptrs[MOE_MAX_R] = {};
  LsaWindow w;
  std::string err;
  moe_status_t st = lsa_window_create(nccl_comm, h->R, h->rank, h->PL.total, &w, ptrs, &err);
  if (st != MOE_OK) return fail(h, st, err);
  // the NCCL window replaces the cudaMalloc one (same layout, zeroed)
  cudaDeviceSynchronize();
  cudaFree(h->pwin);
  h->pwin = (char*)w.buf;
  h->lsa = w;
  if (h->ws) bind_buffers(h);  // token_of_slot lives in the window
  return moe_peer_attach(h, ptrs);
}

moe_status_t moe_peer_import(moe_handle_t h, const void* handles) {
  if (!h || !handles) return MOE_ERR_INVALID_ARG;
  if (!h->use_peer) return fail(h, MOE_ERR_STATE, "not a peer-transport handle");
  void* w[MOE_MAX_R] = {};
  for (int j = 0; j < h->R; ++j) {
    if (j == h->rank) {
      w[j] = h->pwin;
      continue;
    }
    if (h->opened[j]) {
      w[j] = h->wins.p[j];
      continue;
    }
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, (const char*)handles + 64 * j, 64);
    CUDA_TRY(h, cudaIpcOpenMemHandle(&w[j], hd, cudaIpcMemLazyEnablePeerAccess));
    h->opened[j] = true;
    h->wins.p[j] = (char*)w[j];
  }
  return moe_peer_attach(h, w);
}

moe_status_t moe_get_routing(moe_handle_t h, moe_routing_t* out) {
  if (!h || !out) return MOE_ERR_INVALID_ARG;
  if (!h->ws) return fail(h, MOE_ERR_STATE, "workspace not set");
  std::memset(out, 0, sizeof(*out));
  const RouteBufs& r = h->rb;
  out->logits = r.logits;
  out->weights = r.w;
  out->idx = r.idx;
  out->fresh_idx = h->last_cached ? r.fresh_idx : r.idx;
  out->slot_of = r.slot_of;
  out->token_of_slot = r.token_of_slot;
  out->counts = r.counts;
  out->kept = r.kept;
  out->dl = r.dl;
  out->dw = r.dw;
  out->x_buf = buf_x(h);
  out->h_buf = h->ws + h->L.hbuf;
  out->o_buf = buf_o(h);
  out->rows = h->rows;
  for (int j = 0; j <= h->n_local; ++j) out->base_host[j] = h->ct.base[j];
  return MOE_OK;
}

moe_status_t moe_get_stats_async(moe_handle_t h, const moe_stats_t* dst) {
  if (!h || !dst) return MOE_ERR_INVALID_ARG;
  if (!h->ws) return fail(h, MOE_ERR_STATE, "workspace not set");
  if (dst->counts)
    CUDA_TRY(h, cudaMemcpyAsync(dst->counts, h->rb.counts, 4 * h->n, cudaMemcpyDeviceToHost, h->stream));
  if (dst->drops)
    CUDA_TRY(h, cudaMemcpyAsync(dst->drops, h->rb.drops, 8, cudaMemcpyDeviceToHost, h->stream));
  if (dst->hit_count)
    CUDA_TRY(h, cudaMemcpyAsync(dst->hit_count, h->rb.hit_count, 4, cudaMemcpyDeviceToHost, h->stream));
  return MOE_OK;
}

moe_status_t moe_check_device_flags(moe_handle_t h, int32_t* flags_out) {
  if (!h) return MOE_ERR_INVALID_ARG;
  if (!h->ws) return fail(h, MOE_ERR_STATE, "workspace not set");
  int32_t fl = 0;
  CUDA_TRY(h, cudaMemcpyAsync(&fl, h->rb.flags, 4, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  if (flags_out) *flags_out = fl;
  if (fl) {
    CUDA_TRY(h, cudaMemsetAsync(h->rb.flags, 0, 4, h->stream));
    return fail(h, MOE_ERR_DEVICE_FLAG,
                std::string("device flags: ") + ((fl & 1) ? "NaN logit " : "") +
                    ((fl & 2) ? "invalid cached index " : "") +
                    ((fl & 4) ? "sample id out of range " : "") +
                    ((fl & 8) ? "peer barrier timeout" : ""));
  }
  return MOE_OK;
}

moe_status_t moe_profile_enable(moe_handle_t h, int32_t on) {
  if (!h) return MOE_ERR_INVALID_ARG;
  h->prof.on = on != 0;
  return MOE_OK;
}

moe_status_t moe_profile_read(moe_handle_t h, moe_kernel_time_t* out, int32_t max,
                              int32_t* count, int32_t reset) {
  if (!h || !count || (max > 0 && !out)) return MOE_ERR_INVALID_ARG;
  CUDA_TRY(h, cudaDeviceSynchronize());
  std::vector<std::string> order;
  std::map<std::string, std::pair<int64_t, double>> agg;
  for (const auto& r : h->prof.recs) {
    float ms = 0.f;
    CUDA_TRY(h, cudaEventElapsedTime(&ms, r.a, r.b));
    auto it = agg.find(r.name);
    if (it == agg.end()) {
      order.push_back(r.name);
      agg[r.name] = {1, (double)ms};
    } else {
      it->second.first += 1;
      it->second.second += ms;
    }
  }
  int c = 0;
  for (const auto& nm : order) {
    if (c >= max) break;
    std::memset(out[c].name, 0, sizeof(out[c].name));
    std::strncpy(out[c].name, nm.c_str(), sizeof(out[c].name) - 1);
    out[c].launches = agg[nm].first;
    out[c].total_ms = agg[nm].second;
    ++c;
  }
  *count = c;
  if (reset) h->prof.reset();
  return MOE_OK;
}

moe_status_t moe_ep_plan(int32_t R, int32_t rank, int32_t n, const int32_t* cnt_all,
                         const int32_t* cap, int32_t* pre_out, int32_t* kl_out,
                         int32_t* send_off_out, int32_t* kept_local_out, int64_t* drops_out) {
  if (R < 1 || rank < 0 || rank >= R || n < 1 || n % R || !cnt_all || !cap)
    return MOE_ERR_INVALID_ARG;
  EpPlan P;
  ep_make_plan(P, R, rank, n, cnt_all, cap);
  if (pre_out) std::memcpy(pre_out, P.pre.data(), 4 * (size_t)R * n);
  if (kl_out) std::memcpy(kl_out, P.kl.data(), 4 * (size_t)R * n);
  if (send_off_out) std::memcpy(send_off_out, P.send_off.data(), 4 * (size_t)n);
  if (kept_local_out) std::memcpy(kept_local_out, P.kept_local.data(), 4 * (size_t)P.n_local);
  if (drops_out) *drops_out = P.drops;
  return MOE_OK;
}

moe_status_t moe_metrics_enable(moe_handle_t h, int32_t depth) {
  if (!h || depth < 0) return MOE_ERR_INVALID_ARG;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  for (auto& sl : h->mq) {
    if (sl.host) cudaFreeHost(sl.host);
    if (sl.ev) cudaEventDestroy(sl.ev);
  }
  h->mq.assign(depth, {});
  for (auto& sl : h->mq) {
    CUDA_TRY(h, cudaMallocHost(&sl.host, sizeof(moe_metrics_t)));
    std::memset(sl.host, 0, sizeof(moe_metrics_t));
    CUDA_TRY(h, cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming));
  }
  h->mq_head = h->mq_count = 0;
  h->mq_iter = 0;
  return MOE_OK;
}

moe_status_t moe_metrics_pending(moe_handle_t h, int32_t* n) {
  if (!h || !n) return MOE_ERR_INVALID_ARG;
  *n = h->mq_count;
  return MOE_OK;
}

moe_status_t moe_metrics_pop(moe_handle_t h, int32_t block, moe_metrics_t* out, int32_t* got) {
  if (!h || !out || !got) return MOE_ERR_INVALID_ARG;
  *got = 0;
  if (h->mq_count == 0) return MOE_OK;
  auto& sl = h->mq[h->mq_head];
  if (block) {
    CUDA_TRY(h, cudaEventSynchronize(sl.ev));
  } else {
    cudaError_t q = cudaEventQuery(sl.ev);
    if (q == cudaErrorNotReady) return MOE_OK;
    CUDA_TRY(h, q);
  }
  std::memcpy(out, sl.host, sizeof(moe_metrics_t));
  h->mq_head = (h->mq_head + 1) % (int)h->mq.size();
  --h->mq_count;
  *got = 1;
  return MOE_OK;
}

moe_status_t moe_caching_trigger(double hit_fraction, int32_t epoch, int32_t enabled,
                                 double enable_at, double disable_below, int32_t warmup_epochs,
                                 int32_t* new_enabled) {
  if (!new_enabled || disable_below > enable_at) return MOE_ERR_INVALID_ARG;
  int32_t e = enabled ? 1 : 0;
  if (epoch >= warmup_epochs) {
    if (!e && hit_fraction >= enable_at) e = 1;
    else if (e && hit_fraction < disable_below) e = 0;
  }
  *new_enabled = e;
  return MOE_OK;
}

moe_status_t moe_set_balance_loss(moe_handle_t h, float lambda) {
  if (!h || !(lambda >= 0.f)) return MOE_ERR_INVALID_ARG;
  h->balance_lambda = lambda;
  return MOE_OK;
}

moe_status_t moe_get_aux_loss_async(moe_handle_t h, float* host_dst) {
  if (!h || !host_dst) return MOE_ERR_INVALID_ARG;
  if (!h->ws) return fail(h, MOE_ERR_STATE, "workspace not set");
  if (h->balance_lambda == 0.f) {
    *host_dst = 0.f;
    return MOE_OK;
  }
  const float* aux = (const float*)(h->ws + h->L.bal) + (size_t)((h->maxT + 63) / 64) * h->n + 2 * h->n;
  CUDA_TRY(h, cudaMemcpyAsync(host_dst, aux, 4, cudaMemcpyDeviceToHost, h->stream));
  return MOE_OK;
}

moe_status_t moe_set_spec_outputs(moe_handle_t h, void* spec, uint8_t* valid) {
  if (!h || (!spec != !valid)) return MOE_ERR_INVALID_ARG;
  h->spec = spec;
  h->spec_valid = valid;
  return MOE_OK;
}

moe_status_t moe_set_spec_grads(moe_handle_t h, const void* dspec, const float* dw_ext) {
  if (!h) return MOE_ERR_INVALID_ARG;
  h->dspec = dspec;
  h->dw_ext = dw_ext;
  return MOE_OK;
}

moe_status_t moe_vcomm_create(int32_t R, void** comm_out) { return vcomm_create(R, comm_out); }
moe_status_t moe_vcomm_destroy(void* comm) { return vcomm_destroy(comm); }

moe_status_t moe_set_fusion(moe_handle_t h, int32_t flags) {
  if (!h) return MOE_ERR_INVALID_ARG;
  if (flags & ~(MOE_FUSE_GATHER | MOE_FUSE_COMBINE | MOE_FUSE_DX | MOE_FUSE_OTOK |
                MOE_FUSE_COMBINE2 | MOE_FUSE_CDISP))
    return fail(h, MOE_ERR_INVALID_ARG, "unknown fusion flag");
  h->fusion = flags;
  return MOE_OK;
}

moe_status_t moe_launch_count(moe_handle_t h, int64_t* out) {
  if (!h || !out) return MOE_ERR_INVALID_ARG;
  *out = h->launches;
  return MOE_OK;
}

// ------------------------------------------------------------------------------------
// Dynamic capacity policy (SPEC S:449-456 concretisation of P:236; see moe.h)
// ------------------------------------------------------------------------------------
struct moe_policy {
  moe_policy_config_t c;
  std::vector<int32_t> caps;
  std::deque<std::vector<int32_t>> hist;
};

static int32_t policy_clamp(const moe_policy* p, int64_t c) {
  double alpha = (double)c * p->c.n_experts / ((double)p->c.tokens_global * p->c.top_k);
  alpha = std::min(std::max(alpha, p->c.min_alpha), p->c.max_alpha);
  // Eq. 4 with this expert's alpha: max(1, ceil(alpha * T_g * k / n))
  double v = std::ceil(alpha * (double)p->c.tokens_global * p->c.top_k / p->c.n_experts);
  return std::max<int32_t>(1, (int32_t)v);
}

moe_status_t moe_policy_create(const moe_policy_config_t* cfg, const int32_t* init_cap,
                               moe_policy_t* out) {
  if (!cfg || !init_cap || !out || cfg->n_experts < 1 || cfg->top_k < 1 ||
      cfg->tokens_global < 1 || cfg->window < 1 || cfg->min_alpha > cfg->max_alpha)
    return MOE_ERR_INVALID_ARG;
  moe_policy* p = new moe_policy();
  p->c = *cfg;
  p->caps.assign(init_cap, init_cap + cfg->n_experts);
  *out = p;
  return MOE_OK;
}

moe_status_t moe_policy_update(moe_policy_t p, const int32_t* counts, int32_t* new_cap,
                               int32_t* changed) {
  if (!p || !counts || !new_cap || !changed) return MOE_ERR_INVALID_ARG;
  const int n = p->c.n_experts;
  p->hist.emplace_back(counts, counts + n);
  if ((int)p->hist.size() > p->c.window) p->hist.pop_front();
  std::vector<int32_t> nc = p->caps;
  const int W = (int)p->hist.size();
  for (int e = 0; e < n; ++e) {
    int64_t peak = 0, sum = 0;
    for (const auto& hrow : p->hist) {
      peak = std::max<int64_t>(peak, hrow[e]);
      sum += hrow[e];
    }
    int64_t target = (int64_t)std::ceil((1.0 + p->c.headroom) * (double)peak);
    if (p->caps[e] < peak) {
      nc[e] = policy_clamp(p, target);
    } else if (W == p->c.window && ((double)sum / W) / p->caps[e] < p->c.shrink_util) {
      nc[e] = policy_clamp(p, std::max<int64_t>(target, 1));
    }
  }
  *changed = (nc != p->caps) ? 1 : 0;
  if (*changed) p->caps = nc;
  std::memcpy(new_cap, p->caps.data(), sizeof(int32_t) * n);
  return MOE_OK;
}

moe_status_t moe_policy_destroy(moe_policy_t p) {
  delete p;
  return MOE_OK;
}

}  // extern "C"
