/*
 * moe.h -- C ABI of the B200-native DynaMoE MoE-layer hot path.
 *
 * The operation (PAPER.md = /root/reference/PAPER.md, cited as P:line):
 *   Alg. 1: score <- G(x); indices <- argmax_k(score);
 *                       (w_1..w_k) <- normalize(score[indices]); y = sum_i w_i * E_{indices[i]}(x)
 *   Eq. 4: expert capacity C = alpha * batch_size * k / n
 *   P:225:              samples that do not fit an expert's capacity are dropped and
 *                       "ignored during back propagation"
 *   S4.1: dynamic capacity factors  -> moe_set_capacities (a stream-ordered
 *                       "recompile" of the per-expert buffer sizes; weights untouched)
 *   S4.2: sample-assignment caching -> moe_set_cached_assignment (cached
 *                       expert indices drive dispatch so it does not wait for the gate)
 * Readings of points the paper leaves open are SURVEY.md §8(c) readings 1-15, listed in
 * DESIGN.md.  In particular: G is one bias-free linear layer W_g [n x d]; top-k selects on
 * the fp32 logits with ties to the lower expert index; normalize() is sum-normalisation of
 * the selected softmax probabilities (renormalize=1) or the raw probability (renormalize=0);
 * capacity is global and the drop order is token-major (ascending global token index);
 * experts are 2-layer ReLU MLPs  E_e(x) = W2_e relu(W1_e x + b1_e) + b2_e.
 *
 * Conventions
 *  - Every function returns moe_status_t; nothing throws or aborts across the ABI.
 *  - "device" pointers are CUDA device (HBM) pointers on the handle's device; "host"
 *    pointers are ordinary CPU memory.  No torch types appear in any signature.
 *  - Layouts are row-major, torch Linear convention ([out, in]):
 *      x [T, d], w_gate [n, d], w1 [n, f, d], b1 [n, f], w2 [n, d_out, f], b2 [n, d_out],
 *      y [T, d_out], dy [T, d_out], dx [T, d].  All in the layer dtype (fp32 or bf16).
 *  - All GPU work is enqueued on cfg.stream (or the stream set by moe_set_stream) and
 *    is stream-ordered; calls return without synchronising unless stated.  Internal
 *    side streams are joined back onto that stream before a call returns.
 *  - Host-side validation failures return synchronously before any work is enqueued.
 *  - Device-detected errors (NaN logit, invalid cached index) raise a device flag that is
 *    reported as MOE_ERR_DEVICE_FLAG by moe_check_device_flags (which synchronises).
 *  - Ownership: the caller owns every tensor and the workspace; the library owns only its
 *    handle, internal events/side streams.  x and the parameters must stay unchanged
 *    until moe_backward has been enqueued (the backward re-reads them).
 *  - One handle per thread; handles are not reentrant.
 *
 * Environment switches (read once per process; unset = the product configuration, which
 * every test and the bench use unless they say otherwise -- the others exist for A/B timing
 * and diagnosis, DESIGN.md lists what each measured):
 *   MOE_PDL=0          launch without programmatic dependent launch
 *   MOE_FORCE_SIMT=1   bf16 layers on the CUDA-core (SIMT) GEMMs instead of tcgen05
 *   MOE_PEER_RET=0     peer transport: owners' rows read remotely instead of return rows
 *   MOE_TC_1CTA=mask   GEMM kinds (bit per kind) on the 1-CTA instead of the 2-CTA kernel
 *   MOE_TC_SCHED=1     contiguous tile chunk per CTA pair instead of round-robin
 *   MOE_TC_PF=n        GEMM producer prefetches B k-blocks to L2 for the next wave
 *   MOE_TC_DBG, MOE_GATE_DBG   timing-only experiments that SKIP work (wrong results)
 */
#ifndef DYNAMOE_B200_MOE_H
#define DYNAMOE_B200_MOE_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MOE_API __attribute__((visibility("default")))
#else
#define MOE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MOE_OK = 0,
  MOE_ERR_INVALID_ARG = 1,         /* null pointer, bad size, T > max_tokens, capacity < 1 */
  MOE_ERR_CONFIG = 2,              /* unsupported shape: k > n, n > 256, dims not multiples */
  MOE_ERR_STATE = 3,               /* e.g. backward before forward, workspace not set */
  MOE_ERR_WORKSPACE_TOO_SMALL = 4, /* capacities grew: query moe_workspace_size, reallocate */
  MOE_ERR_CUDA = 5,
  MOE_ERR_NCCL = 6,
  MOE_ERR_DEVICE_FLAG = 7          /* a kernel flagged NaN logits or an invalid cached index */
} moe_status_t;

typedef enum { MOE_F32 = 0, MOE_BF16 = 1 } moe_dtype_t;

typedef struct moe_ctx* moe_handle_t;

/* Layer configuration (fixed for the life of a handle). */
typedef struct {
  int32_t n_experts;    /* n, 1..256 */
  int32_t top_k;        /* k, 1..min(n, 8) */
  int32_t d_model;      /* d: multiple of 64 for bf16, of 4 for fp32 */
  int32_t d_ff;         /* f: same rule */
  int32_t d_out;        /* 0 -> d_model; same rule */
  int32_t max_tokens;   /* per-rank upper bound on T */
  int32_t dtype;        /* moe_dtype_t: activation/parameter dtype; logits, weights and
                           every accumulator are fp32 */
  int32_t renormalize;  /* 1: Alg. 1 normalize (sum-norm of selected probs);
                           0: raw softmax probability (Switch-style) */
  int32_t world_size;   /* expert-parallel group size R (n % R == 0) */
  int32_t rank;         /* experts [rank*n/R, (rank+1)*n/R) are local */
  void*   nccl_comm;    /* ncclComm_t of the EP group (e.g. torch ProcessGroupNCCL._comm_ptr()).
                           NULL: single-GPU path (R must be 1).  Non-NULL: expert-parallel path
                           (S8(e)): tokens data-parallel, equal T on every rank, global token
                           index t_g = rank*T + t, GLOBAL capacity (reading 12), exchanges by
                           grouped ncclSend/ncclRecv; R = 1 runs the same path as a loopback.
                           Expert parameter / gradient tensors keep the full [n, ...] shape;
                           only the local experts' slices are read and written. */
  void*   stream;       /* cudaStream_t all work is ordered on (NULL = legacy default) */
  int32_t transport;    /* moe_transport_t of the expert-parallel exchanges (R > 1 or loopback):
                           MOE_TRANSPORT_NCCL: nccl_comm required (above).
                           MOE_TRANSPORT_PEER: device-initiated exchange through peer memory
                           (see "Peer-memory expert parallelism" below);
                           nccl_comm unused (may be NULL), world_size 1..8 */
  int32_t reserved0;    /* must be 0 */
  int64_t window_rows;  /* MOE_TRANSPORT_PEER: rows of each peer-visible expert buffer (bounds
                           sum_local roundup(C_e, 128) for every later moe_set_capacities);
                           0 = the bound for Eq. 4 at alpha = 8 (the policy's maximum) */
} moe_config_t;

typedef enum { MOE_TRANSPORT_NCCL = 0, MOE_TRANSPORT_PEER = 1 } moe_transport_t;

/* Create / destroy a layer handle.  moe_init validates cfg (MOE_ERR_CONFIG) and sets the
   capacities to Eq. 4 with alpha = 1 over T_g = max_tokens * world_size. */
MOE_API moe_status_t moe_init(const moe_config_t* cfg, moe_handle_t* out);
MOE_API moe_status_t moe_destroy(moe_handle_t h);
MOE_API moe_status_t moe_set_stream(moe_handle_t h, void* stream);

/* Eq. 4, host only: cap_out[e] = max(1, ceil(alpha[e] * tokens_global * k / n))
   evaluated in fp64.  alpha: host [n]; cap_out: host [n]. */
MOE_API moe_status_t moe_capacity_from_factors(int32_t n, int64_t tokens_global, int32_t k,
                                       const double* alpha, int32_t* cap_out);

/* Dynamic capacity factors (S4.1).  cap: host [n], each >= 1 (values above the
   global token count are clamped to it; the result is unchanged because an expert can
   receive each token at most once).  Re-lays out the per-expert buffers (row offsets
   base_e = sum_{e'<e} roundup(C_e', 128)) and takes effect at the next moe_forward enqueued
   after this call (the new table travels as kernel arguments: stream-ordered, no sync).
   Returns MOE_ERR_WORKSPACE_TOO_SMALL when the set workspace is too small for the new
   layout; the capacities ARE recorded, so the caller queries moe_workspace_size,
   allocates and calls moe_set_workspace.  With the peer transport, capacities whose
   local expert rows exceed the library-owned peer window (cfg.window_rows) are refused
   with MOE_ERR_CONFIG and NOT recorded (the previous capacities stay in force).
   Weights are never touched. */
MOE_API moe_status_t moe_set_capacities(moe_handle_t h, const int32_t* cap);
MOE_API moe_status_t moe_get_capacities(moe_handle_t h, int32_t* cap_out /* host [n] */);

/* Workspace (caller-owned device memory): saved activations X/H/O, gradient scratch
   dO/dX, routing tables and partial sums.  Size depends on max_tokens and capacities. */
MOE_API moe_status_t moe_workspace_size(moe_handle_t h, size_t* bytes);
MOE_API moe_status_t moe_set_workspace(moe_handle_t h, void* dptr, size_t bytes);

/* Sample-assignment caching (S4.2).  d_idx: device int32 [T x k] expert
   indices (each row k distinct values in [0,n)) read by the NEXT moe_forward; NULL turns
   caching off.  While on, dispatch (histogram, scan, scatter, and in EP the count exchange)
   runs on a side stream from these indices concurrently with the gate; the gate still runs
   and yields the weights normalize(p[t, cached]) (reading 11), the fresh top-k and
   hit_count = #{t : set(fresh_t) == set(cached_t)}.  d_idx must stay valid until that
   forward has been consumed by the stream.  Invalid rows raise the device flag. */
MOE_API moe_status_t moe_set_cached_assignment(moe_handle_t h, const int32_t* d_idx);

/* Per-sample assignment cache (S4.2 P:245-256; SPEC cache_step S:252-257,
   cached_route S:259-267).  d_table: caller-owned device int32 [num_samples x k], row s =
   the experts sample s was last routed to, -1 = unknown (the caller fills it with -1).
   d_sample_ids: device int64 [T], the sample id of each token of the NEXT forwards (the
   caller rewrites it per batch; ids must be distinct within a batch).  mode:
     0  off (the default);
     1  every sample of the batch is known: idx = table[ids] drives dispatch on the side
        stream concurrently with the gate, exactly as moe_set_cached_assignment (a row with
        -1 raises device flag 2 and its pairs are dropped);
     2  fallback: a sample whose row holds -1 is routed by its fresh top-k (counted as a
        miss); known samples use their rows; routing waits for the gate;
     3  observe: routing by the fresh top-k (caching off); hit_count is still measured
        against the remembered rows (the metric that switches caching on).
   Every forward then overwrites table[ids[t]] with the fresh top-k after the gate
   (cache_step).  hit_count (stats, metrics) = known samples whose row equals the
   fresh top-k as a set.  An id outside [0, num_samples) raises device flag 4 (row treated as
   unknown).  Not combinable with moe_set_cached_assignment (MOE_ERR_STATE). */
MOE_API moe_status_t moe_set_assignment_cache(moe_handle_t h, int32_t* d_table,
                                              int64_t num_samples, const int64_t* d_sample_ids,
                                              int32_t mode);

/* Forward.  T <= max_tokens (T may be 0).  All pointers device; y is written
   (y[t] = 0 for a token whose every pair was dropped). */
typedef struct {
  int32_t T;
  const void* x;
  const void* w_gate;
  const void* w1;
  const void* b1;
  const void* w2;
  const void* b2;
  void* y;
} moe_fwd_args_t;
MOE_API moe_status_t moe_forward(moe_handle_t h, const moe_fwd_args_t* a);

/* Backward of sum(dy * y) for the last forward (which it consumes: H is overwritten by dA).
   Gradients overwrite their outputs (accumulate = 0) or add to them (accumulate = 1).
   Expert parallelism: dw1 / db1 / dw2 / db2 are the full [n, ...] tensors; this rank writes
   its own experts' slices, and with accumulate = 0 the other experts' slices are zeroed
   (stream-ordered memsets), so the whole tensor is defined.  Any gradient pointer may be NULL to skip writing it, except that the routing / expert
   chain is always computed.  All pointers device, layer dtype. */
typedef struct {
  const void* dy;
  void* dx;
  void* dw_gate;
  void* dw1;
  void* db1;
  void* dw2;
  void* db2;
  int32_t accumulate;
} moe_bwd_args_t;
MOE_API moe_status_t moe_backward(moe_handle_t h, const moe_bwd_args_t* a);

/* Device views of the last forward's routing (valid until the next forward).
   slot_of[t,r] = position of pair (t,r) inside expert idx[t,r]'s buffer, -1 if dropped;
   token_of_slot[base_e + s] = t_g*k + r for s < kept_e (-1 / unwritten beyond);
   base has n+1 entries (host copy, row offsets of each expert's buffer). */
typedef struct {
  const float* logits;        /* [T x n] fp32 gate logits */
  const float* weights;       /* [T x k] fp32 gate weights w (at the dispatch indices) */
  const int32_t* idx;         /* [T x k] dispatch indices (cached ones in cached mode) */
  const int32_t* fresh_idx;   /* [T x k] fresh top-k of this forward's gate */
  const int32_t* slot_of;     /* [T x k] */
  const int32_t* token_of_slot; /* [rows] */
  const int32_t* counts;      /* [n] pre-drop counts (global over the EP group) */
  const int32_t* kept;        /* [n] min(count, C_e) */
  const float* dl;            /* [T x n] fp32 gradient w.r.t. logits (after backward) */
  const float* dw;            /* [T x k] fp32 gradient w.r.t. gate weights (after backward) */
  const void* x_buf;          /* [rows x d] dispatched expert inputs */
  const void* h_buf;          /* [rows x f] ReLU activations (dA after backward) */
  const void* o_buf;          /* [rows x d_out] expert outputs */
  int64_t rows;               /* total buffer rows */
  int32_t base_host[257];     /* host copy of the row offsets, n+1 entries used */
} moe_routing_t;
MOE_API moe_status_t moe_get_routing(moe_handle_t h, moe_routing_t* out);

/* Per-forward statistics, enqueued as async D2H copies into caller memory (pinned for
   true asynchrony).  Valid once the stream has reached this point (event/stream sync).
   counts: host int32 [n]; drops: host int64 [1]; hit_count: host int32 [1] (cached mode,
   else 0).  Any pointer may be NULL. */
typedef struct {
  int32_t* counts;
  int64_t* drops;
  int32_t* hit_count;
} moe_stats_t;
MOE_API moe_status_t moe_get_stats_async(moe_handle_t h, const moe_stats_t* dst);

/* Synchronises the stream and reports (then clears) the device error flags:
   bit 0 = NaN gate logit, bit 1 = invalid cached index, bit 2 = sample id out of range,
   bit 3 = a peer-transport barrier timed out (a rank never arrived within 20 s; the
   iteration's results are invalid).  flags_out may be NULL. */
MOE_API moe_status_t moe_check_device_flags(moe_handle_t h, int32_t* flags_out);

/* ----------------------------------------------------------------------------------- *
 * Loss variants
 * ----------------------------------------------------------------------------------- */
/* Eq. 3 balance term: B = lambda * n * sum_i T_i G_i with T_i = cnt_i/(T_g k)
   (pre-drop counts, held constant in the backward: stop-gradient) and
   G_i = mean_t p[t,i].  lambda = 0 turns it off.  When on, every forward computes B
   (read with moe_get_aux_loss_async into host fp32 [1]) and the next backward adds dB/dl
   = p (g - <p,g>), g_i = lambda n T_i / T_g, to the gate gradient (i.e. the layer's backward
   returns the gradients of sum(dy * y) + B).  In EP the G sums are all-reduced (fp32). */
MOE_API moe_status_t moe_set_balance_loss(moe_handle_t h, float lambda);
MOE_API moe_status_t moe_get_aux_loss_async(moe_handle_t h, float* host_dst);
/* AggregateSpec (App. A): when set, forwards also write spec [T*k x d_out]
   (layer dtype; row t*k + r = the prediction of the r-th chosen expert for token t, zeros if
   the pair was dropped) and valid [T*k] (uint8, 1 = kept).  Device pointers, caller-owned,
   sized for max_tokens; both NULL = off.  Used with the specification loss (Eq. 2). */
MOE_API moe_status_t moe_set_spec_outputs(moe_handle_t h, void* spec, uint8_t* valid);
/* Extra gradients consumed by the next moe_backward: dspec [T*k x d_out] (layer dtype) w.r.t.
   the spec rows (rows of dropped pairs are ignored) and dw_ext [T x k] fp32 w.r.t. the gate
   weights w (e.g. L(y_hat, O_i) of Eq. 2).  Device pointers or NULL; they persist until reset. */
MOE_API moe_status_t moe_set_spec_grads(moe_handle_t h, const void* dspec, const float* dw_ext);

/* ----------------------------------------------------------------------------------- *
 * Recompile runtime pieces
 * ----------------------------------------------------------------------------------- */
/* Model-metric future queue: App. B pushes one future per launched iteration into a queue
   per metric; its length is the number of launched-but-unexecuted iterations and recompile
   triggers run when it equals Delta_launch.  With depth > 0 every moe_forward appends one
   entry (async D2H into pinned memory + an event, no sync); moe_metrics_pop returns the
   oldest entry once the GPU produced it (block = 1 waits for it) and removes it.  A forward
   issued while `depth` entries are pending fails with MOE_ERR_STATE (the caller must pop:
   this bounds the launch frontier).  depth = 0 disables and clears the queue. */
typedef struct {
  int64_t iteration;      /* forward index since moe_metrics_enable */
  int32_t T;              /* tokens of that forward */
  int32_t hit_count;      /* cached mode: rows whose fresh top-k set equals the cached set */
  int64_t drops;          /* pairs dropped by the capacities */
  float aux_loss;         /* Eq. 3 balance term (0 when off) */
  int32_t counts[256];    /* pre-drop per-expert counts (global in EP), n entries used */
} moe_metrics_t;
MOE_API moe_status_t moe_metrics_enable(moe_handle_t h, int32_t depth);
MOE_API moe_status_t moe_metrics_pending(moe_handle_t h, int32_t* n);
MOE_API moe_status_t moe_metrics_pop(moe_handle_t h, int32_t block, moe_metrics_t* out,
                                     int32_t* got);
/* Caching trigger: switch sample-assignment caching on when hit_fraction >=
   enable_at (paper: 0.96), off when it drops below disable_below (0.90), never before epoch
   warmup_epochs (10).  Host only. */
MOE_API moe_status_t moe_caching_trigger(double hit_fraction, int32_t epoch, int32_t enabled,
                                         double enable_at, double disable_below,
                                         int32_t warmup_epochs, int32_t* new_enabled);

/* Expert-parallel exchange plan (host only, no GPU): from the all-gathered pre-drop counts
   cnt_all [R x n] (row r = rank r's tokens) and the global capacities cap [n], fills
   pre_out [R x n]  global slot of rank r's first pair of expert e (= sum of lower ranks),
   kl_out  [R x n]  kept pairs of rank r for expert e (min(cnt, max(0, cap - pre))),
   send_off_out [n] this rank's send-buffer row offset per expert (prefix of kl[rank]),
   kept_local_out [n/R] global kept count of this rank's experts, drops_out [1].
   Rank r sends kl[r][e] rows to owner(e) = e / (n/R); the owner receives them at rows
   base_e + pre[r][e] of expert e's region.  Any output pointer may be NULL. */
MOE_API moe_status_t moe_ep_plan(int32_t R, int32_t rank, int32_t n, const int32_t* cnt_all,
                                 const int32_t* cap, int32_t* pre_out, int32_t* kl_out,
                                 int32_t* send_off_out, int32_t* kept_local_out,
                                 int64_t* drops_out);

/* Virtual communicator for testing the expert-parallel path on ONE GPU: R ranks run as R
   host threads of one process (one handle per thread, moe_config_t.nccl_comm = *comm_out,
   world_size = R, rank = r); exchanges are device-to-device copies with an event rendezvous
   that reproduces NCCL's grouped send/recv matching, all-gather and (fixed rank order)
   all-reduce semantics.  Every rank must issue the same sequence of layer calls. */
MOE_API moe_status_t moe_vcomm_create(int32_t R, void** comm_out);
MOE_API moe_status_t moe_vcomm_destroy(void* comm);

/* ----------------------------------------------------------------------------------- *
 * Peer-memory expert parallelism (the exchange of S8(e) without the host).
 * With cfg.transport = MOE_TRANSPORT_PEER, moe_init allocates (cudaMalloc, library-owned)
 * this rank's peer window: the X / O / dO / dX rows and token_of_slot of its local experts,
 * a count table, fp32 reduction slots and exchange flags.  Before the first forward every
 * rank attaches the windows of all R ranks (same config and window_rows on every rank):
 *   - in one process (R ranks as threads / streams, e.g. on one GPU): moe_peer_window on
 *     each handle, then moe_peer_attach(h, windows[R]) with windows[rank] = its own;
 *   - across processes (one per GPU): moe_peer_export gives a 64-byte CUDA IPC handle; the
 *     caller all-gathers them (any host channel) and calls moe_peer_import(h, handles[R]),
 *     which opens the peers' windows (peer access over NVLink is enabled lazily).
 * The forward / backward then never synchronise the host: dispatch stores token rows into
 * the owners' X buffers, combine reads O rows from them, the combine backward stores dO rows
 * into them and the gate-input gradient reads dX rows from them; the counts, dW_g and the
 * balance sums are exchanged through the windows; one-block barrier kernels order producer
 * and consumer kernels across ranks.  Return rows (bf16 with d and d_out multiples of 128;
 * MOE_PEER_RET=0 disables): the owners' second expert GEMM and dX GEMM store O / dX rows
 * straight into the TOKEN owner's window at row t*k + r from their epilogues, and combine /
 * gate-dx read them locally; with MOE_FUSE_DX (k = 1) the combine backward also pushes each
 * kept pair's dl pair to the owner, whose dX GEMM returns dx rows (dX + dl W_g).  A barrier
 * whose peer never arrives gives up after 20 s and raises device flag bit 3.  Every rank must call moe_forward / moe_backward the
 * same number of times (the barrier epochs advance in lockstep).  Routing, outputs and
 * gradients equal the NCCL path and the single-GPU path on the concatenated batch
 * (reading 12); dW_g is summed in rank order (identical on every rank). */
MOE_API moe_status_t moe_peer_window(moe_handle_t h, void** window, size_t* bytes);
MOE_API moe_status_t moe_peer_export(moe_handle_t h, void* ipc_handle /* host, 64 bytes */);
MOE_API moe_status_t moe_peer_attach(moe_handle_t h, void* const* windows /* host [R] */);
MOE_API moe_status_t moe_peer_import(moe_handle_t h, const void* handles /* host [R][64] */);
/* The same attachment on an NCCL communicator instead of IPC handles (NCCL >= 2.28
   symmetric memory; collective: every rank of the group calls it, in the same order as
   its other collectives on that communicator).  The window is re-allocated with
   ncclMemAlloc, zeroed, registered with ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC),
   and every rank's mapping is taken from the NCCL device API (ncclGetPeerPointer) of the
   load/store-accessible (LSA, NVLink) team.  nccl_comm: the ncclComm_t of the expert-
   parallel group (size world_size, this rank = cfg.rank), e.g. torch's ProcessGroupNCCL
   communicator; it must outlive the handle (moe_destroy deregisters the window on it).
   Errors: MOE_ERR_NCCL if the library lacks the API or not every rank is in the LSA team
   (the handle then keeps its own window: fall back to moe_peer_import), MOE_ERR_STATE if
   already attached, MOE_ERR_INVALID_ARG if the communicator's size / rank differ. */
MOE_API moe_status_t moe_peer_connect_nccl(moe_handle_t h, void* nccl_comm);

/* N2 fusions of the single-GPU tcgen05 path, a bitmask of moe_fusion_t;
   default MOE_FUSE_COMBINE | MOE_FUSE_DX | MOE_FUSE_OTOK (GATHER is opt-in: on B200 the TMA gather4 stream
   is slower than the dispatch copy it replaces).  GATHER and COMBINE give
   bitwise identical results (same products, same accumulation order); DX see below.
   MOE_FUSE_GATHER: the expert GEMMs that read x rows (H = relu(X W1^T + b1) and
     dW1 = dA^T X) load them straight from the caller's x by TMA gather4 through
     token_of_slot, so the dispatch step (GroupBy) writes only the routing tables and
     no X buffer is materialised.  Applies when world_size == 1 (no EP), dtype bf16, d and f
     multiples of 128 and x 16-byte aligned; else the X buffer path runs.  x must stay
     unchanged until moe_backward has been enqueued (already required above).
   MOE_FUSE_COMBINE (k == 1, world_size == 1, bf16, no AggregateSpec outputs, d_out a
     multiple of 128): the second expert GEMM's epilogue writes y[t] = w[t] O[row]
     (Alg. 1 l.8) next to O and the dispatch zeroes the y rows of dropped tokens, so no
     separate combine pass re-reads O.  With cached indices the gate runs concurrently with
     the routing / dispatch / first GEMM and the second GEMM waits for it (its weights).
     Takes effect at the next moe_forward.
   MOE_FUSE_DX (k == 1, world_size == 1, bf16, d a multiple of 128, dx requested): the
     dispatch backward (dx[t] = dX[row] + dl[t] W_g) runs inside the dX = dA W1 GEMM --
     extra k-blocks accumulate [hi|lo](dl) [W_g; W_g] into the same fp32 accumulator and the
     epilogue writes dx rows directly (no dX buffer, no separate pass); tokens whose pair was
     dropped get dx = dl W_g from a small kernel.  NOT bitwise equal to the unfused path (dX
     is no longer rounded to bf16 before the sum -- one rounding instead of two); within the
     bf16 tolerance of the oracle.
   MOE_FUSE_OTOK (world_size == 1, bf16, d_out a multiple of 128): the second expert GEMM's
     epilogue stores O in (token, choice) order -- row t k + r of the O buffer -- instead of
     expert-region order, so the combine and the combine backward read a token's O rows
     without first resolving its routing slots (the row loads issue together with the
     routing-table loads).  Bitwise equal to the expert-order layout; moe_get_routing's o_buf
     is then [T k x d_out] in token order.
   MOE_FUSE_COMBINE2 (k == 2, with MOE_FUSE_OTOK in effect, no AggregateSpec outputs): the
     combine moves into the second GEMM's epilogue as well -- per (token, column block) a
     counter elects the epilogue that stores its O row second (or alone, when the other
     pair was dropped) to read both stored rows back and write y = w0 O0 + w1 O1 (the
     combine kernel's arithmetic, bitwise equal); the counters live in the workspace and
     reset themselves.  Opt-in (see DESIGN.md §10b for the byte count and measurement).
   MOE_FUSE_CDISP (cached assignments, world_size == 1, bf16, d a multiple of 64): with the
     dispatch indices known before the gate (sample-assignment caching), the
     dispatch (A4) runs inside the gate kernel: its spare warps compute the slots of each
     128-token tile from the cached rows and copy every x k-block from the gate's TMA stage
     to the kept X_buf rows, so x is read once for the gate GEMM and the dispatch; the whole
     forward then stays on the caller's stream (no side-stream fork / join).  Bitwise equal
     to the unfused cached path (same routing tables, same copied rows).  Opt-in: measured
     no faster than the default cached path, where the gate overlaps the routing chain on a
     side stream. */
typedef enum { MOE_FUSE_GATHER = 1, MOE_FUSE_COMBINE = 2, MOE_FUSE_DX = 4,
               MOE_FUSE_OTOK = 8, MOE_FUSE_COMBINE2 = 16, MOE_FUSE_CDISP = 32 } moe_fusion_t;
MOE_API moe_status_t moe_set_fusion(moe_handle_t h, int32_t flags);

/* Number of kernels the library launched since the handle was created (for bench
   accounting of "our kernels in the timed region"). */
MOE_API moe_status_t moe_launch_count(moe_handle_t h, int64_t* out);

/* Per-kernel timing (for the benchmark's roofline): when enabled, every kernel launch is
   bracketed by CUDA events on its stream.  moe_profile_read synchronises, then fills up to
   max entries {name, launches, total_ms} aggregated per kernel name since the last reset. */
typedef struct {
  char name[32];
  int64_t launches;
  double total_ms;
} moe_kernel_time_t;
MOE_API moe_status_t moe_profile_enable(moe_handle_t h, int32_t on);
MOE_API moe_status_t moe_profile_read(moe_handle_t h, moe_kernel_time_t* out, int32_t max,
                                      int32_t* count, int32_t reset);

/* Human-readable description of the last error on this handle (never NULL); with h == NULL,
   why the last moe_init on the calling thread failed (e.g. the peer window allocation). */
MOE_API const char* moe_last_error(moe_handle_t h);

/* ----------------------------------------------------------------------------------- *
 * Dynamic capacity policy (host helper, R1).  The paper leaves the policy open
 * (P:236); this is SPEC's peak-plus-headroom rule: for each
 * expert, peak = max count over the last `window` iterations; grow at once to
 * ceil((1+headroom)*peak) when C_e < peak; shrink to that target only after a full window
 * whose mean count / C_e < shrink_util; alpha_e = C_e*n/(T_g*k) clamped to
 * [min_alpha, max_alpha] and C_e recomputed by Eq. 4.
 * ----------------------------------------------------------------------------------- */
typedef struct moe_policy* moe_policy_t;
typedef struct {
  int32_t n_experts, top_k;
  int64_t tokens_global;
  int32_t window;        /* default 20 */
  double headroom;       /* default 0.15 */
  double shrink_util;    /* default 0.5 */
  double min_alpha;      /* default 0.25 */
  double max_alpha;      /* default 8.0 */
} moe_policy_config_t;
MOE_API moe_status_t moe_policy_create(const moe_policy_config_t* cfg, const int32_t* init_cap,
                               moe_policy_t* out);
/* counts: host [n] observed pre-drop counts of one iteration.  *changed = 1 and
   new_cap (host [n]) filled when a recompile is due, else *changed = 0. */
MOE_API moe_status_t moe_policy_update(moe_policy_t p, const int32_t* counts, int32_t* new_cap,
                               int32_t* changed);
MOE_API moe_status_t moe_policy_destroy(moe_policy_t p);

#ifdef __cplusplus
}
#endif
#endif /* DYNAMOE_B200_MOE_H */
