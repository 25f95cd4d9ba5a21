"""Thin PyTorch binding of the C ABI (include/moe.h): argument marshalling only.

Torch supplies device memory (the workspace and outputs), the current CUDA stream and
process groups; every step of the MoE hot path runs in libdynamoe_b200.so.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L

_TORCH_DT = {"f32": torch.float32, "bf16": torch.bfloat16}


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def capacity_from_factors(alphas, tokens_global: int, k: int):
    """Eq. 4 through the library: max(1, ceil(alpha_e * T_g * k / n))."""
    lib = L.load()
    n = len(alphas)
    a = (C.c_double * n)(*[float(v) for v in alphas])
    out = (C.c_int32 * n)()
    L.check(lib.moe_capacity_from_factors(n, int(tokens_global), int(k), a, out))
    return list(out)


class MoELayer:
    """One DynaMoE MoE layer (Alg. 1 with capacity) on one GPU
    (or one expert-parallel rank).  Parameters are passed per call (torch Linear layout)."""

    def __init__(self, n_experts: int, top_k: int, d_model: int, d_ff: int, d_out: int = 0,
                 max_tokens: int = 4096, dtype: str = "bf16", renormalize: int = 1,
                 world_size: int = 1, rank: int = 0, nccl_comm: int = 0, device=None,
                 transport: str = "nccl", window_rows: int = 0):
        self.lib = L.load()
        dev = torch.device(device if device is not None else "cuda")
        if dev.type != "cuda":
            raise RuntimeError("MoELayer runs only on CUDA devices (no CPU fallback)")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.n, self.k, self.d, self.f = n_experts, top_k, d_model, d_ff
        self.d_out = d_out or d_model
        self.max_tokens = max_tokens
        self.dtype = dtype
        self.tdtype = _TORCH_DT[dtype]
        self.world_size, self.rank = world_size, rank
        import os
        # bf16 layers run the expert FFN and gate contractions on tcgen05 tensor cores
        self.uses_tcgen05 = dtype == "bf16" and os.environ.get("MOE_FORCE_SIMT", "0") != "1"
        # fp32: expert GEMMs on tcgen05 kind::tf32 with split operands (gemm_tf32.cu)
        self.uses_tf32 = (dtype == "f32" and os.environ.get("MOE_FORCE_SIMT", "0") != "1"
                          and d_model % 32 == 0 and d_ff % 32 == 0 and (d_out or d_model) % 32 == 0)
        cfg = L.MoEConfig(n_experts, top_k, d_model, d_ff, d_out, max_tokens, L.DTYPES[dtype],
                          int(renormalize), world_size, rank, C.c_void_p(nccl_comm),
                          C.c_void_p(self._stream()), L.TRANSPORTS[transport], 0,
                          int(window_rows))
        self.transport = transport
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            L.check(self.lib.moe_init(C.byref(cfg), C.byref(h)), None, "moe_init")
        self.h = h
        self.layout_generation = 0   # bumped by every recompile (capacity change)
        # bumped by every call that changes arguments a captured CUDA graph has baked in
        # (capacities, cached indices, assignment cache, fusion, loss variants)
        self.generation = 0
        self._saved = None
        self._fwd_id = 0             # forward counter: a backward must follow its own forward
        self.ws = None
        self._cached_ref = None
        self._alloc_workspace()
        self._pinned = None

    # -- plumbing -------------------------------------------------------------------
    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def _sync_stream(self):
        L.check(self.lib.moe_set_stream(self.h, C.c_void_p(self._stream())), self.h)

    def _alloc_workspace(self):
        sz = C.c_size_t()
        L.check(self.lib.moe_workspace_size(self.h, C.byref(sz)), self.h)
        if self.ws is None or self.ws.numel() < sz.value:
            self.ws = torch.empty(max(sz.value, 256), dtype=torch.uint8, device=self.device)
        self._sync_stream()
        L.check(self.lib.moe_set_workspace(self.h, _ptr(self.ws), self.ws.numel()), self.h,
                "moe_set_workspace")

    def close(self):
        if getattr(self, "h", None):
            self.lib.moe_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- peer-memory expert parallelism (N1) -------------------------------------------
    def peer_window(self) -> int:
        """Device address of this rank's library-owned peer window."""
        w = C.c_void_p()
        L.check(self.lib.moe_peer_window(self.h, C.byref(w), None), self.h)
        return w.value

    def peer_export(self) -> bytes:
        """64-byte CUDA IPC handle of the peer window (for other processes)."""
        buf = C.create_string_buffer(64)
        L.check(self.lib.moe_peer_export(self.h, buf), self.h)
        return buf.raw

    def peer_attach(self, windows):
        """In-process ranks: every rank's window address (own one at index rank)."""
        arr = (C.c_void_p * len(windows))(*windows)
        L.check(self.lib.moe_peer_attach(self.h, arr), self.h, "moe_peer_attach")

    def peer_connect_nccl(self, nccl_comm: int):
        """Cross-process ranks over an NCCL communicator (collective): the window becomes
        NCCL symmetric memory and the peers' mappings come from the NCCL device API."""
        L.check(self.lib.moe_peer_connect_nccl(self.h, C.c_void_p(nccl_comm)), self.h,
                "moe_peer_connect_nccl")
        self.peer_via = "nccl-symmetric-window"

    def peer_import(self, handles):
        """Cross-process ranks: all ranks' IPC handles (list of 64-byte strings)."""
        buf = C.create_string_buffer(b"".join(handles), 64 * len(handles))
        L.check(self.lib.moe_peer_import(self.h, buf), self.h, "moe_peer_import")
        self.peer_via = "cuda-ipc"

    # -- recompile-enabled optimisations ----------------------------------------------
    @property
    def capacities(self):
        out = (C.c_int32 * self.n)()
        L.check(self.lib.moe_get_capacities(self.h, out), self.h)
        return list(out)

    def set_capacities(self, caps):
        """Dynamic capacity factors (S4.1): new per-expert capacities, stream-ordered."""
        arr = (C.c_int32 * self.n)(*[int(c) for c in caps])
        st = self.lib.moe_set_capacities(self.h, arr)
        if st == L.MOE_ERR_WORKSPACE_TOO_SMALL:   # recorded; the layout needs a bigger block
            self._alloc_workspace()
        else:
            L.check(st, self.h, "moe_set_capacities")
            self._sync_stream()
        want = [min(int(c), max(1, self.max_tokens * self.world_size)) for c in caps]
        if self.capacities != want:
            raise RuntimeError(f"moe_set_capacities did not take effect: {self.capacities}")
        self.layout_generation += 1
        self.generation += 1

    def set_capacity_factors(self, alphas, tokens_global=None):
        tg = tokens_global if tokens_global is not None else self.max_tokens * self.world_size
        self.set_capacities(capacity_from_factors(alphas, tg, self.k))

    def set_cached_assignment(self, idx):
        """Sample-assignment caching (S4.2): int32 [T,k] device indices, or None (off)."""
        if idx is not None:
            if idx.dtype != torch.int32 or not idx.is_cuda or not idx.is_contiguous():
                raise ValueError("cached indices must be a contiguous int32 CUDA tensor")
        L.check(self.lib.moe_set_cached_assignment(self.h, _ptr(idx)), self.h)
        self._cached_ref = idx
        self.generation += 1

    def set_assignment_cache(self, table, sample_ids, mode: int):
        """Per-sample assignment cache (N4): table int32 [num_samples, k] (device, -1 =
        unknown), sample_ids int64 [T] (device) of the next forwards; mode 0 off, 1 all
        samples known (overlap with the gate), 2 unknown samples fall back to the gate."""
        if mode:
            if table.dtype != torch.int32 or not table.is_cuda or not table.is_contiguous():
                raise ValueError("table must be a contiguous int32 CUDA tensor")
            if sample_ids.dtype != torch.int64 or not sample_ids.is_cuda:
                raise ValueError("sample_ids must be an int64 CUDA tensor")
            self._ctab_ref = (table, sample_ids)
            L.check(self.lib.moe_set_assignment_cache(self.h, _ptr(table), table.shape[0],
                                                      _ptr(sample_ids), int(mode)), self.h)
        else:
            self._ctab_ref = None
            L.check(self.lib.moe_set_assignment_cache(self.h, None, 0, None, 0), self.h)
        self.generation += 1

    # -- N2 fusions ---------------------------------------------------------------------
    FUSE_GATHER, FUSE_COMBINE, FUSE_DX, FUSE_OTOK, FUSE_COMBINE2, FUSE_CDISP = 1, 2, 4, 8, 16, 32

    def set_fusion(self, flags: int):
        """moe_set_fusion: bitmask of FUSE_GATHER (x rows gathered by the expert GEMMs, no X
        buffer), FUSE_COMBINE (k = 1: y written by the second GEMM's epilogue) and FUSE_DX
        (k = 1: dx = dX + dl W_g written by the dX GEMM) and FUSE_OTOK (O stored in (token,
        choice) order for the combine and its backward), FUSE_COMBINE2 (k = 2: the combine in the
        second GEMM's epilogue too, opt-in), FUSE_CDISP (cached assignments: the dispatch inside
        the gate kernel, opt-in).  Default COMBINE | DX | OTOK."""
        L.check(self.lib.moe_set_fusion(self.h, int(flags)), self.h)
        self.generation += 1

    # -- loss variants (N3) -----------------------------------------------------------
    def set_balance_loss(self, lam: float):
        """Eq. 3 balance term weight (0 = off); the backward then includes dB/dl."""
        L.check(self.lib.moe_set_balance_loss(self.h, float(lam)), self.h)
        self._lam = float(lam)
        self.generation += 1

    def aux_loss(self) -> float:
        """B of the last forward (synchronises)."""
        v = C.c_float()
        self._sync_stream()
        L.check(self.lib.moe_get_aux_loss_async(self.h, C.byref(v)), self.h)
        torch.cuda.current_stream(self.device).synchronize()
        return float(v.value)

    def enable_spec(self, on: bool = True):
        """AggregateSpec outputs for the following forwards (self.spec, self.spec_valid)."""
        if on:
            self.spec = torch.empty(self.max_tokens * self.k, self.d_out, dtype=self.tdtype,
                                    device=self.device)
            self.spec_valid = torch.empty(self.max_tokens * self.k, dtype=torch.uint8,
                                          device=self.device)
            L.check(self.lib.moe_set_spec_outputs(self.h, _ptr(self.spec), _ptr(self.spec_valid)),
                    self.h)
        else:
            self.spec = self.spec_valid = None
            L.check(self.lib.moe_set_spec_outputs(self.h, None, None), self.h)
        self.generation += 1

    def set_spec_grads(self, dspec=None, dw_ext=None):
        """Gradients w.r.t. the spec rows ([T*k, d_out], layer dtype) and the gate weights
        ([T, k] fp32) consumed by the following backwards (None = none)."""
        self._spec_grads = (dspec, dw_ext)
        L.check(self.lib.moe_set_spec_grads(self.h, _ptr(dspec), _ptr(dw_ext)), self.h)
        self.generation += 1

    # -- hot path -------------------------------------------------------------------
    def _check(self, t, shape, name):
        if t.dtype != self.tdtype or tuple(t.shape) != tuple(shape) or not t.is_contiguous() \
                or t.device != self.device:
            raise ValueError(f"{name}: expected contiguous {self.tdtype} {tuple(shape)} on "
                             f"{self.device}, got {t.dtype} {tuple(t.shape)} on {t.device}")

    def forward(self, x, w_gate, w1, b1, w2, b2, y=None):
        T = x.shape[0]
        n, d, f, do = self.n, self.d, self.f, self.d_out
        self._check(x, (T, d), "x")
        self._check(w_gate, (n, d), "w_gate")
        self._check(w1, (n, f, d), "w1")
        self._check(b1, (n, f), "b1")
        self._check(w2, (n, do, f), "w2")
        self._check(b2, (n, do), "b2")
        if y is None:
            y = torch.empty(T, do, dtype=self.tdtype, device=self.device)
        self._sync_stream()
        a = L.FwdArgs(T, _ptr(x), _ptr(w_gate), _ptr(w1), _ptr(b1), _ptr(w2), _ptr(b2), _ptr(y))
        L.check(self.lib.moe_forward(self.h, C.byref(a)), self.h, "moe_forward")
        self._saved = (x, w_gate, w1, b1, w2, b2)   # keep alive until backward (moe.h)
        self._fwd_id += 1
        return y

    def backward(self, dy, grads=None, accumulate=False, need=("dx", "dw_gate", "dw1", "db1",
                                                               "dw2", "db2"), fwd_id=None):
        """Gradients of the LAST forward (the library keeps one saved forward).  fwd_id: the
        value of `self._fwd_id` right after the forward these gradients belong to; a
        mismatch (another forward ran in between) raises instead of mixing batches."""
        if fwd_id is not None and fwd_id != self._fwd_id:
            raise RuntimeError("MoELayer.backward: another forward ran since the forward this "
                               "backward belongs to (the layer saves only the last one)")
        if self._saved is None:
            raise RuntimeError("MoELayer.backward: no saved forward (backward called twice?)")
        x, w_gate, w1, b1, w2, b2 = self._saved
        T = x.shape[0]
        self._check(dy, (T, self.d_out), "dy")
        if grads is None:
            # (EP: the library zeroes the other ranks' expert slices itself, moe.h)
            alloc = torch.zeros if accumulate else torch.empty
            shapes = dict(dx=x.shape, dw_gate=w_gate.shape, dw1=w1.shape, db1=b1.shape,
                          dw2=w2.shape, db2=b2.shape)
            grads = {k: alloc(shapes[k], dtype=self.tdtype, device=self.device) for k in need}
        g = lambda k: _ptr(grads.get(k))  # noqa: E731
        self._sync_stream()
        a = L.BwdArgs(_ptr(dy), g("dx"), g("dw_gate"), g("dw1"), g("db1"), g("dw2"), g("db2"),
                      int(bool(accumulate)))
        L.check(self.lib.moe_backward(self.h, C.byref(a)), self.h, "moe_backward")
        self._saved = None
        return grads

    # -- introspection ----------------------------------------------------------------
    def routing(self, T):
        """Copies of the last forward's routing tables (device tensors)."""
        r = L.Routing()
        L.check(self.lib.moe_get_routing(self.h, C.byref(r)), self.h)
        base = self.ws.data_ptr()

        ws_end = base + self.ws.numel()

        def view(ptr, count, dt):
            nbytes = count * torch.tensor([], dtype=dt).element_size()
            if base <= ptr < ws_end:
                off = ptr - base
                return self.ws[off:off + nbytes].view(dt).clone()
            # peer transport: the expert-major buffers live in the library's peer window
            out = torch.empty(count, dtype=dt, device=self.device)
            torch.cuda.synchronize(self.device)
            if nbytes:
                rt = C.CDLL("libcudart.so.12")
                rc = rt.cudaMemcpy(C.c_void_p(out.data_ptr()), C.c_void_p(ptr),
                                   C.c_size_t(nbytes), 4)  # cudaMemcpyDefault
                if rc != 0:
                    raise RuntimeError(f"cudaMemcpy failed ({rc})")
            return out

        n, k = self.n, self.k
        out = dict(
            logits=view(r.logits, T * n, torch.float32).view(T, n),
            w=view(r.weights, T * k, torch.float32).view(T, k),
            idx=view(r.idx, T * k, torch.int32).view(T, k),
            fresh_idx=view(r.fresh_idx, T * k, torch.int32).view(T, k),
            slot_of=view(r.slot_of, T * k, torch.int32).view(T, k),
            counts=view(r.counts, n, torch.int32),
            kept=view(r.kept, n, torch.int32),
            dl=view(r.dl, T * n, torch.float32).view(T, n),
            dw=view(r.dw, T * k, torch.float32).view(T, k),
            token_of_slot=view(r.token_of_slot, r.rows, torch.int32),
            rows=r.rows,
            base=list(r.base_host)[: n // self.world_size + 1],
        )
        out["x_buf"] = view(r.x_buf, r.rows * self.d, self.tdtype).view(r.rows, self.d)
        out["h_buf"] = view(r.h_buf, r.rows * self.f, self.tdtype).view(r.rows, self.f)
        out["o_buf"] = view(r.o_buf, r.rows * self.d_out, self.tdtype).view(r.rows, self.d_out)
        return out

    def h_snapshot(self):
        """Copy of the H buffer (ReLU outputs of the last forward, expert-region rows of the local
        experts) and the region bases, enqueued on the current stream without any device or
        stream synchronisation (safe between a forward and its backward while peer ranks of
        the same GPU wait in barrier kernels).  Test helper: the backward overwrites H."""
        r = L.Routing()
        L.check(self.lib.moe_get_routing(self.h, C.byref(r)), self.h)
        off = r.h_buf - self.ws.data_ptr()
        nbytes = r.rows * self.f * self.ws.new_empty(0, dtype=self.tdtype).element_size()
        h = self.ws[off:off + nbytes].view(self.tdtype).view(r.rows, self.f).clone()
        return h, list(r.base_host)[: self.n // self.world_size + 1]

    def stats(self):
        """Per-forward statistics (synchronises the stream): counts, drops, hit_count."""
        if self._pinned is None:
            self._pinned = (torch.zeros(self.n, dtype=torch.int32).pin_memory(),
                            torch.zeros(1, dtype=torch.int64).pin_memory(),
                            torch.zeros(1, dtype=torch.int32).pin_memory())
        c, dr, hit = self._pinned
        self._sync_stream()
        s = L.Stats(_ptr(c), _ptr(dr), _ptr(hit))
        L.check(self.lib.moe_get_stats_async(self.h, C.byref(s)), self.h)
        torch.cuda.current_stream(self.device).synchronize()
        return dict(counts=c.tolist(), drops=int(dr.item()), hit_count=int(hit.item()))

    def check_flags(self):
        fl = C.c_int32()
        self._sync_stream()
        st = self.lib.moe_check_device_flags(self.h, C.byref(fl))
        return st, fl.value

    def profile(self, on: bool):
        L.check(self.lib.moe_profile_enable(self.h, int(bool(on))), self.h)

    def profile_read(self, reset=True):
        """{kernel name: (launches, total_ms)} since the last reset (synchronises)."""
        buf = (L.KernelTime * 64)()
        cnt = C.c_int32()
        L.check(self.lib.moe_profile_read(self.h, buf, 64, C.byref(cnt), int(reset)), self.h)
        return {buf[i].name.decode(): (buf[i].launches, buf[i].total_ms) for i in range(cnt.value)}

    def metrics_queue(self, depth: int):
        from .runtime import MetricQueue
        return MetricQueue(self, depth)

    def launch_count(self):
        v = C.c_int64()
        L.check(self.lib.moe_launch_count(self.h, C.byref(v)), self.h)
        return v.value


class CapacityPolicy:
    """Host helper of the dynamic capacity policy in the library (moe_policy_*)."""

    def __init__(self, n, tokens_global, k, capacities, window=20, headroom=0.15,
                 shrink_util=0.5, min_alpha=0.25, max_alpha=8.0):
        self.lib = L.load()
        self.n = n
        cfg = L.PolicyConfig(n, k, tokens_global, window, headroom, shrink_util, min_alpha,
                             max_alpha)
        init = (C.c_int32 * n)(*[int(c) for c in capacities])
        p = C.c_void_p()
        L.check(self.lib.moe_policy_create(C.byref(cfg), init, C.byref(p)))
        self.p = p

    def update(self, counts):
        cin = (C.c_int32 * self.n)(*[int(c) for c in counts])
        cout = (C.c_int32 * self.n)()
        ch = C.c_int32()
        L.check(self.lib.moe_policy_update(self.p, cin, cout, C.byref(ch)))
        return list(cout) if ch.value else None

    def __del__(self):
        try:
            self.lib.moe_policy_destroy(self.p)
        except Exception:
            pass


class MoEFunction(torch.autograd.Function):
    """autograd wrapper: y = MoE(x; W_g, W1, b1, W2, b2) through the C ABI."""

    @staticmethod
    def forward(ctx, layer, x, w_gate, w1, b1, w2, b2):
        ctx.layer = layer
        y = layer.forward(x, w_gate, w1, b1, w2, b2)
        ctx.fwd_id = layer._fwd_id
        return y

    @staticmethod
    def backward(ctx, dy):
        g = ctx.layer.backward(dy.contiguous(), fwd_id=ctx.fwd_id)
        return None, g["dx"], g["dw_gate"], g["dw1"], g["db1"], g["dw2"], g["db2"]


class DynaMoE(torch.nn.Module):
    """nn.Module holding the gate and expert parameters (torch Linear layout)."""

    def __init__(self, n_experts, top_k, d_model, d_ff, d_out=0, max_tokens=4096,
                 dtype="bf16", renormalize=1, device=None):
        super().__init__()
        self.layer = MoELayer(n_experts, top_k, d_model, d_ff, d_out, max_tokens, dtype,
                              renormalize, device=device)
        dev, dt = self.layer.device, self.layer.tdtype
        do = d_out or d_model
        self.w_gate = torch.nn.Parameter(torch.randn(n_experts, d_model, device=dev) * d_model ** -0.5)
        self.w1 = torch.nn.Parameter(torch.randn(n_experts, d_ff, d_model, device=dev) * d_model ** -0.5)
        self.b1 = torch.nn.Parameter(torch.zeros(n_experts, d_ff, device=dev))
        self.w2 = torch.nn.Parameter(torch.randn(n_experts, do, d_ff, device=dev) * d_ff ** -0.5)
        self.b2 = torch.nn.Parameter(torch.zeros(n_experts, do, device=dev))
        for p in self.parameters():
            p.data = p.data.to(dt)

    def forward(self, x):
        return MoEFunction.apply(self.layer, x.contiguous(), self.w_gate, self.w1, self.b1,
                                 self.w2, self.b2)
