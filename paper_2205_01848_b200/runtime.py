"""Recompile runtime around one MoE layer (PAPER App. B).

* The model-metric future queue lives in the C library (moe_metrics_*): every forward pushes
  its routing statistics asynchronously; the queue length is the number of launched but not
  yet consumed iterations.
* RecompileRuntime keeps that length at Delta_launch: after each launch it pops the oldest
  metric (waiting for the GPU only when the queue is longer than Delta_launch), runs the
  user's triggers on the CPU while the GPU keeps executing the already-launched iterations,
  and applies their decisions at the launch frontier (the next launched iteration) -- the
  paper's "graph adjustments take effect at the launch frontier".
* GraphedStep captures one forward+backward of the layer into a CUDA graph; a capacity change
  (a recompile) re-instantiates it, exactly the paper's recompile of a static graph.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L


def caching_trigger(hit_fraction, epoch, enabled, enable_at=0.96, disable_below=0.90,
                    warmup_epochs=10) -> bool:
    """P:353 switching rule (library host helper)."""
    out = C.c_int32()
    L.check(L.load().moe_caching_trigger(float(hit_fraction), int(epoch), int(bool(enabled)),
                                         float(enable_at), float(disable_below),
                                         int(warmup_epochs), C.byref(out)))
    return bool(out.value)


class AssignmentCache:
    """Per-sample assignment cache of one layer (N4; S4.2 P:245-256).

    The table lives on the device (int32 [num_samples, k], -1 = unknown) and is read and
    updated by the library's kernels; the host only tracks WHICH ids have been seen, so it
    can pick the library mode for a batch without a device sync:
      caching off  -> mode 3 (observe: fresh routing, hit metric, remember);
      caching on, every id seen -> mode 1 (cached routing overlaps the gate);
      caching on, some id unseen -> mode 2 (unknown samples fall back to the gate).
    `enabled` is switched by the caching trigger from the per-iteration hit metric."""

    def __init__(self, layer, num_samples: int):
        import numpy as np
        self.layer = layer
        self.table = torch.full((num_samples, layer.k), -1, dtype=torch.int32, device=layer.device)
        self.seen = np.zeros(num_samples, dtype=bool)
        self.ids = torch.empty(max(1, layer.max_tokens), dtype=torch.int64, device=layer.device)
        self.enabled = False
        self.last_mode = 0

    def bind(self, sample_ids):
        """Set the sample ids (host sequence / CPU tensor, distinct) of the next forward."""
        import numpy as np
        ids = np.asarray(sample_ids, dtype=np.int64)
        T = ids.shape[0]
        self.ids[:T].copy_(torch.from_numpy(ids))   # pageable source: host-synchronous copy
        if not self.enabled:
            mode = 3
        elif self.seen[ids].all():
            mode = 1
        else:
            mode = 2
        self.layer.set_assignment_cache(self.table, self.ids, mode)
        self.seen[ids] = True
        self.last_mode = mode
        return mode

    def unbind(self):
        self.layer.set_assignment_cache(None, None, 0)


class MetricQueue:
    """Python view of the library's per-iteration metric queue of one layer."""

    def __init__(self, layer, depth: int):
        self.layer = layer
        self.lib = layer.lib
        L.check(self.lib.moe_metrics_enable(layer.h, int(depth)), layer.h)
        self.depth = depth

    def pending(self) -> int:
        n = C.c_int32()
        L.check(self.lib.moe_metrics_pending(self.layer.h, C.byref(n)), self.layer.h)
        return n.value

    def pop(self, block: bool = True):
        m = L.Metrics()
        got = C.c_int32()
        L.check(self.lib.moe_metrics_pop(self.layer.h, int(block), C.byref(m), C.byref(got)),
                self.layer.h)
        if not got.value:
            return None
        return dict(iteration=m.iteration, T=m.T, hit_count=m.hit_count, drops=m.drops,
                    aux_loss=m.aux_loss, counts=list(m.counts[: self.layer.n]))


class RecompileRuntime:
    """Delta_launch-delayed triggers over one layer's metric queue (App. B).

    triggers: callables f(metrics, runtime) returning None or a dict with optional keys
    'capacities' (list) and 'cached' (tensor or None); decisions apply to the next launch."""

    def __init__(self, layer, delta_launch: int = 1, triggers=()):
        self.layer = layer
        self.delta = int(delta_launch)
        self.queue = MetricQueue(layer, self.delta + 1)
        self.triggers = list(triggers)
        self.log = []            # (metric iteration, launch iteration it takes effect at, decision)
        self.launched = 0

    def before_launch(self):
        """Make room in the queue (the launch frontier may run Delta_launch ahead)."""
        while self.queue.pending() > self.delta:
            self._consume(self.queue.pop(block=True))

    def after_launch(self):
        self.launched += 1
        while self.queue.pending() > self.delta:
            self._consume(self.queue.pop(block=True))

    def _consume(self, m):
        for trig in self.triggers:
            dec = trig(m, self)
            if not dec:
                continue
            if "capacities" in dec:
                self.layer.set_capacities(dec["capacities"])
            if "cached" in dec:
                self.layer.set_cached_assignment(dec["cached"])
            self.log.append((m["iteration"], self.launched, dec))

    def drain(self):
        while self.queue.pending():
            self._consume(self.queue.pop(block=True))


def capacity_trigger(policy):
    """Adapter: the library's dynamic-capacity policy (moe_policy_*) as a runtime trigger."""
    def trig(m, rt):
        new = policy.update(m["counts"])
        return {"capacities": new} if new is not None else None
    return trig


class GraphedStep:
    """forward + backward of a layer captured into one CUDA graph over static tensors.

    A recompile (capacities changed), like any other setter that changes kernel arguments
    (cached indices, assignment cache, fusion flags, loss variants), invalidates the captured
    arguments; `replay()` re-captures when `layer.generation` changed.  The tensors the
    captured arguments point at (cached indices, cache table, spec gradients) are kept
    alive by the capture itself, so a replay never reads memory Python has released."""

    def __init__(self, layer, x, params, dy, grads, y=None):
        self.layer = layer
        self.x, self.params, self.dy, self.grads = x, params, dy, grads
        self.y = y if y is not None else torch.empty(x.shape[0], layer.d_out, dtype=layer.tdtype,
                                                     device=layer.device)
        self.graph = None
        self.gen = None
        self.recapture()

    def _body(self):
        p = self.params
        self.layer.forward(self.x, p["w_gate"], p["w1"], p["b1"], p["w2"], p["b2"], y=self.y)
        self.layer.backward(self.dy, grads=self.grads)

    def recapture(self):
        s = torch.cuda.Stream(self.layer.device)
        s.wait_stream(torch.cuda.current_stream(self.layer.device))
        with torch.cuda.stream(s):
            self._body()                   # warm-up outside capture (attributes, maps)
        torch.cuda.current_stream(self.layer.device).wait_stream(s)
        torch.cuda.synchronize(self.layer.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._body()
        self.graph = g
        self.gen = self.layer.generation
        L = self.layer
        self._pinned_args = (getattr(L, "_cached_ref", None), getattr(L, "_ctab_ref", None),
                             getattr(L, "_spec_grads", None), getattr(L, "spec", None))

    def replay(self):
        if self.gen != self.layer.generation:
            self.recapture()
        self.graph.replay()
        return self.y
