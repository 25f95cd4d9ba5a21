#!/usr/bin/env python
"""Benchmark of the DynaMoE MoE-layer hot path on B200 (driver contract).

A step = one forward + backward of the MoE layer (gate GEMM, softmax/top-k, capacity-bounded
dispatch, expert FFN grouped GEMMs, combine, and every backward incl. weight gradients) over
one batch of synthetic tokens.  Workload at N = 1: BASELINE configs[2] (c3) -- 64 experts,
top-1, d_model 1024, d_ff 4096, 65,536 tokens, bf16, capacity factor 1.0 (the largest config
BASELINE names for one GPU).  At N > 1 (torchrun): BASELINE configs[3] (c4) strong scaling
-- 128 experts, top-2, d_model 2048, d_ff 8192, 262,144 global tokens split over the N ranks,
experts sharded (expert parallelism); `--config c3` / `--config c5` give the weak-scaling
variants (65,536 tokens per GPU), `--config c4` at N = 1 the strong-scaling anchor.  Inputs
exceed the 126 MB L2, so no explicit flush is needed between steps; configs whose inputs
fit the L2 (c1, c2) write 2x the L2 before every timed step and time the steps alone.

Recompile mode (the paper's dynamic-capacity claim): `--regime skewed --capacity
dynamic` runs the capacity policy (reading 14) for `--policy-warmup` steps before timing;
`--capacity static --alpha 7.0` is the paper's static setting.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer fwd+bwd tokens/sec at 1/2/4/8 B200; dispatch/combine HBM GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None,
                    help="c3 at N = 1, c4 (strong scaling) at N > 1 unless given")
    ap.add_argument("--tokens", type=int, default=0, help="override tokens per rank")
    ap.add_argument("--alpha", type=float, default=None, help="static capacity factor")
    ap.add_argument("--cached", action="store_true", help="sample-assignment caching (c5)")
    ap.add_argument("--regime", choices=["uniform", "skewed"], default="uniform",
                    help="routing regime of the synthetic inputs (SURVEY §8(d))")
    ap.add_argument("--capacity", choices=["static", "dynamic"], default=None,
                    help="dynamic: the capacity policy (moe_policy_*) adapts C_e for "
                         "--policy-warmup steps before the timed region (P:221-236)")
    ap.add_argument("--policy-warmup", type=int, default=50)
    ap.add_argument("--emulate-padded", action="store_true",
                    help="TIMING ONLY: expert GEMMs over all C_e rows (MOE_DBG_PAD_GEMM=1), "
                         "what a capacity-padded implementation (the paper's FlexFlow "
                         "operators, P:234, P:370) spends; outputs are not valid")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=8192)
    ap.add_argument("--graph", action="store_true",
                    help="also time the step replayed from a CUDA graph (reported as graph_*)")
    ap.add_argument("--ep", action="store_true",
                    help="force the expert-parallel path at N=1 (loopback)")
    ap.add_argument("--transport", choices=["peer", "nccl"], default="peer",
                    help="expert-parallel exchange: peer = device-initiated through peer "
                         "memory over NVLink (N1, default); nccl = grouped send/recv")
    ap.add_argument("--fusion", choices=["none", "combine", "dx", "otok", "legacy", "default",
                                         "combine2", "all", "cdisp"],
                    default="default",
                    help="N2 fusions (k = 1): combine = y written by the second expert GEMM's "
                         "epilogue; dx = dispatch backward inside the dX GEMM; default = combine+dx+otok; "
                         "otok = O stored in (token, choice) order; legacy = combine+dx; "
                         "combine2 = default + the k = 2 combine in the second GEMM's epilogue; "
                         "all = also gather x rows in the expert GEMMs (TMA gather4); "
                         "cdisp = default + (cached mode) the dispatch inside the gate kernel "
                         "(x read once)")
    a = ap.parse_args()
    if a.emulate_padded:
        os.environ["MOE_DBG_PAD_GEMM"] = "1"
    if a.config is None:
        a.config = "c3" if int(os.environ.get("WORLD_SIZE", "1")) == 1 else "c4"
    if a.capacity is None:
        # BASELINE configs[1] (c2) and configs[4] (c5) run with dynamic capacity factors on;
        # an explicit --alpha asks for a static factor
        a.capacity = "dynamic" if a.config in ("c2", "c5") and a.alpha is None else "static"
    return a


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return dict(hbm=j["hbm_gbs"], bf16=j["bf16_tflops"], bf16_sus=j["bf16_tflops_sustained"],
                    sm_max_mhz=j.get("sm_max_mhz", 1965.0), src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, sm_max_mhz=1965.0, src="fallback")


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML polled every 2 ms
    from a host thread (the timed region can be only tens of ms), nvidia-smi as a fallback."""

    REASONS = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4),
               ("hw_power_brake_slowdown", 0x80)]

    def __init__(self, index, device=None):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop_flag = False
        try:
            import pynvml
            pynvml.nvmlInit()
            h = None
            if device is not None:
                try:
                    import torch
                    pr = torch.cuda.get_device_properties(device)
                    bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                    h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
                except Exception:
                    h = None
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.nvml = (pynvml, h)
        except Exception:
            self.nvml = None

    def start(self):
        if self.nvml is not None:
            # the poller must get the GIL while the main thread enqueues the timed steps: a
            # short switch interval, and the timed region starts only once it is sampling
            self.switch = sys.getswitchinterval()
            sys.setswitchinterval(0.0002)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 1.0:
                time.sleep(0.0005)
            self.rows.clear()
            return
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()
        time.sleep(0.3)  # nvidia-smi start-up

    def _poll(self):
        nv, h = self.nvml
        while not self.stop_flag:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                pw = None
                try:  # instantaneous board power (W); the plain power reading is a 1 s average
                    fv = nv.nvmlDeviceGetFieldValues(h, [nv.NVML_FI_DEV_POWER_INSTANT])[0]
                    if fv.nvmlReturn == 0:
                        pw = fv.value.uiVal / 1000.0
                except Exception:
                    pw = None
                self.rows.append((sm, rs, pw))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.nvml is not None:
            self.stop_flag = True
            self.t.join(timeout=2)
            sys.setswitchinterval(self.switch)
            nv, h = self.nvml
            if not self.rows:
                return None
            sm = sorted(r[0] for r in self.rows)
            pw = sorted(r[2] for r in self.rows if r[2] is not None)
            try:
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            except Exception:
                mx = None
            try:
                lim = nv.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0
            except Exception:
                lim = None
            reasons = sorted({nm for _, rs, _ in self.rows for nm, bit in self.REASONS if rs & bit})
            return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": reasons,
                    "samples": len(sm), "source": "nvml, 2 ms",
                    "power_w": ({"median": round(pw[len(pw) // 2], 1), "max": round(pw[-1], 1),
                                 "limit": lim, "source": "nvml instant"} if pw else None)}
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        if not sm:
            return None
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4)
                          if r[3 + i].lower().startswith("active")})
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# MOE_BENCH_SHARE_GPU=1: run the N > 1 path with every rank on cuda:0 and a gloo process group
# (NCCL refuses two ranks on one device) -- a smoke test of the multi-process bench on one GPU;
# the numbers it prints are not scaling numbers.
SHARE_GPU = os.environ.get("MOE_BENCH_SHARE_GPU", "0") == "1"


def dist_setup(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if SHARE_GPU:  # test hook: every rank on cuda:0 (peer transport over IPC on one device)
        local = 0
    if ws > 1:
        import torch.distributed as dist
        # communicator set-up on stderr (nranks, NVLS / P2P transports) for the run's record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local) if torch.cuda.is_available() else None
        backend = ("nccl" if torch.cuda.is_available() and args.impl == "ours" and not SHARE_GPU
                   else "gloo")
        dist.init_process_group(backend=backend)
        pg = dist
    return ws, rank, local, pg


# ------------------------------------------------------------------------------------------
# algorithmic work per kernel: bytes or FLOPs per launch
# ------------------------------------------------------------------------------------------
def kernel_work(cfg, T, A, s, A_tok=None, gather=False, fcomb=False, fdx=False):
    """A: kept rows of this GPU's experts (GEMM work); A_tok: kept pairs of this GPU's tokens
    (dispatch / combine traffic).  Equal on one GPU.  gather: N2 fusion on (the dispatch
    writes only routing tables + the y rows of dropped tokens; the combine is in FWD2)."""
    n, k, d, f, do = cfg.n_experts, cfg.top_k, cfg.d_model, cfg.d_ff, cfg.d_out
    gf = 2.0 * A * d * f  # one expert GEMM (fwd or dgrad or wgrad) = 2*A*d*f FLOPs
    A = A if A_tok is None else A_tok
    disp = 8 * T * k + 4 * A + ((T - A) * do * s if fcomb else 0)  # routing tables, dropped y rows
    if not gather:
        disp += (T + A) * d * s                                     # + the X row copy
    return {
        # name: (kind, amount)   kind "flop" (tensor/alu) or "byte" (hbm)
        "gate_topk": ("byte", T * d * s + n * d * s + 4 * T * n + 8 * T * k),
        "dispatch": ("byte", disp),
        "zero_pad": ("byte", 0),
        "ffn_gemm1": ("flop", gf), "ffn_gemm2": ("flop", gf),
        "combine_fwd": ("byte", (A + T) * do * s + 8 * T * k),
        "combine_bwd": ("byte", (T + 2 * A) * do * s + 12 * T * k + 8 * T * n),
        "wgrad_w2": ("flop", gf), "dgrad_dA": ("flop", gf),
        "wgrad_w1": ("flop", gf), "dgrad_dX": ("flop", gf),
        # db1 partial reduction (fixed order over 8 partial rows per 256-row m-tile)
        "bias_grad": ("byte", ((A // 256) + n) * 8 * f * 4 + n * f * s),
        # fused (dx): only the dropped tokens, dx = dl W_g (dl row + W_g from L2 + dx row)
        # fused: only the dropped tokens (~5 % at c3) -- a latency-bound pass, no roofline
        "gate_dx": ("latency", 0) if fdx else ("byte", (A + T) * d * s + 4 * T * n + 8 * T * k),
        "route_scan": ("latency", 0), "route_hist": ("latency", 0),
        "gate_dw": ("byte", T * d * s + 4 * T * n),
        "dx_from_ret": ("byte", 2 * A * d * s + 4 * T * k),  # returned dx rows -> dx (peer EP)
    }


def run_ours(args):
    import torch
    from paper_2205_01848_b200 import MoELayer
    from synth import get_config, make_dy, make_layer

    ws, rank, local, dist = dist_setup(args)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = get_config(args.config)
    args.cached = args.cached or args.config == "c5"
    strong = not (cfg.scaling == "weak" or args.config in ("c3", "c5"))
    T = args.tokens or (cfg.tokens // ws if strong else cfg.tokens)
    alpha = args.alpha if args.alpha is not None else cfg.alpha
    n, k, d, f, do = cfg.n_experts, cfg.top_k, cfg.d_model, cfg.d_ff, cfg.d_out
    s = 2 if cfg.dtype == "bf16" else 4
    use_ep = ws > 1 or args.ep
    peer = use_ep and args.transport == "peer"
    comm = 0
    if use_ep and not peer:
        import torch.distributed as tdist
        if not tdist.is_initialized():  # --ep at N = 1: a 1-rank NCCL group (loopback)
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29555")
            tdist.init_process_group("nccl", rank=0, world_size=1)
            dist = tdist
        from paper_2205_01848_b200.dist import nccl_comm_ptr
        comm = nccl_comm_ptr(device=dev)
    # inputs resident in HBM (generated on the device from the seeded recipe); the expert
    # weights are the same on every rank (same seeds), each rank's tokens differ
    g = make_layer(n, d, f, do, T, cfg.dtype, args.regime, device=dev)
    if rank:
        g["x"] = make_layer(n, d, 64, do, T, cfg.dtype, args.regime, device=dev,
                            seed_offset=rank)["x"]
    dy = make_dy(T, do, cfg.dtype, device=dev, seed_offset=rank)
    layer = MoELayer(n, k, d, f, do, T, cfg.dtype, cfg.renormalize, world_size=ws if use_ep else 1,
                     rank=rank if use_ep else 0, nccl_comm=comm, device=dev,
                     transport="peer" if peer else "nccl")
    if peer:  # open every rank's peer window (CUDA IPC handles over the process group)
        if ws > 1:
            from paper_2205_01848_b200.dist import nccl_comm_ptr, peer_connect
            if not peer_connect(layer, strict=False):
                # some rank could not map its peers' windows (no CUDA IPC / P2P on this box):
                # every rank switches to the NCCL transport together (stated in the config)
                print("bench: peer windows unavailable on some rank; using the NCCL transport",
                      file=sys.stderr)
                del layer
                peer = False
                comm = nccl_comm_ptr(device=dev)
                layer = MoELayer(n, k, d, f, do, T, cfg.dtype, cfg.renormalize, world_size=ws,
                                 rank=rank, nccl_comm=comm, device=dev, transport="nccl")
        else:
            layer.peer_attach([layer.peer_window()])
    layer.set_capacity_factors([alpha] * n, T * (ws if use_ep else 1))
    # N2 fusions (moe_set_fusion): gather x rows in the expert GEMMs, combine in FWD2 (k = 1)
    fflags = {"none": 0, "combine": 2, "dx": 4, "otok": 8, "legacy": 6, "default": 14,
              "combine2": 30, "all": 15, "cdisp": 46}[args.fusion]
    tc1 = not use_ep and cfg.dtype == "bf16" and getattr(layer, "uses_tcgen05", False)
    gather = tc1 and bool(fflags & 1) and d % 128 == 0 and f % 128 == 0
    fcomb = tc1 and bool(fflags & 2) and k == 1 and do % 128 == 0
    fdx = tc1 and bool(fflags & 4) and k == 1 and d % 128 == 0
    otok = tc1 and bool(fflags & 8) and do % 128 == 0
    fcomb = fcomb or (otok and bool(fflags & 16) and k == 2)
    cdisp = tc1 and args.cached and bool(fflags & 32) and not gather and d % 64 == 0
    # peer EP (N1): return rows from the GEMM epilogues, and the dispatch backward in the
    # owners' dX GEMMs (k = 1)
    pret = (peer and cfg.dtype == "bf16" and getattr(layer, "uses_tcgen05", False)
            and d % 128 == 0 and do % 128 == 0)
    fdx_ep = pret and bool(fflags & 4) and k == 1
    layer.set_fusion(fflags)
    tdt = layer.tdtype
    grads = dict(dx=torch.empty(T, d, dtype=tdt, device=dev),
                 dw_gate=torch.empty(n, d, dtype=tdt, device=dev),
                 dw1=torch.empty(n, f, d, dtype=tdt, device=dev),
                 db1=torch.empty(n, f, dtype=tdt, device=dev),
                 dw2=torch.empty(n, do, f, dtype=tdt, device=dev),
                 db2=torch.empty(n, do, dtype=tdt, device=dev))
    y = torch.empty(T, do, dtype=tdt, device=dev)
    if args.cached:
        layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"], y=y)
        layer.backward(dy, grads=grads)
        cached_idx = layer.routing(T)["idx"].clone()
        layer.set_cached_assignment(cached_idx)

    # TIMING EXPERIMENT ONLY (MOE_BENCH_L2CLEAN=1, profiled pass): a 2x-L2 read between the
    # forward and the backward writes back and evicts the forward's dirty L2 lines, so the
    # backward's first kernel is timed without the previous kernel's deferred write-back
    l2clean = None

    def step():
        layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"], y=y)
        if l2clean is not None:
            l2clean.sum()
        layer.backward(dy, grads=grads)

    # dynamic capacity factors (S4.1): the library's policy (reading 14) adapts
    # C_e from the observed counts for --policy-warmup steps (recompiles are stream-ordered
    # capacity-table updates, no sync beyond reading the counts); then the timed region runs
    # with the capacities it settled on
    policy = None
    recompiles = 0
    if args.capacity == "dynamic":
        from paper_2205_01848_b200 import CapacityPolicy
        policy = CapacityPolicy(n, T * (ws if use_ep else 1), k, layer.capacities)
        for _ in range(args.policy_warmup):
            step()
            cnt = layer.stats()["counts"]
            new = policy.update(cnt)
            if new is not None:
                layer.set_capacities(new)
                recompiles += 1
        torch.cuda.synchronize(dev)
        time.sleep(2.0)  # the warm-up steps heat the GPU: time from the same rested state
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    stats = layer.stats()
    nl = n // (ws if use_ep else 1)
    e_lo = (rank if use_ep else 0) * nl
    # A: kept rows this GPU's expert GEMMs run over; A_tok: kept pairs of this GPU's tokens
    A = sum(min(c, cap) for c, cap in list(zip(stats["counts"], layer.capacities))[e_lo:e_lo + nl])
    layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"], y=y)
    A_tok = int((layer.routing(T)["slot_of"] >= 0).sum().item())
    layer.backward(dy, grads=grads)
    torch.cuda.synchronize(dev)

    def barrier():
        # drain our stream first: the layer's NCCL exchanges share torch's communicator, and
        # a torch collective must not overlap them on another stream
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if SHARE_GPU else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- timed region (device events on the launching stream) ----------------
    # The headline runs with the library's per-kernel events OFF; a second pass of the same
    # K steps with them on gives the per-kernel table (roofline) below.
    # L2: inputs (x, dy, weights) larger than the L2 stream through it every step; smaller
    # ones (c1, c2) would stay resident, so every timed step then starts after a write of
    # 2x the L2 (outside the step's events) and the time is the sum of the step intervals
    l2_bytes = getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20)
    in_bytes = sum(int(t.numel() * t.element_size())
                   for t in (g["x"], dy, g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"]))
    flush_buf = (torch.empty(2 * l2_bytes, dtype=torch.uint8, device=dev)
                 if in_bytes < 2 * l2_bytes else None)

    def timed_steps(nsteps):
        """[(start, end)] events of nsteps steps: back to back, or each after an L2 flush."""
        evs = []
        prev = torch.cuda.Event(enable_timing=True)
        prev.record(stream)
        for _ in range(nsteps):
            if flush_buf is not None:
                flush_buf.zero_()
                prev = torch.cuda.Event(enable_timing=True)
                prev.record(stream)
            step()
            m = torch.cuda.Event(enable_timing=True)
            m.record(stream)
            evs.append((prev, m))
            prev = m
        return evs

    l0 = layer.launch_count()
    clk = ClockSampler(local, dev)
    barrier()
    clk.start()
    marks = timed_steps(args.steps)  # per-step intervals (median / p10 / p90)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    per_step = sorted(a_.elapsed_time(b_) for a_, b_ in marks)
    ms = (sum(per_step) if flush_buf is not None
          else marks[0][0].elapsed_time(marks[-1][1]))
    q = lambda f: per_step[min(len(per_step) - 1, int(f * (len(per_step) - 1) + 0.5))]  # noqa: E731
    step_stats = {"median": round(q(0.5), 4), "p10": round(q(0.1), 4), "p90": round(q(0.9), 4)}
    barrier()
    launches = layer.launch_count() - l0
    _, dev_flags = layer.check_flags()   # NaN logits / peer-barrier timeout: the run is invalid
    if dev_flags:
        print(f"bench: device error flags {dev_flags} raised in the timed region", file=sys.stderr)
    ms = max_over_ranks(ms)
    ms_step = ms / args.steps
    value = T * ws * args.steps / (ms / 1e3)

    # same starting power state as the headline pass: the B200 drops from 1965 MHz to ~1.25 GHz
    # within ~0.1 s of sustained expert-GEMM load (sw_power_cap), so let it recover first
    time.sleep(2.0)
    layer.profile(True)
    layer.profile_read(reset=True)
    if os.environ.get("MOE_BENCH_L2CLEAN") == "1":
        l2clean = torch.ones(l2_bytes // 2, dtype=torch.float32, device=dev)
    barrier()
    pm = timed_steps(args.steps)
    l2clean = None
    torch.cuda.synchronize(dev)
    prof_ms_step = max_over_ranks(sum(a_.elapsed_time(b_) for a_, b_ in pm)) / args.steps
    barrier()
    ktimes = layer.profile_read(reset=True)
    layer.profile(False)

    graph_ms = None
    if args.graph and not (use_ep and not peer):  # NCCL EP syncs the host per forward
        from paper_2205_01848_b200 import GraphedStep
        gs = GraphedStep(layer, g["x"], g, dy, grads, y=y)
        for _ in range(3):
            gs.replay()
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            gs.replay()
        g1.record(stream)
        torch.cuda.synchronize(dev)
        graph_ms = max_over_ranks(g0.elapsed_time(g1)) / args.steps

    # ---------------- per-kernel rooflines ----------------
    pk = peaks()
    work = kernel_work(cfg, T, A, s, A_tok, gather=gather, fcomb=fcomb, fdx=fdx or fdx_ep)
    sm_peak_tf = 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
    at_max_clock = bool(clocks and clocks.get("sm_mhz") and
                        clocks["sm_mhz"] >= 0.97 * (clocks.get("sm_max_mhz") or pk["sm_max_mhz"]))
    kernels = {}
    for name, (cnt, tot) in ktimes.items():
        avg_ms = tot / max(cnt, 1)
        kind, amt = work.get(name, ("byte", 0))
        ent = {"launches": cnt, "avg_ms": round(avg_ms, 5), "share": None}
        if kind == "latency":
            ent.update(bound="latency")
        elif amt and avg_ms > 0:
            if kind == "byte":
                ach = amt / (avg_ms / 1e3) / 1e9
                ent.update(bound="hbm", achieved=round(ach, 1), peak=pk["hbm"], unit="GB/s",
                           frac=round(ach / pk["hbm"], 4), algorithmic=amt)
            else:
                ach = amt / (avg_ms / 1e3) / 1e12
                tc = layer.tdtype == torch.bfloat16 and getattr(layer, "uses_tcgen05", False)
                tf = layer.tdtype == torch.float32 and getattr(layer, "uses_tf32", False)
                # the burst peak applies while the clock holds its maximum through the timed
                # region (a short region from a rested GPU); the sustained one otherwise
                bpk = pk["bf16"] if at_max_clock else pk["bf16_sus"]
                if tc:
                    peak = bpk
                elif tf:
                    # fp32 GEMMs as split-tf32 on the tensor cores: the tf32 dense peak is the
                    # measured bf16 peak x the guide's nominal ratio (1.1 / 2.25 PF), and every
                    # fp32 product costs 4 tf32 MMAs -> effective fp32 peak = tf32 peak / 4
                    peak = bpk * (1.1 / 2.25) / 4
                else:
                    peak = sm_peak_tf
                ent.update(bound="tensor" if (tc or tf) else "alu", achieved=round(ach, 2),
                           peak=round(peak, 1), unit="TFLOP/s", frac=round(ach / peak, 4),
                           algorithmic=amt)
                if tc:
                    ent.update(frac_burst=round(ach / pk["bf16"], 4),
                               frac_sustained=round(ach / pk["bf16_sus"], 4))
                if tf:
                    ent.update(peak_note="tf32 peak (measured bf16 x 1.1/2.25) / 4 MMAs per fp32 "
                                         "product (split-tf32)")
        kernels[name] = ent
    tot_k = sum(v[1] for v in ktimes.values()) or 1.0
    for name, (cnt, tot) in ktimes.items():
        kernels[name]["share"] = round(tot / tot_k, 4)
    dom = max(ktimes.items(), key=lambda kv: kv[1][1])[0] if ktimes else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if dom and os.path.exists(tp):
        traffic = json.load(open(tp)).get(args.config, {}).get(dom)
    dk = kernels.get(dom, {})
    roofline = {"kernel": dom, "bound": dk.get("bound"), "achieved": dk.get("achieved"),
                "peak": dk.get("peak"), "unit": dk.get("unit"), "frac": dk.get("frac"),
                "traffic": traffic, "peak_source": pk["src"]}
    if "frac_burst" in dk:
        roofline.update(peak_kind="burst" if at_max_clock else "sustained",
                        frac_burst=dk["frac_burst"], frac_sustained=dk["frac_sustained"])
    hbm = {nm: kernels[nm].get("achieved") for nm in ("dispatch", "combine_fwd", "combine_bwd", "gate_dx",
                                                       "dx_from_ret")
           if nm in kernels and kernels[nm].get("achieved") is not None}

    # ---------------- end to end through the public API with host buffers ----------------
    # Every step copies its inputs (x, dy) from pinned host memory and reads its result (y)
    # back; copies run on two copy streams, double-buffered, so step i+1's upload and step
    # i-1's download overlap step i's compute (the way a training loop prefetches batches).
    e2e = None
    if not args.no_e2e:
        x_h = g["x"].cpu().pin_memory()
        dy_h = dy.cpu().pin_memory()
        y_h = [torch.empty(T, do, dtype=tdt).pin_memory() for _ in range(2)]
        x_d = [torch.empty_like(g["x"]) for _ in range(2)]
        dy_d = [torch.empty_like(dy) for _ in range(2)]
        y_d = [torch.empty(T, do, dtype=tdt, device=dev) for _ in range(2)]
        up, down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev = lambda: torch.cuda.Event()  # noqa: E731
        h2d_done = [ev(), ev()]
        comp_done = [ev(), ev()]
        d2h_done = [ev(), ev()]
        for e_ in comp_done + d2h_done:
            e_.record(stream)

        def e2e_run(nsteps, t0=None, t1=None):
            def h2d(i):
                bb = i % 2
                with torch.cuda.stream(up):
                    up.wait_event(comp_done[bb])      # step i-2 no longer reads x_d[bb]/dy_d[bb]
                    x_d[bb].copy_(x_h, non_blocking=True)
                    dy_d[bb].copy_(dy_h, non_blocking=True)
                    h2d_done[bb].record(up)
            if t0 is not None:
                t0.record(up)
            h2d(0)
            for i in range(nsteps):
                bb = i % 2
                if i + 1 < nsteps:
                    h2d(i + 1)
                stream.wait_event(h2d_done[bb])
                stream.wait_event(d2h_done[bb])       # y_d[bb] of step i-2 has been read back
                layer.forward(x_d[bb], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"], y=y_d[bb])
                layer.backward(dy_d[bb], grads=grads)
                comp_done[bb].record(stream)
                with torch.cuda.stream(down):
                    down.wait_event(comp_done[bb])
                    y_h[bb].copy_(y_d[bb], non_blocking=True)
                    d2h_done[bb].record(down)
            if t1 is not None:
                down.wait_event(comp_done[(nsteps - 1) % 2])
                t1.record(down)

        e2e_run(2)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_run(args.steps, e0, e1)
        torch.cuda.synchronize(dev)
        ems = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": round(T * ws * args.steps / (ems / 1e3), 1), "unit": "tokens/s",
               "h2d_bytes_per_step": int(x_h.numel() * x_h.element_size() + dy_h.numel() * dy_h.element_size()),
               "d2h_bytes_per_step": int(y_h[0].numel() * y_h[0].element_size()),
               "overlap": "double-buffered copy streams"}

    # ---------------- CPU oracle baseline (rank 0, N = 1 only) ----------------
    cpu_base = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu_base = cpu_oracle_sample(cfg, g, dy, args.cpu_sample, alpha)

    # expert-parallel exchange: rows that cross to another rank per exchange (this rank's
    # kept pairs whose expert lives elsewhere), NVLink bytes of one token exchange, and the
    # share of the step the peer barriers (wait for peers) took
    exchange = None
    if use_ep:
        rt_ = layer.routing(T)
        nl_ = n // ws
        owner = torch.div(rt_["idx"].long(), nl_, rounding_mode="floor")
        off = int(((rt_["slot_of"] >= 0) & (owner != rank)).sum().item())
        bar = ktimes.get("peer_barrier", (0, 0.0))
        via = getattr(layer, "peer_via", "in-process windows")
        exchange = {"transport": f"peer memory ({via}, device-initiated loads/stores)"
                                 if peer else "NCCL grouped send/recv",
                    "off_rank_rows_per_exchange": off,
                    "nvlink_bytes_per_exchange": off * d * s,
                    "exchanges_per_step": 4,
                    "barrier_share": round(bar[1] / max(prof_ms_step * args.steps, 1e-9), 4),
                    "nccl_debug": os.environ.get("NCCL_DEBUG")}
    if rank == 0:
        padded_flops = 12.0 * d * f * sum(c - min(cnt, c) for cnt, c in zip(stats["counts"], layer.capacities))
        out = {
            "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": cfg.dtype,
            "data": f"synthetic (seeded, {args.regime} regime; random-init weights)",
            "config": {"workload": f"{cfg.name}: {n} experts top-{k}, d_model {d}, d_ff {f}, "
                                   + (f"{T * ws} global tokens ({T}/GPU)" if strong
                                      else f"{T} tokens/GPU")
                                   + f", {cfg.dtype}, "
                                   + (f"dynamic capacity (policy, {args.policy_warmup} steps)"
                                      if policy is not None else f"alpha {alpha}")
                                   + (f", {args.regime} routing" if args.regime != "uniform" else "")
                                   + (", cached assignments" if args.cached else "")
                                   + (", EMULATED capacity-padded GEMMs (timing only)"
                                      if args.emulate_padded else ""),
                       "tokens_per_gpu": T, "n_experts": n, "top_k": k, "d_model": d, "d_ff": f,
                       "capacity_factor": alpha if policy is None else "dynamic",
                       "regime": args.regime, "recompiles": recompiles,
                       "renormalize": cfg.renormalize,
                       "parallelism": (f"ep{ws} (experts sharded, tokens data-parallel, "
                                       + ("peer memory, device-initiated)" if peer else "NCCL)")
                                       if use_ep else "1 GPU"),
                       "l2": (f"inputs {in_bytes / 1e6:.0f} MB < 2x L2: each timed step after "
                              f"a {2 * l2_bytes / 1e6:.0f} MB write (flush), time = sum of steps"
                              if flush_buf is not None else
                              f"inputs {in_bytes / 1e6:.0f} MB > L2 {l2_bytes / 1e6:.0f} MB, "
                              "no flush"),
                       "fusion": "+".join([nm for nm, on in (("gather", gather), ("combine", fcomb),
                                                             ("dx", fdx or fdx_ep),
                                                             ("otok", otok),
                                                             ("cdisp", cdisp),
                                                             ("return_rows", pret)) if on]) or "none",
                       "kept_assignments": A, "drops": stats["drops"],
                       "drop_rate": round(stats["drops"] / max(1, T * k * (ws if use_ep else 1)), 5),
                       "sum_capacity_rows": int(sum(layer.capacities)),
                       "padding_flops_avoided": padded_flops},
            "roofline": roofline,
            "exchange": exchange,
            "device_flags": dev_flags,
            "ms_per_step_profiled": round(prof_ms_step, 4),
            "step_ms": step_stats,
            "hbm_gbs": hbm,
            "kernels": kernels,
            "cpu_baseline": cpu_base,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "graph": (None if graph_ms is None else
                      {"ms_per_step": round(graph_ms, 4),
                       "value": round(T * ws / (graph_ms / 1e3), 1)}),
            "clocks": clocks,
        }
        print(json.dumps(out), flush=True)
    layer.close()   # an NCCL symmetric window is deregistered while the communicator lives
    if dist is not None:
        dist.destroy_process_group()


def _threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        if info:
            return max(i.get("num_threads", 1) for i in info)
    except Exception:
        pass
    return len(os.sched_getaffinity(0))


# The oracle holds fp64 copies of every expert's weights and weight gradients; for the large
# configs (c4: 128 experts of 2 x 2048 x 8192) that is ~70 GB, so above 12 GB the host sample uses
# the first n_sub experts with the per-expert load of the full layer (tokens scaled by
# n_sub / n).  Per token the oracle's work is the same up to the gate (6 d n of 12 k d f FLOPs,
# 0.4 % at c4), so tokens/s of the sub-layer stands for the full layer's.
ORACLE_WEIGHT_BYTES = 12 << 30


def oracle_expert_sample(n, d, f, do, k):
    per = (f * d + do * f) * 8 * 2          # fp64 weights + their gradients, one expert
    return max(k, min(n, ORACLE_WEIGHT_BYTES // per))


def cpu_oracle_sample(cfg, g, dy, tokens, alpha):
    """The fp64 oracle, as it stands, on a bounded sample of the same workload."""
    import numpy as np
    from oracle import moe_oracle as O
    from synth import to_numpy64
    n, k = cfg.n_experts, cfg.top_k
    ns = oracle_expert_sample(n, cfg.d_model, cfg.d_ff, cfg.d_out, k)
    Ts = min(tokens, g["x"].shape[0]) * ns // n
    x = to_numpy64(g["x"][:Ts])
    p = {kk: g[kk][:ns].detach().to("cpu", dtype=__import__("torch").float64).numpy()
         for kk in ("w_gate", "w1", "b1", "w2", "b2")}
    n_all, n = n, ns
    dyn = to_numpy64(dy[:Ts])
    caps = O.capacities_from_factors([alpha] * n, Ts, k)
    t0 = time.perf_counter()
    st = O.moe_forward(x, p, k, caps, cfg.renormalize)
    O.moe_backward(st, dyn)
    dt = time.perf_counter() - t0
    out = {"value": round(Ts / dt, 2), "unit": "tokens/s", "cores": _threads(), "kind": "oracle",
           "sample": (f"{Ts} tokens of {cfg.name} (all {n} experts, alpha {alpha}), fwd+bwd, fp64 NumPy"
                      if n == n_all else
                      f"{Ts} tokens over {n} of {cfg.name}'s {n_all} experts (the full layer's "
                      f"per-expert load), alpha {alpha}, fwd+bwd, fp64 NumPy"),
           "seconds": round(dt, 2)}
    try:  # the same oracle on one core (BLAS limited to one thread), a quarter of the sample
        from threadpoolctl import threadpool_limits
        Ts1 = max(64, Ts // 4)
        caps1 = O.capacities_from_factors([alpha] * n, Ts1, k)
        with threadpool_limits(limits=1):
            t0 = time.perf_counter()
            st = O.moe_forward(x[:Ts1], p, k, caps1, cfg.renormalize)
            O.moe_backward(st, dyn[:Ts1])
            dt1 = time.perf_counter() - t0
        out["single_thread"] = {"value": round(Ts1 / dt1, 2), "cores": 1, "tokens": Ts1,
                                "seconds": round(dt1, 2)}
    except Exception as ex:  # threadpoolctl missing: report the all-core number only
        out["single_thread"] = {"unavailable": str(ex)[:80]}
    return out


def run_reference(args):
    """--impl reference: the fp64 oracle on the host cores (rank 0 only)."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import torch
    try:  # torchrun sets OMP_NUM_THREADS=1: give the BLAS (loaded with numpy) every host core
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=len(os.sched_getaffinity(0)))
    except Exception:
        pass
    from oracle import moe_oracle as O
    from synth import get_config, make_dy, make_layer, to_numpy64
    cfg = get_config(args.config)
    alpha = args.alpha if args.alpha is not None else cfg.alpha
    n, k, d, f, do = cfg.n_experts, cfg.top_k, cfg.d_model, cfg.d_ff, cfg.d_out
    n_all = n
    n = oracle_expert_sample(n, d, f, do, k)   # bounded host memory (see ORACLE_WEIGHT_BYTES)
    # per-step sample: as large as the cpu_baseline sample (--cpu-sample) while the whole
    # K + W run stays within ~150 s of host time, calibrated by one 1024-token step (the
    # oracle has a large per-step fixed cost -- full-size fp64 weight gradients -- so small
    # samples understate its throughput)
    nsteps = args.steps + args.warmup
    cal = make_layer(n, d, f, do, 1024, cfg.dtype, "uniform")
    pc = {kk: cal[kk].to(torch.float64).numpy() for kk in ("w_gate", "w1", "b1", "w2", "b2")}
    t0 = time.perf_counter()
    stc = O.moe_forward(to_numpy64(cal["x"]), pc, k, O.capacities_from_factors([alpha] * n, 1024, k),
                        cfg.renormalize)
    O.moe_backward(stc, to_numpy64(make_dy(1024, do, cfg.dtype)))
    tcal = time.perf_counter() - t0
    del cal, pc, stc
    Ts = int(1024 * 150.0 / max(nsteps * tcal, 1e-6)) // 256 * 256
    Ts = max(256, min(args.cpu_sample, Ts))
    g = make_layer(n, d, f, do, Ts * nsteps, cfg.dtype, "uniform")
    dy = make_dy(Ts * nsteps, do, cfg.dtype)
    p = {kk: g[kk].to(torch.float64).numpy() for kk in ("w_gate", "w1", "b1", "w2", "b2")}
    caps = O.capacities_from_factors([alpha] * n, Ts, k)

    def step(i):
        x = to_numpy64(g["x"][i * Ts:(i + 1) * Ts])
        st = O.moe_forward(x, p, k, caps, cfg.renormalize)
        O.moe_backward(st, to_numpy64(dy[i * Ts:(i + 1) * Ts]))

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    dt = time.perf_counter() - t0
    val = Ts * args.steps / dt
    out = {"impl": "reference", "metric": METRIC, "value": round(val, 2), "unit": "tokens/s",
           "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(dt * 1e3 / args.steps, 2), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{cfg.name}: {n_all} experts top-{k}, d_model {d}, d_ff {f}, "
                                  f"{Ts} tokens/step sample"
                                  + ("" if n == n_all else
                                     f" over {n} of the {n_all} experts (per-expert load of the "
                                     f"full layer)") + f", alpha {alpha}"},
           "cpu_baseline": {"value": round(val, 2), "unit": "tokens/s", "cores": _threads(),
                            "kind": "oracle",
                            "sample": f"{Ts} tokens per step of {cfg.name}"
                                      + ("" if n == n_all else f" over {n} of {n_all} experts")},
           "e2e": {"value": round(val, 2), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
