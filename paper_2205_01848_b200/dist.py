"""Process-group plumbing for expert parallelism: hand torch's NCCL communicator to the C ABI.

torch creates NCCL communicators lazily; one small collective forces creation, after which
ProcessGroupNCCL._comm_ptr() is the ncclComm_t the library enqueues its exchanges on.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def nccl_comm_ptr(group=None, device=None) -> int:
    """ncclComm_t (as an int) of `group` (default: WORLD) for `device` (default: current)."""
    group = group or dist.group.WORLD
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    t = torch.zeros(1, device=dev)
    dist.all_reduce(t, group=group)          # forces communicator creation
    torch.cuda.synchronize(dev)
    backend = group._get_backend(dev)
    ptr = backend._comm_ptr()
    if not ptr:
        raise RuntimeError("ProcessGroupNCCL returned a null communicator")
    return int(ptr)


def peer_connect(layer, group=None, strict=True):
    """Peer-memory transport across processes (one per GPU): all-gather the layers' 64-byte
    CUDA IPC window handles over the process group and open the peers' windows (N1).

    Every rank learns whether EVERY rank opened its peers' windows (one MIN all-reduce), so
    the ranks agree on the outcome.  strict: raise if any rank failed; else return False
    (the caller then builds its layers with the NCCL transport instead)."""
    group = group or dist.group.WORLD
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, layer.peer_export(), group=group)
    err = None
    try:
        layer.peer_import(handles)
    except Exception as e:  # noqa: BLE001 -- reported below, after the ranks agree
        err = e
    on_gpu = dist.get_backend(group) == "nccl"
    flag = torch.tensor([0 if err else 1], dtype=torch.int32,
                        device=torch.device("cuda", torch.cuda.current_device()) if on_gpu else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    ok = bool(flag.item())
    if not ok and strict:
        raise RuntimeError(f"peer windows could not be opened on every rank (this rank: {err!r})")
    return ok


def peer_connect_local(layers):
    """Peer-memory transport for R ranks in ONE process (threads / streams, e.g. one GPU)."""
    wins = [L.peer_window() for L in layers]
    for L in layers:
        L.peer_attach(wins)
