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


def peer_connect(layer, group=None, strict=True, prefer_nccl=True):
    """Peer-memory transport across processes (one per GPU), N1.

    prefer_nccl (NCCL process group): the windows become NCCL symmetric memory registered on
    the group's communicator (moe_peer_connect_nccl; NCCL >= 2.28 device API, every rank in
    one NVLink LSA team).  If any rank cannot, every rank falls back to all-gathering the
    layers' 64-byte CUDA IPC window handles over the process group and opening them.

    Every rank learns whether EVERY rank succeeded (MIN all-reduces), so the ranks agree on
    the outcome.  strict: raise if any rank failed; else return False (the caller then
    builds its layers with the NCCL transport instead)."""
    group = group or dist.group.WORLD
    on_gpu = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if on_gpu else "cpu"
    if prefer_nccl and on_gpu:
        err = None
        try:
            layer.peer_connect_nccl(nccl_comm_ptr(group))
        except Exception as e:  # noqa: BLE001 -- agreed on below
            err = e
        flag = torch.tensor([0 if err else 1], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if bool(flag.item()):
            return True
        if err is None:   # this rank attached but a peer did not: the layer must be rebuilt
            if strict:
                raise RuntimeError("NCCL symmetric windows failed on a peer rank after this "
                                   "rank attached; rebuild the layers, prefer_nccl=False")
            return False
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, layer.peer_export(), group=group)
    err = None
    try:
        layer.peer_import(handles)
    except Exception as e:  # noqa: BLE001 -- reported below, after the ranks agree
        err = e
    flag = torch.tensor([0 if err else 1], dtype=torch.int32, device=dev)
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
