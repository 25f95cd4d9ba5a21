"""ctypes declarations of the C ABI in include/moe.h (argument marshalling only).

Loading fails loudly when the CUDA library has not been built: there is no CPU or
eager-PyTorch fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdynamoe_b200.so")

MOE_OK = 0
STATUS = {0: "MOE_OK", 1: "MOE_ERR_INVALID_ARG", 2: "MOE_ERR_CONFIG", 3: "MOE_ERR_STATE",
          4: "MOE_ERR_WORKSPACE_TOO_SMALL", 5: "MOE_ERR_CUDA", 6: "MOE_ERR_NCCL",
          7: "MOE_ERR_DEVICE_FLAG"}
MOE_ERR_WORKSPACE_TOO_SMALL = 4
MOE_ERR_DEVICE_FLAG = 7
DTYPES = {"f32": 0, "bf16": 1}


class MoEConfig(C.Structure):
    _fields_ = [("n_experts", C.c_int32), ("top_k", C.c_int32), ("d_model", C.c_int32),
                ("d_ff", C.c_int32), ("d_out", C.c_int32), ("max_tokens", C.c_int32),
                ("dtype", C.c_int32), ("renormalize", C.c_int32), ("world_size", C.c_int32),
                ("rank", C.c_int32), ("nccl_comm", C.c_void_p), ("stream", C.c_void_p),
                ("transport", C.c_int32), ("reserved0", C.c_int32), ("window_rows", C.c_int64)]


TRANSPORTS = {"nccl": 0, "peer": 1}


class FwdArgs(C.Structure):
    _fields_ = [("T", C.c_int32), ("x", C.c_void_p), ("w_gate", C.c_void_p), ("w1", C.c_void_p),
                ("b1", C.c_void_p), ("w2", C.c_void_p), ("b2", C.c_void_p), ("y", C.c_void_p)]


class BwdArgs(C.Structure):
    _fields_ = [("dy", C.c_void_p), ("dx", C.c_void_p), ("dw_gate", C.c_void_p),
                ("dw1", C.c_void_p), ("db1", C.c_void_p), ("dw2", C.c_void_p),
                ("db2", C.c_void_p), ("accumulate", C.c_int32)]


class Routing(C.Structure):
    _fields_ = [("logits", C.c_void_p), ("weights", C.c_void_p), ("idx", C.c_void_p),
                ("fresh_idx", C.c_void_p), ("slot_of", C.c_void_p),
                ("token_of_slot", C.c_void_p), ("counts", C.c_void_p), ("kept", C.c_void_p),
                ("dl", C.c_void_p), ("dw", C.c_void_p), ("x_buf", C.c_void_p),
                ("h_buf", C.c_void_p), ("o_buf", C.c_void_p), ("rows", C.c_int64),
                ("base_host", C.c_int32 * 257)]


class Stats(C.Structure):
    _fields_ = [("counts", C.c_void_p), ("drops", C.c_void_p), ("hit_count", C.c_void_p)]


class KernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("total_ms", C.c_double)]


class Metrics(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("T", C.c_int32), ("hit_count", C.c_int32),
                ("drops", C.c_int64), ("aux_loss", C.c_float), ("counts", C.c_int32 * 256)]


class PolicyConfig(C.Structure):
    _fields_ = [("n_experts", C.c_int32), ("top_k", C.c_int32), ("tokens_global", C.c_int64),
                ("window", C.c_int32), ("headroom", C.c_double), ("shrink_util", C.c_double),
                ("min_alpha", C.c_double), ("max_alpha", C.c_double)]


EXPORTS = {
    "moe_init": ([C.POINTER(MoEConfig), C.POINTER(C.c_void_p)], C.c_int),
    "moe_destroy": ([C.c_void_p], C.c_int),
    "moe_set_stream": ([C.c_void_p, C.c_void_p], C.c_int),
    "moe_capacity_from_factors": ([C.c_int32, C.c_int64, C.c_int32, C.POINTER(C.c_double),
                                   C.POINTER(C.c_int32)], C.c_int),
    "moe_set_capacities": ([C.c_void_p, C.POINTER(C.c_int32)], C.c_int),
    "moe_get_capacities": ([C.c_void_p, C.POINTER(C.c_int32)], C.c_int),
    "moe_workspace_size": ([C.c_void_p, C.POINTER(C.c_size_t)], C.c_int),
    "moe_set_workspace": ([C.c_void_p, C.c_void_p, C.c_size_t], C.c_int),
    "moe_set_cached_assignment": ([C.c_void_p, C.c_void_p], C.c_int),
    "moe_set_assignment_cache": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32],
                                 C.c_int),
    "moe_forward": ([C.c_void_p, C.POINTER(FwdArgs)], C.c_int),
    "moe_backward": ([C.c_void_p, C.POINTER(BwdArgs)], C.c_int),
    "moe_get_routing": ([C.c_void_p, C.POINTER(Routing)], C.c_int),
    "moe_get_stats_async": ([C.c_void_p, C.POINTER(Stats)], C.c_int),
    "moe_check_device_flags": ([C.c_void_p, C.POINTER(C.c_int32)], C.c_int),
    "moe_launch_count": ([C.c_void_p, C.POINTER(C.c_int64)], C.c_int),
    "moe_set_fusion": ([C.c_void_p, C.c_int32], C.c_int),
    "moe_last_error": ([C.c_void_p], C.c_char_p),
    "moe_profile_enable": ([C.c_void_p, C.c_int32], C.c_int),
    "moe_profile_read": ([C.c_void_p, C.POINTER(KernelTime), C.c_int32, C.POINTER(C.c_int32),
                          C.c_int32], C.c_int),
    "moe_set_balance_loss": ([C.c_void_p, C.c_float], C.c_int),
    "moe_get_aux_loss_async": ([C.c_void_p, C.POINTER(C.c_float)], C.c_int),
    "moe_set_spec_outputs": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "moe_set_spec_grads": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "moe_metrics_enable": ([C.c_void_p, C.c_int32], C.c_int),
    "moe_metrics_pending": ([C.c_void_p, C.POINTER(C.c_int32)], C.c_int),
    "moe_metrics_pop": ([C.c_void_p, C.c_int32, C.POINTER(Metrics), C.POINTER(C.c_int32)], C.c_int),
    "moe_caching_trigger": ([C.c_double, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_int32,
                             C.POINTER(C.c_int32)], C.c_int),
    "moe_vcomm_create": ([C.c_int32, C.POINTER(C.c_void_p)], C.c_int),
    "moe_vcomm_destroy": ([C.c_void_p], C.c_int),
    "moe_ep_plan": ([C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                     C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                     C.POINTER(C.c_int32), C.POINTER(C.c_int64)], C.c_int),
    "moe_policy_create": ([C.POINTER(PolicyConfig), C.POINTER(C.c_int32), C.POINTER(C.c_void_p)],
                          C.c_int),
    "moe_policy_update": ([C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                           C.POINTER(C.c_int32)], C.c_int),
    "moe_policy_destroy": ([C.c_void_p], C.c_int),
    "moe_peer_window": ([C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)], C.c_int),
    "moe_peer_export": ([C.c_void_p, C.c_void_p], C.c_int),
    "moe_peer_attach": ([C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
    "moe_peer_import": ([C.c_void_p, C.c_void_p], C.c_int),
    "moe_peer_connect_nccl": ([C.c_void_p, C.c_void_p], C.c_int),
}

_lib = None


def load():
    """Load libdynamoe_b200.so (build it first with __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"CUDA library not built: {LIB_PATH} missing "
                           "(run python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(LIB_PATH)
    for name, (argt, rest) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.argtypes = argt
        fn.restype = rest
    _lib = lib
    return lib


class MoEError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def check(status, handle=None, what=""):
    if status != MOE_OK:
        # handle None (moe_init): the library keeps the reason of the last failed init
        msg = load().moe_last_error(handle).decode()
        if msg == "null handle":
            msg = ""
        raise MoEError(status, f"{what} {msg}".strip())
