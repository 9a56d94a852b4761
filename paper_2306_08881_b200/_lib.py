"""ctypes binding of include/acp.h (argument marshalling only).

Loads the in-tree ``lib/libacp.so`` built by ``build.py``. There is no
fallback: if the library is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# ACP_LIB: load another in-tree build instead (A/B runs of two builds)
LIB_PATH = os.environ.get("ACP_LIB") or os.path.join(HERE, "lib", "libacp.so")

ACP_OK, ACP_E_INVAL, ACP_E_CUDA, ACP_E_NCCL, ACP_E_NOMEM, ACP_E_STATE, ACP_E_NONFINITE = range(7)
ACP_NO_EF, ACP_NO_REUSE, ACP_SUM, ACP_POWERSGD, ACP_BUCKETED, ACP_CHECK_FINITE = 1, 2, 4, 8, 16, 32
ACP_ABI_VERSION = 1
(ACP_K_ORTH, ACP_K_PROJ_P, ACP_K_PROJ_Q, ACP_K_DECODE_P, ACP_K_DECODE_Q,
 ACP_K_ALLREDUCE) = range(6)
KERNEL_CLASS_NAMES = ("orth", "proj_p", "proj_q", "decode_p", "decode_q", "allreduce")

EXPORTED = (
    "acp_workspace_bytes", "acp_create", "acp_plan_create", "acp_check_finite", "acp_step", "acp_compress", "acp_decompress",
    "acp_get_state", "acp_set_state", "acp_plan_info", "acp_num_buckets", "acp_bucket_range",
    "acp_profile_enable", "acp_profile_reset", "acp_profile_read", "acp_launch_count",
    "acp_set_graphs", "acp_step_begin", "acp_bucket_ready", "acp_step_end",
    "acp_symmetric_bytes", "acp_attach_symmetric",
    "acp_destroy", "acp_last_error", "acp_abi_version", "acp_nccl_unique_id",
    "acp_nccl_comm_create", "acp_nccl_comm_destroy",
)


class AcpConfig(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32),
        ("num_tensors", C.c_int32),
        ("rows", C.POINTER(C.c_int64)),
        ("cols", C.POINTER(C.c_int64)),
        ("rank", C.c_int32),
        ("world_size", C.c_int32),
        ("nccl_comm", C.c_void_p),
        ("seed", C.c_uint64),
        ("q0_host", C.POINTER(C.c_float)),
        ("default_bucket_bytes", C.c_int64),
        ("flags", C.c_uint32),
        ("device", C.c_int32),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_size_t),
    ]


class AcpError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"acp status {status}: {msg}")
        self.status = status


_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (or paper_2306_08881_b200/build.py) first")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, i32, i64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
    fpp = C.POINTER(C.c_void_p)
    sig = {
        "acp_workspace_bytes": [C.POINTER(AcpConfig), C.POINTER(sz)],
        "acp_create": [C.POINTER(AcpConfig), C.POINTER(vp)],
        "acp_plan_create": [C.POINTER(AcpConfig), C.POINTER(vp)],
        "acp_check_finite": [vp, vp],
        "acp_step": [vp, i32, fpp, vp],
        "acp_compress": [vp, i32, fpp, C.POINTER(vp), C.POINTER(i64), vp],
        "acp_decompress": [vp, i32, fpp, vp],
        "acp_get_state": [vp, i32, vp, vp, vp, vp],
        "acp_set_state": [vp, i32, vp, vp, vp, vp],
        "acp_plan_info": [vp, i32, C.POINTER(i64)],
        "acp_num_buckets": [vp, i32, C.POINTER(i32)],
        "acp_bucket_range": [vp, i32, i32, C.POINTER(i64), C.POINTER(i64)],
        "acp_profile_enable": [vp, i32],
        "acp_set_graphs": [vp, i32],
        "acp_step_begin": [vp, i32, fpp, vp],
        "acp_bucket_ready": [vp, i32, vp],
        "acp_step_end": [vp, vp],
        "acp_symmetric_bytes": [vp, C.POINTER(i64)],
        "acp_attach_symmetric": [vp, vp, vp, fpp, i32, i64],
        "acp_profile_reset": [vp],
        "acp_profile_read": [vp, i32, C.POINTER(C.c_double), C.POINTER(i64), C.POINTER(C.c_double)],
        "acp_launch_count": [vp, C.POINTER(i64)],
        "acp_destroy": [vp],
        "acp_nccl_unique_id": [C.POINTER(C.c_uint8)],
        "acp_nccl_comm_create": [C.POINTER(C.c_uint8), i32, i32, i32, C.POINTER(vp)],
        "acp_nccl_comm_destroy": [vp],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    lib.acp_last_error.argtypes = []
    lib.acp_last_error.restype = C.c_char_p
    lib.acp_abi_version.argtypes = []
    lib.acp_abi_version.restype = C.c_int32
    if lib.acp_abi_version() != ACP_ABI_VERSION:
        raise ImportError("libacp.so ABI version mismatch")
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != ACP_OK:
        msg = _lib.acp_last_error().decode() if _lib is not None else ""
        raise AcpError(status, msg)
