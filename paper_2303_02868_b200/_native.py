"""ctypes binding of the C-ABI in include/hm_page.h (libhm_page.so).

This is the only door to native code.  There is no Python or CPU fallback:
a missing library raises NativeError, and every non-zero status is turned
into the matching hiermem-style exception.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import AllocationError, ConfigError, MoveError, NativeError, ProtocolError

LIB_PATH = Path(__file__).resolve().parent / "libhm_page.so"
if os.environ.get("HM_LIB_VARIANT"):   # measurement builds only (tools/build_variants.sh)
    LIB_PATH = LIB_PATH.with_name(f"libhm_page_{os.environ['HM_LIB_VARIANT']}.so")

HM_OK, HM_ERR_CONFIG, HM_ERR_ALLOCATION, HM_ERR_MOVE, HM_ERR_PROTOCOL, HM_ERR_KEY, \
    HM_ERR_CUDA, HM_ERR_INVALID = range(8)

DT_F16, DT_BF16, DT_F32 = 1, 2, 3
DTYPE_CODES = {"fp16": DT_F16, "float16": DT_F16, "bf16": DT_BF16, "bfloat16": DT_BF16,
               "fp32": DT_F32, "float32": DT_F32}
TIER_CODES = {"GPU": 0, "CPU": 1, "SSD": 2}
KIND_CODES = {"param16": 0, "grad16": 1, "optim32": 2, "activation16": 3}

# Descriptor layouts (must match the C structs in include/hm_page.h).
ADAM_CHUNK = np.dtype([("g_off", "<u8"), ("s_off", "<u8"), ("p_off", "<u8"),
                       ("n", "<u4"), ("slot", "<u4")])
GROUP_LAUNCH = np.dtype([("g_shift", "<u8"), ("p_shift", "<u8"), ("group", "<u4"),
                         ("flag", "<u4")])
GROUP_RT_BYTES = 16
SEG_CHUNK = np.dtype([("src_off", "<u8"), ("dst_off", "<u8"), ("n", "<u4"), ("slot", "<u4")])
COPY_DESC = np.dtype([("src_off", "<u8"), ("dst_off", "<u8"), ("bytes", "<u8")])
assert ADAM_CHUNK.itemsize == 32 and GROUP_LAUNCH.itemsize == 24
assert SEG_CHUNK.itemsize == 24 and COPY_DESC.itemsize == 24


class LaunchOpts(C.Structure):
    """hm_launch_opts: per-launch tuning; -1 = the process default."""
    _fields_ = [("adam_threads", C.c_int32), ("adam_variant", C.c_int32), ("grid_ctas", C.c_int32),
                ("ag_publish", C.c_int32), ("reduce_width", C.c_int32), ("reduce_wide", C.c_int32)]

    def __init__(self, adam_threads=-1, adam_variant=-1, grid_ctas=-1, ag_publish=-1,
                 reduce_width=-1, reduce_wide=-1):
        super().__init__(adam_threads, adam_variant, grid_ctas, ag_publish, reduce_width, reduce_wide)


class AdamHyperC(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("one_minus_beta1", C.c_float),
                ("beta2", C.c_float), ("one_minus_beta2", C.c_float), ("eps", C.c_float),
                ("inv_scale", C.c_float), ("max_norm", C.c_float)]


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_INT = C.c_int
_I64P = C.POINTER(C.c_int64)
_OPTS = C.POINTER(LaunchOpts)

# name -> (restype, argtypes); the set of symbols declared in include/hm_page.h.
SIGNATURES = {
    "hm_last_error": (C.c_char_p, []),
    "hm_last_error_bytes": (None, [_I64P, _I64P]),
    "hm_abi_version": (_INT, []),
    "hm_device_chunk_elems": (_INT, []),
    "hm_pt_create": (_INT, [C.POINTER(_P)]),
    "hm_pt_destroy": (_INT, [_P]),
    "hm_pt_add_pool": (_INT, [_P, _INT, _I64, _I64, _I64]),
    "hm_pt_allocate": (_INT, [_P, _INT, _INT, _I64, _I64P]),
    "hm_pt_release": (_INT, [_P, _I64, _I64P]),
    "hm_pt_page_move": (_INT, [_P, _I64, _INT, _I64P]),
    "hm_pt_tensor_merge": (_INT, [_P, _I64, _I64P]),
    "hm_pt_num_pools": (_INT, [_P]),
    "hm_pt_pool_info": (_INT, [_P, _INT, _I64P]),
    "hm_pt_allocated_pages": (_I64, [_P, _INT, _I64P, _I64]),
    "hm_pt_free_pages": (_I64, [_P, _INT, _I64P, _I64]),
    "hm_pt_page_info": (_INT, [_P, _I64, _I64P]),
    "hm_pt_tensor_ids": (_I64, [_P, _I64P, _I64]),
    "hm_pt_tensor_info": (_INT, [_P, _I64, _I64P]),
    "hm_pt_tensor_pages": (_I64, [_P, _I64, _I64P, _I64]),
    "hm_pt_tensor_segments": (_I64, [_P, _I64, _I64P, _I64]),
    "hm_adam_step": (_INT, [_P, _I64, _P, _I32, _P, _P, _INT, _P, _P, _P, _P, _INT,
                            C.POINTER(AdamHyperC), _P, _I64, _I64, _P, _P, _P, _P, _INT, _P, _P,
                            _OPTS, _P]),
    "hm_set_adam_threads": (_INT, [_INT]),
    "hm_set_adam_variant": (_INT, [_INT]),
    "hm_set_dp_reduce_ctas": (_INT, [_INT]),
    "hm_set_dp_reduce_width": (_INT, [_INT]),
    "hm_set_dp_reduce_wide": (_INT, [_INT]),
    "hm_set_ag_publish": (_INT, [_INT]),
    "hm_set_dp_update_ctas": (_INT, [_INT]),
    "hm_adam_prologue": (_INT, [_P, _I32, _P, C.POINTER(AdamHyperC), _P, _I64, _I64, _P, _P, _P,
                                _P, _INT, _P, _P, _P]),
    "hm_adam_main": (_INT, [_P, _I64, _P, _P, _P, _INT, _P, _P, _P, _P, _INT,
                            C.POINTER(AdamHyperC), _OPTS, _P]),
    "hm_adam_layer": (_INT, [_P, _I64, _P, _P, _INT, _P, _P, _P, _P, C.POINTER(AdamHyperC), _P, _I64,
                             _P, _P, _P, _P, _P, _P, _P, _P]),
    "hm_dp_reduce_check": (_INT, [_P, _INT, _P, _P, _INT, _P, _I64, _P, _P, _OPTS, _P]),
    "hm_dp_flags_merge": (_INT, [_P, _P, _INT, _INT, _P, _P, _P]),
    "hm_adam_main_ag": (_INT, [_P, _I64, _P, _P, _P, _INT, _P, _P, _P, _P, _INT, _P, _INT,
                               C.POINTER(AdamHyperC), _OPTS, _P]),
    "hm_dp_onepass_update": (_INT, [_P, _I64, _P, _P, _P, _I64, _P, _P, _INT, _INT, _P, _P, _P, _P,
                                     C.POINTER(AdamHyperC), _OPTS, _P]),
    "hm_dp_push_grad": (_INT, [_P, _I64, _P, _P, _I64, _P]),
    "hm_dp_onepass_recv_update": (_INT, [_P, _I64, _P, _P, _P, _I64, _P, _P, _I64, _INT, _INT, _P, _INT, _INT,
                                          _P, _P, _P, _P, C.POINTER(AdamHyperC), _P]),
    "hm_dp_onepass_finalize": (_INT, [_P, _INT, _INT, _P, _P, _P, _P, _P, _P]),
    "hm_dp_republish_rejected": (_INT, [_P, _I64, _P, _P, _P, _I64, _P, _P, _INT, _INT, _P]),
    "hm_accumulate": (_INT, [_P, _INT, _P, _INT, _P, _I64, _INT, _P, _P, _P, _P, _P, _OPTS, _P]),
    "hm_stats_take": (_INT, [_P, _I32, _P, _P, _P, _P, _P]),
    "hm_cast": (_INT, [_P, _INT, _P, _INT, _P, _I64, _P]),
    "hm_reduce_stats": (_INT, [_P, _INT, _P, _I64, _P, _P, _P, _P]),
    "hm_copy_runs": (_INT, [_P, _P, _P, _I64, _P]),
    "hm_memcpy_runs": (_INT, [_P, _P, _P, _I64, _INT, _P]),
    "hm_spin": (_INT, [_I64, _P]),
    "hm_host_alloc": (_INT, [_I64, C.POINTER(_P)]),
    "hm_host_free": (_INT, [_P]),
}

_lib = None


def lib():
    """Load libhm_page.so once; fail loudly if it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (no CPU fallback exists)")
        handle = C.CDLL(os.fspath(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    return lib().hm_last_error().decode(errors="replace")


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == HM_OK:
        return
    msg = last_error()
    if rc == HM_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == HM_ERR_ALLOCATION:
        req, avail = C.c_int64(), C.c_int64()
        lib().hm_last_error_bytes(C.byref(req), C.byref(avail))
        raise AllocationError(msg, req.value, avail.value)
    if rc == HM_ERR_MOVE:
        raise MoveError(msg)
    if rc == HM_ERR_PROTOCOL:
        raise ProtocolError(msg)
    if rc == HM_ERR_KEY:
        raise KeyError(msg)
    raise NativeError(f"libhm_page error {rc}: {msg}")


def i64_buf(n: int):
    return (C.c_int64 * max(n, 1))()


def stream_ptr(stream) -> int:
    """cudaStream_t of a torch stream (0 = legacy default)."""
    return int(stream.cuda_stream) if stream is not None else 0
