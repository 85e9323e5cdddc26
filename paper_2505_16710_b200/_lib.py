"""ctypes binding of libseco.so (include/seco.h).  Argument marshalling only:
every step of the hot path runs inside the library's CUDA kernels.  Fails loudly
if the library is missing -- there is no fallback of any kind."""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, os.environ.get("SECO_LIB_VARIANT", "libseco.so"))

SECO_OK, SECO_ERR_ARG, SECO_ERR_UNSUPPORTED, SECO_ERR_CUDA = 0, 1, 2, 3
SECO_BF16, SECO_FP32_DEBUG = 0, 1
SPACO_PAPER, SPACO_HT, SPACO_BERNOULLI = 0, 1, 2

EXPORTS = ("seco_workspace_size", "seco_chunk_forward", "seco_chunk_backward", "spaco_chunk_skip",
           "spaco_sample_and_scale",
           "seco_lora_workspace_size", "seco_lora_grad",
           "seco_status_string", "seco_last_error", "seco_last_launch_count", "seco_debug_bwd_schedule",
           "seco_debug_fwd_schedule",
           "seco_debug_check_enabled", "seco_debug_check_word", "seco_debug_check_selftest")


class SecoShape(ctypes.Structure):
    _fields_ = [("hq", ctypes.c_int32), ("hkv", ctypes.c_int32), ("d", ctypes.c_int32),
                ("chunk", ctypes.c_int32), ("num_chunks", ctypes.c_int32),
                ("softmax_scale", ctypes.c_float), ("dtype", ctypes.c_int32),
                ("q_head_stride", ctypes.c_int64), ("q_row_stride", ctypes.c_int64),
                ("kv_head_stride", ctypes.c_int64), ("kv_row_stride", ctypes.c_int64),
                ("flags", ctypes.c_int32)]


SECO_FLAG_DETERMINISTIC = 1
SECO_FLAG_PREV_INDEPENDENT = 2


class LoraShape(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int32), ("n_in", ctypes.c_int32), ("n_out", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("dtype", ctypes.c_int32), ("ldx", ctypes.c_int64), ("ldy", ctypes.c_int64),
                ("flags", ctypes.c_int32)]


class SecoError(RuntimeError):
    pass


_lib = None


def load():
    """Load libseco.so (built in-tree by ``python -m paper_2505_16710_b200.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SecoError(f"{LIB_PATH} is missing: build it with `python -m paper_2505_16710_b200.build` "
                        "(there is no fallback path)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, f32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_float, ctypes.c_size_t
    P = ctypes.POINTER
    lib.seco_workspace_size.argtypes = [P(SecoShape)]
    lib.seco_workspace_size.restype = sz
    lib.seco_chunk_forward.argtypes = [P(SecoShape), i32, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.seco_chunk_forward.restype = i32
    lib.seco_chunk_backward.argtypes = [P(SecoShape), i32, vp, vp, vp, vp, vp, vp, f32, f32,
                                        vp, vp, vp, vp, vp, sz, vp]
    lib.seco_chunk_backward.restype = i32
    lib.spaco_chunk_skip.argtypes = [P(SecoShape), i32, vp, vp, vp, vp, vp]
    lib.spaco_chunk_skip.restype = i32
    lib.spaco_sample_and_scale.argtypes = [i32, i32, ctypes.c_uint64, f32, i32, P(i32), P(i32), P(f32), P(f32)]
    lib.spaco_sample_and_scale.restype = i32
    lib.seco_lora_workspace_size.argtypes = [P(LoraShape)]
    lib.seco_lora_workspace_size.restype = sz
    lib.seco_lora_grad.argtypes = [P(LoraShape), vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.seco_lora_grad.restype = i32
    lib.seco_status_string.argtypes = [i32]
    lib.seco_status_string.restype = ctypes.c_char_p
    lib.seco_last_error.argtypes = []
    lib.seco_last_error.restype = ctypes.c_char_p
    lib.seco_last_launch_count.argtypes = []
    lib.seco_last_launch_count.restype = i32
    if hasattr(lib, "seco_debug_check_word"):
        lib.seco_debug_check_enabled.argtypes = []
        lib.seco_debug_check_enabled.restype = i32
        lib.seco_debug_check_word.argtypes = []
        lib.seco_debug_check_word.restype = ctypes.c_uint64
        lib.seco_debug_check_selftest.argtypes = [vp]
        lib.seco_debug_check_selftest.restype = i32
    if hasattr(lib, "seco_debug_bwd_schedule"):      # (older experiment variants lack it)
        lib.seco_debug_bwd_schedule.argtypes = [i32, i32, i32, i32, i32, P(i32)]
        lib.seco_debug_bwd_schedule.restype = i32
    if hasattr(lib, "seco_debug_fwd_schedule"):
        lib.seco_debug_fwd_schedule.argtypes = [P(SecoShape), i32, i32, P(i32)]
        lib.seco_debug_fwd_schedule.restype = i32
    _lib = lib
    return lib


def check(status: int, what: str):
    if status != SECO_OK:
        lib = load()
        raise SecoError(f"{what}: {lib.seco_status_string(status).decode()}: {lib.seco_last_error().decode()}")
