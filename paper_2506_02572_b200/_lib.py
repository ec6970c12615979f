"""ctypes loader for libhata.so (the C ABI in include/hata.h).

Argument marshalling only: no arithmetic of the method happens in Python.
If the shared library is missing this module raises -- there is no CPU or
PyTorch fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# HATA_LIB=libhata_trace.so selects the diagnostics build (tools/trace_decode.py)
LIB_PATH = os.path.join(_HERE, os.environ.get("HATA_LIB", "libhata.so"))

HATA_OK = 0
HATA_F32 = 0
HATA_BF16 = 1
HATA_OPT_SELECTION_HINT = 0
HATA_OPT_PDL = 1
HATA_OPT_COOPERATIVE = 2

c_i32 = ctypes.c_int
c_i64 = ctypes.c_int64
c_ptr = ctypes.c_void_p
c_f32 = ctypes.c_float
c_size = ctypes.c_size_t


class Strides(ctypes.Structure):
    _fields_ = [("sb", c_i64), ("sh", c_i64), ("st", c_i64)]


_SIGS = {
    "hata_hash_keys": (c_i32, [c_ptr, Strides, c_i32, c_ptr, c_i32, c_i32, c_i32, c_i32, c_i64, c_i64, c_i64,
                               c_ptr, Strides, c_ptr]),
    "hata_prefill_write": (c_i32, [c_ptr, c_ptr, Strides, c_ptr, c_ptr, Strides, c_i32, c_ptr, c_i32, c_i32, c_i32,
                                   c_i32, c_i64, c_i64, c_i64, c_ptr, Strides, c_ptr]),
    "hata_append": (c_i32, [c_ptr, c_ptr, c_i32, c_ptr, c_ptr, c_ptr, Strides, c_ptr, Strides, c_ptr, c_i64, c_i32,
                            c_i32, c_i32, c_i32, c_ptr]),
    "hata_decode_topk_attn": (c_i32, [c_ptr, c_ptr, c_ptr, Strides, c_i32, c_ptr, Strides, c_ptr, c_i32, c_i32,
                                      c_i32, c_i32, c_i32, c_ptr, c_i64, c_i32, c_f32, c_ptr, c_i32, c_ptr, c_ptr,
                                      c_ptr, c_ptr, c_size, c_ptr]),
    "hata_decode_step": (c_i32, [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, Strides, c_i32, c_ptr, Strides, c_ptr, c_i32,
                                 c_i32, c_i32, c_i32, c_i32, c_ptr, c_i64, c_i64, c_i32, c_f32, c_ptr, c_i32, c_ptr,
                                 c_ptr, c_ptr, c_ptr, c_size, c_ptr]),
    "hata_decode_step_paged": (c_i32, [c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, Strides, c_i32, c_ptr, Strides, c_ptr,
                                       c_i32, c_i32, c_ptr, c_i32, c_i32, c_i32, c_i32, c_i32, c_ptr, c_i64, c_i32,
                                       c_f32, c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_size, c_ptr]),
    "hata_decode_workspace_size": (c_size, [c_i32, c_i32, c_i32, c_i32, c_i32, c_i64, c_i32, c_i32]),
    "hata_decode_ranks": (c_i32, [c_i32, c_i32, c_i32, c_i32, c_i32, c_i64, c_i32, c_i32]),
    "hata_shard_candidates": (c_i32, [c_ptr, c_i32, c_ptr, Strides, c_ptr, c_i32, c_i32, c_i32, c_i32, c_i32, c_ptr,
                                      c_i64, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_size, c_ptr]),
    "hata_shard_select": (c_i32, [c_ptr, c_ptr, c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_ptr, c_i64,
                                  c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "hata_shard_partial_attn": (c_i32, [c_ptr, c_ptr, c_ptr, Strides, c_i32, c_ptr, c_ptr, c_i32, c_i32, c_i32,
                                        c_i32, c_i32, c_f32, c_i32, c_ptr, c_ptr]),
    "hata_shard_combine": (c_i32, [c_ptr, c_i32, c_i32, c_i32, c_i32, c_ptr, c_i32, c_ptr]),
    "hata_set_option": (c_i32, [c_i32, c_i32]),
    "hata_status_string": (ctypes.c_char_p, [c_i32]),
    "hata_last_error": (ctypes.c_char_p, []),
    "hata_version": (ctypes.c_char_p, []),
    "hata_debug_trace": (c_i32, [c_ptr]),
    "hata_debug_timestamp": (c_i32, [c_ptr, c_ptr]),
}
EXPORTS = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load libhata.so once; raise (never fall back) if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"libhata.so not found at {path}; build it with `python -m paper_2506_02572_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class HataError(RuntimeError):
    pass


def check(status: int, what: str):
    if status != HATA_OK:
        lib = load()
        raise HataError(f"{what}: {lib.hata_status_string(status).decode()} "
                        f"{lib.hata_last_error().decode()}".strip())
