"""ctypes binding of the C ABI declared in include/slp_b200.h.

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``)
at ``paper_1805_01407_b200/_lib/libslp_b200.so``.  There is no fallback: if
the library is missing every entry point raises ``NativeLibraryMissing``.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SLP_LIB") or os.path.join(_HERE, "_lib", "libslp_b200.so")  # SLP_LIB: A/B builds

# status codes (include/slp_b200.h)
SLP_OK = 0
SLP_ERR_INVALID = -1
SLP_ERR_UNKNOWN_GENERATOR = -2
SLP_ERR_UNSUPPORTED = -3
SLP_ERR_ZERO_STATE = -4
SLP_ERR_CUDA = -5
SLP_ERR_ALGEBRA = -6
SLP_ERR_BUFFER = -7

OUT_NATIVE, OUT_U64, OUT_F64, OUT_F32 = 0, 1, 2, 3
STREAM_MAJOR, POSITION_MAJOR = 0, 1
FUSE_INT, FUSE_F64, FUSE_EXACT = 1, 2, 4

u64p = ctypes.POINTER(ctypes.c_uint64)
vp = ctypes.c_void_p


class NativeLibraryMissing(RuntimeError):
    pass


class Gf2Error(Exception):
    """Internal GF(2) self-check failure (mirrors slprng.gf2.Gf2Error, gf2.py:48-53)."""


class CudaError(RuntimeError):
    pass


class GenInfo(ctypes.Structure):
    _fields_ = [
        ("id", ctypes.c_int32), ("family", ctypes.c_int32), ("k", ctypes.c_int32),
        ("w", ctypes.c_int32), ("a", ctypes.c_int32), ("b", ctypes.c_int32), ("c", ctypes.c_int32),
        ("scrambler", ctypes.c_int32), ("word_i", ctypes.c_int32), ("word_j", ctypes.c_int32),
        ("R", ctypes.c_int32), ("S", ctypes.c_uint64), ("T", ctypes.c_uint64), ("name", ctypes.c_char * 32),
    ]


class Checksum(ctypes.Structure):
    _fields_ = [
        ("sum_lo", ctypes.c_uint64), ("sum_hi", ctypes.c_uint64), ("xor_all", ctypes.c_uint64),
        ("low_sum", ctypes.c_uint64), ("count", ctypes.c_uint64), ("fsum", ctypes.c_double),
    ]


CHECKSUM_BYTES = ctypes.sizeof(Checksum)

# name -> (restype, argtypes); the exported surface of include/slp_b200.h
SIGNATURES = {
    "slp_num_generators": (ctypes.c_int, []),
    "slp_generator_id": (ctypes.c_int, [ctypes.c_char_p]),
    "slp_generator_info": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(GenInfo)]),
    "slp_register_generator": (ctypes.c_int, [ctypes.POINTER(GenInfo)]),
    "slp_char_poly": (ctypes.c_int, [ctypes.c_int, u64p, ctypes.c_int]),
    "slp_jump_poly": (ctypes.c_int, [ctypes.c_int, u64p, ctypes.c_int, u64p, ctypes.c_int]),
    "slp_init_plan_poly": (ctypes.c_int64, [ctypes.c_int, u64p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, u64p,
                                            ctypes.c_int]),
    "slp_host_jump": (ctypes.c_int, [ctypes.c_int, u64p, ctypes.c_int, u64p]),
    "slp_engine_char_poly": (ctypes.c_int, [ctypes.c_int] * 6 + [u64p, ctypes.c_int]),
    "slp_engine_jump_poly": (ctypes.c_int, [ctypes.c_int] * 6 + [u64p, ctypes.c_int, u64p, ctypes.c_int]),
    "slp_init_substreams": (ctypes.c_int, [ctypes.c_int, u64p, ctypes.c_uint64, u64p, ctypes.c_int, vp,
                                           ctypes.c_uint64, ctypes.c_uint64, vp]),
    "slp_jump_states": (ctypes.c_int, [ctypes.c_int, u64p, ctypes.c_int, vp, ctypes.c_uint64, vp,
                                       ctypes.c_uint64, ctypes.c_uint64, vp]),
    "slp_split_factor": (ctypes.c_int64, [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64]),
    "slp_split_substreams": (ctypes.c_int, [ctypes.c_int, vp, ctypes.c_uint64, ctypes.c_uint64, u64p, ctypes.c_int,
                                            ctypes.c_uint64, vp, ctypes.c_uint64, vp]),
    "slp_fill": (ctypes.c_int, [ctypes.c_int, vp, vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                ctypes.c_int, ctypes.c_int, vp, ctypes.c_uint64, vp]),
    "slp_laned_fill": (ctypes.c_int, [ctypes.c_int, u64p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, vp, vp,
                                      vp]),
    "slp_fill_checksum": (ctypes.c_int, [ctypes.c_int, vp, vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_int, vp, ctypes.c_uint64, vp, vp, ctypes.c_size_t, vp]),
    "slp_fused_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_uint64]),
    "slp_fused": (ctypes.c_int, [ctypes.c_int, vp, vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.c_int, vp, vp, ctypes.c_size_t, vp]),
    "slp_hwd_count": (ctypes.c_int, [ctypes.c_int, vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                     ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, u64p, u64p, u64p, vp]),
    "slp_device_cache_bytes": (ctypes.c_size_t, [ctypes.c_int]),
    "slp_set_fill_pace": (ctypes.c_int, [ctypes.c_int]),
    "slp_status_str": (ctypes.c_char_p, [ctypes.c_int]),
    "slp_last_error": (ctypes.c_char_p, []),
    "slp_build_info": (ctypes.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


def lib():
    """The loaded library (raises NativeLibraryMissing if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} is not built; run `make` in the repo root or __graft_entry__.build()")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def status_error(rc: int, what: str) -> Exception:
    L = lib()
    msg = f"{what}: {L.slp_status_str(rc).decode()}"
    detail = L.slp_last_error().decode()
    if detail:
        msg += f" ({detail})"
    if rc == SLP_ERR_UNKNOWN_GENERATOR:
        return KeyError(msg)
    if rc in (SLP_ERR_INVALID, SLP_ERR_ZERO_STATE, SLP_ERR_UNSUPPORTED, SLP_ERR_BUFFER):
        return ValueError(msg)
    if rc == SLP_ERR_ALGEBRA:
        return Gf2Error(msg)
    return CudaError(msg)


def check(rc: int, what: str):
    if rc != SLP_OK:
        raise status_error(rc, what)


def int_to_words(x: int, nwords: int | None = None):
    """Little-endian u64 words of a non-negative Python int (ctypes array)."""
    if x < 0:
        raise ValueError("negative integer")
    n = max(1, (x.bit_length() + 63) // 64) if nwords is None else nwords
    arr = (ctypes.c_uint64 * n)()
    for i in range(n):
        arr[i] = (x >> (64 * i)) & 0xFFFFFFFFFFFFFFFF
    return arr, n


def words_to_int(arr) -> int:
    v = 0
    for i in range(len(arr)):
        v |= int(arr[i]) << (64 * i)
    return v
