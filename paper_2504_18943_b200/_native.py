"""ctypes binding of the C ABI in ``include/ltlsynth_b200.h``.

This is the binding INTEGRATION.md describes for a reference maintainer: plain
pointers and sizes, no torch types.  Loading fails loudly -- there is no CPU
fallback behind it, and the in-tree shared library must have been built with
``python -c "import __graft_entry__ as g; g.build()"`` (nvcc, sm_100a).
"""

from __future__ import annotations

import ctypes
import os
import pathlib

# LTLB200_LIB selects a tuning variant built by _build.build_native(defines=..., out=...)
LIB_PATH = pathlib.Path(os.environ.get("LTLB200_LIB") or pathlib.Path(__file__).resolve().parent / "_lib" / "libltlsynth_b200.so")

OK, TIME_BUDGET, MEMORY_BUDGET = 0, 1, 2
ERR_ARGUMENT, ERR_CUDA, ERR_UNSUPPORTED = -1, -2, -3
ABI_VERSION = 2

# every symbol include/ltlsynth_b200.h declares
EXPORTED_SYMBOLS = (
    "ltlb200_abi_version",
    "ltlb200_last_error",
    "ltlb200_device_count",
    "ltlb200_create",
    "ltlb200_set_weights",
    "ltlb200_set_regex",
    "ltlb200_destroy",
    "ltlb200_reset",
    "ltlb200_trim",
    "ltlb200_expand_level",
    "ltlb200_route_begin",
    "ltlb200_exchange_recv",
    "ltlb200_owner_reduce",
    "ltlb200_winners_export",
    "ltlb200_level_commit",
    "ltlb200_level_abort",
    "ltlb200_seps_copy",
    "ltlb200_key_bytes",
    "ltlb200_now",
    "ltlb200_level_info",
    "ltlb200_level_candidates",
    "ltlb200_holds_separator",
    "ltlb200_num_levels",
    "ltlb200_level_copy",
    "ltlb200_level_device",
    "ltlb200_entry",
    "ltlb200_approx_bytes",
    "ltlb200_get_stats",
)


class NativeEngineError(RuntimeError):
    """The CUDA engine is missing, unusable, or reported an error."""


class Stats(ctypes.Structure):
    _fields_ = [
        ("constructed", ctypes.c_uint64),
        ("unique", ctypes.c_uint64),
        ("kernel_launches", ctypes.c_uint64),
        ("enumerate_ms", ctypes.c_double),
        ("finalize_ms", ctypes.c_double),
        ("enumerate_launches", ctypes.c_uint64),
        ("enumerate_candidates", ctypes.c_uint64),
        ("table_slots", ctypes.c_uint64),
        ("table_rebuilds", ctypes.c_uint64),
        ("device_bytes", ctypes.c_uint64),
        ("h2d_bytes", ctypes.c_uint64),
        ("d2h_bytes", ctypes.c_uint64),
        ("row_bytes", ctypes.c_uint32),
        ("key_bytes", ctypes.c_uint32),
        ("alloc_ms", ctypes.c_double),
        ("rebuild_host_ms", ctypes.c_double),
        ("create_ms", ctypes.c_double),
        ("route_ms", ctypes.c_double),
        ("probe_ms", ctypes.c_double),
        ("routed_records", ctypes.c_uint64),
        ("received_records", ctypes.c_uint64),
        ("tiny_ms", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None


def load():
    """Load the shared library and declare its prototypes (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeEngineError(
            f"{LIB_PATH} is missing: build the CUDA engine first (__graft_entry__.build()); "
            "this package has no CPU fallback"
        )
    try:
        L = ctypes.CDLL(str(LIB_PATH))
    except OSError as err:
        raise NativeEngineError(f"cannot load {LIB_PATH}: {err}") from err
    i32, i64, u32, u64, p, dbl = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64,
                                  ctypes.c_void_p, ctypes.c_double)
    L.ltlb200_abi_version.restype = ctypes.c_int
    L.ltlb200_last_error.restype = ctypes.c_char_p
    L.ltlb200_device_count.restype = ctypes.c_int
    L.ltlb200_create.restype = p
    L.ltlb200_create.argtypes = [i32, i32, p, p, p, i32, i32, u64, p]
    L.ltlb200_set_weights.restype = ctypes.c_int
    L.ltlb200_set_weights.argtypes = [p, p]
    L.ltlb200_set_regex.restype = ctypes.c_int
    L.ltlb200_set_regex.argtypes = [p, i32, p, p, u64]
    L.ltlb200_destroy.argtypes = [p]
    L.ltlb200_destroy.restype = None
    L.ltlb200_trim.restype = None
    L.ltlb200_trim.argtypes = [i32]
    L.ltlb200_reset.restype = ctypes.c_int
    L.ltlb200_reset.argtypes = [p]
    L.ltlb200_expand_level.restype = ctypes.c_int
    L.ltlb200_expand_level.argtypes = [p, i32, u32, i32, i64, u64, dbl,
                                       ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)]
    pu64 = ctypes.POINTER(u64)
    pp = ctypes.POINTER(p)
    L.ltlb200_route_begin.restype = ctypes.c_int
    L.ltlb200_route_begin.argtypes = [p, i32, u32, i32, dbl, i32, i32, pu64, pu64, pp, pp, pu64, pu64]
    L.ltlb200_exchange_recv.restype = ctypes.c_int
    L.ltlb200_exchange_recv.argtypes = [p, u64, pp, pp]
    L.ltlb200_owner_reduce.restype = ctypes.c_int
    L.ltlb200_owner_reduce.argtypes = [p, u64, pu64, pp, pu64]
    L.ltlb200_winners_export.restype = ctypes.c_int
    L.ltlb200_winners_export.argtypes = [p, u64, pu64, pp, pp]
    L.ltlb200_level_abort.restype = ctypes.c_int
    L.ltlb200_level_abort.argtypes = [p]
    L.ltlb200_level_commit.restype = ctypes.c_int
    L.ltlb200_level_commit.argtypes = [p, u64, p, u64, p, i32, i64, u64, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.ltlb200_seps_copy.restype = i64
    L.ltlb200_seps_copy.argtypes = [p, p, u64]
    L.ltlb200_key_bytes.restype = i32
    L.ltlb200_key_bytes.argtypes = [p]
    L.ltlb200_now.restype = dbl
    L.ltlb200_level_info.restype = ctypes.c_int
    L.ltlb200_level_info.argtypes = [p, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.ltlb200_level_candidates.restype = ctypes.c_int
    L.ltlb200_level_candidates.argtypes = [p, i32, ctypes.c_uint32, ctypes.POINTER(i64)]
    L.ltlb200_holds_separator.restype = i32
    L.ltlb200_holds_separator.argtypes = [p]
    L.ltlb200_num_levels.restype = i32
    L.ltlb200_num_levels.argtypes = [p]
    L.ltlb200_level_copy.restype = ctypes.c_int
    L.ltlb200_level_copy.argtypes = [p, i32, i64, i64, p, p, p, p]
    L.ltlb200_level_device.restype = ctypes.c_int
    L.ltlb200_level_device.argtypes = [p, i32, pp, pp]
    L.ltlb200_entry.restype = ctypes.c_int
    L.ltlb200_entry.argtypes = [p, i64, ctypes.POINTER(i32), ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.ltlb200_approx_bytes.restype = u64
    L.ltlb200_approx_bytes.argtypes = [p]
    L.ltlb200_get_stats.restype = ctypes.c_int
    L.ltlb200_get_stats.argtypes = [p, ctypes.POINTER(Stats)]
    if L.ltlb200_abi_version() != ABI_VERSION:
        raise NativeEngineError("libltlsynth_b200.so was built from a different header version; rebuild it")
    _lib = L
    return L


def last_error() -> str:
    return load().ltlb200_last_error().decode("utf-8", "replace")


def check(status: int, what: str) -> int:
    if status < 0:
        raise NativeEngineError(f"{what} failed (status {status}): {last_error()}")
    return status
