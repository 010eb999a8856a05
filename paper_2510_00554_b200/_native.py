"""ctypes binding of ``lib/libsentinel_b200.so`` (C ABI: include/sentinel_b200.h).

The library is the only implementation of the hashing path: if it cannot be
loaded, every hashing entry point raises ``ResourceError`` -- nothing falls
back to the CPU.
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, c_char_p, c_int, c_size_t, c_uint32, c_uint64, c_void_p
from pathlib import Path
from typing import Optional

from .errors import ResourceError, raise_for_status

import os

# SNT_LIB_PATH lets kernel experiments (tools/) load an alternative build of the same ABI
LIB_PATH = Path(os.environ.get("SNT_LIB_PATH") or Path(__file__).resolve().parent / "lib" / "libsentinel_b200.so")

SNT_LEVELS_TO_ROOT = 0xFFFFFFFF
SCHEDULE_PERSISTENT, SCHEDULE_FUSED, SCHEDULE_GRID = 0, 1, 2
SAMPLES_UNKNOWN, SAMPLES_UNIFORM, SAMPLES_RAGGED = 0, 1, 2      # snt_samples_shape
ABI_VERSION = 3

# name -> (restype, argtypes); mirrors include/sentinel_b200.h one to one
SIGNATURES = {
    "snt_strerror": (c_char_p, [c_int]),
    "snt_last_cuda_error": (c_char_p, []),
    "snt_abi_version": (c_uint32, []),
    "snt_debug_launch_count": (c_uint64, []),
    "snt_digest_len": (c_uint32, [c_int]),
    "snt_model_plan_create": (c_int, [POINTER(c_void_p), POINTER(c_uint64), c_uint32, c_uint32, c_void_p,
                                      POINTER(c_void_p)]),
    "snt_model_plan_destroy": (None, [c_void_p]),
    "snt_model_plan_leaf_count": (c_uint64, [c_void_p]),
    "snt_model_plan_total_bytes": (c_uint64, [c_void_p]),
    "snt_merkle_schedule": (c_int, [c_int]),
    "snt_debug_fused_trace": (None, [c_void_p]),
    "snt_merkle_work_bytes": (c_size_t, [c_int, c_uint64]),
    "snt_merkle_work_init": (c_int, [c_void_p, c_size_t, c_void_p]),
    "snt_memcpy_h2d_batch": (c_int, [c_void_p, c_void_p, c_void_p, c_uint32, c_void_p]),
    "snt_gather_chunk_bytes": (c_uint32, []),
    "snt_gather_spans": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_uint32, c_uint64, c_uint32, c_void_p,
                                 c_void_p]),
    "snt_merkle_leaves": (c_int, [c_void_p, c_int, c_uint64, c_uint64, c_void_p, c_void_p]),
    "snt_merkle_inplace": (c_int, [c_void_p, c_int, c_uint64, c_uint64, c_uint32, c_void_p, c_void_p,
                                   c_size_t, c_void_p, c_void_p]),
    "snt_hash_blocks": (c_int, [c_int, c_void_p, c_void_p, c_void_p, c_uint64, c_void_p, c_void_p]),
    "snt_merkle_reduce_levels": (c_int, [c_int, c_void_p, c_uint64, c_uint64, c_uint64, c_uint32,
                                         c_void_p, c_size_t, c_void_p, c_void_p]),
    "snt_merkle_root": (c_int, [c_int, c_void_p, c_uint64, c_void_p, c_size_t, c_void_p, c_void_p]),
    "snt_lthash_samples": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_uint64, c_uint32,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "snt_device_reads_pinned_host": (c_int, []),
    "snt_lthash_samples_shaped": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_uint64, c_uint32,
                                          c_void_p, c_void_p, c_void_p, c_void_p, c_uint32, c_void_p]),
    "snt_lthash_rows": (c_int, [c_void_p, c_uint64, c_uint64, c_void_p, c_void_p, c_void_p, c_uint32,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "snt_lthash_model": (c_int, [c_void_p, c_uint64, c_uint64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "snt_lthash_model_layers": (c_int, [c_void_p, c_uint64, c_uint64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "snt_merkle_roots_segmented": (c_int, [c_int, c_void_p, POINTER(c_uint64), c_uint32, c_void_p, c_void_p,
                                           c_size_t, c_void_p, c_void_p]),
    "snt_lt_reduce": (c_int, [c_void_p, c_uint64, c_void_p, c_void_p]),
    "snt_lt_finalize": (c_int, [c_void_p, c_uint32, c_void_p, c_void_p]),
}

_lib: Optional[ctypes.CDLL] = None


def load() -> ctypes.CDLL:
    """Load the native library once; raise ``ResourceError`` if it is absent or stale."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ResourceError(
            f"native library {LIB_PATH} is missing; build it with "
            "`python -m paper_2510_00554_b200.build` (there is no CPU fallback)")
    try:
        lib = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:
        raise ResourceError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (restype, argtypes) in SIGNATURES.items():
        try:
            fn = getattr(lib, name)
        except AttributeError as exc:
            raise ResourceError(f"{LIB_PATH} does not export {name}; rebuild it") from exc
        fn.restype = restype
        fn.argtypes = argtypes
    if lib.snt_abi_version() != ABI_VERSION:
        raise ResourceError(f"{LIB_PATH} has ABI {lib.snt_abi_version()}, expected {ABI_VERSION}; rebuild it")
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    """Map a ``snt_status`` to the reference's exception classes (errors.py:4-33)."""
    if status == 0:
        return
    lib = load()
    detail = lib.snt_strerror(status).decode()
    if status == -5:
        cuda = lib.snt_last_cuda_error().decode()
        if cuda:
            detail += f" ({cuda})"
    raise_for_status(status, what, detail)
