"""ctypes binding of libhinm_b200.so (the C ABI in include/hinm_b200.h).

This is the same binding a maintainer would add to the reference.  The
library is required: if it is missing or unloadable every device entry point raises
:class:`DeviceError` -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HINM_B200_LIB", os.path.join(_HERE, "libhinm_b200.so"))

c_int, c_i64, c_vp, c_size = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t

STATUS_TO_EXCEPTION = {
    1: E.ShapeMismatch,
    2: IndexError,
    3: E.InvariantViolation,
    4: E.GroupingError,
    5: E.BudgetError,
    6: E.DimensionError,
    7: ValueError,
    8: E.DeviceError,
    9: E.DeviceError,
    10: E.DimensionError,
}

HINM_ORDER_SIGMA, HINM_ORDER_ORIGINAL = 0, 1
HINM_SELECT_SCORES, HINM_SELECT_MASK = 0, 1
HINM_UNPACK_REFERENCE_VIEW, HINM_UNPACK_OPERAND_IMAGE = 0, 1


class PackStruct(ctypes.Structure):
    """Mirror of hinm_pack_t (``group`` points at the union-group pseudo pack, if built)."""


PackStruct._fields_ = [
    ("m", ctypes.c_int32), ("n", ctypes.c_int32), ("V", ctypes.c_int32),
    ("N", ctypes.c_int32), ("M", ctypes.c_int32), ("T", ctypes.c_int32),
    ("total_keep", c_i64),
    ("tile_ptr", c_vp), ("vec_idx", c_vp), ("nm_pos", c_vp), ("kept_bf16", c_vp),
    ("sigma_o", c_vp),
    ("kpad_cap", c_i64), ("meta_words_cap", c_i64),
    ("tile_kofs", c_vp), ("tile_eofs", c_vp), ("gidx", c_vp), ("a_vals", c_vp),
    ("a_meta", c_vp),
    ("group", ctypes.POINTER(PackStruct)), ("pair", ctypes.c_int32), ("rows", ctypes.c_int32),
    ("image", ctypes.c_int32),
]
IMAGE_AUTO, IMAGE_TILES, IMAGE_GROUPS = 0, 1, 2


class ChainStep(ctypes.Structure):
    """Mirror of hinm_chain_step_t."""

    _fields_ = [("pack", ctypes.POINTER(PackStruct)), ("src", ctypes.c_int32),
                ("dst", ctypes.c_int32), ("out_order", ctypes.c_int32)]


_SIGNATURES = {
    "hinm_version": ([], ctypes.c_char_p),
    "hinm_status_string": ([c_int], ctypes.c_char_p),
    "hinm_compress_workspace": ([c_int, c_int, c_int, c_int, ctypes.POINTER(c_size)], c_int),
    "hinm_pack_capacity": ([c_int, c_int, c_int, c_i64, ctypes.POINTER(c_i64),
                            ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)], c_int),
    "hinm_vector_prune": ([c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_int, c_int, c_int,
                           c_int, c_i64, c_vp, c_vp, c_vp, c_vp, c_size, c_vp], c_int),
    "hinm_nm_select": ([c_int, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp,
                        c_vp, c_int, c_int, c_int, c_int, c_int, c_i64, c_vp, c_vp, c_vp, c_vp,
                        c_vp], c_int),
    "hinm_pack_build": ([ctypes.POINTER(PackStruct), c_vp], c_int),
    "hinm_compress_bf16": ([c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, ctypes.POINTER(PackStruct),
                            c_vp, c_vp, c_size, c_vp], c_int),
    "hinm_unpack_to_reference": ([ctypes.POINTER(PackStruct), c_int, c_vp, c_vp, c_vp, c_vp, c_vp,
                                  c_vp], c_int),
    "hinm_spmm_bf16": ([ctypes.POINTER(PackStruct), c_vp, c_i64, c_int, c_vp, c_i64, c_int, c_vp],
                       c_int),
    "hinm_spmm_simt_f32": ([ctypes.POINTER(PackStruct), c_vp, c_i64, c_int, c_vp, c_i64, c_int,
                            c_vp], c_int),
    "hinm_chain_workspace": ([ctypes.POINTER(c_i64), c_int, c_int, ctypes.POINTER(c_size)], c_int),
    "hinm_chain_run_host": ([ctypes.POINTER(ChainStep), c_int, ctypes.POINTER(c_i64), c_int, c_int,
                             c_vp, c_i64, c_int, c_vp, c_i64, c_int, c_vp, c_size, c_vp], c_int),
    "hinm_last_launch_count": ([], c_int),
    "hinm_last_image": ([], c_int),
    "hinm_stream_fence": ([c_vp], c_int),
    "hinm_icp_costs": ([c_vp, c_int, c_int, c_vp, c_vp, c_int, c_int, c_int, c_vp, c_vp], c_int),
    "hinm_lex_assignment": ([c_vp, c_int, c_vp], c_int),
    "hinm_ocp_workspace": ([c_int, c_int, c_int, ctypes.POINTER(c_size)], c_int),
    "hinm_sq_dists": ([c_vp, c_int, c_vp, c_int, c_int, c_vp, c_vp], c_int),
    "hinm_group_workspace": ([ctypes.POINTER(PackStruct), ctypes.POINTER(c_size)], c_int),
    "hinm_group_plan": ([ctypes.POINTER(PackStruct), c_vp, c_size, c_vp, c_vp], c_int),
    "hinm_group_build": ([ctypes.POINTER(PackStruct), c_vp, c_size, ctypes.POINTER(PackStruct), c_vp], c_int),
    "hinm_ocp_costs": ([c_vp, c_vp, c_int, c_int, c_int, c_i64, ctypes.c_double, c_vp, c_vp, c_size, c_vp],
                       c_int),
}
EXPORTED = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


def load(path: str | None = None):
    """Load (once) and type the shared library; raises DeviceError when unavailable."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise E.DeviceError(
                f"native library {p} not built; run `python -m paper_2407_20496_b200.build`")
        try:
            lib = ctypes.CDLL(p)
        except OSError as exc:  # pragma: no cover - depends on the host
            raise E.DeviceError(f"cannot load {p}: {exc}") from exc
        for name, (argtypes, restype) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = restype
        if path is None:
            _lib = lib
        return lib


def check(status: int, what: str) -> None:
    """Raise the reference exception class that corresponds to a C-ABI status."""
    if status == 0:
        return
    lib = load()
    msg = lib.hinm_status_string(status).decode()
    exc = STATUS_TO_EXCEPTION.get(status, E.DeviceError)
    raise exc(f"{what}: {msg} (status {status})")
