"""The C-ABI library loads on a CPU-only host and exports every symbol include/hinm_b200.h
declares (no compute calls -- there is no GPU here)."""

import ctypes
import os
import re

from conftest import ROOT


def _lib_path():
    from paper_2407_20496_b200.build import LIB, build

    if not os.path.exists(LIB):
        build()
    return LIB


def declared_functions():
    hdr = open(os.path.join(ROOT, "include", "hinm_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(hinm_[a-z0-9_]+)\s*\(", hdr)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("hinm_vector_prune", "hinm_nm_select", "hinm_pack_build",
                     "hinm_compress_bf16", "hinm_spmm_bf16"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib_path())
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_types_every_symbol():
    from paper_2407_20496_b200 import _lib

    assert set(_lib.EXPORTED) == set(declared_functions())
    lib = _lib.load(_lib_path())
    assert lib.hinm_version().decode().startswith("hinm_b200")
    assert lib.hinm_status_string(3).decode() == "invariant violation"


def test_host_only_queries_without_gpu():
    from paper_2407_20496_b200 import _lib

    lib = _lib.load(_lib_path())
    kc, mc, ac = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    assert lib.hinm_pack_capacity(4096, 11008, 64, 64 * 5504, ctypes.byref(kc), ctypes.byref(mc),
                                  ctypes.byref(ac)) == 0
    assert kc.value == 64 * 5504 + 64 * 64
    assert ac.value == 64 * kc.value // 2
    assert lib.hinm_pack_capacity(100, 10, 64, 0, None, None, None) == 6  # m % V -> DimensionError


def test_status_codes_map_to_reference_exceptions():
    import pytest

    from paper_2407_20496_b200 import _lib, errors as E

    _lib.load(_lib_path())
    for code, exc in ((1, E.ShapeMismatch), (3, E.InvariantViolation), (4, E.GroupingError),
                      (5, E.BudgetError), (6, E.DimensionError)):
        with pytest.raises(exc):
            _lib.check(code, "x")
    _lib.check(0, "ok")


def test_sass_has_tcgen05_and_tma():
    """The SpMM kernel is compiled to tcgen05 MMA (UTCHMMA), TMEM (LDTM / UTCCP), bulk copies
    (UBLKCP, the A / metadata image), cp.async gather (LDGSTS) and 256-bit Y stores."""
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        import pytest

        pytest.skip("cuobjdump not available")
    sass = subprocess.run([cuobjdump, "-sass", _lib_path()], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "UTCCP", "LDTM", "UBLKCP", "LDGSTS", "ENL2.256"):
        assert mnem in sass, mnem
