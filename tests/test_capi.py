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


def test_group_image_host_queries_without_gpu():
    """hinm_group_workspace validates the pack and sizes the plan / build workspace on the host;
    configurations outside the union-group image are rejected before any device work."""
    from paper_2407_20496_b200 import _lib

    lib = _lib.load(_lib_path())
    dummy = ctypes.c_int32(0)
    st = _lib.PackStruct()
    st.m, st.n, st.V, st.N, st.M, st.T = 11008, 4096, 64, 2, 4, 11008 // 64
    for f in ("tile_ptr", "vec_idx", "nm_pos", "kept_bf16"):
        setattr(st, f, ctypes.addressof(dummy))
    nb = ctypes.c_size_t()
    assert lib.hinm_group_workspace(ctypes.byref(st), ctypes.byref(nb)) == 0
    U = -(-11008 // 256)
    assert nb.value >= st.T * 4096 * 2 + U * 4096 * 32 + U * 4096 * 16
    st.V = 128  # V = 128 has no union-group image
    assert lib.hinm_group_workspace(ctypes.byref(st), ctypes.byref(nb)) == 10
    st.V, st.N = 64, 1  # 1:4 is not 2:4
    assert lib.hinm_group_workspace(ctypes.byref(st), ctypes.byref(nb)) == 10
    assert lib.hinm_last_image() == 0


def test_sass_has_cta_pair_mma():
    """The union-group path is compiled to the CTA-pair instruction forms: 2-CTA sparse MMA, the
    pair's TMEM copies and multicast commits (UTCHMMA.2CTA, UTCBAR.2CTA.MULTICAST)."""
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        import pytest

        pytest.skip("cuobjdump not available")
    sass = subprocess.run([cuobjdump, "-sass", _lib_path()], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA.2CTA", "UTCBAR.2CTA.MULTICAST"):
        assert mnem in sass, mnem


def test_product_library_has_only_validated_knobs():
    """The product library reads only the documented tuning knobs (each validated: an unknown value
    is an error, results are unchanged); the timing-only / diagnostic switches whose results are
    garbage (HINM_PAIR_DBG, HINM_SP2, HINM_CHAIN_NOCOMPUTE, HINM_COMPRESS_PDL, ...) and the
    timing-only kernel variants exist only in the experiments build."""
    blob = open(_lib_path(), "rb").read()
    knobs = sorted(set(re.findall(rb"HINM_[A-Z0-9_]+", blob)))
    assert [k.decode() for k in knobs] == ["HINM_BN", "HINM_GATHER", "HINM_GROUPS", "HINM_GW", "HINM_KS",
                                           "HINM_PAIR_GW", "HINM_PAIR_KS", "HINM_PDL", "HINM_Y_V8"]
