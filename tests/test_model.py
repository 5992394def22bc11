"""Host-side config / type semantics (mirrors the reference's test_model.py cases)."""

from fractions import Fraction

import numpy as np
import pytest

import paper_2407_20496_b200 as H


def test_validate_derived_counts():
    v = H.validate_config(H.HiNMConfig(64, 2, 4, 0.5), (4096, 11008))
    assert (v.num_tiles, v.tile_keep, v.total_keep) == (64, 5504, 64 * 5504)


@pytest.mark.parametrize("cfg,shape,exc", [
    (H.HiNMConfig(0, 2, 4, 0.5), (8, 8), ValueError),
    (H.HiNMConfig(4, 0, 4, 0.5), (8, 8), ValueError),
    (H.HiNMConfig(4, 5, 4, 0.5), (8, 8), ValueError),
    (H.HiNMConfig(4, 4, 4, 0.5), (8, 8), ValueError),       # N == M only allowed for M == 1
    (H.HiNMConfig(4, 2, 4, 1.0), (8, 8), ValueError),
    (H.HiNMConfig(4, 2, 4, -0.1), (8, 8), ValueError),
    (H.HiNMConfig(4, 2, 4, 0.5, tie_break="random"), (8, 8), ValueError),
    (H.HiNMConfig(4, 2, 4, 0.5, tile_rows=8), (8, 8), H.DimensionError),
    (H.HiNMConfig(3, 2, 4, 0.5), (8, 8), H.DimensionError),
    (H.HiNMConfig(4, 2, 4, 0.3), (8, 10), H.DimensionError),  # 7 vectors
    (H.HiNMConfig(4, 2, 4, 0.5), (8, 12), H.DimensionError),  # 6 % 4
    (H.HiNMConfig(4, 2, 4, 0.5, ocp_sample_schedule=(5,)), (8, 8), ValueError),
])
def test_validate_errors(cfg, shape, exc):
    with pytest.raises(exc):
        H.validate_config(cfg, shape)


def test_vector_only_mode_allowed():
    H.validate_config(H.HiNMConfig(2, 1, 1, 0.5), (4, 2))


def test_float_sparsity_is_rational():
    v = H.validate_config(H.HiNMConfig(4, 1, 2, 0.6), (4, 20))
    assert v.tile_keep == 8
    assert H.composed_sparsity(0.5, 2, 4) == Fraction(3, 4)
    assert H.composed_sparsity(0.6, 1, 1) == Fraction(3, 5)


def test_default_schedule():
    assert H.default_sample_schedule(64, 3) == (32, 26, 20)
    assert min(H.default_sample_schedule(4, 30)) == 1


def test_value_types():
    with pytest.raises(H.InvariantViolation):
        H.DenseMatrix(np.array([[1.0, np.nan]]))
    with pytest.raises(H.InvariantViolation):
        H.SaliencyMatrix(np.array([[1.0, -1.0]]))
    with pytest.raises(H.DimensionError):
        H.DenseMatrix(np.ones(3))
    with pytest.raises(H.InvariantViolation):
        H.MaskPair(np.ones((3, 4), bool), np.ones((4, 4), bool))
    g = H.GyroPermutation(np.array([1, 0]), (np.array([2, 2]),))
    with pytest.raises(H.InvariantViolation):
        g.validate((2, 4))
    with pytest.raises(H.InvariantViolation):
        H.GyroPermutation(np.array([0, 0]), ()).validate((2, 4))


def test_exit_codes():
    assert H.exit_code_for(H.ShapeMismatch("x")) == 3
    assert H.exit_code_for(H.BudgetError("x")) == 2
    assert H.exit_code_for(H.SizeGuard("x")) == 4


def test_hnmw_roundtrip(tmp_path):
    from paper_2407_20496_b200.io import read_hnmw, write_hnmw

    a = np.arange(12, dtype=np.float64).reshape(3, 4) / 7
    write_hnmw(tmp_path / "a.hnmw", a)
    assert np.array_equal(read_hnmw(tmp_path / "a.hnmw"), a.astype(np.float32).astype(np.float64))
    (tmp_path / "b.hnmw").write_bytes(b"XXXX" + bytes(12))
    with pytest.raises(H.FormatError):
        read_hnmw(tmp_path / "b.hnmw")


def test_dropin_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(H.DeviceError):
        H.vector_prune(np.ones((4, 8)), H.HiNMConfig(2, 1, 2, 0.5), np.arange(4))


# values produced by the reference's hinm.model.count_permutation_space (model.py:249-267);
# the large case is pinned by its bit length and its residue mod 2**61 - 1
@pytest.mark.parametrize("args,exact,residue,bits", [
    ((8, 8, 4, 4), 2450, 2450, 12),
    ((16, 32, 4, 4), 623138617594693176539062500, 420383145671866053, 90),
    ((6, 8, 2, 2), 4725, 4725, 13),
    ((4, 4, 1, 1), 4, 4, 3),
    ((768, 3072, 64, 4), None, 206401976091169948, 24066),
])
def test_count_permutation_space(args, exact, residue, bits):
    v = H.count_permutation_space(*args)
    if exact is not None:
        assert v == exact
    assert v % (2 ** 61 - 1) == residue and v.bit_length() == bits


@pytest.mark.parametrize("args", [(0, 4, 1, 1), (6, 8, 4, 2), (8, 6, 4, 4)])
def test_count_permutation_space_errors(args):
    with pytest.raises(H.DimensionError):
        H.count_permutation_space(*args)


def test_reference_names_exported():
    for name in ("Partition", "ScheduleState", "assignment_cost", "count_permutation_space"):
        assert name in H.__all__ and hasattr(H, name)
