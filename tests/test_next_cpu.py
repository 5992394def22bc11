"""§8(f) rows 2 and 4 on the CPU: the reference's on-disk formats (files written by the
reference, tests/golden/io/) and group-order freedom (shuffle_encoding / kept_triples against
the reference's outputs for the same generator, tests/golden/next.npz).  Generator:
tests/golden/make_golden_next.py."""

import filecmp
import os

import numpy as np
import pytest

from paper_2407_20496_b200 import io as hio
from paper_2407_20496_b200.model import GyroPermutation, HiNMConfig
from paper_2407_20496_b200.pruning import HiNMEncoding, TileEncoding
from paper_2407_20496_b200.spmm import kept_triples, shuffle_encoding

GOLD = os.path.join(os.path.dirname(__file__), "golden")
IOD = os.path.join(GOLD, "io")


@pytest.fixture(scope="module")
def nxt():
    return np.load(os.path.join(GOLD, "next.npz"))


def test_config_roundtrip_bytes(tmp_path):
    cfg = hio.load_config(os.path.join(IOD, "config.json"))
    assert cfg == HiNMConfig(4, 2, 4, 0.5, ocp_sample_schedule=(2, 1), seed=3)
    hio.save_config(cfg, tmp_path / "c.json")
    assert filecmp.cmp(tmp_path / "c.json", os.path.join(IOD, "config.json"), shallow=False)


def test_config_rejects_unknown_and_missing():
    with pytest.raises(ValueError, match="unknown config keys"):
        hio.config_from_dict({"vector_size": 4, "nm_keep": 2, "nm_group": 4,
                              "vector_sparsity": 0.5, "bogus": 1})
    with pytest.raises(ValueError, match="missing required key"):
        hio.config_from_dict({"vector_size": 4, "nm_keep": 2, "nm_group": 4})


def test_encoding_roundtrip_bytes(tmp_path):
    enc = hio.load_encoding(os.path.join(IOD, "encoding.json"))
    assert enc.shape == (16, 32) and len(enc.tiles) == 4
    hio.save_encoding(enc, tmp_path / "e.json")
    assert filecmp.cmp(tmp_path / "e.json", os.path.join(IOD, "encoding.json"), shallow=False)


def test_encoding_missing_key(tmp_path):
    p = tmp_path / "bad.json"
    p.write_text('{"rows": 1, "cols": 1, "tiles": []}')
    from paper_2407_20496_b200.errors import InvariantViolation
    with pytest.raises(InvariantViolation):
        hio.load_encoding(p)


def test_permutation_roundtrip_bytes(tmp_path):
    sig = hio.load_permutation(os.path.join(IOD, "permutation.json"))
    assert isinstance(sig, GyroPermutation) and len(sig.sigma_i) == 4
    hio.save_permutation(sig, tmp_path / "p.json")
    assert filecmp.cmp(tmp_path / "p.json", os.path.join(IOD, "permutation.json"), shallow=False)


def test_dump_json_matches_reference(tmp_path):
    hio.dump_json({"b": 1.0 / 3.0, "a": [np.float64(2.0) / 7.0, np.int64(5)], "c": {"z": 1e-12}},
                  tmp_path / "r.json")
    assert filecmp.cmp(tmp_path / "r.json", os.path.join(IOD, "report.json"), shallow=False)


def test_chain_manifest():
    paths = hio.load_chain_manifest(os.path.join(IOD, "chain.json"))
    assert paths == [os.path.realpath(os.path.join(IOD, "encoding.json"))] * 2


def _enc(z, tag, which):
    m, n, V, N, M = (int(x) for x in z[f"{tag}_meta"])
    T = m // V
    tiles = [TileEncoding(z[f"{tag}_{which}_t{t}_vi"], z[f"{tag}_{which}_t{t}_nm"],
                          z[f"{tag}_{which}_t{t}_kv"]) for t in range(T)]
    return HiNMEncoding(shape=(m, n), config=HiNMConfig(V, N, M, 0.5), sigma_o=z[f"{tag}_sigma_o"],
                        tiles=tiles)


@pytest.mark.parametrize("tag", ["s24", "s14"])
def test_shuffle_encoding_matches_reference(nxt, tag):
    enc = _enc(nxt, tag, "enc")
    ref = _enc(nxt, tag, "sh")
    got = shuffle_encoding(enc, np.random.default_rng(7))
    for g, r in zip(got.tiles, ref.tiles):
        assert np.array_equal(g.vector_index, r.vector_index)
        assert np.array_equal(g.nm_index, r.nm_index)
        assert np.array_equal(g.kept_values, r.kept_values)


@pytest.mark.parametrize("tag", ["s24", "s14"])
def test_kept_triples(nxt, tag):
    enc = _enc(nxt, tag, "enc")
    trip = kept_triples(enc)
    assert len(trip) == int(nxt[f"{tag}_ntriples"])
    assert kept_triples(shuffle_encoding(enc, np.random.default_rng(3))) == trip
