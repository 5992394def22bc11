"""On-disk formats of the reference (pkg/src/hinm/io.py) and their bridge to the device pack.

* HNMW binary matrices (io.py:19-49): magic 'HNMW', u32 version=1, u32 rows, u32 cols, then
  rows*cols little-endian float32, row-major.
* Config JSON (io.py:55-104): exactly the HiNMConfig keys; unknown keys and missing required
  keys raise ValueError.
* Deterministic JSON reports (io.py:110-135): floats at 9 significant digits, sorted keys,
  2-space indent, trailing newline -- byte-identical reruns.
* Encoding JSON (io.py:147-195) and permutation JSON (io.py:198-212): same schema, so files
  written here load in the reference and vice versa (tests/test_io.py pins this against files
  the reference wrote, tests/golden/io/).
* Device bridge (no reference analogue): ``save_pack`` writes a DevicePack's reference view as
  encoding JSON; ``load_pack`` reads encoding JSON straight into a DevicePack with its tcgen05
  operand image, so the unchanged CLI artefacts drive the GPU path.

Host I/O only: no numerics here.
"""

from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np

from .errors import FormatError, InvariantViolation
from .model import GyroPermutation, HiNMConfig, as_values

_HDR = struct.Struct("<4sIII")


# ------------------------------------------------------------------------------------- HNMW
def write_hnmw(path, matrix) -> None:
    v = as_values(matrix)
    if v.ndim != 2:
        raise FormatError(f"HNMW stores 2-D matrices, got shape {v.shape}")
    with open(path, "wb") as fh:
        fh.write(_HDR.pack(b"HNMW", 1, v.shape[0], v.shape[1]))
        fh.write(np.ascontiguousarray(v, dtype="<f4").tobytes())


def read_hnmw(path) -> np.ndarray:
    raw = Path(path).read_bytes()
    if len(raw) < _HDR.size:
        raise FormatError(f"{path}: truncated header")
    magic, version, rows, cols = _HDR.unpack_from(raw)
    if magic != b"HNMW":
        raise FormatError(f"{path}: bad magic {magic!r}")
    if version != 1:
        raise FormatError(f"{path}: unsupported version {version}")
    if len(raw) != _HDR.size + 4 * rows * cols:
        raise FormatError(f"{path}: expected {_HDR.size + 4 * rows * cols} bytes, found {len(raw)}")
    return np.frombuffer(raw, dtype="<f4", offset=_HDR.size).reshape(rows, cols).astype(np.float64)


# -------------------------------------------------------------------------------- config JSON
CONFIG_KEYS = ("vector_size", "nm_keep", "nm_group", "vector_sparsity", "tile_rows",
               "ocp_sample_schedule", "ocp_max_iters", "icp_max_iters", "seed", "tie_break")
_REQUIRED = ("vector_size", "nm_keep", "nm_group", "vector_sparsity")


def config_from_dict(data: dict) -> HiNMConfig:
    """HiNMConfig from its JSON object (io.py:69-79)."""
    extra = sorted(set(data) - set(CONFIG_KEYS))
    if extra:
        raise ValueError(f"unknown config keys: {extra}")
    missing = [k for k in _REQUIRED if k not in data]
    if missing:
        raise ValueError(f"config is missing required key {missing[0]!r}")
    kw = dict(data)
    if kw.get("ocp_sample_schedule") is not None:
        kw["ocp_sample_schedule"] = tuple(kw["ocp_sample_schedule"])
    return HiNMConfig(**kw)


def config_to_dict(cfg: HiNMConfig) -> dict:
    d = {k: getattr(cfg, k) for k in CONFIG_KEYS}
    if d["ocp_sample_schedule"] is not None:
        d["ocp_sample_schedule"] = list(d["ocp_sample_schedule"])
    return d


def load_config(path) -> HiNMConfig:
    data = load_json(path)
    if not isinstance(data, dict):
        raise ValueError(f"{path}: config JSON must be an object")
    return config_from_dict(data)


def save_config(cfg: HiNMConfig, path) -> None:
    _write_sorted(config_to_dict(cfg), path)


# ---------------------------------------------------------------------- deterministic JSON
def _canonical(obj, sig: int):
    if isinstance(obj, (float, np.floating)):
        return float(f"{float(obj):.{sig}g}")
    if isinstance(obj, np.integer):
        return int(obj)
    if isinstance(obj, np.ndarray):
        return _canonical(obj.tolist(), sig)
    if isinstance(obj, dict):
        return {k: _canonical(v, sig) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_canonical(v, sig) for v in obj]
    return obj


def _write_sorted(obj, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(obj, fh, indent=2, sort_keys=True)
        fh.write("\n")


def dump_json(obj, path, sig: int = 9) -> None:
    """Floats at `sig` significant digits, sorted keys: byte-stable reruns (io.py:126-135)."""
    _write_sorted(_canonical(obj, sig), path)


def load_json(path):
    with open(path, "r", encoding="utf-8") as fh:
        return json.load(fh)


# ------------------------------------------------------------------------------ encoding JSON
def encoding_to_dict(enc) -> dict:
    return {
        "rows": int(enc.shape[0]), "cols": int(enc.shape[1]),
        "config": config_to_dict(enc.config),
        "sigma_o": np.asarray(enc.sigma_o).tolist(),
        "tiles": [{"vector_index": np.asarray(t.vector_index).tolist(),
                   "nm_index": np.asarray(t.nm_index).tolist(),
                   "kept_values": np.asarray(t.kept_values, dtype=np.float64).tolist()}
                  for t in enc.tiles],
    }


def save_encoding(enc, path) -> None:
    """Encoding JSON (io.py:164-170): repr floats, which round-trip float64 exactly."""
    _write_sorted(encoding_to_dict(enc), path)


def encoding_from_dict(data, where="encoding"):
    from .pruning import HiNMEncoding, TileEncoding

    try:
        cfg = config_from_dict(data["config"])
        tiles = [TileEncoding(vector_index=np.asarray(t["vector_index"], dtype=np.int64),
                              nm_index=np.asarray(t["nm_index"], dtype=np.int64),
                              kept_values=np.asarray(t["kept_values"], dtype=np.float64))
                 for t in data["tiles"]]
        return HiNMEncoding(shape=(int(data["rows"]), int(data["cols"])), config=cfg,
                            sigma_o=np.asarray(data["sigma_o"], dtype=np.int64), tiles=tiles)
    except KeyError as exc:
        raise InvariantViolation(f"{where}: encoding JSON missing key {exc}") from exc


def load_encoding(path):
    return encoding_from_dict(load_json(path), str(path))


# --------------------------------------------------------------------------- permutation JSON
def permutation_to_dict(sigma: GyroPermutation) -> dict:
    return {"sigma_o": np.asarray(sigma.sigma_o).tolist(),
            "sigma_i": [np.asarray(o).tolist() for o in sigma.sigma_i]}


def save_permutation(sigma: GyroPermutation, path) -> None:
    _write_sorted(permutation_to_dict(sigma), path)


def load_permutation(path) -> GyroPermutation:
    data = load_json(path)
    return GyroPermutation(sigma_o=np.asarray(data["sigma_o"], dtype=np.int64),
                           sigma_i=tuple(np.asarray(o, dtype=np.int64) for o in data["sigma_i"]))


def load_chain_manifest(path) -> list[str]:
    """{"layers": [relative encoding paths]} -> absolute paths (io.py:215-220)."""
    data = load_json(path)
    if not isinstance(data, dict) or "layers" not in data:
        raise ValueError(f"{path}: chain manifest must be an object with a 'layers' list")
    base = Path(path).parent
    return [str((base / layer).resolve()) for layer in data["layers"]]


# ------------------------------------------------------------------------- device pack bridge
def save_pack(pack, path) -> None:
    """Write a DevicePack (GPU compressor output) as reference encoding JSON."""
    from .pruning import encoding_from_pack

    save_encoding(encoding_from_pack(pack), path)


def load_pack(path, device=None):
    """Encoding JSON -> DevicePack (reference view + tcgen05 operand image) on `device`."""
    from .pruning import _torch, pack_from_encoding

    torch = _torch()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    return pack_from_encoding(load_encoding(path), dev)


__all__ = ["write_hnmw", "read_hnmw", "CONFIG_KEYS", "config_from_dict", "config_to_dict",
           "load_config", "save_config", "dump_json", "load_json", "encoding_to_dict",
           "encoding_from_dict", "save_encoding", "load_encoding", "permutation_to_dict",
           "save_permutation", "load_permutation", "load_chain_manifest", "save_pack",
           "load_pack"]
