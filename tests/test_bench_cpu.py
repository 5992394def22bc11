"""CPU: bench.py's reference arm (the reference's own CPU path from oracle/_ref, or the oracle port
when that package is absent) prints one JSON line with the driver contract's keys, on the same
metric / unit / scaling as the GPU arm."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--cpu-tokens", "8", *extra],
                       capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


_LINE = {}


def _default_line():
    if not _LINE:
        _LINE.update(_run())
    return dict(_LINE)


def test_reference_arm_contract():
    line = _default_line()
    assert line["impl"] == "reference"
    assert line["unit"] == "TFLOP/s" and line["higher_is_better"] is True
    assert line["metric"].startswith("HiNM SpMM effective TFLOPS")
    assert line["value"] > 0 and line["steps"] == 1 and line["scaling"] == "strong"
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert "sample" in cb
    assert line["e2e"] == {"value": line["value"], "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_reference_arm_runs_the_reference_package_when_installed():
    line = _default_line()
    if os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "hinm")):
        assert line["cpu_baseline"]["kind"] == "reference"


def test_reference_arm_nonzero_rank_is_silent():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--cpu-tokens", "8"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env={**os.environ, "RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0 and r.stdout.strip() == ""
