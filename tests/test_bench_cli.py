"""bench.py process plumbing on CPU: `--gpus N` launches N ranks (torch.distributed.run, gloo
dry run: no kernels) and rank 0 reports n_gpus = N; strong scaling splits the global tokens."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_gpus_2_spawns_two_ranks_strong():
    out = _run("--gpus", "2", "--dry-run")
    assert out["n_gpus"] == 2 and out["scaling"] == "strong"
    assert out["global_tokens"] == 16384 and out["tokens_rank0"] == 8192
    assert out["max_over_ranks"] == 2.0        # max over both ranks' values


def test_gpus_2_weak():
    out = _run("--gpus", "2", "--dry-run", "--weak")
    assert out["n_gpus"] == 2 and out["scaling"] == "weak" and out["tokens_rank0"] == 16384


def test_gpus_1_no_spawn():
    out = _run("--dry-run")
    assert out["n_gpus"] == 1 and out["tokens_rank0"] == 16384


def test_world_mismatch_fails_loudly():
    env = {**os.environ, "WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
