"""Sustained time / power of the union-group SpMM (LLaMA up, 16k tokens) for several library builds:
python scripts/power_variants.py lib1.so [lib2.so ...] (each in a fresh process)."""
import os, sys, subprocess, json
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = open(os.path.join(root, "scripts", "power_split.py")).read().split("code = r'''")[1].split("''' % root")[0] % root
for lib in sys.argv[1:]:
    env = dict(os.environ, HINM_B200_LIB=lib)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    out = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
    print(os.path.basename(lib), out, flush=True)
