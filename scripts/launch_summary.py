"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python scripts/launch_summary.py gpurun_out/launches_bench.csv profiles/r01_launches.txt
"""
import collections
import csv
import sys


def main():
    src, out = sys.argv[1], sys.argv[2]
    lines = [ln for ln in open(src) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = name.split("(")[0][:90] if "hinm" in name or "k_" in name else name[:60]
        ns = float(r["Metric Value"]) * (1e3 if r["Metric Unit"] == "us" else 1e6 if r["Metric Unit"] == "ms" else 1)
        a = agg.setdefault(short, [0, 0.0, r["Grid Size"], r["Block Size"]])
        a[0] += 1
        a[1] += ns
    tot = sum(a[1] for a in agg.values())
    with open(out, "w") as fh:
        fh.write(f"# launch list summary of {src}\n# ncu --metrics gpu__time_duration.sum "
                 f"--clock-control none (cold-cache, serialised): per-launch times\n")
        fh.write(f"{'kernel':92s} {'n':>5s} {'avg_us':>10s} {'total_us':>11s} {'share':>7s}  grid/block\n")
        for k, (n, ns, g, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"{k:92s} {n:5d} {ns / n / 1e3:10.2f} {ns / 1e3:11.1f} {ns / tot:7.1%}  {g}/{b}\n")
    print(open(out).read())


if __name__ == "__main__":
    main()
