"""Write profiles/spmm_dram_traffic.json (bench.py's roofline.traffic) from an ncu --set full
capture of one k_hinm_spmm launch:

    python scripts/traffic_json.py gpurun_out/prof.ncu-rep "<what was captured>"
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, what = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, v = rows[0], rows[2]
    get = lambda k: float(v[h.index(k)].replace(",", ""))
    # ncu reports these two in the unit shown in row 1 (Mbyte / Gbyte)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    units = rows[1]
    rd = get("dram__bytes_read.sum") * scale[units[h.index("dram__bytes_read.sum")]]
    wr = get("dram__bytes_write.sum") * scale[units[h.index("dram__bytes_write.sum")]]
    res = {"dram_bytes_per_launch": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
           "kernel": v[h.index("Kernel Name")], "source": os.path.basename(rep),
           "note": f"ncu --set full, one launch: {what}"}
    with open(os.path.join(ROOT, "profiles", "spmm_dram_traffic.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
