"""Summarise an ncu report (.ncu-rep) into a small text file for profiles/.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r1_spmm_up.txt [title]
"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "kernel duration"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active (% of elapsed)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->L1/SMEM bytes"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum.per_second", "L2->L1/SMEM bandwidth"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed", "L2->SM ingress % of peak"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("dram__bytes.sum.per_second", "DRAM bandwidth"),
    ("l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed", "SMEM bank reads %"),
    ("l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed", "SMEM bank writes %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "LSU wavefronts %"),
    ("smsp__inst_executed.sum", "instructions executed"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__sass_inst_executed_op_ldgsts.sum", "LDGSTS instructions"),
    ("lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed", "L2 sectors from SMs % (avg slice)"),
    ("lts__t_sectors_srcunit_tex.max.pct_of_peak_sustained_elapsed", "L2 sectors from SMs % (max slice)"),
    ("lts__lts2xbar_cycles_active.avg.pct_of_peak_sustained_elapsed", "L2->xbar return % (avg slice)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe cycles active %"),
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    with open(out, "w") as fh:
        fh.write(f"# {title}\n# source: {rep} (ncu --set full --clock-control none)\n")
        for r in rows[2:]:
            d = {h: (u, v) for h, u, v in zip(hdr, units, r)}
            fh.write(f"\n## kernel: {d.get('Kernel Name', ('', '?'))[1][:120]}\n")
            for k, label in KEYS:
                if k in d:
                    fh.write(f"{label:40s} {d[k][1]:>22s} {d[k][0]}\n")
    print(open(out).read())


if __name__ == "__main__":
    main()
