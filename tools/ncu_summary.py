"""Condense an ncu --set full report into the numbers the roofline cites.

usage: python tools/ncu_summary.py <report.ncu-rep> [algorithmic_bytes_per_launch]
Prints duration, FMA-pipe / issue utilisation, DRAM traffic, occupancy and the
top stall reasons (read here, on the CPU box, with `ncu -i`).
"""

import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (us, cold, serialised)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA-pipe inst issue % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM read (MB)"),
    ("dram__bytes_write.sum", "DRAM write (MB)"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid size"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem store bank conflicts"),
]


def main(path: str, algo_bytes: float | None = None) -> None:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"kernel: {d.get('Kernel Name', '?')}")
        for k, label in KEYS:
            if k in d:
                print(f"  {label:38s} {d[k]} {u.get(k, '')}")
        rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        if rd and wr:
            scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
            tot = float(rd) * scale.get(u["dram__bytes_read.sum"], 1) + float(wr) * scale.get(u["dram__bytes_write.sum"], 1)
            print(f"  {'DRAM traffic per launch (bytes)':38s} {tot:.0f}")
            if algo_bytes:
                print(f"  {'traffic / algorithmic bytes':38s} {tot / algo_bytes:.3f}")
        stalls = [(h, float(v)) for h, v in zip(hdr, vals)
                  if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and v]
        tot = sum(v for _, v in stalls) or 1.0
        print("  stall reasons (pc sampling):")
        for h, v in sorted(stalls, key=lambda x: -x[1])[:8]:
            print(f"    {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
