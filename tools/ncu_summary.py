"""Summarise ncu reports for profiles/ (runs on the CPU box).

    python tools/ncu_summary.py OUT_PREFIX REPORT.ncu-rep [REPORT2 ...]

Writes OUT_PREFIX.md: per-kernel duration, DRAM bytes, issue / pipe
utilisation (FMA, LSU, tensor), shared-memory wavefronts and conflicts,
occupancy, top stall reasons.  (profiles/ncu_traffic.json, which bench.py
reads, is written from launch lists by tools/traffic_json.py.)
"""

import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefront util %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "uniform pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    argv = sys.argv[1:]
    prefix, reps = argv[0], argv[1:]
    lines = ["# ncu summary", ""]
    for rep in reps:
        hdr, units, rows = raw(rep)
        lines.append(f"## {os.path.basename(rep)}")
        for row in rows:
            name = row[hdr.index("Kernel Name")]
            lines.append(f"### `{name}`")
            vals = {}
            for key, label in KEYS:
                if key in hdr:
                    i = hdr.index(key)
                    lines.append(f"- {label}: {row[i]} {units[i]}")
                    vals[key] = (row[i], units[i])
            st = {}
            for i, h in enumerate(hdr):
                if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                    try:
                        st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(row[i])
                    except ValueError:
                        pass
            tot = sum(st.values()) or 1.0
            top = sorted(st.items(), key=lambda x: -x[1])[:6]
            lines.append("- top stall reasons: " + ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in top))
            lines.append("")
    with open(prefix + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print(prefix + ".md")


if __name__ == "__main__":
    main()
