"""Summarise an ncu --set full report into a small text file for profiles/.

usage: python scripts/ncu_summary.py report.ncu-rep out.txt
"""
import csv
import re
import subprocess
import sys

KEYS = r"^(Kernel Name|gpu__time_duration.sum|dram__bytes_(read|write).sum|launch__(grid_size|block_size|registers_per_thread|occupancy_limit_\w+|shared_mem_per_block_dynamic)|sm__warps_active.avg.pct_of_peak_sustained_active|smsp__issue_active.avg.pct_of_peak_sustained_active|sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active|sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active|sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active|lts__t_sector_hit_rate.pct|l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum|smsp__inst_executed.sum|smsp__pcsamp_warps_issue_stalled_\w+|dram__throughput.avg.pct_of_peak_sustained_elapsed|sm__throughput.avg.pct_of_peak_sustained_elapsed)$"

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
out = []
for h, u, v in zip(hdr, units, vals):
    if re.match(KEYS, h) and v not in ("", "0") or h == "Kernel Name":
        out.append(f"{h:70s} {v} {u}".rstrip())
open(sys.argv[2], "w").write("\n".join(out) + "\n")
print("\n".join(out[:12]))
