"""Pipe utilisation and warp-stall breakdown of the kernels in an `ncu --set full` report.

    python tools/ncu_stalls.py gpurun_out/r2/prof_render.ncu-rep 'k_blend_fp32' > profiles/...

Per kernel (first launch matching the pattern): issue-slot use, the FMA / ALU / LSU / XU /
FP64 pipes, shared-memory wavefronts and their pipe share, and the stall reasons as warp-cycles
per issued instruction (ncu's smsp__average_warps_issue_stalled_*_per_issue_active)."""
from __future__ import annotations

import csv
import io
import re
import subprocess
import sys

PIPES = [
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe (inst) %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe (cycles) %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed", "smem pipe %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "registers"),
    ("gpu__time_duration.sum", "duration"),
]


def main(path, pattern):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kn = hdr.index("Kernel Name")
    seen = set()
    print(f"Pipe utilisation and stall reasons from `{path}` (first launch per kernel)\n")
    for r in rows[2:]:
        name = r[kn].split("(")[0]
        if not re.search(pattern, name) or name in seen:
            continue
        seen.add(name)
        print(f"### `{name}`\n\n| counter | value |\n|---|---:|")
        for m, label in PIPES:
            if m in hdr:
                i = hdr.index(m)
                print(f"| {label} | {r[i]} {units[i]} |")
        stalls = []
        for i, h in enumerate(hdr):
            mm = re.match(r"smsp__average_warps_issue_stalled_(.+)_per_issue_active\.ratio$", h)
            if mm and r[i]:
                try:
                    stalls.append((float(r[i]), mm.group(1)))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("\n| stall reason | warp-cycles per issued instruction |\n|---|---:|")
        for v, s in stalls[:12]:
            print(f"| {s} | {v:.3f} |")
        print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ".")
