"""Summarise an `ncu --set full` report (read here, no GPU) into a markdown table.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/ncu_full_<kernel>_rN.md

Per launch: duration, DRAM bytes read/written (the roofline `traffic`), DRAM and SM
throughput, issue-slot and FMA-pipe utilisation, shared-memory wavefronts, occupancy and
registers -- the counters DESIGN.md §3 cites for each kernel.
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def rows(report: str):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head, units = r[0], r[1]
    for row in r[2:]:
        yield {h: (v, u) for h, u, v in zip(head, units, row)}


def main(report: str):
    cols = [m for m in METRICS]
    print(f"ncu --set full summary of `{report}`\n")
    print("| kernel | " + " | ".join(label for _, label in cols) + " |")
    print("|---|" + "---:|" * len(cols))
    for d in rows(report):
        name = d.get("Kernel Name", ("?", ""))[0].split("(")[0]
        cells = []
        for m, _ in cols:
            v, u = d.get(m, ("n/a", ""))
            cells.append(f"{v} {u}".strip())
        print(f"| `{name}` | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
