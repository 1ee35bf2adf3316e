#!/usr/bin/env python
"""Key metrics of an `ncu --set full` capture (reads the report via
`ncu -i … --page raw --csv`).  Usage: ncu_full_summary.py report.ncu-rep [title]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occ limit (regs, blocks)"),
    ("launch__occupancy_limit_shared_mem", "occ limit (smem, blocks)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM, active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active % (of active cycles)"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe inst % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-inst"),
    ("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "DMUL thread-inst"),
    ("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thread-inst"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("smsp__average_warp_latency_issue_stalled_barrier", "stall barrier"),
]


def main(path, title=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    lines = raw.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    print(f"# {title}")
    for d in data:
        kname = d[hdr.index("Kernel Name")]
        print(f"## {kname[:120]}")
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"  {label:42s} {d[i]} {units[i]}")
        stalls = [(h, d[i]) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warp_latency_issue_stalled_") is False
                  and h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        tops = sorted(((float(v.replace(",", "") or 0), h) for h, v in stalls), reverse=True)[:8]
        if tops:
            print("  top stall reasons (pc samples):")
            for v, h in tops:
                print(f"    {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):32s} {v:.0f}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
