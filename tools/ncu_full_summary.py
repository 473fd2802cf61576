#!/usr/bin/env python3
"""Selected metrics of every kernel in an `ncu --set full` report, one column per launch (CSV on stdout).

    ncu -i gpurun_out/x.ncu-rep --page raw --csv | python tools/ncu_full_summary.py > profiles/rNN_x_summary.csv
"""
import csv
import re
import sys

KEEP = [
    r"^Grid Size$", r"^Block Size$", r"^gpu__time_duration\.sum$", r"^smsp__inst_executed\.sum$",
    r"^launch__registers_per_thread$", r"^launch__occupancy_limit_registers$", r"^launch__occupancy_limit_shared_mem$",
    r"^sm__warps_active\.avg\.pct_of_peak_sustained_active$", r"^smsp__issue_active\.avg\.pct_of_peak_sustained_active$",
    r"^dram__bytes_read\.sum$", r"^dram__bytes_write\.sum$", r"^dram__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed$", r"^lts__t_sector_hit_rate\.pct$", r"^lts__t_sectors\.sum$",
    r"^lts__t_sectors_srcunit_tex_op_read\.sum$", r"^lts__t_sectors_srcunit_tex_op_read_lookup_hit\.sum$",
    r"^smsp__thread_inst_executed_per_inst_executed\.ratio$", r"^l1tex__data_bank_conflicts_pipe_lsu_mem_shared\.sum$",
    r"^smsp__average_warps_issue_stalled_.*_per_issue_active\.ratio$",
    r"^sm__inst_executed_pipe_(alu|fma|lsu|xu|adu|cbu|uniform)\.avg\.pct_of_peak_sustained_active$",
    r"^l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate\.pct$", r"^l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum\.pct_of_peak_sustained_elapsed$",
    r"^sm__throughput\.avg\.pct_of_peak_sustained_elapsed$",
]


def main() -> int:
    rows = list(csv.reader(sys.stdin))
    hdr, units, data = rows[0], rows[1], rows[2:]
    name_i = hdr.index("Kernel Name")
    out = csv.writer(sys.stdout)
    out.writerow(["metric", "unit"] + [f"{r[name_i][:40]} #{k}" for k, r in enumerate(data)])
    for i, col in enumerate(hdr):
        if any(re.match(p, col) for p in KEEP):
            out.writerow([col, units[i]] + [r[i] for r in data])
    return 0


if __name__ == "__main__":
    sys.exit(main())
