"""Summarise `ncu --page raw --csv` exports into a small JSON keyed by kernel.

    python tools/ncu_summary.py out.json raw1.csv [raw2.csv ...]
"""
import csv
import json
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]


def main():
    out, paths = sys.argv[1], sys.argv[2:]
    res = {}
    for path in paths:
        rows = list(csv.reader(open(path)))
        hdr, units = rows[0], rows[1]
        name_i = hdr.index("Kernel Name")
        for vals in rows[2:]:
            d = {}
            for k in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    d[k] = f"{vals[i]} {units[i]}".strip()
            res.setdefault(vals[name_i], []).append(d)
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    for k, v in res.items():
        t = v[0].get("gpu__time_duration.sum")
        print(f"{k[:90]}: {len(v)} launch(es), first {t}")


if __name__ == "__main__":
    main()
