"""One-line-per-metric digest of `ncu --page raw --csv` exports (the binding
unit of a kernel): duration, issue, LSU, DRAM, L2 hit, warps, stalls.

    python tools/ncu_brief.py raw1.csv [raw2.csv ...]
"""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "us"),
        ("smsp__inst_executed.sum", "warp instr"),
        ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue % active"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "lsu smem %"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bank conflicts"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
        ("dram__bytes_read.sum", "dram rd"), ("dram__bytes_write.sum", "dram wr"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu pipe %"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
        ("launch__registers_per_thread", "regs"), ("launch__occupancy_limit_shared_mem", "occ smem"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block")]
STALLS = ["long_scoreboard", "short_scoreboard", "barrier", "mio_throttle", "math_pipe_throttle",
          "wait", "not_selected", "dispatch_stall", "lg_throttle", "no_instruction",
          "branch_resolving", "selected"]


def main():
    for path in sys.argv[1:]:
        rows = list(csv.reader(open(path)))
        hdr, units = rows[0], rows[1]
        for vals in rows[2:]:
            name = vals[hdr.index("Kernel Name")][:70]
            print(f"== {path}: {name}")
            for k, lab in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    print(f"  {lab:16s} {vals[i]} {units[i]}")
            st = []
            for s in STALLS:
                k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
                if k in hdr:
                    st.append(f"{s}={float(vals[hdr.index(k)]):.2f}")
            print("  stalls/issue   ", " ".join(st))


if __name__ == "__main__":
    main()
