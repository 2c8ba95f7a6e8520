"""Per-(config, kernel) ncu figures for bench.py's roofline record.

    python tools/ncu_roofline.py profiles/ncu_roofline_r02.json CONFIG KERNEL raw.csv [launches_per_call]

Reads one `ncu --set full --page raw --csv` export (one launch of KERNEL,
captured on the bench workload of CONFIG) and merges into the JSON:
duration, DRAM bytes read + written (`traffic`), the binding fractions
(instruction issue, shared-memory LSU wavefronts, DRAM throughput, each of
its peak), L2 hit rate and the bank-conflict share of the shared-memory
wavefronts.  bench.py keys its lookup by (config, kernel), so a capture of
one configuration is never reused for another.
"""
import csv
import json
import os
import sys


def num(hdr, vals, units, key, scale_units=True):
    if key not in hdr:
        return None
    i = hdr.index(key)
    v = vals[i].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return None
    if scale_units:
        u = units[i].strip()
        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1,
              "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}.get(u, 1)
    return x


def main():
    out, config, kernel, raw = sys.argv[1:5]
    per_call = int(sys.argv[5]) if len(sys.argv) > 5 else 1
    rows = list(csv.reader(open(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    g = lambda k: num(hdr, vals, units, k)  # noqa: E731
    rd = g("dram__bytes_read.sum") or 0.0
    wr = g("dram__bytes_write.sum") or 0.0
    wf = g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    bc = g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
    rec = {
        "kernel_name": vals[hdr.index("Kernel Name")],
        "us": g("gpu__time_duration.sum"),
        "dram_bytes": rd + wr,
        "issue_frac": (g("sm__issue_active.avg.pct_of_peak_sustained_elapsed") or 0) / 100,
        "lsu_shared_frac": (g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed") or 0) / 100,
        "dram_frac": (g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed") or 0) / 100,
        "l2_hit": (g("lts__t_sector_hit_rate.pct") or 0) / 100,
        "bank_conflict_share": (bc / wf) if (wf and bc is not None) else None,
        "warp_instructions": g("smsp__inst_executed.sum"),
        "achieved_occupancy": (g("sm__warps_active.avg.pct_of_peak_sustained_active") or 0) / 100,
        "launches_per_call": per_call,
        "source_csv": os.path.basename(raw),
    }
    d = {}
    if os.path.exists(out):
        with open(out) as fh:
            d = json.load(fh)
    d.setdefault(config, {})[kernel] = rec
    d["_note"] = ("one `ncu --set full --clock-control none` launch per (config, kernel), captured "
                  "on bench.py's own workload (tools/ncu_capture.sh); cold-cache and serialised, "
                  "so compare shares and fractions, not absolute times, with the bench line")
    with open(out, "w") as fh:
        json.dump(d, fh, indent=1, sort_keys=True)
    print(config, kernel, json.dumps(rec))


if __name__ == "__main__":
    main()
