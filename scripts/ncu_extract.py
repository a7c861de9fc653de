"""Turn an `ncu -i X.ncu-rep --page raw --csv` export into the tracked per-kernel summary bench.py reads.

    python scripts/ncu_extract.py gpurun_out/r02x_raw.csv profiles/r02x_kernels.csv [profiles/ncu_kernels.json]

Writes (1) a compact CSV with the metrics the round summaries quote, one row per profiled launch, and
(2) optionally the JSON `bench.py` reads for `roofline.traffic` / `issue_frac` (first launch of every kernel):
{kernel: {"dram_bytes": read + write, "dram_read_bytes", "dram_write_bytes", "inst_executed", "time_us",
"issue_active_pct", ...}, "_source": csv path}.  Sizes are converted to bytes from the unit row.
"""
import csv
import json
import re
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_sectors_srcunit_tex_op_red.sum", "sm__cycles_elapsed.max", "smsp__cycles_active.avg",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
    "smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio",
    "smsp__average_warp_latency_issue_stalled_barrier.ratio",
    "smsp__average_warp_latency_issue_stalled_mio_throttle.ratio",
    "smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio",
    "smsp__average_warp_latency_issue_stalled_not_selected.ratio",
    "smsp__average_warp_latency_issue_stalled_wait.ratio",
    "smsp__average_warp_latency_issue_stalled_branch_resolving.ratio",
    "sm__inst_executed_pipe_fp64.sum", "sm__inst_executed_pipe_lsu.sum", "sm__inst_executed_pipe_alu.sum",
    "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_xu.sum",
]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6,
         "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3, "second": 1e6}


def short_name(full: str) -> str:
    m = re.search(r"(k_[a-z_0-9]+(?:<[^>]*>)?)", full)
    return m.group(1) if m else full[:48]


def main():
    src, out_csv = sys.argv[1], sys.argv[2]
    out_json = sys.argv[3] if len(sys.argv) > 3 else None
    rows = list(csv.reader(open(src)))
    hdr, units = rows[0], rows[1]
    col = {}
    for i, h in enumerate(hdr):
        col.setdefault(h, i)
    kcol = col["Kernel Name"]
    have = [m for m in METRICS if m in col]
    table, first = [], {}
    for r in rows[2:]:
        if len(r) <= kcol:
            continue
        name = short_name(r[kcol])
        rec = {"kernel": name}
        for m in have:
            try:
                v = float(r[col[m]].replace(",", ""))
            except ValueError:
                continue
            rec[m] = v * SCALE.get(units[col[m]], 1.0)
        table.append(rec)
        first.setdefault(name, rec)
    with open(out_csv, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel"] + have)
        for rec in table:
            w.writerow([rec["kernel"]] + [("%.6g" % rec[m]) if m in rec else "" for m in have])
    if out_json:
        js = {"_source": out_csv, "_units": "bytes, microseconds, counts, percent"}
        for name, rec in first.items():
            base = name.split("<")[0]
            js[base] = {
                "instantiation": name,
                "time_us": rec.get("gpu__time_duration.sum"),
                "dram_read_bytes": rec.get("dram__bytes_read.sum"),
                "dram_write_bytes": rec.get("dram__bytes_write.sum"),
                "dram_bytes": (rec.get("dram__bytes_read.sum") or 0.0) + (rec.get("dram__bytes_write.sum") or 0.0),
                "inst_executed": rec.get("smsp__inst_executed.sum"),
                "issue_active_pct": rec.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "l1tex_pct": rec.get("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
                "registers": rec.get("launch__registers_per_thread"),
            }
        with open(out_json, "w") as f:
            json.dump(js, f, indent=1)
    print(f"{len(table)} launches, {len(have)} metrics -> {out_csv}" + (f", {out_json}" if out_json else ""))


if __name__ == "__main__":
    main()
