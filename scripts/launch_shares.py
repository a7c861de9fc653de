"""Per-kernel launch counts, average durations and shares from an
`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv <cmd>` launch list.

    python scripts/launch_shares.py gpurun_out/r02h_launches.csv > profiles/r02h_launch_shares.txt
"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[1:]:
    m = re.search(r"(k_[a-z_0-9]+)", r[ki])
    key = m.group(1) if m else "(library) " + r[ki][:60]
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] in ("ns", "nsecond") else v * 1e3 if r[ui] in ("ms", "msecond") else v
    agg[key].append(v)
mine = sum(sum(v) for k, v in agg.items() if k.startswith("k_"))
print(f"{'kernel':58s} launches   avg us   share of this repo's kernels")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    share = f"{100 * sum(v) / mine:5.1f}%" if k.startswith("k_") else "  (torch: L2 flush / bench set-up, outside the hot path)"
    print(f"{k:58s} {len(v):5d} {sum(v) / len(v):9.1f}   {share}")
