"""Per-source-line instruction counts and warp-stall samples from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass` (development aid).

    python scripts/ncu_stalls.py src.csv [kernel substring] [top N]
"""
import csv
import sys

path = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 45
rows = list(csv.reader(open(path)))
hdr, fn, cur_file, out = None, None, "", {}
for r in rows:
    if not r:
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or fn is None or kfilter not in fn or r[0] == "":
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr, r))

    def num(k):
        try:
            return float(d.get(k, "0"))
        except ValueError:
            return 0.0
    o = out.setdefault((cur_file, line), {"src": r[1][:88], "inst": 0.0, "tinst": 0.0, "samp": 0.0})
    o["inst"] += num("Instructions Executed")
    o["tinst"] += num("Thread Instructions Executed")
    o["samp"] += num("# Samples")
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k:
            o[k] = o.get(k, 0.0) + num(k)
tot = sum(o["samp"] for o in out.values()) or 1.0
print(f"total samples {tot:.0f}, warp instructions {sum(o['inst'] for o in out.values()) / 1e6:.1f} M")
stalls = {}
for o in out.values():
    for k, v in o.items():
        if k.startswith("stall_"):
            stalls[k] = stalls.get(k, 0.0) + v
print("stall shares:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:12]))
for (f, line), o in sorted(out.items(), key=lambda kv: -kv[1]["samp"])[:top]:
    best = sorted([(v, k) for k, v in o.items() if k.startswith("stall_")], reverse=True)[:3]
    act = o["tinst"] / o["inst"] if o["inst"] else 0.0
    print(f"{f}:{line:4d} inst {o['inst'] / 1e6:6.2f}M act {act:4.1f} samp {100 * o['samp'] / tot:4.1f}%  "
          f"{' '.join(f'{k[6:]}:{100 * v / tot:.1f}' for v, k in best)} | {o['src']}")
