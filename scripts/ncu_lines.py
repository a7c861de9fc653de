"""Summarise an `ncu --page source --csv --print-source cuda,sass` export per source line
(development aid): instructions executed, avg active threads, stall samples."""
import csv
import sys

path = sys.argv[1]
kernel_filter = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
rows = list(csv.reader(open(path)))
fn = None
hdr = None
out = {}
for r in rows:
    if not r:
        continue
    if r[0] == "Function Name":
        fn = r[1]; continue
    if r[0] == "File Path":
        cur_file = r[1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or fn is None or kernel_filter not in fn:
        continue
    if r[0] == "":  # sass row
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr, r))
    def num(k):
        try: return float(d.get(k, "0"))
        except ValueError: return 0.0
    key = (fn[:60], cur_file.split("/")[-1], line)
    o = out.setdefault(key, [0, 0, 0, r[1][:110]])
    o[0] += num("Instructions Executed"); o[1] += num("Thread Instructions Executed"); o[2] += num("# Samples")
tot_i = sum(v[0] for v in out.values()); tot_s = sum(v[2] for v in out.values())
print(f"total inst {tot_i/1e6:.1f} M, samples {tot_s:.0f}")
for k, v in sorted(out.items(), key=lambda kv: -kv[1][2])[:top]:
    act = v[1] / v[0] if v[0] else 0
    print(f"{k[1]}:{k[2]:4d} inst {v[0]/1e6:7.2f}M ({100*v[0]/tot_i:4.1f}%) act {act:4.1f} samp {100*v[2]/tot_s:4.1f}%  {v[3]}")
