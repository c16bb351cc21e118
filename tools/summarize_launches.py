"""Summarize an ncu --csv launch list: last step's kernels with times (us)."""
import csv
import sys

path = sys.argv[1]
last_n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
sel = data[-last_n:]
tot = 0.0
for d in sel:
    v = float(d["Metric Value"]) / 1e3
    tot += v
    print(f"{v:10.1f}  {d['Grid Size']:>16}  {d['Kernel Name'][:90]}")
print(f"total {tot:.1f} us over {len(sel)} launches")
