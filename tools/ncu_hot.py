"""Per-CUDA-source-line stall samples (or another source-page column, e.g.
"Instructions Executed") of one kernel: ncu_hot.py rep kernel [top] [column]."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
col = sys.argv[4] if len(sys.argv) > 4 else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
agg, cur = {}, None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        si = hdr.index(col)
        continue
    if not hdr or len(r) <= si:
        continue
    if r[0]:  # a CUDA source line
        cur = (r[0], r[1].strip()[:100])
        agg.setdefault(cur, 0)
    elif cur:
        try:
            agg[cur] += int(r[si])
        except ValueError:
            pass
tot = sum(agg.values())
print("total samples", tot)
for (ln, t), s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{s:8d} {100*s/max(tot,1):5.1f}%  L{ln}: {t}")
