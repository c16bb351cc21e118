"""Markdown table + per-launch DRAM traffic JSON of the hot kernels in an
ncu --set full report: python tools/ncu_table.py rep.ncu-rep out.md traffic.json"""
import csv
import json
import re
import subprocess
import sys

rep, out_md, out_json = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
SC = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3}


def g(r, k):
    i = hdr.index(k)
    return float(r[i].replace(",", "")) * SC.get(units[i], 1.0)


def short(nm, rd):
    m = re.search(r"(k_\w+)(<[^>(]*>)?", nm)
    base, targs = m.group(1), m.group(2) or ""
    if base in ("k_rle_write_fast", "k_rle_tiles_fast"):
        return base + ("<u16> (residual)" if "short" in targs else "<u32> (grid)")
    if base == "k_dec_out":
        if targs.startswith("<0"):
            return base + "<P64> (grid)"
        if targs.startswith("<5"):
            return base + "<Q32> (grid)"
        return base + "<RECOMPOSE> (residual)"
    if base == "k_dec_agg":
        return base + (" (residual)" if rd > 1e8 else " (grid)")
    return base


lines, seen = [], set()
for r in rows[2:]:
    rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
    s = short(r[hdr.index("Kernel Name")], rd)
    if s in seen:
        continue
    seen.add(s)
    lines.append((s, g(r, "gpu__time_duration.sum"), rd, wr, g(r, "lts__t_sector_hit_rate.pct"),
                  g(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                  g(r, "l1tex__throughput.avg.pct_of_peak_sustained_active")))
md = ["| kernel | ncu us | DRAM read GB | DRAM write GB | L2 hit % | issue active % | L1TEX % |",
      "|---|---|---|---|---|---|---|"]
for s, t, rd, wr, hit, iss, l1 in lines:
    md.append(f"| {s} | {t:.1f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | {hit:.1f} | {iss:.1f} | {l1:.1f} |")
open(out_md, "w").write("\n".join(md) + "\n")
names = {"k_gather_fwd": "k_gather_fwd", "k_bucket_tma": "k_bucket", "k_resid_codes": "k_resid_codes", "k_resid_codes_sr": "k_resid_codes",
         "k_dec_agg (residual)": "k_dec_agg", "k_dec_out<RECOMPOSE> (residual)": "k_dec_out",
         "k_dec_out<P64> (grid)": "k_dec_out_grid", "k_dec_out<Q32> (grid)": "k_dec_out_grid"}
d = {names[s]: rd + wr for s, t, rd, wr, *_ in lines if s in names}
d["k_rle_write"] = sum(rd + wr for s, t, rd, wr, *_ in lines if s.startswith("k_rle_write_fast"))
json.dump(d, open(out_json, "w"), indent=1)
print("\n".join(md))
print(d)
