"""Stall-reason totals (and top stalled SASS lines) from an .ncu-rep source page."""
import csv, io, subprocess, sys
rep = sys.argv[1]
import os
k = (["-k", "regex:" + os.environ["NCU_K"]] + (["--kernel-name-base", "mangled"] if os.environ.get("NCU_MANGLED") else [])) if os.environ.get("NCU_K") else []  # one kernel of a multi-kernel report
txt = subprocess.run(["ncu", "-i", rep] + k + ["--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: 0 for r in reasons}
lines = []
for r in rows[2:]:
    if len(r) < len(hdr): continue
    try:
        vals = {k: int(r[ix[k]] or 0) for k in reasons}
    except ValueError:
        continue
    for k, v in vals.items(): tot[k] += v
    lines.append((sum(vals.values()), r[ix["Source"]].strip()[:70], max(vals, key=vals.get)))
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v: print(f"{k:28s} {v:8d} {100*v/s:5.1f}%")
print("top stalled instructions:")
for n, src, why in sorted(lines, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"  {n:7d} {why:22s} {src}")
