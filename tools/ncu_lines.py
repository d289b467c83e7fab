"""Executed warp instructions per CUDA source line from an .ncu-rep (cuda,sass source page)."""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None; line = None; src = {}; cnt = defaultdict(int); hdr = None
for r in csv.reader(io.StringIO(txt)):
    if not r: continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = {h: i for i, h in enumerate(r)}; continue
    if r[0].isdigit():
        line = (f, int(r[0])); src[line] = r[1].strip(); continue
    if hdr and len(r) > 7 and r[2].startswith("0x"):
        v = r[7]
        try: cnt[line] += int(v)
        except ValueError: pass
tot = sum(cnt.values())
print("total warp instructions", tot)
byfile = defaultdict(int)
for (fn, _), v in cnt.items(): byfile[fn] += v
print({k: round(v / tot, 3) for k, v in byfile.items()})
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k, v in sorted(cnt.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{100*v/tot:5.1f}% {k[0]}:{k[1]:4d} {src.get(k, '')[:90]}")
