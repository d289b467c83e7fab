"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file X)
into per-kernel launch counts, total time and shares (profiles/<round>_launches.txt).

    python tools/ncu_launches.py launches.csv "<command that produced it>" [exclude_substr ...]
"""
import csv
import re
import sys
from collections import defaultdict

path, cmd = sys.argv[1], sys.argv[2]
excl = sys.argv[3:]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).replace("holo::", "").replace("(anonymous namespace)::", "")
    name = re.sub(r"<unnamed>::", "", name)[:60]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"# ncu launch list: {cmd}")
print("# (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)")
print(f"# {sum(cnt.values())} launches, {T:.1f} us total")
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:60s} {cnt[k]:8d} {tot[k]:12.1f} {100 * tot[k] / T:6.1f}%")
keep = {k: v for k, v in tot.items() if not any(e in k for e in excl)}
S = sum(keep.values())
if excl:
    print(f"# shares within the solve (excluding {', '.join(excl)}): " +
          ", ".join(f"{k} {100 * v / S:.1f}%" for k, v in sorted(keep.items(), key=lambda kv: -kv[1])[:6]))
