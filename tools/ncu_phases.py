"""Per-source-line share of warp-stall samples and executed instructions for one
kernel of an .ncu-rep, attributing inlined code to the line of `fn_range`
(the function whose body lines we care about) it was inlined from.
usage: ncu_phases.py report.ncu-rep sass_with_inline_info.txt kernel_substr call_lines lo hi [n]
(sass: nvdisasm -gi -c of the same build)"""
import csv, io, re, subprocess, sys

rep, sass, ksub, calls, lo, hi = sys.argv[1:7]
n_top = int(sys.argv[7]) if len(sys.argv) > 7 else 40
calls = set(int(c) for c in calls.split(","))
lo, hi = int(lo), int(hi)
txt = open(sass).read().split("\n")
start = [i for i, l in enumerate(txt) if l.startswith(".text.") and ksub in l][0]
amap, pending, last = {}, [], None
for l in txt[start + 1:]:
    if l.startswith(".text.") or l.startswith("//----"):
        break
    if "//## File" in l:
        pending.append(l)
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if not m:
        continue
    if pending:
        ln = None
        for c in pending:
            mm = re.search(r'line (\d+) inlined at "[^"]*", line (\d+)', c)
            if mm and int(mm.group(2)) in calls:
                ln = int(mm.group(1))
        if ln is None:
            for c in pending:
                mm = re.search(r'line (\d+)', c)
                if mm and lo <= int(mm.group(1)) <= hi:
                    ln = int(mm.group(1))
            if ln is None:
                mm = re.search(r'line (\d+)', pending[-1])
                ln = ("outer", int(mm.group(1)) if mm else -1)
        last = ln
    amap[int(m.group(1), 16)] = last
    pending = []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [(int(r[0], 16), int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), int(r[ix["Instructions Executed"]] or 0))
        for r in rows[2:] if len(r) >= len(hdr) and r[0].startswith("0x")]
base = data[0][0]
acc = {}
for a, s, n in data:
    k = amap.get(a - base)
    x = acc.setdefault(k, [0, 0])
    x[0] += s
    x[1] += n
ts = sum(v[0] for v in acc.values())
tn = sum(v[1] for v in acc.values())
print(f"samples {ts}  instructions {tn}")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1][0])[:n_top]:
    print(f"{str(k):14s} {100 * v[0] / ts:5.1f}% time {100 * v[1] / tn:5.1f}% instr")
