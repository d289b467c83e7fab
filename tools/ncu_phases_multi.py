"""Per-source-line stall samples for every kernel of a multi-kernel .ncu-rep
(inline-aware: code inlined from prox_tile is attributed to its prox_strip.cu
line).  usage: ncu_phases_multi.py report.ncu-rep nvdisasm_gi.sass lo hi [n]"""
import csv, io, re, subprocess, sys, collections
rep, sass, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
n_top = int(sys.argv[5]) if len(sys.argv) > 5 else 15
txt = open(sass).read().split("\n")
maps = {}  # kernel mangled substring -> {offset: line}
cur = None
for l in txt:
    if l.startswith(".text."):
        cur = {}; maps[l.split()[0]] = cur; pend = []; last = None; continue
    if cur is None: continue
    if "//## File" in l: pend.append(l); continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if not m: continue
    if pend:
        ln = None
        for c in pend:
            for mm in re.finditer(r'line (\d+)', c):
                v = int(mm.group(1))
                if lo <= v <= hi and ln is None: ln = v
        last = ln if ln is not None else ("outer",)
        pend = []
    cur[int(m.group(1), 16)] = last
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks = []; kname = None; hdr = None
for r in rows:
    if r and r[0] == "Kernel Name":
        if kname != r[1]: blocks.append([r[1], []]); kname = r[1]
        continue
    if r and r[0] == "Address": hdr = {h: i for i, h in enumerate(r)}; continue
    if hdr and r and r[0].startswith("0x"):
        blocks[-1][1].append((int(r[0], 16), int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0), int(r[hdr["Instructions Executed"]] or 0)))
for name, data in blocks:
    args = re.search(r"k_prox_strip<([^>]*)>", name)
    key = None
    if args:
        v = [re.sub(r"\(\w+\)", "", x).strip() for x in args.group(1).split(",")]
        kinds = ["b", "i", "b", "b", "i", "b"]  # TV, PH, RM, FAST, TT, ORD
        mang = "".join(f"L{k}{x}E" for k, x in zip(kinds, v))
        key = [k for k in maps if f"k_prox_stripI{mang}" in k]
    if not key: print("no map for", name[:60]); continue
    amap = maps[key[0]]; base = data[0][0]
    acc = collections.defaultdict(lambda: [0, 0])
    for a, s, n in data:
        k = amap.get(a - base); acc[k][0] += s; acc[k][1] += n
    ts = sum(v[0] for v in acc.values()); tn = sum(v[1] for v in acc.values())
    print(f"== {name[:70]}  samples {ts} instr {tn}")
    for k, v in sorted(acc.items(), key=lambda kv: -kv[1][0])[:n_top]:
        print(f"   {str(k):10s} {100*v[0]/ts:5.1f}% time {100*v[1]/tn:5.1f}% instr")
