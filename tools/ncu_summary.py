"""Summarise an .ncu-rep (details page + SASS instruction mix) as text for profiles/."""
import csv
import os
import io
import subprocess
import sys

# NCU_K=<regex>: one kernel of a multi-kernel report
_K = ["-k", "regex:" + os.environ["NCU_K"]] if os.environ.get("NCU_K") else []
from collections import Counter

SECTIONS = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Compute Workload Analysis",
            "Occupancy", "Launch Statistics", "Scheduler Statistics", "Warp State Statistics")


def run(args):
    return subprocess.run(["ncu", "-i", args[0]] + _K + args[1:], capture_output=True, text=True).stdout


def main(rep):
    out = []
    det = run([rep, "--page", "details", "--csv"])
    rows = list(csv.reader(io.StringIO(det)))
    hdr = rows[0]
    kernel = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if kernel is None:
            kernel = d.get("Kernel Name")
            out.append(f"kernel: {kernel}")
        if d.get("Section Name") in SECTIONS and d.get("Metric Name"):
            out.append(f"{d['Section Name'][:28]:28s} | {d['Metric Name'][:48]:48s} | {d['Metric Value']} {d['Metric Unit']}")
    raw = run([rep, "--page", "raw", "--csv"])
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        h, v = rr[0], rr[2]
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                    "sm__inst_executed.sum", "launch__registers_per_thread"):
            for i, name in enumerate(h):
                if name == key:
                    out.append(f"raw | {key} | {v[i]} {rr[1][i]}")
    src = run([rep, "--page", "source", "--csv", "--print-source", "sass"])
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2:
        sh = srows[1]
        ix = {k: i for i, k in enumerate(sh)}
        ops, tot = Counter(), 0
        for r in srows[2:]:
            if len(r) < len(sh):
                continue
            try:
                n = int(r[ix["Instructions Executed"]])
            except ValueError:
                continue
            toks = r[ix["Source"]].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            ops[op.split(".")[0]] += n
            tot += n
        out.append(f"SASS warp-instructions executed: {tot}")
        for op, n in ops.most_common(20):
            out.append(f"  {op:10s} {n:14d}  {100.0 * n / tot:5.1f}%")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
