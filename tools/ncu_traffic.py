"""DRAM traffic of one captured launch (ncu --set full) -> profiles/<round>_traffic.json.

    python tools/ncu_traffic.py REP KERNEL_CLASS VOXELS_IN_LAUNCH [OUT]

bench.py reports roofline.traffic = dram_bytes_per_voxel x voxels per launch.
"""
import csv
import io
import json
import os
import subprocess
import sys

# NCU_K=<regex>: one kernel of a multi-kernel report
_K = ((["-k", "regex:" + os.environ["NCU_K"]] + (["--kernel-name-base", "mangled"] if os.environ.get("NCU_MANGLED") else []))
      if os.environ.get("NCU_K") else [])

rep, cls, vox = sys.argv[1], sys.argv[2], int(sys.argv[3])
out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(os.path.dirname(__file__), "..", "profiles", "r01_traffic.json")
rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep] + _K + ["--page", "raw", "--csv"], capture_output=True,
                                                  text=True).stdout)))
d = dict(zip(rows[0], rows[2]))
unit = dict(zip(rows[0], rows[1]))


def num(k):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
             "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit.get(k, "byte"), 1)
    return float(d[k].replace(",", "")) * scale


rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
data = json.load(open(out)) if os.path.exists(out) else {}
data[cls] = {"dram_bytes_per_voxel": (rd + wr) / vox, "read_bytes": rd, "write_bytes": wr, "voxels": vox,
             "kernel": d.get("Kernel Name"), "duration_ns": num("gpu__time_duration.sum"), "report": os.path.basename(rep)}
json.dump(data, open(out, "w"), indent=1)
print(json.dumps(data[cls]))
