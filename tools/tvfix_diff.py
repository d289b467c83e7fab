"""Where do the tvfix (54-row tiles) and 52-row-tile proxes differ?  One prox
of a random stack through holo_op_prox_fl with HOLO_PROX_TVFIX=1 / 0."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_04884_b200 import VolumeGeometry  # noqa: E402
from paper_1904_04884_b200.engine import HoloEngine  # noqa: E402

ny = nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
nz = 4
rng = np.random.default_rng(1)
v = (rng.standard_normal((nz, ny, nx)) + 1j * rng.standard_normal((nz, ny, nx))).astype(np.complex64)
eng = HoloEngine(VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9))
out = {}
for fix in ("1", "0"):
    os.environ["HOLO_PROX_TVFIX"] = fix
    out[fix] = eng.prox_fl(v, 0.3, 0.2, 5)
a, b = out["1"], out["0"]
d = np.abs(a - b)
print("max |diff|", d.max(), "differing", int((d > 0).sum()), "of", d.size)
rows = np.nonzero(d.max(axis=(0, 2)) > 0)[0]
cols = np.nonzero(d.max(axis=(0, 1)) > 0)[0]
print("rows with differences:", rows[:60].tolist(), "...", len(rows))
print("cols with differences:", cols[:60].tolist(), "...", len(cols))
