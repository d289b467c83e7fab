import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs on the GPU box)")
    config.addinivalue_line("markers", "slow: minutes of CPU; set HOLO_SLOW=1 to run")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("HOLO_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow oracle check; HOLO_SLOW=1 to run")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))


def geom_of(arr):
    from oracle.holo_oracle import Geometry
    nx, ny, nz, pitch, dz, z0, lam = arr
    return Geometry(int(nx), int(ny), int(nz), pitch, dz, z0, lam)


def dense_from_golden(d):
    g = geom_of(d["geom"])
    x = np.zeros((g.nz, g.ny, g.nx), dtype=np.complex128)
    x[d["k"], d["r"], d["c"]] = d["v"]
    return x


def rel_l2(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


FISTA_CASES = ["fista_64", "fista_64_tvheavy", "fista_64_stall", "fista_64_backtrack", "fista_64_fixed_stop",
               "fista_64_diverge", "fista_64_zero", "fista_128", "fista_c1",
               "fista_64_real", "fista_64_real_tv", "fista_128_real"]


def fista_kwargs(d):
    lam = d["lam"]
    step = float(d["step_in"])
    return dict(lam_l1=float(lam[0]), lam_tv=float(lam[1]), max_iters=int(d["iters"]), inner=int(d["inner"]),
                policy=str(d["policy"]), step_size=None if step < 0 else step, stop_tol=float(d["stop_tol"]),
                real=bool(d["real"]) if "real" in d else False)
