"""Bounds-checked build (make checked; common.cuh HOLO_CHECKS) as the
compute-sanitizer substitute: compute-sanitizer is closed on the GPU pool.

tools/checked_solve.py runs small solves over every kernel family -- the
single-pass and multi-pass strip prox, the generic prox, the packed real
engine, plane skipping, the in-process rank group's peer-memory plane sum and
the guard fix-up, the mixed-radix passes of general plane sides -- once with the normal library and once with the checked one,
in which every kernel tests its global indices and tensor-copy frames against
the buffers' bounds, the prox / FFT kernels fill their shared memory with NaN
before use and the engine fills fresh device buffers with 0xFF (NaN).  The two
runs must print the same histories and solution hashes (a never-written slot
or allocation that reached the output would have turned it into NaN) and the
checked run must report no violations."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1904_04884_b200", "libholo_b200_checked.so")


def _run(lib):
    env = dict(os.environ)
    if lib:
        env["HOLO_LIB_PATH"] = lib
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checked_solve.py")], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    return [ln for ln in r.stdout.splitlines() if ln.strip()]


def test_checked_build_matches_and_reports_no_violations():
    if not os.path.exists(CHECKED):
        raise FileNotFoundError(f"{CHECKED} missing: run `make checked` (or __graft_entry__.build())")
    normal = _run(None)
    checked = _run(CHECKED)
    assert normal[-1] == "checked-build 0 check-bits 0x0", normal[-1]
    assert checked[-1] == "checked-build 1 check-bits 0x0", checked[-1]
    assert normal[:-1] == checked[:-1]
    assert len(normal) == 10
