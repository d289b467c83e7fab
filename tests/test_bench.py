"""CPU: bench.py's reference arm keeps the driver's JSON contract (one line,
metric/unit/config matching the GPU arm, impl=reference, cpu_baseline and an
e2e object with zero host<->device bytes), times the reference itself when
the driver's install is present, and `--gpus N` relaunches under torchrun."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAVE_REF = os.path.isfile(os.path.join(ROOT, "baseline", "_ref", "holotrack", "solver.py"))


def _json_lines(out):
    return [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]


def _check_line(d):
    assert d["impl"] == "reference"
    assert d["unit"] == "voxel-iter/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["metric"].startswith("voxel-iterations/sec")
    assert d["cpu_baseline"]["kind"] == ("reference" if HAVE_REF else "port")
    assert d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "voxel-iter/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("c1: 256x256x64")
    assert "2 FISTA iterations" in d["config"]["sample"]


def test_reference_arm_json_contract():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _json_lines(out)
    assert len(lines) == 1
    _check_line(lines[0])
    assert lines[0]["n_gpus"] == 1


def test_reference_arm_non_zero_rank_is_silent():
    """Under torchrun (N > 1) only rank 0 runs the CPU reference; the other
    ranks exit 0 without work or output."""
    env = dict(os.environ, OMP_NUM_THREADS="1", RANK="1", LOCAL_RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=120,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert not _json_lines(out)


def test_gpus_flag_self_launches_torchrun():
    """`bench.py --gpus 2` with no WORLD_SIZE relaunches itself under torchrun
    with 2 ranks (here the reference arm, so no GPU is needed): rank 0
    prints the one line with n_gpus = 2, rank 1 stays silent."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--gpus", "2", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _json_lines(out)
    assert len(lines) == 1
    _check_line(lines[0])
    assert lines[0]["n_gpus"] == 2


def test_gpu_arm_rejects_world_mismatch():
    """The GPU arm refuses to report n_gpus it did not run (WORLD_SIZE set by
    a launcher that disagrees with --gpus)."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert out.returncode != 0
    assert "WORLD_SIZE" in out.stderr
