"""bench.py parses and answers --help without a GPU (driver contract smoke)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_help():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "--gpus" in r.stdout and "--impl" in r.stdout


def test_graft_entry_imports():
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; assert callable(g.build) and callable(g.smoke)"],
                       cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_reference_arm_line():
    """`--impl reference` prints the contract's JSON line (CPU only, small sample)."""
    import json
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1", "--ref-sample", "3000"], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    assert len(r.stdout.strip().splitlines()) == 1   # stdout is the one JSON line
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]



@pytest.mark.gpu
def test_bench_line_contract():
    """The default arm's JSON line carries every key the driver reads."""
    import json
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline"], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "clocks", "roofline"):
        assert k in d, k
    assert d["value"] > 1e9 and d["gpu_launches"] > 0 and d["steps"] == 3
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 8 * d["config"]["nodes_per_rank"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_bench_sharded_step_on_one_gpu():
    """The node-range sharded step (the N > 1 bench path: per layer one NCCL
    all-reduce of its grid per step) runs end to end on one GPU (`--sharded`);
    stdout holds only the JSON line even with NCCL's version banner on."""
    import json
    env = dict(os.environ, NCCL_DEBUG="VERSION")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--sharded", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline", "--workload", "cfg2"], capture_output=True, text=True, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert len(r.stdout.strip().splitlines()) == 1, r.stdout[:500]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 1 and d["value"] > 1e8 and "sharded" in d["config"]["parallelism"]
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
