"""bench.py parses and answers --help without a GPU (driver contract smoke)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_help():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "--gpus" in r.stdout and "--impl" in r.stdout


def test_graft_entry_imports():
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; assert callable(g.build) and callable(g.smoke)"],
                       cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
