"""pytest plugin: import THIS package under the reference's name, so the
reference's own test files exercise the B200 backend as a drop-in
(`import multilap` -> paper_2007_05239_b200, submodules likewise).

    python -m pytest -p integration.pytest_as_multilap <multilap tests>
"""

import importlib
import sys

SUBMODULES = ("errors", "kernels", "fastsum", "graphs", "krylov", "powermean", "allencahn", "datapipe", "config",
              "cli", "runner", "csvio", "nfft")


def _alias():
    # at plugin import: the reference's conftest.py imports multilap before any hook runs
    pkg = importlib.import_module("paper_2007_05239_b200")
    sys.modules["multilap"] = pkg
    for sub in SUBMODULES:
        try:
            sys.modules["multilap." + sub] = importlib.import_module("paper_2007_05239_b200." + sub)
        except ImportError:
            pass


_alias()
_start = [0]


def pytest_configure(config):
    from paper_2007_05239_b200 import _lib
    _start[0] = int(_lib.lib().mlb_launch_count())


def pytest_sessionfinish(session, exitstatus):
    from paper_2007_05239_b200 import _lib
    print(f"\n[as-multilap] libmlb kernel launches during the reference tests: "
          f"{int(_lib.lib().mlb_launch_count()) - _start[0]}")
