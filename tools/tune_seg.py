"""Spread + reduction time of the config-2 RGB layer vs segment size (MLB_SEG_POINTS)."""
import math, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import math, os, sys
sys.path.insert(0, %r)
import numpy as np, torch, synth
from paper_2007_05239_b200 import _lib, with_shift
torch.cuda.set_device(0)
wl = synth.config2_segmentation(seed=0)
G = synth.build_graph(wl, device=0, layer_ids=[0])
lay = with_shift(G.layers[0], math.log(2.0)); b = lay.weights._bindings[0]; lib = _lib.lib()
v = torch.from_numpy(np.random.default_rng(1).standard_normal(wl.n)).cuda()
grid = torch.empty(b.stats()["grid_cells"], dtype=torch.float64, device="cuda")
def t(f, reps=20):
    for _ in range(3): f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): f()
    e.record(); e.synchronize(); return s.elapsed_time(e) / reps * 1e3
ts = t(lambda: lib.mlb_spread(b.ptr, _lib.ptr(v), _lib.ptr(grid), _lib.MLB_USE_ISD | _lib.MLB_SPREAD_ONLY, _lib.stream_ptr()))
tr = t(lambda: lib.mlb_reduce(b.ptr, _lib.ptr(grid), _lib.stream_ptr()))
print(os.environ.get("MLB_SEG_POINTS"), b.stats()["segments"], f"spread {ts:.1f} us  reduce {tr:.1f} us  sum {ts+tr:.1f}")
''' % ROOT
for sp in sys.argv[1:]:
    env = dict(os.environ, MLB_SEG_POINTS=sp)
    print(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout.strip())
