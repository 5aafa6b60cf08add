"""Break the e2e step into H2D, compute, D2H (CUDA events) -- profiling aid."""
import math, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch, synth
from paper_2007_05239_b200 import LaplacianBatch, MultilayerGraph, with_shift
torch.cuda.set_device(0)
wl = synth.config2_segmentation(seed=0)
G = synth.build_graph(wl, device=0)
G = MultilayerGraph(tuple(with_shift(l, math.log(2.0)) for l in G.layers))
b = LaplacianBatch(G)
n, T = wl.n, G.T
vp = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).pin_memory()
yp = torch.empty((T, n), dtype=torch.float64, pin_memory=True)
vd = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(5):
    b.apply(vp, out=yp)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
def timeit(fn, reps=20):
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record(); ev[1].synchronize()
    return ev[0].elapsed_time(ev[1]) / reps * 1e3
print("H2D 2MB        %.1f us" % timeit(lambda: vd.copy_(vp, non_blocking=True)))
print("D2H 2MB        %.1f us" % timeit(lambda: yp[0].copy_(vd, non_blocking=True)))
print("D2H 4MB        %.1f us" % timeit(lambda: yp.copy_(b._y, non_blocking=True)))
print("compute (run)  %.1f us" % timeit(lambda: b._run()))
print("apply (e2e)    %.1f us" % timeit(lambda: b.apply(vp, out=yp)))
t0 = time.perf_counter()
for _ in range(20):
    b.apply(vp, out=yp)
print("apply wall     %.1f us" % ((time.perf_counter() - t0) / 20 * 1e6))
# host-side split of one apply (whole-step graph path)
import time as _t
key = (vp.data_ptr(), yp.data_ptr())
print("whole-step graph cached:", key in b._full)
g, cnt = b._full[key]
main = torch.cuda.current_stream()
ts = []
for _ in range(20):
    t0 = _t.perf_counter(); g.replay(); t1 = _t.perf_counter(); main.synchronize(); t2 = _t.perf_counter()
    ts.append((t1 - t0, t2 - t1))
ts = np.array(ts) * 1e6
print("replay launch %.1f us, wait %.1f us (median)" % tuple(np.median(ts, axis=0)))
ev[0].record(); g.replay(); ev[1].record(); ev[1].synchronize()
print("whole-step graph device time %.1f us" % (ev[0].elapsed_time(ev[1]) * 1e3))
