"""When should the cheap d=2 layer start relative to the d=3 layer's stages?
(profiling aid: stage hooks, two streams, CUDA events; not the product path)"""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch, synth
import bench
from paper_2007_05239_b200 import _lib

torch.cuda.set_device(0)
lib = _lib.lib()
wl = synth.config2_segmentation(seed=0)
layers = bench.build_layers(wl, 0, math.log(2.0))
n = wl.n
B = [l.weights._bindings[0] for l in layers]
v = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
g = [torch.empty(b.stats()["grid_cells"], dtype=torch.float64, device="cuda") for b in B]
g2 = [torch.empty_like(x) for x in g]
y = [torch.empty_like(v) for _ in B]
hi = torch.cuda.Stream(priority=-1)
lo = torch.cuda.Stream(priority=0)
main = torch.cuda.current_stream()
E = lambda: torch.cuda.Event(enable_timing=True)


def stages(t, s):
    sp = _lib.C.c_void_p(s.cuda_stream)
    yield lambda: lib.mlb_spread(B[t].ptr, _lib.ptr(v), _lib.ptr(g[t]), _lib.MLB_USE_ISD, sp)
    yield lambda: lib.mlb_convolve(B[t].ptr, _lib.ptr(g[t]), _lib.ptr(g2[t]), sp)
    yield lambda: lib.mlb_gather(B[t].ptr, _lib.ptr(g2[t]), _lib.ptr(y[t]), 0, sp)


def run(after):
    """after = index of the d=3 stage after whose launch the d=2 layer may start
    (-1: at once; 3: after the whole d=3 layer; None: d=3 alone)."""
    e0, e3, e2 = E(), E(), E()
    fork = torch.cuda.Event()
    gate = torch.cuda.Event()
    e0.record(main)
    fork.record(main)
    hi.wait_event(fork)
    lo.wait_event(fork)
    if after == -1:
        gate.record(main)
    for k, st in enumerate(stages(0, hi)):
        with torch.cuda.stream(hi):
            st()
            if after == k:
                gate.record(hi)
    e3.record(hi)
    if after is not None:
        lo.wait_event(gate)
        for st in stages(1, lo):
            with torch.cuda.stream(lo):
                st()
    e2.record(lo)
    main.wait_stream(hi)
    main.wait_stream(lo)
    return e0, e3, e2


for after in (None, -1, 0, 1, 2):
    rows = []
    for rep in range(40):
        e0, e3, e2 = run(after)
        torch.cuda.synchronize()
        if rep >= 10:
            rows.append((e0.elapsed_time(e3), e0.elapsed_time(e2)))
    r = np.median(np.array(rows), axis=0) * 1e3
    print(f"d2 starts after d3 stage {after}: d3 done {r[0]:6.1f} us, d2 done {r[1]:6.1f} us")
