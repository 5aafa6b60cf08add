"""Time the d=3 spread kernel of config 2 with parts switched off (profiling aid)."""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import synth
from paper_2007_05239_b200 import _lib, with_shift
torch.cuda.set_device(0)
wl = synth.config2_segmentation(seed=0)
LID = int(os.environ.get("LAYER", "0"))
G = synth.build_graph(wl, device=0, layer_ids=[LID])
lay = with_shift(G.layers[0], math.log(2.0))
b = lay.weights._bindings[0]
lib = _lib.lib()
v = torch.from_numpy(np.random.default_rng(1).standard_normal(wl.n)).cuda()
grid = torch.empty(b.stats()["grid_cells"], dtype=torch.float64, device="cuda")


def timed(fn, reps=20):
    """Device time per call: `reps` calls captured in one CUDA graph (host launch cost excluded)."""
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / reps * 1e3
for name, bits in [("full", 0), ("no-accumulate", 1 << 16), ("no-windows", 1 << 17), ("no-flush", 1 << 18),
                   ("none", (1 << 16) | (1 << 17) | (1 << 18)), ("no-tile-io", 1 << 19),
                   ("none+no-tile-io", (1 << 16) | (1 << 17) | (1 << 18) | (1 << 19))]:
    f = _lib.MLB_USE_ISD | _lib.MLB_SPREAD_ONLY | bits
    for _ in range(3):
        lib.mlb_spread(b.ptr, _lib.ptr(v), _lib.ptr(grid), f, _lib.stream_ptr())
    print(f"{name:15s} {timed(lambda: lib.mlb_spread(b.ptr, _lib.ptr(v), _lib.ptr(grid), f, _lib.stream_ptr())):8.1f} us")
print(b.stats())
grid2 = torch.empty_like(grid)
lib.mlb_spread(b.ptr, _lib.ptr(v), _lib.ptr(grid), _lib.MLB_USE_ISD, _lib.stream_ptr())
lib.mlb_convolve(b.ptr, _lib.ptr(grid), _lib.ptr(grid2), _lib.stream_ptr())
y = torch.empty_like(v)
for name, bits in [("gather full", 0), ("gather no-contraction", 1 << 16), ("gather no-windows", 1 << 17),
                   ("gather none", (1 << 16) | (1 << 17)), ("gather none+no-staging", (1 << 16) | (1 << 17) | (1 << 18)),
                   ("gather no-staging", 1 << 18)]:
    for _ in range(3):
        lib.mlb_gather(b.ptr, _lib.ptr(grid2), _lib.ptr(y), bits, _lib.stream_ptr())
    print(f"{name:22s} {timed(lambda: lib.mlb_gather(b.ptr, _lib.ptr(grid2), _lib.ptr(y), bits, _lib.stream_ptr())):8.1f} us")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
lib.mlb_spread(b.ptr, _lib.ptr(v), _lib.ptr(grid), _lib.MLB_USE_ISD | _lib.MLB_SPREAD_ONLY, _lib.stream_ptr())
for _ in range(3):
    lib.mlb_reduce(b.ptr, _lib.ptr(grid), _lib.stream_ptr())
print(f"reduce (merge + R2)     {timed(lambda: lib.mlb_reduce(b.ptr, _lib.ptr(grid), _lib.stream_ptr())):8.1f} us")
print(f"convolve                {timed(lambda: lib.mlb_convolve(b.ptr, _lib.ptr(grid), _lib.ptr(grid2), _lib.stream_ptr())):8.1f} us")
