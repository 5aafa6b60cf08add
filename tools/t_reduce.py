import math, os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, synth
from paper_2007_05239_b200 import _lib, with_shift
torch.cuda.set_device(0)
wl = synth.config2_segmentation(seed=0)
G = synth.build_graph(wl, device=0, layer_ids=[0])
b = G.layers[0].weights._bindings[0]
lib = _lib.lib()
v = torch.from_numpy(np.random.default_rng(1).standard_normal(wl.n)).cuda()
grid = torch.empty(b.stats()["grid_cells"], dtype=torch.float64, device="cuda")
lib.mlb_spread(b.ptr, _lib.ptr(v), _lib.ptr(grid), _lib.MLB_USE_ISD | _lib.MLB_SPREAD_ONLY, _lib.stream_ptr())

s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3): lib.mlb_reduce(b.ptr, _lib.ptr(grid), _lib.stream_ptr())
s.record()
for _ in range(20): lib.mlb_reduce(b.ptr, _lib.ptr(grid), _lib.stream_ptr())
e.record(); e.synchronize()
print("reduce", s.elapsed_time(e) / 20 * 1e3, "us")
