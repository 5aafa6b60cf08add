"""Step time of each layer alone vs both layers (streams) -- profiling aid."""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch, synth
from paper_2007_05239_b200 import LaplacianBatch, MultilayerGraph, with_shift
torch.cuda.set_device(0)
wl = synth.config2_segmentation(seed=0)
G = synth.build_graph(wl, device=0)
layers = [with_shift(l, math.log(2.0)) for l in G.layers]
v = torch.from_numpy(np.random.default_rng(1).standard_normal(wl.n)).cuda()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for name, ls in [("d3 only", layers[:1]), ("d2 only", layers[1:]), ("both", layers)]:
    b = LaplacianBatch(MultilayerGraph(tuple(ls)))
    b._v.copy_(v)
    for _ in range(5):
        b._run()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    tot = 0.0
    for i in range(30):
        flush.fill_(float(i))
        ev[0].record(); b._run(); ev[1].record(); ev[1].synchronize()
        tot += ev[0].elapsed_time(ev[1])
    print(f"{name:8s} {tot / 30 * 1e3:7.1f} us/step")
