"""Config 4: does a concurrent PCIe copy slow the step's kernels (or the
kernels the copy)?  CUDA events per stream; profiling aid for the e2e leg."""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch, synth

from paper_2007_05239_b200 import LaplacianBatch, MultilayerGraph
from paper_2007_05239_b200.graphs import apply_sym_laplacian_dev

torch.cuda.set_device(0)
wl = synth.config4_large(seed=0)
from paper_2007_05239_b200 import with_shift
G = synth.build_graph(wl, device=0)
layers = [with_shift(l, math.log(2.0)) for l in G.layers]
n, T = wl.n, len(layers)
vd = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
yd = torch.empty((T, n), dtype=torch.float64, device="cuda")
host = torch.empty(n, dtype=torch.float64, pin_memory=True)
hsrc = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).pin_memory()
dbuf = torch.empty(n, dtype=torch.float64, device="cuda")
E = lambda: torch.cuda.Event(enable_timing=True)
sc, sx = torch.cuda.Stream(), torch.cuda.Stream()


def layer_run(t, s):
    with torch.cuda.stream(s):
        e0, e1 = E(), E()
        e0.record(s)
        apply_sym_laplacian_dev(layers[t], vd, yd[t])
        e1.record(s)
    return e0, e1


def copy_run(kind, s):
    with torch.cuda.stream(s):
        e0, e1 = E(), E()
        e0.record(s)
        if kind == "d2h":
            host.copy_(dbuf, non_blocking=True)
        else:
            dbuf.copy_(hsrc, non_blocking=True)
        e1.record(s)
    return e0, e1


res = {}
for rep in range(8):
    for t in range(T):
        for mode in ("alone", "d2h", "h2d"):
            torch.cuda.synchronize()
            ev = layer_run(t, sc)
            cv = copy_run(mode, sx) if mode != "alone" else None
            torch.cuda.synchronize()
            if rep >= 2:
                res.setdefault(f"layer{t}_{mode}", []).append(ev[0].elapsed_time(ev[1]))
                if cv:
                    res.setdefault(f"copy_{mode}_with_layer{t}", []).append(cv[0].elapsed_time(cv[1]))
    for mode in ("d2h", "h2d"):
        torch.cuda.synchronize()
        cv = copy_run(mode, sx)
        torch.cuda.synchronize()
        if rep >= 2:
            res.setdefault(f"copy_{mode}_alone", []).append(cv[0].elapsed_time(cv[1]))
print({k: round(float(np.median(v)), 3) for k, v in res.items()})

# both directions at once (PCIe full duplex?)
sy = torch.cuda.Stream()
dbuf2 = torch.empty(n, dtype=torch.float64, device="cuda")
host2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
bi = []
for rep in range(6):
    torch.cuda.synchronize()
    a = copy_run("h2d", sx)
    with torch.cuda.stream(sy):
        e0, e1 = E(), E()
        e0.record(sy)
        host2.copy_(dbuf2, non_blocking=True)
        e1.record(sy)
    torch.cuda.synchronize()
    bi.append((round(a[0].elapsed_time(a[1]), 3), round(e0.elapsed_time(e1), 3)))
print("bidirectional (h2d ms, d2h ms):", bi)

# drift of the pinned-buffer copy rates after allocation
import time
t0 = time.time()
drift = []
while time.time() - t0 < float(os.environ.get("DRIFT_S", "0")):
    for mode in ("h2d", "d2h"):
        torch.cuda.synchronize()
        cv = copy_run(mode, sx)
        torch.cuda.synchronize()
        drift.append((round(time.time() - t0, 1), mode, round(cv[0].elapsed_time(cv[1]), 3)))
    time.sleep(1.0)
print(drift)
