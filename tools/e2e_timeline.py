"""Timeline of one end-to-end step (H2D, per-layer compute, per-layer D2H),
CUDA events on each stream, non-graph path -- profiling aid."""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch, synth
import bench
from paper_2007_05239_b200 import LaplacianBatch, MultilayerGraph

torch.cuda.set_device(0)
wl = synth.config4_large(seed=0) if os.environ.get("CFG4") else synth.config2_segmentation(seed=0)
from paper_2007_05239_b200 import with_shift
layers = [with_shift(l, math.log(2.0)) for l in synth.build_graph(wl, device=0).layers]
n, T = wl.n, len(layers)
b = LaplacianBatch(MultilayerGraph(tuple(layers)))
vp = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).pin_memory()
yp = torch.empty((T, n), dtype=torch.float64, pin_memory=True)
for _ in range(50):
    b.apply(vp, out=yp)
torch.cuda.synchronize()
main = torch.cuda.current_stream()
E = lambda: torch.cuda.Event(enable_timing=True)
rows = []
DEFER = os.environ.get("DEFER")
ONLY = os.environ.get("ONLY")
for rep in range(30):
    e0, eh = E(), E()
    ec = [E() for _ in range(T)]
    ed = [E() for _ in range(T)]
    e0.record(main)
    if not os.environ.get("NOH2D"):
        b._v.copy_(vp, non_blocking=True)
    eh.record(main)
    b._fork.record(main)
    for t, (s, j) in enumerate(zip(b._streams, b._joins)):
        s.wait_event(b._fork)
        with torch.cuda.stream(s):
            if ONLY is None or int(ONLY) == t:
                b._layer(t)
            ec[t].record(s)
            if not DEFER:
                yp[t].copy_(b._y[t], non_blocking=True)
            ed[t].record(s)
        j.record(s)
    for j in b._joins:
        main.wait_event(j)
    main.synchronize()
    rows.append([e0.elapsed_time(eh)] + [e0.elapsed_time(e) for e in ec] + [e0.elapsed_time(e) for e in ed])
r = np.median(np.array(rows), axis=0) * 1e3
ev = [E(), E()]
ev[0].record(main)
for _ in range(20):
    b._run()
ev[1].record(main); ev[1].synchronize()
print("_run back-to-back %.1f us" % (ev[0].elapsed_time(ev[1]) / 20 * 1e3))
rr = []
for _ in range(20):
    ev[0].record(main); b._run(); ev[1].record(main); ev[1].synchronize()
    rr.append(ev[0].elapsed_time(ev[1]) * 1e3)
print("_run isolated %.1f us" % np.median(rr))
print("H2D done %.1f us" % r[0])
for t in range(T):
    print("layer %d (d=%d): compute done %.1f us, D2H done %.1f us" % (t, layers[t].weights.plan.d if hasattr(layers[t].weights, "plan") else -1, r[1 + t], r[1 + T + t]))
