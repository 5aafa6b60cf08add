"""Does the e2e number depend on what ran before it?  (profiling aid)

Measures LaplacianBatch.apply (pinned host in/out) the way bench.py does, at
several points: cold, after a long device-only soak, after an idle pause.
"""
import math, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch, synth
import bench
from paper_2007_05239_b200 import LaplacianBatch, MultilayerGraph

torch.cuda.set_device(0)
wl = synth.config2_segmentation(seed=0)
layers = bench.build_layers(wl, 0, math.log(2.0))
n, T = wl.n, len(layers)
batch = LaplacianBatch(MultilayerGraph(tuple(layers)))
v_host = np.random.default_rng(1000).standard_normal(n)
v_pin = torch.from_numpy(v_host).pin_memory()
y_pin = torch.empty((T, n), dtype=torch.float64, pin_memory=True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def e2e(reps=20, tag=""):
    for _ in range(5):
        batch.apply(v_pin, out=y_pin)
    torch.cuda.synchronize()
    ev[0].record()
    t0 = time.perf_counter()
    for _ in range(reps):
        batch.apply(v_pin, out=y_pin)
    ev[1].record(); ev[1].synchronize()
    wall = (time.perf_counter() - t0) / reps * 1e6
    dev = ev[0].elapsed_time(ev[1]) / reps * 1e3
    print(f"{tag:28s} device {dev:7.1f} us/step  wall {wall:7.1f} us/step", flush=True)


batch._v.copy_(v_pin.cuda())
for _ in range(5):
    batch._run()
torch.cuda.synchronize()
for i in range(3):
    e2e(tag=f"cold {i}")
t = time.perf_counter()
while time.perf_counter() - t < 0.6:
    for _ in range(20):
        batch._run()
    torch.cuda.synchronize()
for i in range(3):
    e2e(tag=f"after soak {i}")
time.sleep(0.5)
for i in range(3):
    e2e(tag=f"after idle 0.5s {i}")
for reps in (3, 10, 50, 200):
    e2e(reps=reps, tag=f"reps={reps}")
# the bench's clock sampler (nvidia-smi -lms 100) around a device-only soak
cs = bench.ClockSampler(0)
cs.start()
t = time.perf_counter()
while time.perf_counter() - t < 0.6:
    for _ in range(20):
        batch._run()
    torch.cuda.synchronize()
print("clocks", cs.stop())
for i in range(3):
    e2e(tag=f"after sampler {i}")
time.sleep(1.0)
for i in range(3):
    e2e(tag=f"after sampler + 1s {i}")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for i in range(20):
    flush.fill_(float(i)); batch._run()
torch.cuda.synchronize()
for i in range(3):
    e2e(tag=f"after flush loop {i}")

vd = torch.empty(n, dtype=torch.float64, device="cuda")
for nm, fn in (("h2d", lambda: batch._v.copy_(v_pin, non_blocking=True)),
               ("d2h", lambda: y_pin.copy_(batch._y, non_blocking=True))):
    ev[0].record()
    for _ in range(20):
        fn()
    ev[1].record(); ev[1].synchronize()
    print(nm, "us:", ev[0].elapsed_time(ev[1]) / 20 * 1e3)
