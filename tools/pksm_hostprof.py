"""Host-side profile of one warm config-3 power-mean apply (cProfile), to see
where the lockstep PKSM spends host time per step (profiling aid).

    python tools/pksm_hostprof.py
"""
import cProfile
import math
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
from paper_2007_05239_b200 import PowerMeanConfig, with_shift
from paper_2007_05239_b200.graphs import MultilayerGraph
from paper_2007_05239_b200.powermean import apply_Lp_power_dev

wl = synth.CONFIGS[3](seed=0)
G = synth.build_graph(wl, device=0)
g = MultilayerGraph(tuple(with_shift(l, math.log(2.0)) for l in G.layers))
v = torch.from_numpy(np.random.default_rng(0).standard_normal(wl.n)).cuda()
cfg = PowerMeanConfig(p=-1.0)
for _ in range(3):
    apply_Lp_power_dev(g, cfg, v)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    apply_Lp_power_dev(g, cfg, v)
torch.cuda.synchronize()
print("warm apply ms", (time.perf_counter() - t0) / 5 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    apply_Lp_power_dev(g, cfg, v)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
