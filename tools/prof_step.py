"""Small driver for ncu: build a workload's layers, run a few fused
normalized-Laplacian steps (no timing, no CPU baseline).

    python tools/prof_step.py [steps] [side|cfg4]   (default: 3 steps of config 2 at 512)
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
from paper_2007_05239_b200 import with_shift
from paper_2007_05239_b200.graphs import apply_sym_laplacian_dev


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    which = sys.argv[2] if len(sys.argv) > 2 else "512"
    torch.cuda.set_device(0)
    if which == "cfg4":
        wl = synth.config4_large(seed=0)
    else:
        wl = synth.config2_segmentation(seed=0, side=int(which))
    G = synth.build_graph(wl, device=0)
    layers = [with_shift(l, math.log(2.0)) for l in G.layers]
    v = torch.from_numpy(np.random.default_rng(1).standard_normal(wl.n)).cuda()
    ys = [torch.empty_like(v) for _ in layers]
    for _ in range(steps):
        for lay, y in zip(layers, ys):
            apply_sym_laplacian_dev(lay, v, y)
    torch.cuda.synchronize()
    for lay in layers:
        print(lay.weights._bindings[0].stats())


if __name__ == "__main__":
    main()
