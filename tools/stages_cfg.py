"""Stage split (spread / reduce / convolve / gather) of every layer of a config (profiling aid).

    python tools/stages_cfg.py [--config 4]
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    args = ap.parse_args()
    import bench
    from paper_2007_05239_b200 import with_shift
    torch.cuda.set_device(0)
    wl = synth.CONFIGS[args.config](seed=0)
    G = synth.build_graph(wl, device=0)
    layers = [with_shift(l, math.log(2.0)) for l in G.layers]
    v = torch.from_numpy(np.random.default_rng(1).standard_normal(wl.n)).cuda()
    for st in bench.stage_breakdown(torch, [l.weights for l in layers], v, reps=10):
        st.pop("stats", None)
        print({k: (round(x * 1e3, 1) if k.endswith("_ms") else x) for k, x in st.items()})


if __name__ == "__main__":
    main()
