"""Where does a PKSM solve spend its time?  Wall time per Krylov step against
the device time of the same work (profiling aid).

    python tools/pksm_profile.py [--config 2]
"""
import argparse
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    from paper_2007_05239_b200 import with_shift
    from paper_2007_05239_b200.krylov import PksmStats, pksm_layer_dev, pksm_layers_dev
    torch.cuda.set_device(0)
    wl = synth.CONFIGS[args.config](seed=0)
    G = synth.build_graph(wl, device=0)
    layers = [with_shift(l, math.log(2.0)) for l in G.layers]
    v = torch.from_numpy(np.random.default_rng(1).standard_normal(wl.n)).cuda()
    out = torch.zeros_like(v)
    for name, fn in [("per-layer", lambda: [pksm_layer_dev(l, -1.0, v, out) for l in layers]),
                     ("lockstep", lambda: pksm_layers_dev(layers, -1.0, v, out))]:
        fn()
        torch.cuda.synchronize()
        PksmStats.reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        e1.synchronize()
        wall = time.perf_counter() - t0
        steps = sum(PksmStats.steps)
        print(f"{name:10s} wall {wall / steps * 1e6:7.1f} us/step ({steps} layer steps), "
              f"events {e0.elapsed_time(e1) * 1e3 / steps:7.1f} us/step")
    # device cost of one step's work, back to back (no host round trip)
    lay = layers[0]
    from paper_2007_05239_b200.graphs import apply_sym_laplacian_dev
    from paper_2007_05239_b200.krylov import cgs2
    dim = 50
    V = torch.randn((dim, wl.n), dtype=torch.float64, device="cuda")
    h = torch.empty(2 * dim + 3, dtype=torch.float64, device="cuda")
    for s in (5, 10, 20):
        y = torch.empty_like(v)
        for _ in range(3):
            apply_sym_laplacian_dev(lay, V[s], y)
            cgs2(V, s + 1, y, h[: s + 1], h[dim:dim + s + 1], h[dim + s + 1:dim + s + 2])
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            apply_sym_laplacian_dev(lay, V[s], y)
        e1.record()
        e1.synchronize()
        tm = e0.elapsed_time(e1) / 20 * 1e3
        e0.record()
        for _ in range(20):
            cgs2(V, s + 1, y, h[: s + 1], h[dim:dim + s + 1], h[dim + s + 1:dim + s + 2])
        e1.record()
        e1.synchronize()
        tc = e0.elapsed_time(e1) / 20 * 1e3
        t0 = time.perf_counter()
        for _ in range(20):
            apply_sym_laplacian_dev(lay, V[s], y)
            cgs2(V, s + 1, y, h[: s + 1], h[dim:dim + s + 1], h[dim + s + 1:dim + s + 2])
        host = (time.perf_counter() - t0) / 20 * 1e6
        torch.cuda.synchronize()
        print(f"s={s:2d}: matvec {tm:6.1f} us, cgs2 {tc:6.1f} us (device); host issue time of both {host:6.1f} us")


if __name__ == "__main__":
    main()
