"""BASELINE configs[4]: matvec micro-benchmark.

n points uniform in the ball of radius 0.21875 (the reference rejects 0.25),
v ~ N(0,1) (x drawn before v, one default_rng(0) stream), Gaussian sigma in
{0.05, 0.2} (box units), N in {16, 32, 64}, m in {3, 4, 6}, p = 8; R
normalized-Laplacian matvecs timed (CUDA events) after warm-up with a
prebuilt binding and degrees; accuracy of W v against the exact O(n^2) sum
(GPU direct kernel) on a 2,000-target subsample (default_rng(1)).

    python tools/bench_micro.py [--n 1e5,1e6,1e7] [--d 1,2,3] [--reps 100] [--quick]
"""

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth


def exact_rows(points, v, sigma, rows):
    """(W v)[rows] exactly: kernel sums of the sampled targets against all points (GPU)."""
    X = torch.from_numpy(points).cuda()
    vd = torch.from_numpy(v).cuda()
    out = np.empty(len(rows))
    for lo in range(0, len(rows), 256):
        r = torch.from_numpy(rows[lo:lo + 256]).cuda()
        d2 = torch.cdist(X[r], X).pow(2)
        K = torch.exp(-d2 / sigma ** 2)
        out[lo:lo + 256] = (K @ vd - vd[r]).cpu().numpy()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="100000,1000000,10000000")
    ap.add_argument("--d", default="1,2,3")
    ap.add_argument("--N", default="16,32,64")
    ap.add_argument("--m", default="3,4,6")
    ap.add_argument("--sigma", default="0.05,0.2")
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--quick", action="store_true", help="one (N, m, sigma) per (n, d)")
    args = ap.parse_args()
    from paper_2007_05239_b200 import KernelSpec, KernelWeights, build_layer, build_plan, with_shift
    from paper_2007_05239_b200.graphs import apply_sym_laplacian_dev
    torch.cuda.set_device(0)
    combos = []
    for n in [int(float(x)) for x in args.n.split(",")]:
        for d in [int(x) for x in args.d.split(",")]:
            if args.quick:
                combos.append((n, d, 32, 4, 0.2))
                continue
            for N in [int(x) for x in args.N.split(",")]:
                for m in [int(x) for x in args.m.split(",")]:
                    for s in [float(x) for x in args.sigma.split(",")]:
                        combos.append((n, d, N, m, s))
    for n, d, N, m, sigma in combos:
        x, v = synth.config5_micro(n, d, seed=0)
        kern = KernelSpec("gaussian", sigma)
        t0 = time.perf_counter()
        plan = build_plan(kern, d=d, N=N, m_nfft=m, p_nfft=8)
        w = KernelWeights(x, kern, plan=plan)
        layer = with_shift(build_layer(w), math.log(2.0))
        torch.cuda.synchronize()
        t_bind = time.perf_counter() - t0
        vd = torch.from_numpy(v).cuda()
        y = torch.empty_like(vd)
        for _ in range(3):
            apply_sym_laplacian_dev(layer, vd, y)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(args.reps):
            apply_sym_laplacian_dev(layer, vd, y)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / args.reps
        rows = np.sort(np.random.default_rng(1).choice(n, size=min(2000, n), replace=False))
        Wv = w.matvec(vd)[torch.from_numpy(rows).cuda()].cpu().numpy()
        ex = exact_rows(x, v, sigma, rows)
        err = float(np.linalg.norm(Wv - ex) / np.linalg.norm(ex))
        print(json.dumps({"n": n, "d": d, "N": N, "m": m, "sigma": sigma, "ms_per_matvec": ms,
                          "node_layers_per_s": n / (ms * 1e-3), "bind_s": t_bind,
                          "rel_err_vs_direct_2000": err}), flush=True)
        del layer, w, plan
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
