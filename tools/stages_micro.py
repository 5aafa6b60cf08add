"""Stage times + HBM / FP64 fractions of the spread and gather kernels on the
config-5 micro-benchmark points (uniform ball, n = 1e7 by default).

    python tools/stages_micro.py [--n 1e7] [--d 1,2] [--N 64] [--m 4] [--sigma 0.2]
"""
import argparse
import json
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
    ap.add_argument("--n", default="1e7")
    ap.add_argument("--d", default="1,2")
    ap.add_argument("--N", type=int, default=64)
    ap.add_argument("--m", default="4")
    ap.add_argument("--sigma", type=float, default=0.2)
    ap.add_argument("--sorted", action="store_true", help="vectors in the binding's cell order (the solvers' order)")
    a = ap.parse_args()
    import bench
    from paper_2007_05239_b200 import KernelSpec, KernelWeights, build_layer, build_plan
    torch.cuda.set_device(0)
    n = int(float(a.n))
    hbm = bench._peaks()[0]
    fp64 = bench.measure_fp64_peak(torch, "cuda:0")
    for d in [int(x) for x in a.d.split(",")]:
        for m in [int(x) for x in a.m.split(",")]:
            x, v = synth.config5_micro(n, d, seed=0)
            kern = KernelSpec("gaussian", a.sigma)
            plan = build_plan(kern, d=d, N=a.N, m_nfft=m, p_nfft=8)
            layer = build_layer(KernelWeights(x, kern, plan=plan))
            vd = torch.from_numpy(v).cuda()
            st = bench.stage_breakdown(torch, [layer.weights], vd, reps=10, sorted_order=a.sorted)
            rows = bench.kernel_table(st, "micro", hbm, fp64)
            for r in rows:
                if r["kernel"] in ("spread", "gather"):
                    print(json.dumps({"order": "sorted" if a.sorted else "node", "d": d, "m": m, "N": a.N, "n": n, "kernel": r["kernel"], "us": round(r["ms"] * 1e3, 1),
                                      "hbm_frac": round(r["hbm_frac"], 3), "fp64_frac": round(r["fp64_frac"], 3)}))


if __name__ == "__main__":
    main()
