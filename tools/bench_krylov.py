"""CGS2 / GEMV throughput of the Krylov kernels vs the HBM roofline.

    python tools/bench_krylov.py [--n 262144] [--cols 10,25,50]

cgs2 over s columns reads V twice for V^T w and twice for w -= V h:
4 * 8 n s bytes (+ w traffic, 8 n per pass).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=262144)
    ap.add_argument("--cols", default="10,25,50")
    args = ap.parse_args()
    from paper_2007_05239_b200.krylov import cgs2, gemv_n, gemv_t
    n = args.n
    for s in [int(x) for x in args.cols.split(",")]:
        V = torch.randn(s, n, dtype=torch.float64, device="cuda")
        w = torch.randn(n, dtype=torch.float64, device="cuda")
        h = torch.empty(2 * s + 3, dtype=torch.float64, device="cuda")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        res = {}
        for name, fn, nbytes in [
            ("gemv_t", lambda: gemv_t(V, n, s, w, h[:s]), 8 * n * (s + 1)),
            ("gemv_n", lambda: gemv_n(V, n, s, h[:s], w), 8 * n * (s + 1)),
            ("cgs2", lambda: cgs2(V, s, w, h[:s], h[s:2 * s], h[2 * s:2 * s + 1]), 8 * n * (4 * s + 4)),
        ]:
            for _ in range(3):
                fn()
            ev[0].record()
            for _ in range(20):
                fn()
            ev[1].record()
            ev[1].synchronize()
            ms = ev[0].elapsed_time(ev[1]) / 20
            res[name] = {"us": ms * 1e3, "GBps": nbytes / (ms * 1e-3) / 1e9}
        print(json.dumps({"n": n, "cols": s, **res}))


if __name__ == "__main__":
    main()
