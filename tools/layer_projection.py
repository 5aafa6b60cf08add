"""Per-rank compute of the layer round-robin power-mean operator (config 3:
52 feature-grouped layers), on ONE GPU.

    python tools/layer_projection.py [--worlds 2 4 8] [--reps 5] [--out file.json]

dist.LayerParallelGraph gives rank r the layers t = r, r + N, ...; one outer
Lanczos step of power_mean_eigs applies M_p^p = (1/T) sum_t PKSM_t(v) with
each rank solving its own layers' PKSMs (lockstep when it holds >= 4 layers)
and one all-gather of the per-layer results.  For every world size N and
rank r this times that rank's share -- apply_Lp_power_dev on the sub-graph
of its layers, warm (graphs captured), CUDA events, the ranks one after the
other -- on a seeded vector.  The all-gather (52 x 40,000 doubles = 16.6 MB
summed over ranks, NVLink) is not measured here; the projection adds an
assumed time and says so.
"""

import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--allgather-us", type=float, default=60.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch

    import synth
    from paper_2007_05239_b200 import MultilayerGraph, PowerMeanConfig, with_shift
    from paper_2007_05239_b200.powermean import apply_Lp_power_dev
    wl = synth.CONFIGS[3](seed=0)
    G = synth.build_graph(wl, device=0)
    delta = math.log(2.0)
    layers = [with_shift(lay, delta) for lay in G.layers]
    cfg = PowerMeanConfig(p=wl.p_mean)
    v = torch.from_numpy(np.random.default_rng(4).standard_normal(wl.n)).cuda()
    res = {"workload": wl.name, "n": wl.n, "layers": len(layers), "allgather_us_assumed": a.allgather_us,
           "worlds": {}}

    def time_apply(sub):
        for _ in range(2):   # warm: graph capture, pools
            apply_Lp_power_dev(sub, cfg, v)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            apply_Lp_power_dev(sub, cfg, v)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    for N in [1] + list(a.worlds):
        per_rank = [time_apply(MultilayerGraph(tuple(layers[r::N]))) for r in range(N)]
        worst = max(per_rank)
        proj = worst + (a.allgather_us * 1e-3 if N > 1 else 0.0)
        res["worlds"][N] = {"per_rank_ms": per_rank, "max_ms": worst, "projected_ms": proj}
        print(N, ["%.2f" % x for x in per_rank], "projected %.2f ms" % proj, flush=True)
    base = res["worlds"][1]["projected_ms"]
    for N, r in res["worlds"].items():
        r["projected_speedup"] = base / r["projected_ms"]
    out = json.dumps(res, indent=1)
    print(out)
    if a.out:
        with open(a.out, "w") as f:
            f.write(out)


if __name__ == "__main__":
    main()
