"""End-to-end solver benchmark: feature layers -> power-mean eigenpairs -> Allen-Cahn.

    python tools/bench_solver.py [--config 1|2|3] [--side S]

Prints one JSON line with stage times, the number of layer matvecs inside
the eigensolver (effective node*layers/s in the solver, SURVEY 8(d)
"Eigensolve" timing) and the classification accuracy.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--side", type=int, default=0)
    ap.add_argument("--k", type=int, default=0)
    args = ap.parse_args()
    from paper_2007_05239_b200 import (AllenCahnParams, PowerMeanConfig, _lib, allen_cahn_solve, power_mean_eigs,
                                       predict_labels, sample_labels)
    from paper_2007_05239_b200.krylov import PksmStats
    torch.cuda.set_device(0)
    gen = synth.CONFIGS[args.config]
    wl = gen(seed=0, side=args.side) if args.side else gen(seed=0)
    k = args.k or wl.k
    t0 = time.perf_counter()
    G = synth.build_graph(wl, device=0)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    PksmStats.reset()
    l0 = _lib.lib().mlb_launch_count()
    stats = {}
    t0 = time.perf_counter()
    basis = power_mean_eigs(G, PowerMeanConfig(p=wl.p_mean), k=k, seed=0, return_device=True, stats=stats)
    torch.cuda.synchronize()
    t_eig = time.perf_counter() - t0
    layer_mv = int(sum(PksmStats.steps)) + 4 * len(G.layers)  # + degree / probe applies are not counted here
    first_steps = int(sum(PksmStats.steps))
    # a second, identical eigensolve: the steady state (step graphs already captured)
    PksmStats.reset()
    t0 = time.perf_counter()
    power_mean_eigs(G, PowerMeanConfig(p=wl.p_mean), k=k, seed=0, return_device=True)
    torch.cuda.synchronize()
    t_eig_warm = time.perf_counter() - t0
    warm_steps = int(sum(PksmStats.steps))
    PksmStats.steps = [first_steps]
    labels = sample_labels(wl.truth, wl.label_fraction, seed=0)
    t0 = time.perf_counter()
    res = allen_cahn_solve(basis, labels, AllenCahnParams(max_iter=wl.ac_max_iter), return_device=True)
    pred = predict_labels(res.scores).cpu().numpy()
    t_ac = time.perf_counter() - t0
    acc = float(np.mean(pred == wl.truth))
    # the raw batched matvec rate of the same layers (every layer's shifted
    # L_sym of one vector per step, LaplacianBatch), for the in-solver ratio
    from paper_2007_05239_b200 import LaplacianBatch, MultilayerGraph, with_shift
    batch = LaplacianBatch(MultilayerGraph(tuple(with_shift(l, math.log(2.0)) for l in G.layers)))
    vv = torch.from_numpy(np.random.default_rng(3).standard_normal(wl.n)).cuda()
    for _ in range(3):
        batch.apply_dev(vv)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        batch.apply_dev(vv)
    e1.record()
    e1.synchronize()
    raw_rate = wl.n * len(G.layers) * reps / (e0.elapsed_time(e1) * 1e-3)
    out = {
        "workload": wl.name, "n": wl.n, "layers": len(G.layers), "k": k,
        "t_build_s": t_build, "t_eig_s": t_eig, "t_ac_s": t_ac,
        "outer_matvecs": stats.get("matvecs"), "restarts": stats.get("restarts"),
        "pksm_calls": len(PksmStats.steps), "layer_matvecs": int(sum(PksmStats.steps)),
        "node_layers_per_s_in_solver": wl.n * sum(PksmStats.steps) / t_eig if t_eig > 0 else None,
        "raw_batched_node_layers_per_s": raw_rate,
        "in_solver_over_raw": (wl.n * sum(PksmStats.steps) / t_eig) / raw_rate if t_eig > 0 else None,
        "t_eig_warm_s": t_eig_warm,
        "in_solver_warm_node_layers_per_s": wl.n * warm_steps / t_eig_warm,
        "in_solver_warm_over_raw": (wl.n * warm_steps / t_eig_warm) / raw_rate,
        "ac_iterations": res.iterations, "ac_converged": res.converged, "accuracy": acc,
        "values": [float(x) for x in basis.values], "libmlb_launches": int(_lib.lib().mlb_launch_count() - l0),
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
