"""Per-rank compute of the node-range-sharded config-4 step, on ONE GPU.

    python tools/shard_projection.py [--worlds 2 4 8] [--steps 20] [--out file.json]

For each world size N and each rank r, binds only rank r's node range
[r n/N, (r+1) n/N) of both config-4 layers (box map of ALL nodes, as
dist.shard_feature_groups does) and times that rank's sharded step --
both spreads, the convolutions and both fused gathers -- with NO collective
(comm=None), CUDA events on the launching stream, 256 MB L2 flush between
steps.  The ranks run one after the other, never concurrently, so no kernel
waits on another rank.  This is the compute half of an N-GPU step only: the
NCCL all-reduce of the 702 KB grid buffer over NVLink is not measured here
(one GPU), so the projection adds it as a stated estimate, and says so.
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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--allreduce-us", type=float, default=30.0,
                    help="assumed NCCL all-reduce time of the grid buffer (not measured: one GPU)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch

    import synth
    from paper_2007_05239_b200 import KernelSpec
    from paper_2007_05239_b200.dist import ShardedKernelGraph, shard_feature_groups
    wl = synth.CONFIGS[4](seed=0)
    groups = [(ls.columns, KernelSpec(ls.family, ls.sigma), dict(N=ls.N, m_nfft=ls.m, p_nfft=ls.p))
              for ls in wl.layers]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    rng = np.random.default_rng(3)
    delta = math.log(2.0)
    res = {"workload": wl.name, "n": wl.n, "allreduce_us_assumed": a.allreduce_us, "worlds": {}}

    import time

    def time_step(sg, v, ys):
        for _ in range(3):
            sg.lsym(v, ys)
        torch.cuda.synchronize()
        tot = 0.0
        cpu = 0.0
        for _ in range(a.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            sg.lsym(v, ys)
            e1.record()
            cpu += time.perf_counter() - t0
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        # the same step replayed from a captured CUDA graph (no host issue time inside)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            sg.lsym(v, ys)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            sg.lsym(v, ys)
        gt = 0.0
        for _ in range(a.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            e1.synchronize()
            gt += e0.elapsed_time(e1)
        return tot / a.steps, cpu / a.steps * 1e3, gt / a.steps

    for N in [1] + list(a.worlds):
        per_rank, cpu_ms, graph_ms = [], [], []
        for r in range(N):
            lo, hi, pts, kerns, plans = shard_feature_groups(wl.X, groups, r, N)
            sg = ShardedKernelGraph(pts, kerns, plans, wl.n, lo, hi, comm=None, shift=delta, device=0).build()
            v = torch.from_numpy(rng.standard_normal(hi - lo)).cuda()
            ys = [torch.empty_like(v) for _ in range(len(wl.layers))]
            t_ev, t_cpu, t_graph = time_step(sg, v, ys)
            per_rank.append(t_ev)
            cpu_ms.append(t_cpu)
            graph_ms.append(t_graph)
            if r == 0:
                import bench
                st = bench.stage_breakdown(torch, sg.weights, v)
                stages0 = [{k: x[k] for k in ("d", "n", "spread_ms", "reduce_ms", "convolve_ms", "gather_ms")}
                           for x in st]
            del sg, v, ys
            torch.cuda.empty_cache()
        worst = max(per_rank)
        proj = worst + (a.allreduce_us * 1e-3 if N > 1 else 0.0)
        res["worlds"][N] = {"per_rank_compute_ms": per_rank, "max_compute_ms": worst,
                            "host_issue_ms": cpu_ms, "graph_replay_ms": graph_ms,
                            "projected_step_ms": proj, "rank0_stages_ms": stages0,
                            "projected_value": wl.n * len(wl.layers) / (proj * 1e-3)}
        print(N, ["%.3f" % x for x in per_rank], "projected %.3f ms" % proj, "host issue",
              ["%.3f" % x for x in cpu_ms], "graph", ["%.3f" % x for x in graph_ms], flush=True)
    base = res["worlds"][1]["projected_step_ms"]
    for N, r in res["worlds"].items():
        r["projected_speedup"] = base / r["projected_step_ms"]
    # the bench's N > 1 step replays one captured graph per rank (lsym_graph):
    # the same projection on the graph-replay times
    if 1 in res["worlds"]:
        gbase = max(res["worlds"][1]["graph_replay_ms"])
        for N, r in res["worlds"].items():
            r["projected_step_graph_ms"] = max(r["graph_replay_ms"]) + (a.allreduce_us * 1e-3 if N > 1 else 0.0)
            r["projected_speedup_graph"] = gbase / r["projected_step_graph_ms"]
    out = json.dumps(res, indent=1)
    print(out)
    if a.out:
        with open(a.out, "w") as f:
            f.write(out)


if __name__ == "__main__":
    main()
