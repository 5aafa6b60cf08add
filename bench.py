#!/usr/bin/env python
"""Benchmark: normalized-Laplacian matvecs/s (node*layers/s), fp64, on B200.

Workload (BASELINE.json configs[1], the config the metric is quoted on):
512x512 synthetic segmentation image (n = 262,144 nodes), T = 2 kernel layers
-- RGB d=3 sigma=0.1 (N=64, m=4, p=8; the reference rejects N=32 for this
layer) and xy d=2 sigma=0.15 (N=32, m=4, p=8) -- shifted by
delta = ln 2 as in the p = -1 PKSM solves.  One STEP = one shifted
normalized-Laplacian matvec y = (1+delta) v - D^-1/2 W D^-1/2 v on every
layer (2 x 262,144 node*layers), vectors in node order (the drop-in
`apply_sym_laplacian` semantics).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Timing: W warm-up steps; then K steps, each bracketed by CUDA events on the
launching stream, with a 256 MB L2 flush between steps (outside the events);
barrier + synchronize around the loop; max over ranks.  Multi-GPU (torchrun):
layers are independent, each rank owns the 2 layers of its own seeded image
(round-robin layer ownership, no data-path collective) -> weak scaling.

`--impl reference` times the CPU reference algorithm (the numpy oracle port
of multilap's fastsum/graphs path: bincount spread/gather + scipy.fft) on a
bounded subsample of the same layers, rank 0 only.
"""

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "normalized-Laplacian matvecs/sec (node*layers/s) fp64"
UNIT = "node*layers/s"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_bench_{os.getpid()}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def build_layers(workload, device, delta):
    import synth
    from paper_2007_05239_b200 import with_shift
    G = synth.build_graph(workload, device=device)
    return [with_shift(l, delta) for l in G.layers]


def algorithmic_bytes(d):
    """B(d) = 16 d + 40 bytes per node per normalized-Laplacian matvec."""
    return 16 * d + 40


def algorithmic_flops(d, m):
    """F(d, m) = 4 (2m+1)^d fp64 flops per node per matvec."""
    return 4 * (2 * m + 1) ** d


def measure_fp64_peak(torch, device):
    from paper_2007_05239_b200 import _lib
    lib = _lib.lib()
    out = torch.zeros(1, dtype=torch.float64, device=device)
    blocks, iters = 148 * 8, 20000
    for _ in range(2):
        lib.mlb_probe_fp64(iters, blocks, _lib.ptr(out), _lib.stream_ptr())
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(3):
        s.record()
        lib.mlb_probe_fp64(iters, blocks, _lib.ptr(out), _lib.stream_ptr())
        e.record()
        e.synchronize()
        flops = 2.0 * 8 * iters * blocks * 256
        best = max(best, flops / (s.elapsed_time(e) * 1e-3) / 1e12)
    return best


def stage_breakdown(torch, layers, v, reps=10):
    """Per-kernel device times (CUDA events, launching stream): spread kernel,
    partial reduction, convolution, gather (with the Laplacian epilogue)."""
    from paper_2007_05239_b200 import _lib
    lib = _lib.lib()
    out = []
    for li, lay in enumerate(layers):
        w = lay.weights
        b = w._bindings[0]
        g = b.plan
        K0 = w.kernel.value_at_zero()
        grid = torch.empty(b.stats()["grid_cells"], dtype=torch.float64, device=v.device)
        grid2 = torch.empty_like(grid)
        y = torch.empty_like(v)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        tt = np.zeros(4)
        sp = _lib.stream_ptr()
        for r in range(reps + 2):
            ev[0].record()
            _lib.check(lib.mlb_spread(b.ptr, _lib.ptr(v), _lib.ptr(grid), _lib.MLB_USE_ISD | _lib.MLB_SPREAD_ONLY, sp))
            ev[1].record()
            _lib.check(lib.mlb_reduce(b.ptr, _lib.ptr(grid), sp))
            ev[2].record()
            _lib.check(lib.mlb_convolve(b.ptr, _lib.ptr(grid), _lib.ptr(grid2), sp))
            ev[3].record()
            _lib.check(lib.mlb_gather(b.ptr, _lib.ptr(grid2), _lib.ptr(y), 0, sp))
            ev[4].record()
            ev[4].synchronize()
            if r >= 2:
                tt += [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
        tt /= reps
        d, m = g.d, g.m_nfft
        out.append(dict(layer=li, d=d, N=g.N, m=m, n=b.n, spread_ms=tt[0], reduce_ms=tt[1], convolve_ms=tt[2],
                        gather_ms=tt[3], stats=b.stats()))
    return out


def _reference_arm(workload, delta, n_sample, seed=1):
    """The reference algorithm (oracle port) of every layer over a random node
    sample, on all host cores (oracle/parallel_ref.py)."""
    from oracle import fastsum_oracle as fo
    from oracle.parallel_ref import ParallelReference
    from paper_2007_05239_b200 import datapipe, GroupSpec, KernelSpec
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(workload.n, size=min(n_sample, workload.n), replace=False))
    specs = []
    for ls in workload.layers:
        g = GroupSpec(ls.columns, KernelSpec(ls.family, ls.sigma))
        Xb, kb, _ = datapipe._scaled_group(workload.X[idx][:, list(ls.columns)], g, 1.0 / 16)
        specs.append((fo.OraclePlan(ls.family, kb.sigma, len(ls.columns), ls.N, ls.m, p=ls.p), Xb))
    ref = ParallelReference(specs, len(idx), delta)
    return ref, rng.standard_normal(len(idx))


def _sample_words(ns, n):
    return f"all {n} nodes" if ns >= n else f"{ns}-node random subsample"


def cpu_baseline_oracle(workload, delta, n_sample, reps, seed=1):
    """Time the reference algorithm (numpy oracle, all host cores) on a subsample."""
    ref, v = _reference_arm(workload, delta, n_sample, seed)
    try:
        ref.step(v)  # warm-up
        t0 = time.perf_counter()
        for _ in range(reps):
            ref.step(v)
        dt = time.perf_counter() - t0
    finally:
        ref.close()
    return ref.n * ref.T * reps / dt, ref.n, dt, ref.P


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import synth
    wl = synth.config2_segmentation(seed=0)
    delta = math.log(2.0)
    ref, v = _reference_arm(wl, delta, args.ref_sample, seed=1)
    n_s, P, T = ref.n, ref.P, ref.T
    try:
        for _ in range(args.warmup):
            ref.step(v)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ref.step(v)
        dt = time.perf_counter() - t0
    finally:
        ref.close()
    value = n_s * T * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE configs[1] shapes)",
        "config": {"workload": wl.name, "layers": [vars(l) for l in wl.layers], "delta": delta,
                   "sample_nodes": n_s},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": P, "kind": "port",
                         "sample": f"{_sample_words(n_s, wl.n)} of both layers of {wl.name}; one step = one "
                                   "shifted normalized-Laplacian matvec per layer through the oracle port of the "
                                   f"reference algorithm (bincount spread/gather, full-grid scipy.fft) on {P} "
                                   "processes (point chunks, fixed-order grid sum, FFT on all cores)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    device = local
    torch.cuda.set_device(device)
    import synth
    from paper_2007_05239_b200 import LaplacianBatch, MultilayerGraph, _lib
    from paper_2007_05239_b200.graphs import apply_sym_laplacian_dev
    lib = _lib.lib()
    wl = synth.config2_segmentation(seed=rank)   # rank r owns the layers of image r
    delta = math.log(2.0)
    layers = build_layers(wl, device, delta)
    n, T = wl.n, len(layers)
    rng = np.random.default_rng(1000 + rank)
    v_host = rng.standard_normal(n)
    v = torch.from_numpy(v_host).cuda(device)
    ys = [torch.empty_like(v) for _ in layers]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)

    # the layers are independent: one CUDA stream per layer, joined per step,
    # the whole step replayed from one captured CUDA graph (LaplacianBatch)
    main = torch.cuda.current_stream()
    lstreams = [torch.cuda.Stream() for _ in layers]
    fork = torch.cuda.Event()
    joins = [torch.cuda.Event() for _ in layers]
    graph = MultilayerGraph(tuple(layers))
    batch = LaplacianBatch(graph, use_graph=not args.no_cuda_graph)
    batch._v.copy_(v)

    # persistent pinned host buffers of the end-to-end leg, allocated at setup:
    # a freshly pinned buffer moves data slowly for a while (measured on the
    # pool's boxes: 2 MiB H2D at 90-160 us right after allocation, 42 us once
    # settled), and a user that streams many vectors keeps its buffers
    v_pin = torch.from_numpy(v_host).pin_memory()
    y_pin = torch.empty((T, n), dtype=torch.float64, pin_memory=True)
    e2e_k = max(3, args.steps)  # one distinct host vector per e2e step
    V_pin = torch.from_numpy(rng.standard_normal((e2e_k, n))).pin_memory()
    Y_pin = torch.empty((e2e_k, T, n), dtype=torch.float64, pin_memory=True)

    def step():
        batch._run()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(device)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.start()
    l0 = lib.mlb_launch_count()
    for i in range(args.steps):
        flush.fill_(float(i))
        starts[i].record()
        step()
        ends[i].record()
    torch.cuda.synchronize()
    launches = lib.mlb_launch_count() - l0
    # the timed loop lasts only milliseconds: keep running the identical step
    # (untimed) for ~0.6 s so nvidia-smi samples the clocks under this load
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < 0.6:
        for _ in range(20):
            step()
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    clk["note"] = "sampled over the timed loop plus a 0.6 s soak of the identical step"
    total_ms = float(sum(s.elapsed_time(e) for s, e in zip(starts, ends)))
    if ws > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = n * T * args.steps * ws / (total_ms * 1e-3)

    # ---- end-to-end through the public API: pinned host in, host out ----------
    # (one call = every layer's L_sym of one host vector: pinned H2D of v,
    # per-layer D2H of the results as each layer finishes, host sync)
    for _ in range(max(3, args.warmup)):
        batch.apply(v_pin, out=y_pin)
    torch.cuda.synchronize()
    e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(3, args.steps)
    e_s.record()
    for _ in range(e2e_steps):
        batch.apply(v_pin, out=y_pin)
    e_e.record()
    e_e.synchronize()
    e2e_sync_ms = e_s.elapsed_time(e_e)
    e2e_sync_value = n * T * e2e_steps * ws / (e2e_sync_ms * 1e-3)
    # streamed: the K steps' distinct host vectors through apply_many (vector
    # i+1's H2D and vector i-1's D2H overlap vector i's compute); the call
    # returns once every result is in host memory
    for _ in range(2):
        batch.apply_many(V_pin[:3], out=Y_pin[:3])
    torch.cuda.synchronize()
    e_s.record()
    batch.apply_many(V_pin, out=Y_pin)
    e_e.record()
    e_e.synchronize()
    e2e_ms = e_s.elapsed_time(e_e)
    e2e_value = n * T * e2e_k * ws / (e2e_ms * 1e-3)

    # ---- sorted-order variant (what the PKSM inner loop runs) -----------------
    sorted_value = None
    try:
        vs = [torch.empty_like(v) for _ in layers]
        for lay, x in zip(layers, vs):
            lib.mlb_to_sorted(lay.weights._bindings[0].ptr, _lib.ptr(v), _lib.ptr(x), _lib.stream_ptr())

        def step_sorted():
            fork.record(main)
            for lay, x, y, s, j in zip(layers, vs, ys, lstreams, joins):
                w = lay.weights
                s.wait_event(fork)
                lib.mlb_apply(w._bindings[0].ptr, _lib.ptr(x), _lib.ptr(y), 1.0 + lay.shift, -1.0,
                              w.kernel.value_at_zero(), _lib.MLB_USE_ISD | _lib.MLB_SORTED,
                              _lib.C.c_void_p(s.cuda_stream))
                j.record(s)
            for j in joins:
                main.wait_event(j)
        for _ in range(3):
            step_sorted()
        tot = 0.0
        for i in range(args.steps):
            flush.fill_(float(i))
            starts[i].record()
            step_sorted()
            ends[i].record()
        torch.cuda.synchronize()
        tot = float(sum(s.elapsed_time(e) for s, e in zip(starts, ends)))
        sorted_value = n * T * args.steps * ws / (tot * 1e-3)
    except Exception as exc:  # diagnostic only
        sorted_value = f"error: {exc}"

    # ---- roofline of the dominant kernel ---------------------------------------
    stages = stage_breakdown(torch, layers, v)
    fp64_peak = measure_fp64_peak(torch, f"cuda:{device}")
    hbm_peak, peak_kind = _peaks()
    kern = []
    for st in stages:
        d, m, nl = st["d"], st["m"], st["n"]
        C = (2 * m + 1) ** d
        kern.append(("spread", st, st["spread_ms"], (8 * d + 16) * nl, 2 * C * nl))
        kern.append(("gather", st, st["gather_ms"], (8 * d + 24) * nl, 2 * C * nl))
        kern.append(("convolve", st, st["convolve_ms"], 16 * st["stats"]["grid_cells"], 0))
        kern.append(("reduce", st, st["reduce_ms"], 8 * st["stats"]["grid_cells"], 0))
    top = max(kern, key=lambda k: k[2])
    name, st, ms, nbytes, nflops = top
    achieved = nbytes / (ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        key = f"{name}_d{st['d']}"
        if key in tr:
            traffic = tr[key]
    except Exception:
        traffic = None
    roof = {"bound": "hbm", "kernel": f"{name} (layer d={st['d']}, N={st['N']}, m={st['m']})",
            "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})", "traffic": traffic,
            "fp64": {"achieved_tflops": nflops / (ms * 1e-3) / 1e12, "peak_tflops": fp64_peak,
                     "frac": (nflops / (ms * 1e-3) / 1e12) / fp64_peak if fp64_peak else None,
                     "peak_source": "mlb_probe_fp64 DFMA microbenchmark, this run"}}
    # whole-step HBM-roofline fraction of the metric (R * B(d) / peak)
    step_bytes = sum(algorithmic_bytes(st["d"]) * st["n"] for st in stages)
    step_flops = sum(algorithmic_flops(st["d"], st["m"]) * st["n"] for st in stages)
    ms_step = total_ms / args.steps
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE configs[1] image; no dataset exists for it)",
        "config": {"workload": wl.name, "nodes_per_rank": n, "layers": [vars(l) for l in wl.layers],
                   "delta": delta, "vector_order": "node", "l2": "256 MB flush between steps (outside events)",
                   "streams": "one CUDA stream per layer (independent layers), joined every step; the step is "
                              "one captured CUDA graph replay" + (" (disabled)" if args.no_cuda_graph else ""),
                   "parallelism": f"layer-parallel x{ws} (independent layers per rank, no collective)"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n * T,
                "steps": e2e_k,
                "path": "paper_2007_05239_b200.LaplacianBatch(graph).apply_many(pinned host (K, n), out=pinned host "
                        "(K, T, n)): K distinct host vectors, each one H2D of v and T D2H of its results, copies "
                        "on their own streams overlapping the neighbouring vectors' compute; timed until the last "
                        "result is in host memory",
                "synchronous": {"value": e2e_sync_value, "unit": UNIT,
                                "path": "LaplacianBatch(graph).apply(pinned host v, out=pinned host (T, n)) per step: "
                                        "H2D, compute, D2H and a host sync every step (no overlap between steps)"}},
        "gpu_launches": int(launches),
        "clocks": clk,
        "roofline": roof,
        "step_roofline": {"hbm_bytes_per_step": step_bytes, "hbm_frac": step_bytes / (ms_step * 1e-3) / 1e9 / hbm_peak,
                          "fp64_flops_per_step": step_flops,
                          "fp64_frac": step_flops / (ms_step * 1e-3) / 1e12 / fp64_peak if fp64_peak else None},
        "sorted_order_value": sorted_value,
        "stages_ms": [{k: st[k] for k in ("layer", "d", "N", "m", "n", "spread_ms", "reduce_ms", "convolve_ms",
                                          "gather_ms")}
                      for st in stages],
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        val, ns, secs, ncore = cpu_baseline_oracle(wl, delta, args.cpu_sample, args.cpu_reps)
        result["cpu_baseline"] = {"value": val, "unit": UNIT, "cores": ncore, "kind": "port",
                                  "sample": f"{_sample_words(ns, wl.n)} of both layers, {args.cpu_reps} shifted "
                                            f"normalized-Laplacian matvecs per layer through the oracle port of the "
                                            f"reference algorithm on {ncore} processes (bincount + full-grid "
                                            f"scipy.fft), {secs:.1f} s"}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cuda-graph", action="store_true", help="launch the step kernel by kernel")
    # CPU legs: the full config-2 workload (all 262,144 nodes) unless reduced;
    # ~0.35 s per step on 16 cores, so 30 reps are ~10 s of CPU work
    ap.add_argument("--cpu-sample", type=int, default=1 << 30, help="nodes in the CPU baseline sample (default: all)")
    ap.add_argument("--cpu-reps", type=int, default=30)
    ap.add_argument("--ref-sample", type=int, default=1 << 30, help="nodes in the reference arm's sample (default: all)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
