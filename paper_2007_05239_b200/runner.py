"""Command-line pipelines on the B200 path (runner.py of the reference,
SURVEY 8(f) rank 3): `fastsum-bench`, `eig` and `classify` with the
reference's config keys, output files and report.json layout, every layer,
eigensolve and Allen-Cahn run on the GPU.  Stage wall times go to
report["times"]; fastsum-bench adds device-only (CUDA event) times beside
the host-API times the reference reports.

`segment-image` (PNG decoding / mask writing) and `sbm-bench` (stochastic
block model edge-list graphs) are outside the hot path (not on the
NFFT matvec path) and raise ConfigError naming the supported commands.
"""

import json
import os
import time
from contextlib import contextmanager

import numpy as np

from . import fastsum
from .allencahn import AllenCahnParams, LabelData, allen_cahn_solve, predict_labels
from .csvio import load_features_csv, load_labels_csv, write_matrix_csv, write_predictions_csv
from .datapipe import GroupingSpec, GroupSpec, feature_group, sample_labels
from .errors import ConfigError
from .graphs import MultilayerGraph, build_layer, load_edge_list
from .kernels import KernelSpec
from .powermean import PowerMeanConfig, power_mean_eigs


class Stopwatch:
    """Accumulated wall time per named stage plus the total (runner.py:58-78)."""

    def __init__(self):
        self.times = {}
        self._t0 = time.perf_counter()

    @contextmanager
    def stage(self, name):
        t = time.perf_counter()
        try:
            yield
        finally:
            self.times[name] = self.times.get(name, 0.0) + time.perf_counter() - t

    def report(self):
        out = {k: round(v, 6) for k, v in self.times.items()}
        out["total"] = round(time.perf_counter() - self._t0, 6)
        return out


def _out_dir(path):
    os.makedirs(path, exist_ok=True)
    return path


def _write_report(out_dir, report):
    path = os.path.join(out_dir, "report.json")
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(report, fh, indent=2)
        fh.write("\n")
    return path


def fastsum_params(cfg):
    f = cfg["fastsum"]
    return {"N": int(f["N"]), "m_nfft": int(f["m"]), "eps_b": float(f["eps_b"]), "p_nfft": int(f["p"]),
            "rho": float(f["rho"])}


def grouping_from_config(groups):
    return GroupingSpec(tuple(
        GroupSpec(columns=tuple(g["columns"]), kernel=KernelSpec(g.get("family", "gaussian"), float(g["sigma"])),
                  mode=g.get("mode", "fastsum-box"), per_component=bool(g.get("per_component", False)))
        for g in groups))


def _device(cfg):
    import torch
    dev = int(cfg.get("gpu", {}).get("device", 0) or 0)
    torch.cuda.set_device(dev)
    return dev


def _graph(cfg, watch):
    icfg = cfg["input"]
    if not (icfg["features_csv"] or icfg["edge_lists"] is not None):
        raise ConfigError("no graph input: set input.features_csv or input.edge_lists")
    device = _device(cfg)
    if icfg["features_csv"]:
        with watch.stage("load"):
            X = load_features_csv(icfg["features_csv"])
        if cfg["grouping"]["groups"] is None:
            raise ConfigError("feature input needs grouping.groups")
        with watch.stage("graph"):
            return feature_group(X, grouping_from_config(cfg["grouping"]["groups"]),
                                 fastsum_params=fastsum_params(cfg), device=device)
    paths = icfg["edge_lists"]
    if not paths:
        raise ConfigError("input.edge_lists must list at least one file")
    with watch.stage("graph"):
        n = icfg["n_nodes"]
        if n is None:  # common node count = the largest layer's
            ws = [load_edge_list(p) for p in paths]
            n = max(w.n for w in ws)
            ws = [w if w.n == n else load_edge_list(p, n) for w, p in zip(ws, paths)]
        else:
            ws = [load_edge_list(p, int(n)) for p in paths]
        return MultilayerGraph(tuple(build_layer(w) for w in ws))


def _eigs(graph, cfg, seed, watch):
    e, pw = cfg["eig"], cfg["power"]
    with watch.stage("eig"):
        return power_mean_eigs(
            graph, PowerMeanConfig(p=float(pw["p"]), delta=pw["delta"], dense_limit=int(pw["dense_limit"])),
            k=int(e["k"]), tol=float(e["tol"]),
            max_subspace=None if e["max_subspace"] is None else int(e["max_subspace"]),
            max_restarts=int(e["max_restarts"]), krylov_dim=int(cfg["pksm"]["krylov_dim"]),
            inner_tol=float(cfg["pksm"]["tol"]), seed=seed)


def _labels(cfg, n, truth, seed):
    icfg = cfg["input"]
    omega0 = icfg["omega0"] if icfg["omega0"] is not None else cfg["ac"]["omega0"]
    if icfg["labels_csv"]:
        ids = load_labels_csv(icfg["labels_csv"], n=n)
        if ids.max() < 0:
            raise ConfigError(f"{icfg['labels_csv']}: no labeled nodes")
        m = int(ids.max()) + 1
        if truth is not None:
            m = max(m, int(truth.max()) + 1)
        return LabelData.from_class_ids(ids, max(m, 2), omega0)
    if icfg["label_fraction"] is not None:
        if truth is None:
            raise ConfigError("input.label_fraction needs input.truth_csv")
        return sample_labels(truth, float(icfg["label_fraction"]), (seed, 1), omega0)
    raise ConfigError("classification needs input.labels_csv, or input.truth_csv with input.label_fraction")


def run_eig(cfg, seed, out_dir=".", threads=1):
    """k smallest power-mean eigenvalues -> eigenvalues.csv (+ eigenvectors.csv)."""
    watch = Stopwatch()
    graph = _graph(cfg, watch)
    basis = _eigs(graph, cfg, seed, watch)
    out_dir = _out_dir(out_dir)
    outputs = {}
    with watch.stage("write"):
        outputs["eigenvalues"] = os.path.join(out_dir, "eigenvalues.csv")
        write_matrix_csv(outputs["eigenvalues"], basis.values)
        if cfg["output"]["write_vectors"]:
            outputs["eigenvectors"] = os.path.join(out_dir, "eigenvectors.csv")
            write_matrix_csv(outputs["eigenvectors"], basis.vectors)
    report = {"command": "eig", "seed": seed, "n": graph.n, "layers": graph.T, "p": float(cfg["power"]["p"]),
              "k": basis.k, "eigenvalues": [float(x) for x in basis.values], "times": watch.report(),
              "outputs": outputs, "config": cfg, "backend": "b200"}
    outputs["report"] = _write_report(out_dir, report)
    return report


def run_classify(cfg, seed, out_dir=".", threads=1):
    """Eigensolve + Allen-Cahn -> predictions.csv (+ scores, eigenvectors)."""
    watch = Stopwatch()
    graph = _graph(cfg, watch)
    truth = None
    if cfg["input"]["truth_csv"]:
        truth = load_labels_csv(cfg["input"]["truth_csv"], n=graph.n)
        if truth.min() < 0:
            raise ConfigError(f"{cfg['input']['truth_csv']}: ground truth must assign a class to every node")
    labels = _labels(cfg, graph.n, truth, seed)
    if labels.n != graph.n:
        raise ConfigError(f"{labels.n} labels for a graph on {graph.n} nodes")
    basis = _eigs(graph, cfg, seed, watch)
    a = cfg["ac"]
    with watch.stage("ac"):
        result = allen_cahn_solve(basis, labels, AllenCahnParams(
            epsilon=float(a["epsilon"]), omega0=float(a["omega0"]), c=None if a["c"] is None else float(a["c"]),
            dt=float(a["dt"]), tolerance=float(a["tolerance"]), max_iter=int(a["max_iter"])))
    pred = predict_labels(result.scores)
    out_dir = _out_dir(out_dir)
    outputs = {}
    with watch.stage("write"):
        outputs["predictions"] = os.path.join(out_dir, "predictions.csv")
        write_predictions_csv(outputs["predictions"], pred)
        if cfg["output"]["write_scores"]:
            outputs["scores"] = os.path.join(out_dir, "scores.csv")
            write_matrix_csv(outputs["scores"], result.scores)
        if cfg["output"]["write_vectors"]:
            outputs["eigenvectors"] = os.path.join(out_dir, "eigenvectors.csv")
            write_matrix_csv(outputs["eigenvectors"], basis.vectors)
    report = {"command": "classify", "seed": seed, "n": graph.n, "layers": graph.T, "classes": labels.m,
              "p": float(cfg["power"]["p"]), "k": basis.k, "eigenvalues": [float(x) for x in basis.values],
              "iterations": result.iterations, "converged": result.converged}
    if truth is not None:
        hits = pred == truth
        unl = ~labels.labeled_mask
        report["accuracy"] = float(np.mean(hits))
        report["misclassification"] = 1.0 - report["accuracy"]
        report["accuracy_unlabeled"] = float(np.mean(hits[unl])) if unl.any() else report["accuracy"]
    report.update({"times": watch.report(), "outputs": outputs, "config": cfg, "backend": "b200"})
    outputs["report"] = _write_report(out_dir, report)
    return report


def _box_points(rng, n, d, eps_b):
    hw = fastsum.box_halfwidth(eps_b)
    return rng.uniform(-hw, hw, size=(n, d))


def _device_time(binding, plan, v, reps):
    """Median device time (CUDA events) of W v on resident vectors."""
    import torch
    vd = torch.from_numpy(np.ascontiguousarray(v)).cuda()
    y = torch.empty_like(vd)
    fastsum.apply_binding(binding, vd, y, -plan.K0, 1.0, 0.0, 0)
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fastsum.apply_binding(binding, vd, y, -plan.K0, 1.0, 0.0, 0)
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e-3)
    return float(np.median(ts))


def run_fastsum_bench(cfg, seed, out_dir=".", threads=1):
    """Accuracy vs the exact sum at accuracy_n, then a size sweep of one
    prebuilt-binding apply (runner.py:484-581); same CSV / table outputs."""
    import torch
    _device(cfg)
    watch = Stopwatch()
    b = cfg["bench"]["fastsum"]
    kernel = KernelSpec(family=b["family"], sigma=float(b["sigma"]))
    params = fastsum_params(cfg)
    reps = int(b["repetitions"])
    if reps < 1:
        raise ConfigError("bench.fastsum.repetitions must be >= 1")
    accuracy = []
    with watch.stage("accuracy"):
        acc_n = int(b["accuracy_n"])
        for d in [int(x) for x in b["accuracy_dims"]]:
            rng = np.random.default_rng((seed, 101, d))
            pts = _box_points(rng, acc_n, d, params["eps_b"])
            v = rng.standard_normal(acc_n)
            plan = fastsum.build_plan(kernel, d=d, **params)
            binding = fastsum.bind_points(plan, pts)
            t0 = time.perf_counter()
            fast = fastsum.fastsum_apply(None, v, plan, binding=binding)
            t_fast = time.perf_counter() - t0
            t0 = time.perf_counter()
            exact = fastsum.direct_apply(pts, v, kernel)
            t_direct = time.perf_counter() - t0
            accuracy.append({"d": d, "n": acc_n, "rel_error": float(np.linalg.norm(fast - exact) / np.linalg.norm(exact)),
                             "t_fast": round(t_fast, 6), "t_direct": round(t_direct, 6)})
    d_s = int(b["d"])
    sizes = [int(n) for n in b["sizes"]]
    with_direct = bool(b["with_direct"])
    scaling = {"d": d_s, "sizes": sizes, "t_fast": [], "t_direct": [], "t_fast_device": []}
    with watch.stage("scaling"):
        plan = fastsum.build_plan(kernel, d=d_s, **params)
        for n in sizes:
            rng = np.random.default_rng((seed, 202, n))
            pts = _box_points(rng, n, d_s, params["eps_b"])
            v = rng.standard_normal(n)
            binding = fastsum.bind_points(plan, pts)
            fastsum.fastsum_apply(None, v, plan, binding=binding)  # warm-up
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                fastsum.fastsum_apply(None, v, plan, binding=binding)
                ts.append(time.perf_counter() - t0)
            scaling["t_fast"].append(float(np.median(ts)))
            scaling["t_fast_device"].append(_device_time(binding, plan, v, reps))
            if with_direct:
                ts = []
                for _ in range(reps):
                    t0 = time.perf_counter()
                    fastsum.direct_apply(pts, v, kernel)
                    torch.cuda.synchronize()
                    ts.append(time.perf_counter() - t0)
                scaling["t_direct"].append(float(np.median(ts)))
    out_dir = _out_dir(out_dir)
    acc_path = os.path.join(out_dir, "fastsum_accuracy.csv")
    with open(acc_path, "w", encoding="utf-8") as fh:
        fh.write("d,n,rel_error,t_fast,t_direct\n")
        for r in accuracy:
            fh.write(f"{r['d']},{r['n']},{r['rel_error']:.3e},{r['t_fast']:.6f},{r['t_direct']:.6f}\n")
    scale_path = os.path.join(out_dir, "fastsum_scaling.csv")
    with open(scale_path, "w", encoding="utf-8") as fh:
        fh.write("n,t_fast_median" + (",t_direct_median" if with_direct else "") + ",t_fast_device_median\n")
        for i, n in enumerate(sizes):
            cols = [f"{n}", f"{scaling['t_fast'][i]:.6f}"]
            if with_direct:
                cols.append(f"{scaling['t_direct'][i]:.6f}")
            cols.append(f"{scaling['t_fast_device'][i]:.6f}")
            fh.write(",".join(cols) + "\n")
    txt_path = os.path.join(out_dir, "fastsum_bench.txt")
    with open(txt_path, "w", encoding="utf-8") as fh:
        fh.write(f"kernel {kernel.family}, sigma {kernel.sigma:g} (box units), N={params['N']}, "
                 f"m={params['m_nfft']}, median of {reps} (B200)\n\naccuracy (n={int(b['accuracy_n'])}):\n")
        for r in accuracy:
            fh.write(f"  d={r['d']}  rel_error={r['rel_error']:.3e}  fast {r['t_fast']:.4f}s  "
                     f"direct {r['t_direct']:.4f}s\n")
        fh.write(f"\nscaling (d={d_s}, apply with prebuilt binding):\n")
        for i, n in enumerate(sizes):
            line = f"  n={n:<8d} fast {scaling['t_fast'][i]:.4f}s (device {scaling['t_fast_device'][i] * 1e6:.1f} us)"
            if with_direct:
                line += f"  direct {scaling['t_direct'][i]:.4f}s"
            fh.write(line + "\n")
    report = {"command": "fastsum-bench", "seed": seed, "accuracy": accuracy, "scaling": scaling,
              "times": watch.report(), "config": cfg, "backend": "b200",
              "outputs": {"accuracy_csv": acc_path, "scaling_csv": scale_path, "table": txt_path}}
    report["outputs"]["report"] = _write_report(out_dir, report)
    return report


def _unsupported(name):
    def run(cfg, seed, out_dir=".", threads=1):
        raise ConfigError(f"{name} is not part of the B200 backend (supported: fastsum-bench, eig, classify)")
    return run


run_segment_image = _unsupported("segment-image")
run_sbm_bench = _unsupported("sbm-bench")
