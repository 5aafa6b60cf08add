"""Command-line pipelines on the B200 path (runner.py of the reference,
SURVEY 8(f) rank 3): `fastsum-bench`, `eig`, `classify` and `segment-image`
with the reference's config keys, output files and report.json layout, every
layer, eigensolve and Allen-Cahn run on the GPU.  Stage times are measured
with the device drained at each stage boundary (kernels launched
asynchronously are charged to the stage that issued them); fastsum-bench adds
CUDA-event device times beside the host-API times the reference reports.

`sbm-bench` (stochastic block model edge-list graphs, no kernel layers) is
outside the NFFT hot path and raises ConfigError.
"""

import json
import os
import time

import numpy as np

from . import fastsum
from .allencahn import AllenCahnParams, LabelData, allen_cahn_solve, predict_labels
from .csvio import load_features_csv, load_labels_csv, write_matrix_csv, write_predictions_csv
from .datapipe import (GroupingSpec, GroupSpec, feature_group, image_features, load_image, masks_from_labels,
                       sample_labels, save_image)
from .errors import ConfigError, FormatError
from .graphs import MultilayerGraph, build_layer, load_edge_list
from .kernels import KernelSpec
from .powermean import PowerMeanConfig, power_mean_eigs

# default image grouping (runner.py:51-57): colour over all pixels, pixel
# coordinates per image (the spatial kernel stays block diagonal)
SEGMENT_GROUPS = ({"columns": [0, 1, 2], "family": "gaussian", "sigma": 1.0, "mode": "unit-box"},
                  {"columns": [3, 4], "family": "gaussian", "sigma": 4.0, "mode": "unit-box",
                   "per_component": True})
# composite-mask colours (runner.py:45-49)
PALETTE = np.array([(230, 25, 75), (60, 180, 75), (255, 225, 25), (0, 130, 200), (245, 130, 48),
                    (145, 30, 180), (70, 240, 240), (240, 50, 230), (210, 245, 60), (170, 110, 40)], dtype=np.uint8)


class StageClock:
    """Per-stage seconds + total for report["times"] (runner.py:60-78).  The
    device is synchronised when a stage closes so asynchronous GPU work is
    charged to the stage that launched it."""

    def __init__(self):
        self.start = time.perf_counter()
        self.acc = {}

    def __call__(self, name):
        clock = self

        class _Stage:
            def __enter__(self):
                self.t = time.perf_counter()

            def __exit__(self, *exc):
                _drain()
                clock.acc[name] = clock.acc.get(name, 0.0) + time.perf_counter() - self.t
                return False
        return _Stage()

    def report(self):
        rep = {k: round(v, 6) for k, v in self.acc.items()}
        rep["total"] = round(time.perf_counter() - self.start, 6)
        return rep


def _drain():
    try:
        import torch
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.synchronize()
    except Exception:
        pass


def _out_dir(path):
    os.makedirs(path, exist_ok=True)
    return path


def _finish(out_dir, report, clock, outputs):
    """Attach times / outputs and write report.json (runner.py:84-90)."""
    report.update(times=clock.report(), outputs=outputs, backend="b200")
    path = os.path.join(out_dir, "report.json")
    outputs["report"] = path
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(report, fh, indent=2)
        fh.write("\n")
    return report


def fastsum_params(cfg):
    f = cfg["fastsum"]
    return dict(N=int(f["N"]), m_nfft=int(f["m"]), eps_b=float(f["eps_b"]), p_nfft=int(f["p"]), rho=float(f["rho"]))


def grouping_from_config(groups):
    def one(g):
        kern = KernelSpec(g.get("family", "gaussian"), float(g["sigma"]))
        return GroupSpec(columns=tuple(g["columns"]), kernel=kern, mode=g.get("mode", "fastsum-box"),
                         per_component=bool(g.get("per_component", False)))
    return GroupingSpec(tuple(one(g) for g in groups))


def _device(cfg):
    import torch
    dev = int(cfg.get("gpu", {}).get("device", 0) or 0)
    torch.cuda.set_device(dev)
    return dev


def _edge_list_graph(paths, n_nodes):
    if not paths:
        raise ConfigError("input.edge_lists must list at least one file")
    if n_nodes is not None:
        return MultilayerGraph(tuple(build_layer(load_edge_list(p, int(n_nodes))) for p in paths))
    first = [load_edge_list(p) for p in paths]          # a common node count: the largest layer's
    n = max(w.n for w in first)
    return MultilayerGraph(tuple(build_layer(w if w.n == n else load_edge_list(p, n)) for w, p in zip(first, paths)))


def _graph(cfg, clock, features=None, components=None):
    """Kernel layers from features (argument or input.features_csv) or edge-list layers."""
    icfg = cfg["input"]
    if features is None and not icfg["features_csv"] and icfg["edge_lists"] is None:
        raise ConfigError("no graph input: set input.features_csv or input.edge_lists")
    device = _device(cfg)
    if features is None and icfg["features_csv"]:
        with clock("load"):
            features = load_features_csv(icfg["features_csv"])
    if features is not None:
        groups = cfg["grouping"]["groups"]
        if groups is None:
            raise ConfigError("feature input needs grouping.groups")
        with clock("graph"):
            return feature_group(features, grouping_from_config(groups), components=components,
                                 fastsum_params=fastsum_params(cfg), device=device)
    if icfg["edge_lists"] is not None:
        with clock("graph"):
            return _edge_list_graph(icfg["edge_lists"], icfg["n_nodes"])
    raise ConfigError("no graph input: set input.features_csv or input.edge_lists")


def _eigs(graph, cfg, seed, clock):
    e, pw = cfg["eig"], cfg["power"]
    with clock("eig"):
        return power_mean_eigs(
            graph, PowerMeanConfig(p=float(pw["p"]), delta=pw["delta"], dense_limit=int(pw["dense_limit"])),
            k=int(e["k"]), tol=float(e["tol"]),
            max_subspace=None if e["max_subspace"] is None else int(e["max_subspace"]),
            max_restarts=int(e["max_restarts"]), krylov_dim=int(cfg["pksm"]["krylov_dim"]),
            inner_tol=float(cfg["pksm"]["tol"]), seed=seed)


def _truth(cfg, n):
    path = cfg["input"]["truth_csv"]
    if not path:
        return None
    t = load_labels_csv(path, n=n)
    if t.min() < 0:
        raise ConfigError(f"{path}: ground truth must assign a class to every node")
    return t


def _labels(cfg, n, truth, seed):
    """Known labels (runner.py:157-174): an explicit label file wins; else a
    sampled fraction of the ground truth (stream (seed, 1))."""
    icfg = cfg["input"]
    omega0 = cfg["ac"]["omega0"] if icfg["omega0"] is None else icfg["omega0"]
    path, frac = icfg["labels_csv"], icfg["label_fraction"]
    if not path and frac is None:
        raise ConfigError("classification needs input.labels_csv, or input.truth_csv with input.label_fraction")
    if not path:
        if truth is None:
            raise ConfigError("input.label_fraction needs input.truth_csv")
        return sample_labels(truth, float(frac), (seed, 1), omega0)
    ids = load_labels_csv(path, n=n)
    if ids.max() < 0:
        raise ConfigError(f"{path}: no labeled nodes")
    classes = int(max(ids.max(), -1 if truth is None else truth.max())) + 1
    return LabelData.from_class_ids(ids, max(classes, 2), omega0)


def _ac_params(cfg):
    a = cfg["ac"]
    return AllenCahnParams(epsilon=float(a["epsilon"]), omega0=float(a["omega0"]),
                           c=None if a["c"] is None else float(a["c"]), dt=float(a["dt"]),
                           tolerance=float(a["tolerance"]), max_iter=int(a["max_iter"]))


def _scores(pred, truth, labels):
    """accuracy / misclassification / accuracy on unlabelled nodes (runner.py:208-217)."""
    if truth is None:
        return {}
    hits = pred == truth
    acc = float(hits.mean())
    unl = ~labels.labeled_mask
    return {"accuracy": acc, "misclassification": 1.0 - acc,
            "accuracy_unlabeled": float(hits[unl].mean()) if unl.any() else acc}


def _classify(graph, cfg, seed, clock, truth):
    labels = _labels(cfg, graph.n, truth, seed)
    if labels.n != graph.n:
        raise ConfigError(f"{labels.n} labels for a graph on {graph.n} nodes")
    basis = _eigs(graph, cfg, seed, clock)
    with clock("ac"):
        result = allen_cahn_solve(basis, labels, _ac_params(cfg))
    return labels, basis, result, predict_labels(result.scores)


def _summary(command, seed, graph, labels, basis, result, cfg):
    return {"command": command, "seed": seed, "n": graph.n, "layers": graph.T, "classes": labels.m,
            "p": float(cfg["power"]["p"]), "k": basis.k, "eigenvalues": [float(x) for x in basis.values],
            "iterations": result.iterations, "converged": result.converged}


def run_eig(cfg, seed, out_dir=".", threads=1):
    """k smallest power-mean eigenvalues -> eigenvalues.csv (+ eigenvectors.csv)."""
    clock = StageClock()
    graph = _graph(cfg, clock)
    basis = _eigs(graph, cfg, seed, clock)
    out_dir = _out_dir(out_dir)
    outputs = {"eigenvalues": os.path.join(out_dir, "eigenvalues.csv")}
    with clock("write"):
        write_matrix_csv(outputs["eigenvalues"], basis.values)
        if cfg["output"]["write_vectors"]:
            outputs["eigenvectors"] = os.path.join(out_dir, "eigenvectors.csv")
            write_matrix_csv(outputs["eigenvectors"], basis.vectors)
    report = {"command": "eig", "seed": seed, "n": graph.n, "layers": graph.T, "p": float(cfg["power"]["p"]),
              "k": basis.k, "eigenvalues": [float(x) for x in basis.values], "config": cfg}
    return _finish(out_dir, report, clock, outputs)


def _write_classification(out_dir, cfg, clock, pred, result, basis):
    outputs = {"predictions": os.path.join(out_dir, "predictions.csv")}
    with clock("write"):
        write_predictions_csv(outputs["predictions"], pred)
        if cfg["output"]["write_scores"]:
            outputs["scores"] = os.path.join(out_dir, "scores.csv")
            write_matrix_csv(outputs["scores"], result.scores)
        if cfg["output"].get("write_vectors") and basis is not None:
            outputs["eigenvectors"] = os.path.join(out_dir, "eigenvectors.csv")
            write_matrix_csv(outputs["eigenvectors"], basis.vectors)
    return outputs


def run_classify(cfg, seed, out_dir=".", threads=1):
    """Eigensolve + Allen-Cahn -> predictions.csv (+ scores, eigenvectors)."""
    clock = StageClock()
    graph = _graph(cfg, clock)
    truth = _truth(cfg, graph.n)
    labels, basis, result, pred = _classify(graph, cfg, seed, clock, truth)
    out_dir = _out_dir(out_dir)
    outputs = _write_classification(out_dir, cfg, clock, pred, result, basis)
    report = _summary("classify", seed, graph, labels, basis, result, cfg)
    report.update(_scores(pred, truth, labels))
    report["config"] = cfg
    return _finish(out_dir, report, clock, outputs)


def run_segment_image(cfg, seed, out_dir=".", threads=1):
    """Pixel classification of RGB images (runner.py:271-333): colour and
    per-image spatial kernel layers on the GPU, power-mean eigenbasis,
    Allen-Cahn; predictions / scores CSV and per-class + composite PNG masks."""
    clock = StageClock()
    images = cfg["input"]["images"]
    if not images:
        raise ConfigError("segment-image needs input.images")
    paths = [images] if isinstance(images, str) else list(images)
    with clock("load"):
        X, comps, shapes = image_features([load_image(p) for p in paths])
    cfg_g = cfg if cfg["grouping"]["groups"] is not None else \
        {**cfg, "grouping": {**cfg["grouping"], "groups": [dict(g) for g in SEGMENT_GROUPS]}}
    graph = _graph(cfg_g, clock, features=X, components=comps)
    truth = _truth(cfg, graph.n)
    labels, basis, result, pred = _classify(graph, cfg, seed, clock, truth)
    out_dir = _out_dir(out_dir)
    outputs = _write_classification(out_dir, {**cfg, "output": {**cfg["output"], "write_vectors": False}}, clock,
                                    pred, result, None)
    if cfg["output"]["write_masks"]:
        with clock("write"):
            colours = PALETTE[np.arange(labels.m) % len(PALETTE)]
            for i, mask in enumerate(masks_from_labels(pred, shapes)):
                for c in range(labels.m):
                    key = f"mask_img{i}_class{c + 1}"
                    outputs[key] = os.path.join(out_dir, key + ".png")
                    save_image(outputs[key], np.where(mask == c, 255, 0))
                outputs[f"composite_img{i}"] = os.path.join(out_dir, f"composite_img{i}.png")
                save_image(outputs[f"composite_img{i}"], colours[mask])
    report = _summary("segment-image", seed, graph, labels, basis, result, cfg)
    report["images"] = [list(sh) for sh in shapes]
    report.update(_scores(pred, truth, labels))
    report["config"] = cfg
    return _finish(out_dir, report, clock, outputs)


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
    clock = StageClock()
    b = cfg["bench"]["fastsum"]
    kernel = KernelSpec(family=b["family"], sigma=float(b["sigma"]))
    params = fastsum_params(cfg)
    reps = int(b["repetitions"])
    if reps < 1:
        raise ConfigError("bench.fastsum.repetitions must be >= 1")
    accuracy = []
    with clock("accuracy"):
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
    with clock("scaling"):
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
    # the reference's CSV exactly (a drop-in consumer parses it); the device
    # times go to their own file and report.json
    scale_path = os.path.join(out_dir, "fastsum_scaling.csv")
    with open(scale_path, "w", encoding="utf-8") as fh:
        fh.write("n,t_fast_median" + (",t_direct_median" if with_direct else "") + "\n")
        for i, n in enumerate(sizes):
            cols = [f"{n}", f"{scaling['t_fast'][i]:.6f}"]
            if with_direct:
                cols.append(f"{scaling['t_direct'][i]:.6f}")
            fh.write(",".join(cols) + "\n")
    dev_path = os.path.join(out_dir, "fastsum_scaling_device.csv")
    with open(dev_path, "w", encoding="utf-8") as fh:
        fh.write("n,t_fast_device_median\n")
        for i, n in enumerate(sizes):
            fh.write(f"{n},{scaling['t_fast_device'][i]:.6f}\n")
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
    report = {"command": "fastsum-bench", "seed": seed, "accuracy": accuracy, "scaling": scaling, "config": cfg}
    return _finish(out_dir, report, clock, {"accuracy_csv": acc_path, "scaling_csv": scale_path,
                                            "scaling_device_csv": dev_path, "table": txt_path})


def _unsupported(name):
    def run(cfg, seed, out_dir=".", threads=1):
        raise ConfigError(f"{name} is not part of the B200 backend "
                          "(supported: fastsum-bench, eig, classify, segment-image)")
    return run


run_sbm_bench = _unsupported("sbm-bench")
