"""End-to-end golden runs of the REAL reference for BASELINE configs 2, 3 and a
reduced config 4 (build container only; TEST INFRASTRUCTURE, never imported by
the product).

    python oracle/gen_golden_cfg.py --config 2            (~2-3 h of one core)
    python oracle/gen_golden_cfg.py --config 3            (~1-2 h)
    python oracle/gen_golden_cfg.py --config 4 --side 400 (~2 h)

Same recipe as oracle/gen_golden_cfg1.py: the seeded synth.py workload, one
`multilap.datapipe.feature_group` call per layer (each layer keeps its own
plan: synth.py records the N corrections the reference forces), then
`power_mean_eigs(G, PowerMeanConfig(p=-1), k, seed=0)` (ref powermean.py:130-189),
`sample_labels(truth, fraction, seed=0)` (ref datapipe.py:367-385) and
`allen_cahn_solve(basis, labels, AllenCahnParams(max_iter=...))`
(ref allencahn.py:172-229).

Config 4 runs at a reduced side (`--side`, same generator, same N=64 m=5
plans): the full 3162^2 image needs a 213 GB reference binding (SURVEY
§8(c)).  Its full-size matvec parity is pinned separately by the C chunked
oracle (oracle/c/mlb_oracle.c).

The output keeps what the parity tests check and stays small:
eigenvalues, the Allen-Cahn predicted labels, iterations, the degrees of
every layer (all nodes when n x layers <= 2e5, else a 4096-node seeded sample), and a
sketch of the eigenvector subspace: P z = Phi (Phi^T z) for two seeded
Gaussian z (float32), which compares projectors independently of the
eigenvectors' signs / rotations inside clusters.
"""

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.environ.get("MULTILAP_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import multilap  # noqa: E402,F401
from multilap import allencahn, datapipe, graphs, powermean  # noqa: E402
from multilap.kernels import KernelSpec  # noqa: E402

import synth  # noqa: E402


def sketch_seeds(n):
    """The two seeded probe vectors of the subspace sketch (tests regenerate them)."""
    return np.random.default_rng(12345).standard_normal((n, 2))


def degree_sample(n):
    return np.sort(np.random.default_rng(777).choice(n, size=min(n, 4096), replace=False))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True, choices=(2, 3, 4))
    ap.add_argument("--side", type=int, default=None)
    ap.add_argument("--max-iter", type=int, default=None)
    a = ap.parse_args()
    kw = {} if a.side is None else {"side": a.side}
    wl = synth.CONFIGS[a.config](seed=0, **kw)
    t0 = time.time()
    layers = []
    for ls in wl.layers:
        spec = datapipe.GroupingSpec((datapipe.GroupSpec(ls.columns, KernelSpec(ls.family, ls.sigma)),))
        G = datapipe.feature_group(wl.X, spec, fastsum_params=dict(N=ls.N, m_nfft=ls.m, p_nfft=ls.p))
        layers.append(G.layers[0])
    t_build = time.time() - t0
    G = graphs.MultilayerGraph(tuple(layers))
    count = [0]
    for lay in layers:  # count the layer matvecs inside the solver
        w = lay.weights
        orig = w.matvec

        def counted(v, orig=orig):
            count[0] += 1
            return orig(v)
        w.matvec = counted
    t0 = time.time()
    basis = powermean.power_mean_eigs(G, powermean.PowerMeanConfig(p=wl.p_mean), k=wl.k, seed=0)
    t_eig = time.time() - t0
    n_matvecs = count[0]
    labels = datapipe.sample_labels(wl.truth, wl.label_fraction, seed=0)
    params = allencahn.AllenCahnParams(max_iter=a.max_iter or wl.ac_max_iter)
    t0 = time.time()
    res = allencahn.allen_cahn_solve(basis, labels, params)
    t_ac = time.time() - t0
    pred = allencahn.predict_labels(res.scores)
    n = wl.n
    Z = sketch_seeds(n)
    sketch = (basis.vectors @ (basis.vectors.T @ Z)).astype(np.float32)
    if n * len(layers) <= 200_000:
        deg_idx = np.arange(n)
    else:   # a seeded 4096-node sample keeps the fixture small
        deg_idx = degree_sample(n)
    degs = np.stack([lay.degrees[deg_idx] for lay in layers])
    tag = f"cfg{a.config}" + ("" if a.side is None else f"_side{a.side}")
    out = os.path.join(ROOT, "tests", "golden", f"golden_{tag}.npz")
    np.savez_compressed(
        out, values=basis.values, pred=pred.astype(np.int16), sketch=sketch,
        deg_idx=deg_idx.astype(np.int64), degrees=degs,
        iters=np.array([res.iterations, int(res.converged)]),
        times=np.array([t_build, t_eig, t_ac]), n_matvecs=np.array([n_matvecs]),
        side=np.array([a.side or -1]), max_iter=np.array([params.max_iter]))
    acc = float(np.mean(pred == wl.truth))
    print(f"wrote {out}: build {t_build:.1f}s eig {t_eig:.1f}s ({n_matvecs} layer matvecs) "
          f"AC {t_ac:.2f}s ({res.iterations} it) accuracy {acc:.4f} values {basis.values}", flush=True)


if __name__ == "__main__":
    main()
