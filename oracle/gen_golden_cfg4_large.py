"""Config 4 at side 1000 (n = 10^6) end to end: the REAL reference's solvers
(multilap power_mean_eigs / sample_labels / allen_cahn_solve, feature scaling
by multilap.datapipe.scale_for_fastsum) with the layers' W v computed by the
multi-process oracle of the reference algorithm (oracle/parallel_ref.py:
bincount spread / scipy FFT / bincount gather on point chunks, pinned to the
reference's own fastsum outputs at <= 1e-13 in tests/test_oracle_golden.py).
multilap's own KernelWeights would need a 21 GB binding and ~5 h of one core
for this size; the chunked processes give the same arithmetic up to the
summation order of the grid.  Build container only; TEST INFRASTRUCTURE.

    python oracle/gen_golden_cfg4_large.py [--side 1000] [--procs 8]   (~1 h)
"""

import argparse
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.environ.get("MULTILAP_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from multilap import allencahn, datapipe, graphs, powermean  # noqa: E402

import synth  # noqa: E402
from oracle import fastsum_oracle as fo  # noqa: E402
from oracle.gen_golden_cfg import degree_sample, sketch_seeds  # noqa: E402
from oracle.parallel_ref import ParallelReference  # noqa: E402


class ParallelWeights:
    """The reference weights protocol {n, matvec, materialize} over one layer
    of a ParallelReference (W v with zero diagonal)."""

    def __init__(self, ref, li):
        self.ref, self.li, self.n = ref, li, ref.n

    def matvec(self, v):
        v = np.asarray(v, dtype=float)
        self.ref.S["v"][:] = v
        self.ref._apply(self.li, False, "degrees")   # the "degrees" mode returns gather - K0 (for v = 1)
        K0 = self.ref.S["layers"][self.li][0].K0
        return self.ref.S["deg"][self.li] + K0 - K0 * v   # W v = gather - K0 v (fastsum.py:497)

    def materialize(self):
        raise NotImplementedError


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=1000)
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    a = ap.parse_args()
    wl = synth.config4_large(seed=0, side=a.side)
    t0 = time.time()
    specs = []
    for ls in wl.layers:
        Xb, info = datapipe.scale_for_fastsum(wl.X[:, list(ls.columns)])
        sigma_box = ls.sigma / info.factor                 # mode "fastsum-box" (datapipe.py:126-133)
        specs.append((fo.OraclePlan(ls.family, sigma_box, len(ls.columns), ls.N, ls.m, p=ls.p), Xb))
    ref = ParallelReference(specs, wl.n, math.log(2.0), procs=a.procs)
    try:
        layers = [graphs.build_layer(ParallelWeights(ref, li)) for li in range(len(specs))]
        t_build = time.time() - t0
        count = [0]
        for lay in layers:
            w = lay.weights
            orig = w.matvec

            def counted(v, orig=orig):
                count[0] += 1
                return orig(v)
            w.matvec = counted
        G = graphs.MultilayerGraph(tuple(layers))
        t0 = time.time()
        basis = powermean.power_mean_eigs(G, powermean.PowerMeanConfig(p=wl.p_mean), k=wl.k, seed=0)
        t_eig = time.time() - t0
    finally:
        ref.close()
    labels = datapipe.sample_labels(wl.truth, wl.label_fraction, seed=0)
    params = allencahn.AllenCahnParams(max_iter=wl.ac_max_iter)
    t0 = time.time()
    res = allencahn.allen_cahn_solve(basis, labels, params)
    t_ac = time.time() - t0
    pred = allencahn.predict_labels(res.scores)
    n = wl.n
    sketch_idx = np.arange(0, n, 8, dtype=np.int64)   # every 8th row keeps the fixture ~1 MB
    sketch = (basis.vectors @ (basis.vectors.T @ sketch_seeds(n)))[sketch_idx].astype(np.float32)
    deg_idx = degree_sample(n)
    degs = np.stack([lay.degrees[deg_idx] for lay in layers])
    out = os.path.join(ROOT, "tests", "golden", f"golden_cfg4_side{a.side}.npz")
    np.savez_compressed(out, values=basis.values, pred=pred.astype(np.int8), sketch=sketch, sketch_idx=sketch_idx,
                        deg_idx=deg_idx.astype(np.int64), degrees=degs,
                        iters=np.array([res.iterations, int(res.converged)]),
                        times=np.array([t_build, t_eig, t_ac]), n_matvecs=np.array([count[0]]),
                        side=np.array([a.side]), max_iter=np.array([params.max_iter]),
                        hybrid=np.array([1]))
    print(f"wrote {out}: build {t_build:.1f}s eig {t_eig:.1f}s ({count[0]} layer matvecs, {a.procs} processes) "
          f"AC {t_ac:.2f}s ({res.iterations} it) accuracy {np.mean(pred == wl.truth):.4f} values {basis.values}",
          flush=True)


if __name__ == "__main__":
    main()
