"""Config-1 end-to-end golden vectors from the REAL reference (build container only).

    python oracle/gen_golden_cfg1.py        (~2 minutes of CPU)

BASELINE configs[0] (the reference's CPU-runnable case): 100x100 synthetic
image (synth.config1_toy, seed 0), layers RGB d=3 sigma=0.1 and xy d=2
sigma=0.2, m=4, p_nfft=8; the RGB layer uses N=64 because the reference
rejects N=16 for it (negative NFFT degrees), xy keeps N=16.
Power mean p=-1, k=10 eigenpairs, 2% labels (sample_labels seed 0),
Allen-Cahn defaults.  Layers are built one feature_group call each so every
layer keeps its own plan.  Output: tests/golden/golden_cfg1.npz.
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.environ.get("MULTILAP_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import multilap  # noqa: E402
from multilap import allencahn, datapipe, graphs, powermean  # noqa: E402
from multilap.kernels import KernelSpec  # noqa: E402

import synth  # noqa: E402


def main():
    wl = synth.config1_toy(seed=0)
    layers = []
    for ls in wl.layers:
        spec = datapipe.GroupingSpec((datapipe.GroupSpec(ls.columns, KernelSpec(ls.family, ls.sigma)),))
        G = datapipe.feature_group(wl.X, spec, fastsum_params=dict(N=ls.N, m_nfft=ls.m, p_nfft=ls.p))
        layers.append(G.layers[0])
    G = graphs.MultilayerGraph(tuple(layers))
    t0 = time.time()
    basis = powermean.power_mean_eigs(G, powermean.PowerMeanConfig(p=-1.0), k=wl.k, seed=0)
    t_eig = time.time() - t0
    labels = datapipe.sample_labels(wl.truth, wl.label_fraction, seed=0)
    t0 = time.time()
    res = allencahn.allen_cahn_solve(basis, labels, allencahn.AllenCahnParams())
    t_ac = time.time() - t0
    pred = allencahn.predict_labels(res.scores)
    ids = np.where(labels.labeled_mask, np.argmax(labels.F, axis=1), -1)
    out = os.path.join(ROOT, "tests", "golden", "golden_cfg1.npz")
    np.savez_compressed(out, X=wl.X, truth=wl.truth, deg0=layers[0].degrees, deg1=layers[1].degrees,
                        values=basis.values, vectors=basis.vectors, label_ids=ids, scores=res.scores,
                        iters=np.array([res.iterations, int(res.converged)]), pred=pred,
                        times=np.array([t_eig, t_ac]))
    acc = float(np.mean(pred == wl.truth))
    print(f"wrote {out}: eig {t_eig:.1f}s, AC {t_ac:.2f}s ({res.iterations} it), accuracy {acc:.4f}, "
          f"values {basis.values}")


if __name__ == "__main__":
    main()
