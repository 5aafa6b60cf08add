"""Parity at the headline size: BASELINE configs[1] (512 x 512 segmentation,
n = 262,144, RGB d=3 N=64 m=4 + xy d=2 N=32 m=4) through the GPU path
against the reference algorithm run on every host core over ALL nodes
(oracle/parallel_ref.py: the oracle's bincount spread / full-grid FFT /
gather, one fixed point chunk per worker).  North-star tolerance: matvecs
within 1e-8 relative; observed ~1e-13."""

import math

import numpy as np
import pytest

from oracle import fastsum_oracle as fo

pytestmark = pytest.mark.gpu


def test_config2_full_size_matches_parallel_reference():
    import torch

    import synth
    from oracle import fastsum_oracle as fo
    from oracle.parallel_ref import ParallelReference
    from paper_2007_05239_b200 import KernelSpec, LaplacianBatch, MultilayerGraph, datapipe, with_shift
    wl = synth.config2_segmentation(seed=0)
    delta = math.log(2.0)
    G = synth.build_graph(wl, device=0)
    graph = MultilayerGraph(tuple(with_shift(layer, delta) for layer in G.layers))
    specs = []
    for ls in wl.layers:
        Xb, kb = datapipe.box_points(wl.X[:, list(ls.columns)], KernelSpec(ls.family, ls.sigma))
        specs.append((fo.OraclePlan(ls.family, kb.sigma, len(ls.columns), ls.N, ls.m, p=ls.p), Xb))
    ref = ParallelReference(specs, wl.n, delta, start_method="forkserver")  # this process runs CUDA
    try:
        v = np.random.default_rng(3).standard_normal(wl.n)
        want = [y.copy() for y in ref.step(v)]
        # the reference's degrees (W 1) against the layers' device degrees
        for t, layer in enumerate(G.layers):
            deg = layer.degrees
            assert np.linalg.norm(deg - ref.S["deg"][t]) <= 1e-12 * np.linalg.norm(ref.S["deg"][t])
    finally:
        ref.close()
    got = LaplacianBatch(graph).apply(torch.from_numpy(v).pin_memory()).numpy()
    for t in range(graph.T):
        err = np.linalg.norm(got[t] - want[t]) / np.linalg.norm(want[t])
        assert err < 1e-11, (t, err)


def test_config4_full_size_matches_c_oracle():
    """BASELINE configs[3] at FULL size (3162 x 3162, n = 9,998,244; RGB d=3
    and xy d=2, N=64, m=5): the layers' degrees and L_sym v for two seeded
    vectors through the GPU path (the m=5 d=3 spread, the grouped d=2 lanes
    of n >= 2^20, heavy-cell block splitting, the batched two-stream step)
    against the C restatement of the reference spread / gather on every host
    core with the scipy FFT stage (oracle/c_oracle.py; the chunked oracle of
    SURVEY 8(c): the reference binding would need 213 GB).  North-star bar:
    1e-8 relative; observed ~1e-13."""
    import torch

    import synth
    from oracle import c_oracle as co
    from paper_2007_05239_b200 import KernelSpec, LaplacianBatch, MultilayerGraph, datapipe, with_shift
    wl = synth.config4_large(seed=0)
    delta = math.log(2.0)
    G = synth.build_graph(wl, device=0)
    graph = MultilayerGraph(tuple(with_shift(layer, delta) for layer in G.layers))
    rng = np.random.default_rng(44)
    V = rng.standard_normal((2, wl.n))
    batch = LaplacianBatch(graph)
    got = [batch.apply(torch.from_numpy(v).pin_memory()).numpy().copy() for v in V]
    for t, ls in enumerate(wl.layers):
        Xb, kb = datapipe.box_points(wl.X[:, list(ls.columns)], KernelSpec(ls.family, ls.sigma))
        op = fo.OraclePlan(ls.family, kb.sigma, len(ls.columns), ls.N, ls.m, p=ls.p)
        deg, L = co.laplacian_layer(op, Xb, V, delta)
        derr = np.linalg.norm(G.layers[t].degrees - deg) / np.linalg.norm(deg)
        assert derr <= 1e-10, (t, derr)
        for k in range(2):
            err = np.linalg.norm(got[k][t] - L[k]) / np.linalg.norm(L[k])
            assert err <= 1e-8, (t, k, err)
            # the kernel part alone, D^-1/2 W D^-1/2 v = (1+delta) v - L v (the diagonal term would hide its error)
            kw, kw_ref = (1.0 + delta) * V[k] - got[k][t], (1.0 + delta) * V[k] - L[k]
            kerr = np.linalg.norm(kw - kw_ref) / np.linalg.norm(kw_ref)
            assert kerr <= 1e-8, (t, k, kerr)
            print(f"config 4 layer {t} vector {k}: L_sym rel err {err:.2e}, D^-1/2 W D^-1/2 v rel err {kerr:.2e} "
                  f"(degrees {derr:.2e})")
