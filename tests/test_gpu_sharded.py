"""Node-range sharding on the GPU: dist.ShardedKernelGraph.

* NCCL at world size 1 (the only size one GPU allows): the step runs its
  all-reduce and must equal the unsharded LaplacianBatch step bitwise (same
  kernels, a one-rank sum is the identity).
* Two ranks emulated on one GPU WITHOUT collectives (each half binds its own
  nodes; the test sums the two ranks' grids itself, then every rank finishes
  its nodes): degrees and L_sym match the unsharded layers and the oracle,
  i.e. the partitioning is right by construction for the NCCL all-reduce.
"""

import math
import os
import socket

import numpy as np
import pytest

from oracle import fastsum_oracle as fo
from oracle import solvers_oracle as so

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _groups(wl):
    from paper_2007_05239_b200 import KernelSpec
    return [(ls.columns, KernelSpec(ls.family, ls.sigma), dict(N=ls.N, m_nfft=ls.m, p_nfft=ls.p)) for ls in wl.layers]


def _small_cfg4(side=96):
    import synth
    return synth.config4_large(seed=0, side=side)


def test_sharded_graph_nccl_world1_equals_unsharded():
    import torch
    import torch.distributed as dist

    import synth
    from paper_2007_05239_b200 import LaplacianBatch, MultilayerGraph, with_shift
    from paper_2007_05239_b200.dist import Comm, ShardedKernelGraph, shard_feature_groups
    wl = _small_cfg4()
    delta = math.log(2.0)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        lo, hi, pts, kerns, plans = shard_feature_groups(wl.X, _groups(wl), 0, 1)
        sg = ShardedKernelGraph(pts, kerns, plans, wl.n, lo, hi, comm=Comm(), shift=delta, device=0).build()
        G = synth.build_graph(wl, device=0)
        for t, layer in enumerate(G.layers):
            assert np.array_equal(sg.degrees[t].cpu().numpy(), layer.degrees)
        v = torch.from_numpy(np.random.default_rng(5).standard_normal(wl.n)).cuda()
        ys = [torch.empty_like(v) for _ in range(wl.layers.__len__())]
        sg.lsym(v, ys)
        ref = LaplacianBatch(MultilayerGraph(tuple(with_shift(lay, delta) for lay in G.layers))).apply_dev(v)
        for t in range(len(ys)):
            assert torch.equal(ys[t], ref[t]), t
        # the step replayed from a captured CUDA graph (NCCL all-reduces inside)
        # equals the eager step bitwise, replay after replay
        yg = [torch.empty_like(v) for _ in range(len(ys))]
        for _ in range(3):
            sg.lsym_graph(v, yg)
        assert sg._graphs[(v.data_ptr(), tuple(y.data_ptr() for y in yg))][0] is not None   # captured
        for t in range(len(ys)):
            assert torch.equal(yg[t], ref[t]), t
        # the streamed host-in / host-out form: every vector's results equal
        # the per-vector step bitwise
        V = torch.from_numpy(np.random.default_rng(6).standard_normal((5, wl.n))).pin_memory()
        Y = sg.lsym_many(V)
        for i in range(5):
            sg.lsym(V[i].cuda(), ys)
            for t in range(len(ys)):
                assert torch.equal(Y[i, t], ys[t].cpu()), (i, t)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,lattice", [(2, False), (3, False), (2, True), (3, True)])
def test_sharded_graph_emulated_ranks_match_oracle(world, lattice):
    """(lattice: the xy layer on the d = 2 lattice items, forced at this size;
    the rank boundaries cut image rows -> partial-run segments)"""
    import torch

    from paper_2007_05239_b200.dist import ShardedKernelGraph, shard_feature_groups
    wl = _small_cfg4(side=80)
    delta = math.log(2.0)
    ranks = []
    os.environ["MLB_LATTICE"] = "1" if lattice else "0"
    try:
        for r in range(world):
            lo, hi, pts, kerns, plans = shard_feature_groups(wl.X, _groups(wl), r, world)
            ranks.append(ShardedKernelGraph(pts, kerns, plans, wl.n, lo, hi, comm=None, shift=delta, device=0))
    finally:
        del os.environ["MLB_LATTICE"]
    for sg in ranks:   # the d = 2 (xy) layer runs on lattice items exactly when forced
        assert [w._bindings[0].stats()["lattice_items"] > 0 for w in sg.weights] == [False, lattice]
    T = len(wl.layers)

    def emulated_step(vs, coef_of, flags):
        outs = [[torch.empty_like(v) for _ in range(T)] for v in vs]
        for sg, v in zip(ranks, vs):
            sg.spread_local(v, flags)
        total = sum(sg.grids for sg in ranks)            # the all-reduce, done by the test
        for sg, v, ys in zip(ranks, vs, outs):
            sg.grids.copy_(total)
            sg.finish(v, ys, coef_of(sg), flags)
        return outs

    ones = [torch.ones(sg.n_local, dtype=torch.float64, device="cuda") for sg in ranks]
    degs = emulated_step(ones, lambda sg: [(-k0, 1.0, 0.0) for k0 in sg.K0], 0)
    for sg, dg in zip(ranks, degs):
        sg.set_degrees(dg)
    rng = np.random.default_rng(11)
    v = rng.standard_normal(wl.n)
    vs = [torch.from_numpy(v[sg.lo:sg.hi].copy()).cuda() for sg in ranks]
    from paper_2007_05239_b200 import _lib
    outs = emulated_step(vs, lambda sg: [(1.0 + delta, -1.0, k0) for k0 in sg.K0], _lib.MLB_USE_ISD)
    got = [np.concatenate([o[t].cpu().numpy() for o in outs]) for t in range(T)]
    got_deg = [np.concatenate([dg[t].cpu().numpy() for dg in degs]) for t in range(T)]
    from paper_2007_05239_b200 import KernelSpec, datapipe
    for t, ls in enumerate(wl.layers):
        Xb, kb = datapipe.box_points(wl.X[:, list(ls.columns)], KernelSpec(ls.family, ls.sigma))
        op = fo.OraclePlan(ls.family, kb.sigma, len(ls.columns), ls.N, ls.m, p=ls.p)
        b = fo.bind(op, Xb)
        lay = so.OracleLayer(lambda x, op=op, b=b: fo.fastsum(op, x, binding=b), wl.n)
        deg = lay.matvec(np.ones(wl.n))
        assert _rel(got_deg[t], deg) < 1e-12
        ref = so.sym_laplacian(lay.shifted(delta), v)
        assert _rel(got[t], ref) < 1e-11, (t, _rel(got[t], ref))


def test_sharded_eigensolver_and_allen_cahn_nccl_world1():
    """sharded.sharded_power_mean_eigs + sharded_allen_cahn through the NCCL
    process group (world size 1: every reduction is a real collective call)
    against the single-GPU power_mean_eigs / allen_cahn_solve of the same
    graph: eigenvalues <= 1e-9, projectors <= 1e-7, identical labels."""
    import torch
    import torch.distributed as dist

    import synth
    from paper_2007_05239_b200 import (AllenCahnParams, LabelData, PowerMeanConfig, allen_cahn_solve,
                                       power_mean_eigs, predict_labels, sample_labels)
    from paper_2007_05239_b200.dist import Comm, ShardedKernelGraph, shard_feature_groups
    from paper_2007_05239_b200.powermean import SpectralBasis
    from paper_2007_05239_b200.sharded import ShardContext, sharded_allen_cahn, sharded_power_mean_eigs
    wl = _small_cfg4(side=64)
    delta = math.log(2.0)
    k = 4
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        comm = Comm()
        lo, hi, pts, kerns, plans = shard_feature_groups(wl.X, _groups(wl), 0, 1)
        sg = ShardedKernelGraph(pts, kerns, plans, wl.n, lo, hi, comm=comm, shift=delta, device=0).build()
        ctx = ShardContext(comm, wl.n, lo, hi, device=0)
        vals, vecs = sharded_power_mean_eigs(ctx, sg.layer_ops(), PowerMeanConfig(p=-1.0), k, seed=0)
        G = synth.build_graph(wl, device=0)
        ref = power_mean_eigs(G, PowerMeanConfig(p=-1.0), k, seed=0)
        assert np.max(np.abs(vals - ref.values) / np.abs(ref.values)) <= 1e-9
        V = vecs.cpu().numpy()
        z = np.random.default_rng(3).standard_normal((wl.n, 2))
        d = np.linalg.norm(V @ (V.T @ z) - ref.vectors @ (ref.vectors.T @ z)) / np.linalg.norm(z)
        assert d <= 1e-7, d
        lab = sample_labels(wl.truth, 0.02, seed=0)
        U, it, conv = sharded_allen_cahn(ctx, vals, vecs, LabelData(F=lab.F, fidelity=lab.fidelity, m=lab.m),
                                         AllenCahnParams(max_iter=100))
        res = allen_cahn_solve(SpectralBasis(values=vals, vectors=V), lab, AllenCahnParams(max_iter=100))
        assert it == res.iterations and conv == res.converged
        assert np.abs(U.cpu().numpy() - res.scores).max() <= 1e-12
        assert np.array_equal(predict_labels(U.cpu().numpy()), predict_labels(res.scores))
    finally:
        dist.destroy_process_group()
