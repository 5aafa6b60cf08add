"""Node-range sharded solvers (paper_2007_05239_b200/sharded.py) at world
size 2 over gloo on CPU, against the single-process oracle.

Each rank owns half of the nodes of BOTH layers (one d=2, one d=3); its
layer engine is the numpy oracle on its own points with the grid summed over
the ranks (dist.ShardedLayer), the Krylov / Allen-Cahn algebra is torch on
CPU slices, every global sum one all-reduce.  The GPU path runs the same
solver code with libmlb as the engine and the algebra (tests/test_gpu_sharded.py).

Checks: power_mean_eigs at p = -1 and p = 1 (eigenvalues <= 1e-7, the
north-star bar; projectors <= 1e-6), Allen-Cahn scores / iterations /
labels in the oracle's eigenbasis, and every rank's identical decisions.
"""

import math
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fastsum_oracle as fo
from oracle import solvers_oracle as so

K = 4


class OracleEngine:
    def __init__(self, plan, points_local):
        self.plan = plan
        self.b = fo.bind(plan, points_local)

    def spread(self, x):
        return torch.from_numpy(fo.spread(self.b, np.asarray(x)).copy())

    def convolve(self, g):
        return fo.convolve_grid(self.plan, g.numpy())

    def gather(self, g):
        return fo.gather(self.b, g)

    def ones(self, n):
        return np.ones(n)

    def new_grid(self):
        return torch.zeros(self.plan.ng ** self.plan.d, dtype=torch.float64)


def _problem():
    rng = np.random.default_rng(321)
    n = 700
    g = rng.standard_normal((n, 2))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    pts2 = g * (0.21875 * rng.random(n) ** 0.5)[:, None]
    pts3 = np.clip(rng.normal(0, 0.06, size=(n, 3)), -0.21875, 0.21875)
    truth = (pts2[:, 0] > 0).astype(int) + 2 * (pts3[:, 0] > 0).astype(int)
    return pts2, pts3, truth


def _plans():
    return fo.OraclePlan("gaussian", 0.2, 2, 32, 4, p=8), fo.OraclePlan("gaussian", 0.15, 3, 16, 4, p=8)


def _labels(truth):
    from paper_2007_05239_b200.datapipe import sample_labels
    return sample_labels(truth, 0.05, seed=0)


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2007_05239_b200 import AllenCahnParams, LabelData, PowerMeanConfig
    from paper_2007_05239_b200.dist import Comm, ShardedLayer, shard_range
    from paper_2007_05239_b200.sharded import ShardContext, sharded_allen_cahn, sharded_power_mean_eigs
    comm = Comm()
    pts2, pts3, truth = _problem()
    n = len(truth)
    lo, hi = shard_range(n, rank, world)
    delta = math.log(2.0)
    out = {"lo": lo, "hi": hi}
    ctx = ShardContext(comm, n, lo, hi, device=None)
    for p, shift in ((-1.0, delta), (1.0, 0.0)):
        layers = []
        for plan, pts in zip(_plans(), (pts2, pts3)):
            lay = ShardedLayer(OracleEngine(plan, pts[lo:hi]), n, lo, hi, comm, K0=1.0, shift=shift).build()

            def lsym(x, lay=lay):
                return torch.from_numpy(np.asarray(lay.apply_lsym(x.numpy()), dtype=np.float64))

            def weighted(x, lay=lay):
                return torch.from_numpy(np.asarray(lay.isd * lay.matvec(lay.isd * x.numpy()), dtype=np.float64))
            layers.append((lsym, weighted))
        vals, vecs = sharded_power_mean_eigs(ctx, layers, PowerMeanConfig(p=p), K, seed=0)
        out[f"vals{int(p)}"] = vals
        out[f"vecs{int(p)}"] = vecs.numpy()
    # Allen-Cahn in the oracle's p = -1 eigenbasis (so its parity is separate from the eigensolver's)
    ref_layers = _oracle_layers(delta)
    rv, rV = so.power_mean_eigs(ref_layers, -1.0, K, seed=0)
    lab = _labels(truth)
    local = LabelData(F=lab.F[lo:hi], fidelity=lab.fidelity[lo:hi], m=lab.m)
    U, it, conv = sharded_allen_cahn(ctx, rv, rV[lo:hi], local, AllenCahnParams(max_iter=150))
    out.update(U=U.numpy(), it=it, conv=int(conv))
    np.savez(os.path.join(outdir, f"r{rank}.npz"), **out)
    dist.destroy_process_group()


def _oracle_layers(shift):
    pts2, pts3, truth = _problem()
    n = len(truth)
    p2, p3 = _plans()
    return [so.OracleLayer(lambda x: fo.fastsum(p2, x, points=pts2), n).shifted(shift),
            so.OracleLayer(lambda x: fo.fastsum(p3, x, points=pts3), n).shifted(shift)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _proj_dist(A, B, z):
    return np.linalg.norm(A @ (A.T @ z) - B @ (B.T @ z)) / np.linalg.norm(z)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_eigensolver_and_allen_cahn_two_ranks(world):
    """World sizes 2 and 3 (uneven node ranges) against the single-process oracle."""
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _free_port(), td), nprocs=world, join=True)
        parts = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(world)]
    pts2, pts3, truth = _problem()
    n = len(truth)
    z = np.random.default_rng(9).standard_normal((n, 3))
    for p in (-1, 1):
        ref_vals, ref_vecs = so.power_mean_eigs(_oracle_layers(math.log(2.0) if p < 0 else 0.0), float(p), K, seed=0)
        vals = parts[0][f"vals{p}"]
        for q in parts[1:]:
            assert np.array_equal(vals, q[f"vals{p}"])                   # identical on every rank
        assert np.max(np.abs(vals - ref_vals) / np.abs(ref_vals)) <= 1e-7, (p, vals, ref_vals)
        vecs = np.concatenate([q[f"vecs{p}"] for q in parts])
        assert _proj_dist(vecs, ref_vecs, z) <= 1e-6
    rv, rV = so.power_mean_eigs(_oracle_layers(math.log(2.0)), -1.0, K, seed=0)
    lab = _labels(truth)
    U_ref, it_ref, conv_ref = so.allen_cahn(rv, rV, lab.F, lab.fidelity, max_iter=150)
    U = np.concatenate([q["U"] for q in parts])
    assert all(int(q["it"]) == it_ref for q in parts)
    assert bool(parts[0]["conv"]) == conv_ref
    assert np.abs(U - U_ref).max() <= 1e-9
    assert np.array_equal(so.predict(U), so.predict(U_ref))
