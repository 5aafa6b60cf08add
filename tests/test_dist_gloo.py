"""Multi-process (gloo, world_size 2, CPU) tests of the partitioning logic in
paper_2007_05239_b200/dist.py, with the per-rank compute supplied by the
numpy oracle (the GPU engine is libmlb; the logic under test is identical).

Checks: node-range sharded Laplacian == single-process oracle; sharded PKSM
== oracle PKSM; layer round-robin M_p^p v == oracle.
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


class OracleEngine:
    """spread / convolve / gather of this rank's points on the full ng^d torus grid."""

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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    rng = np.random.default_rng(123)
    n = 900
    g = rng.standard_normal((n, 2))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    pts = g * (0.21875 * rng.random(n) ** 0.5)[:, None]
    pts3 = np.clip(rng.normal(0, 0.06, size=(n, 3)), -0.21875, 0.21875)
    v = rng.standard_normal(n)
    return pts, pts3, v


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2007_05239_b200.dist import (Comm, LayerParallelGraph, ShardedLayer, shard_range, sharded_pksm)
    comm = Comm()
    pts, pts3, v = _problem()
    n = len(v)
    lo, hi = shard_range(n, rank, world)
    plan = fo.OraclePlan("gaussian", 0.2, 2, 32, 4, p=8)
    delta = math.log(2.0)
    lay = ShardedLayer(OracleEngine(plan, pts[lo:hi]), n, lo, hi, comm, K0=1.0, shift=delta).build()
    y = lay.apply_lsym(v[lo:hi])
    yp = sharded_pksm(lay, -1.0, v[lo:hi])
    # layer round-robin over two oracle layers (one d=2, one d=3)
    plan3 = fo.OraclePlan("gaussian", 0.15, 3, 16, 4, p=8)
    full = [so.OracleLayer(lambda x: fo.fastsum(plan, x, points=pts), n).shifted(delta),
            so.OracleLayer(lambda x: fo.fastsum(plan3, x, points=pts3), n).shifted(delta)]
    local = [full[t] if t % world == rank else None for t in range(2)]
    lpg = LayerParallelGraph(2, n, local, comm,
                             pksm=lambda layer, p, x: torch.from_numpy(so.pksm(layer, p, x.numpy())))
    z = lpg.apply_Lp_power(-1.0, torch.from_numpy(v)).numpy()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), lo=lo, hi=hi, y=y, yp=yp, z=z,
             deg=lay.degrees)
    dist.destroy_process_group()


def test_two_rank_partitionings_match_oracle():
    world = 2
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _free_port(), td), nprocs=world, join=True)
        parts = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(world)]
        pts, pts3, v = _problem()
        n = len(v)
        plan = fo.OraclePlan("gaussian", 0.2, 2, 32, 4, p=8)
        delta = math.log(2.0)
        ref_layer = so.OracleLayer(lambda x: fo.fastsum(plan, x, points=pts), n).shifted(delta)
        y = np.concatenate([p["y"] for p in parts])
        deg = np.concatenate([p["deg"] for p in parts])
        ref = so.sym_laplacian(ref_layer, v)
        assert np.linalg.norm(deg - ref_layer.degrees) <= 1e-13 * np.linalg.norm(ref_layer.degrees)
        assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
        yp = np.concatenate([p["yp"] for p in parts])
        refp = so.pksm(ref_layer, -1.0, v)
        assert np.linalg.norm(yp - refp) <= 1e-10 * np.linalg.norm(refp)
        plan3 = fo.OraclePlan("gaussian", 0.15, 3, 16, 4, p=8)
        full = [ref_layer, so.OracleLayer(lambda x: fo.fastsum(plan3, x, points=pts3), n).shifted(delta)]
        refz = so.apply_Lp_power(full, -1.0, v)
        for p in parts:   # every rank holds the identical layer sum
            assert np.linalg.norm(p["z"] - refz) <= 1e-12 * np.linalg.norm(refz)
        assert np.array_equal(parts[0]["z"], parts[1]["z"])
