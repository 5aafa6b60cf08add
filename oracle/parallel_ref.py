"""Multi-process CPU reference arm (TEST / BENCHMARK INFRASTRUCTURE ONLY).

The reference algorithm of the normalized-Laplacian matvec
(fastsum.py:389-406 spread / gather by bincount, :492-495 rfftn * fused *
irfftn on the full ng^d grid; graphs.py:197-201 the Laplacian) run on every
host core, as bench.py's `--impl reference` arm is asked to: the sample's
points are split into one contiguous chunk per worker process (bound once);
per layer and step the workers spread their chunk into private full grids,
sum the grids slice-wise in a fixed worker order, the main process runs the
FFT stage with scipy.fft on all cores, and the workers gather their chunk and
finish the Laplacian.  Same arithmetic as oracle/fastsum_oracle.py up to the
order of the grid sum.  Only bench.py (the reference arm, the CPU baseline)
and the tests use it.
"""

import multiprocessing as mp
import os

import numpy as np
import scipy.fft as sfft

from . import fastsum_oracle as fo


class _Shared:
    """A float64 array in shared memory: the RawArray travels to the workers
    (inherited under fork, passed by handle under forkserver), each side
    makes its own numpy view."""

    def __init__(self, shape):
        self.shape = tuple(int(x) for x in shape)
        self.raw = mp.RawArray("d", max(int(np.prod(self.shape)), 1))

    def view(self):
        n = int(np.prod(self.shape))
        return np.frombuffer(self.raw, dtype=np.float64, count=n).reshape(self.shape)


def _views(R):
    """Replace every _Shared in the (nested) dict / lists by its numpy view."""
    if isinstance(R, _Shared):
        return R.view()
    if isinstance(R, dict):
        return {k: _views(v) for k, v in R.items()}
    if isinstance(R, list):
        return [_views(v) for v in R]
    return R


def _worker(rank, R, conn):
    """One fixed chunk of the sample: bind once, then serve phase commands."""
    S = _views(R)
    lo, hi = S["bounds"][rank], S["bounds"][rank + 1]
    P = len(S["bounds"]) - 1
    bindings = [fo.bind(plan, pts[lo:hi], sort=False) if hi > lo else None for plan, pts in S["layers"]]
    conn.send("ready")
    while True:
        msg = conn.recv()
        if msg is None:
            return
        op, li = msg[0], msg[1]
        plan = S["layers"][li][0]
        b = bindings[li]
        if op == "spread":
            part = S["parts"][li][rank]
            if b is None:
                part[:] = 0.0
            else:
                x = S["v"][lo:hi]
                if msg[2]:
                    x = S["isd"][li][lo:hi] * x
                part[:] = fo.spread(b, x)
        elif op == "sum":  # grid slice [g0, g1) summed over the workers in a fixed order
            parts = S["parts"][li]
            G = parts.shape[1]
            g0, g1 = G * rank // P, G * (rank + 1) // P
            acc = parts[0, g0:g1].copy()
            for w in range(1, P):
                acc += parts[w, g0:g1]
            S["grid"][li][g0:g1] = acc
        elif op == "gather" and b is not None:
            if msg[2] == "degrees":  # W 1 = gather - K0 (graphs.py:176-177)
                S["deg"][li][lo:hi] = fo.gather(b, S["conv"][li]) - plan.K0
            else:  # (1 + delta) v - isd * W (isd v),  W x = gather - K0 x
                v = S["v"][lo:hi]
                isd = S["isd"][li][lo:hi]
                wx = fo.gather(b, S["conv"][li]) - plan.K0 * (isd * v)
                S["y"][li][lo:hi] = (1.0 + msg[3]) * v - isd * wx
        conn.send("ok")


class ParallelReference:
    """The shifted normalized-Laplacian matvec of several kernel layers over
    one node sample, on `procs` worker processes (default: every core)."""

    def __init__(self, layer_specs, n, delta, procs=None, start_method="fork"):
        """layer_specs: [(OraclePlan, points n x d in box units)].  `start_method`
        "forkserver" starts the workers from a clean interpreter (callers whose
        process already runs CUDA threads, e.g. the GPU tests)."""
        ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        self.P = P = int(procs or ncpu)
        self.n, self.delta, self.T = n, float(delta), len(layer_specs)
        bounds = [n * r // P for r in range(P + 1)]
        R = {
            "layers": [(plan, np.ascontiguousarray(pts)) for plan, pts in layer_specs],
            "bounds": bounds,
            "v": _Shared((n,)),
            "isd": [_Shared((n,)) for _ in layer_specs],
            "deg": [_Shared((n,)) for _ in layer_specs],
            "y": [_Shared((n,)) for _ in layer_specs],
            "parts": [_Shared((P, plan.ng ** plan.d)) for plan, _ in layer_specs],
            "grid": [_Shared((plan.ng ** plan.d,)) for plan, _ in layer_specs],
            "conv": [_Shared((plan.ng ** plan.d,)) for plan, _ in layer_specs],
        }
        self.S = S = _views(R)
        ctx = mp.get_context(start_method)
        if start_method == "forkserver":
            ctx.set_forkserver_preload(["numpy", "scipy.fft", "oracle.fastsum_oracle"])
        self.conns, self.procs = [], []
        for r in range(P):
            a, b = ctx.Pipe()
            pr = ctx.Process(target=_worker, args=(r, R, b), daemon=True)
            pr.start()
            self.conns.append(a)
            self.procs.append(pr)
        for c in self.conns:
            if c.recv() != "ready":
                raise RuntimeError("reference worker failed to start")
        # degrees W 1 (graphs.py:176-177), then D^-1/2
        S["v"][:] = 1.0
        for li in range(self.T):
            self._apply(li, False, "degrees")
            deg = S["deg"][li]
            if np.any(deg <= 1e-300):
                raise fo.OracleError("zero degree in the reference sample")
            S["isd"][li][:] = 1.0 / np.sqrt(deg)

    def _all(self, msg):
        for c in self.conns:
            c.send(msg)
        for c in self.conns:
            c.recv()

    def _apply(self, li, use_isd, mode):
        plan = self.S["layers"][li][0]
        self._all(("spread", li, use_isd))
        self._all(("sum", li))
        with sfft.set_workers(self.P):
            self.S["conv"][li][:] = fo.convolve_grid(plan, self.S["grid"][li])
        self._all(("gather", li, mode, self.delta))

    def step(self, v):
        """L_t v for every layer t -> list of arrays (views of shared memory)."""
        self.S["v"][:] = v
        for li in range(self.T):
            self._apply(li, True, "laplacian")
        return self.S["y"]

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except (BrokenPipeError, OSError):
                pass
        for pr in self.procs:
            pr.join(timeout=5)


def check_against_serial(layer_specs, delta, v, procs=2, start_method="fork"):
    """Max relative deviation of the parallel arm from the serial oracle (tests)."""
    from . import solvers_oracle as so
    par = ParallelReference(layer_specs, len(v), delta, procs=procs, start_method=start_method)
    try:
        ys = [y.copy() for y in par.step(v)]
    finally:
        par.close()
    worst = 0.0
    for (plan, pts), y in zip(layer_specs, ys):
        b = fo.bind(plan, pts)
        lay = so.OracleLayer(lambda x, plan=plan, b=b: fo.fastsum(plan, x, binding=b), len(v)).shifted(delta)
        ref = so.sym_laplacian(lay, v)
        worst = max(worst, float(np.linalg.norm(y - ref) / np.linalg.norm(ref)))
    return worst
