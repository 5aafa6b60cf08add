"""ctypes front of oracle/c/mlb_oracle.c (TEST INFRASTRUCTURE ONLY).

The chunked reference oracle of SURVEY 8(c) for sizes where the numpy
restatement's binding does not fit in RAM (config 4: n = 9,998,244, d = 3,
m = 5 would need a 213 GB reference binding): spread / gather in C on all host
threads with the weights formed on the fly (fastsum.py:333-406 arithmetic),
the FFT stage in scipy exactly as oracle/fastsum_oracle.convolve_grid
(fastsum.py:492-495).  Pinned against the reference goldens in
tests/test_oracle_golden.py.  Only tests/, __graft_entry__ and bench.py's CPU
legs may use it.
"""

import ctypes as C
import os
import subprocess

import numpy as np
import scipy.fft as sfft

from . import fastsum_oracle as fo

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libmlb_oracle.so")
_lib = None


def build(force=False):
    """make -C oracle/c (gcc, pthreads); a no-op when the library is current."""
    src = os.path.join(HERE, "c", "mlb_oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(src) > os.path.getmtime(LIB):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "c")], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        P, I, I64, D = C.c_void_p, C.c_int, C.c_int64, C.c_double
        L.mlbo_window.restype = D
        L.mlbo_window.argtypes = [D, I, D]
        for name in ("mlbo_spread", "mlbo_gather"):
            fn = getattr(L, name)
            fn.restype = I
            fn.argtypes = [I, I, I, D, D, P, I64, P, I, P, I]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def window(t, m, b):
    return np.array([lib().mlbo_window(float(x), int(m), float(b)) for x in np.ravel(t)])


def spread(plan, points, V, threads=0, scale=None):
    """(nv, ng^d) grids of the rows of V (nv x n) over the box points."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    V = np.ascontiguousarray(np.atleast_2d(V), dtype=np.float64)
    n = pts.shape[0]
    G = plan.ng ** plan.d
    grid = np.empty((V.shape[0], G))
    sc = plan.ball_scale if scale is None else scale
    rc = lib().mlbo_spread(plan.d, plan.ng, plan.m, plan.b, sc, _ptr(pts), n, _ptr(V), V.shape[0], _ptr(grid),
                           int(threads))
    if rc:
        raise RuntimeError(f"mlbo_spread failed ({rc})")
    return grid


def gather(plan, points, grids, threads=0, scale=None):
    pts = np.ascontiguousarray(points, dtype=np.float64)
    grids = np.ascontiguousarray(np.atleast_2d(grids), dtype=np.float64)
    n = pts.shape[0]
    Y = np.empty((grids.shape[0], n))
    sc = plan.ball_scale if scale is None else scale
    rc = lib().mlbo_gather(plan.d, plan.ng, plan.m, plan.b, sc, _ptr(pts), n, _ptr(grids), grids.shape[0], _ptr(Y),
                           int(threads))
    if rc:
        raise RuntimeError(f"mlbo_gather failed ({rc})")
    return Y


def fastsum_many(plan, points, V, threads=0):
    """W v (zero diagonal, fastsum.py:475-497) for every row v of V, one pass
    over the points for all rows."""
    pts = fo.check_box(points, plan.eps_b)
    V = np.atleast_2d(np.asarray(V, dtype=np.float64))
    grids = spread(plan, pts, V, threads)
    workers = os.cpu_count() or 1
    with sfft.set_workers(workers):
        conv = np.stack([fo.convolve_grid(plan, g) for g in grids])
    return gather(plan, pts, conv, threads) - plan.K0 * V


def laplacian_layer(plan, points, V, delta, threads=0):
    """(degrees, rows of (1+delta) v - D^-1/2 W D^-1/2 v) for the rows of V
    (graphs.py:168-183, :197-201): two passes, W 1 then W (isd v)."""
    pts = fo.check_box(points, plan.eps_b)
    n = pts.shape[0]
    deg = fastsum_many(plan, pts, np.ones((1, n)), threads)[0]
    if np.any(deg <= 1e-300):
        raise fo.OracleError("zero degree")
    isd = 1.0 / np.sqrt(deg)
    V = np.atleast_2d(np.asarray(V, dtype=np.float64))
    W = fastsum_many(plan, pts, isd[None, :] * V, threads)
    return deg, (1.0 + delta) * V - isd[None, :] * W
