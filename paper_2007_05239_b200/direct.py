"""Exact O(n^2) kernel sums on the GPU (direct_apply, fastsum.py:500-553).

Used for KernelWeights without a plan (groups wider than 3 columns, mode
"none") and as the accuracy reference of the fastsum benches.
"""

import numpy as np

from . import _lib
from .errors import ConfigError


def _torch():
    import torch
    return torch


def _family(kernel):
    return 0 if kernel.family == "gaussian" else 1


def direct_sum_dev(X, v, kernel, y, alpha, beta, gamma, s=None, accumulate=False):
    """y (=|+=) alpha v + s (beta sum_j K s_j v_j + gamma s v), sum incl. j = i."""
    n, d = X.shape
    _lib.check(_lib.lib().mlb_direct(_lib.ptr(X), n, d, _family(kernel), float(kernel.sigma), _lib.ptr(v),
                                     _lib.ptr(s), _lib.ptr(y), float(alpha), float(beta), float(gamma),
                                     int(accumulate), _lib.stream_ptr()))
    return y


def direct_apply(points, v, kernel, block_rows=None):
    """W v with exact kernel weights, zero diagonal."""
    torch = _torch()
    x = np.asarray(points, dtype=float)
    if x.ndim != 2:
        raise ConfigError(f"points must be a 2-d array, got shape {x.shape}")
    n = x.shape[0]
    host = not isinstance(v, torch.Tensor)
    vv = np.asarray(v, dtype=float) if host else v
    if tuple(vv.shape) != (n,):
        raise ConfigError("v must be a vector matching the number of points")
    if n == 0:
        return np.zeros(0)
    dev = torch.cuda.current_device()
    Xd = torch.from_numpy(np.ascontiguousarray(x)).to(f"cuda:{dev}")
    vd = torch.from_numpy(np.ascontiguousarray(vv)).to(f"cuda:{dev}") if host else \
        vv.to(device=f"cuda:{dev}", dtype=torch.float64).contiguous()
    y = torch.empty_like(vd)
    direct_sum_dev(Xd, vd, kernel, y, -kernel.value_at_zero(), 1.0, 0.0)
    return y.cpu().numpy() if host else y


def direct_apply_dev(weights, v, y, alpha, beta, gamma, s=None, accumulate=False):
    """Block-diagonal direct apply for KernelWeights without a plan."""
    torch = _torch()
    cache = weights.__dict__.setdefault("_direct_blocks", {})
    for bi, idx in enumerate(weights._blocks):
        key = (bi, v.device.index)
        if key not in cache:
            Xb = torch.from_numpy(np.ascontiguousarray(weights.points[idx])).to(v.device)
            ib = torch.from_numpy(idx.astype(np.int64)).to(v.device)
            cache[key] = (Xb, ib)
        Xb, ib = cache[key]
        if len(weights._blocks) == 1:
            direct_sum_dev(Xb, v, weights.kernel, y, alpha, beta, gamma, s, accumulate)
            continue
        vb = v.index_select(0, ib).contiguous()
        sb = None if s is None else s.index_select(0, ib).contiguous()
        yb = y.index_select(0, ib).contiguous() if accumulate else torch.empty_like(vb)
        direct_sum_dev(Xb, vb, weights.kernel, yb, alpha, beta, gamma, sb, accumulate)
        y.index_copy_(0, ib, yb)
    return y


def direct_at_targets(points, v, kernel, targets):
    """Exact (W v)[t] for the target rows `targets` (zero diagonal), one
    device pass over all sources per target tile (mlb_direct_targets): the
    reference's accuracy check of fastsum against direct_apply
    (runner.py:496-512) on a target sample when n is too large for O(n^2)."""
    torch = _torch()
    x = np.ascontiguousarray(points, dtype=float)
    v = np.ascontiguousarray(v, dtype=float)
    tg = np.asarray(targets, dtype=np.int64)
    if x.ndim != 2 or v.shape != (x.shape[0],):
        raise ConfigError("points / v shapes do not match")
    dev = torch.cuda.current_device()
    Xd = torch.from_numpy(x).to(f"cuda:{dev}")
    vd = torch.from_numpy(v).to(f"cuda:{dev}")
    Xt = torch.from_numpy(np.ascontiguousarray(x[tg])).to(f"cuda:{dev}")
    yt = torch.empty(len(tg), dtype=torch.float64, device=f"cuda:{dev}")
    lib = _lib.lib()
    work = torch.empty(max(int(lib.mlb_direct_targets_work_size(len(tg))), 1), dtype=torch.float64,
                       device=f"cuda:{dev}")
    _lib.check(lib.mlb_direct_targets(_lib.ptr(Xd), x.shape[0], x.shape[1], _family(kernel), float(kernel.sigma),
                                      _lib.ptr(vd), _lib.ptr(Xt), len(tg), _lib.ptr(yt), _lib.ptr(work),
                                      _lib.stream_ptr()))
    return yt.cpu().numpy() - kernel.value_at_zero() * v[tg]
