"""Multiclass Allen-Cahn classifier in the eigenbasis -- drop-in for multilap.allencahn.

One convexity-splitting iteration (allencahn.py:172-223):
    R  = (1 + c dt) U - dt/(2 eps) T(U) - dt omega (U - F)
    Vc = Phi^T R / (1 + c dt + eps dt lambda)
    U+ = proj_simplex(Phi Vc)
runs as the libmlb kernel sequence mlb_ac_step2: one pass over Phi per
iteration (the projection of iteration t and the right-hand side of t+1
share the staged, double-buffered Phi tile; fixed-order Phi^T R reduction);
the host only reads the two maxima of the stopping rule each iteration.
"""

import ctypes as C
from dataclasses import dataclass

import os

import numpy as np

from . import _lib
from .errors import ConfigError, NumericalError
from .powermean import SpectralBasis


def _torch():
    import torch
    return torch


@dataclass(frozen=True)
class LabelData:
    """One-hot F plus per-node fidelity (allencahn.py:32-70)."""

    F: np.ndarray
    fidelity: np.ndarray
    m: int

    @classmethod
    def from_class_ids(cls, ids, m, omega0):
        ids = np.asarray(ids)
        if m < 2:
            raise ConfigError(f"need at least 2 classes, got m={m}")
        if ids.ndim != 1:
            raise ConfigError("class ids must form a vector")
        if ids.max(initial=-1) >= m:
            raise ConfigError(f"class id {ids.max()} out of range for m={m}")
        if ids.min(initial=0) < -1:
            raise ConfigError("class ids must be >= -1 (-1 = unlabeled)")
        if omega0 <= 0:
            raise ConfigError(f"omega0 must be positive, got {omega0}")
        n = ids.shape[0]
        F = np.zeros((n, m))
        lab = ids >= 0
        F[np.flatnonzero(lab), ids[lab]] = 1.0
        return cls(F=F, fidelity=np.where(lab, float(omega0), 0.0), m=m)

    @property
    def n(self):
        return self.F.shape[0]

    @property
    def labeled_mask(self):
        return self.fidelity > 0


@dataclass(frozen=True)
class AllenCahnParams:
    """Scheme parameters (allencahn.py:73-102); c defaults to omega0 + 3/eps."""

    epsilon: float = 5e-3
    omega0: float = 1000.0
    c: float | None = None
    dt: float = 0.01
    tolerance: float = 1e-6
    max_iter: int = 300

    def __post_init__(self):
        if self.epsilon <= 0 or self.dt <= 0:
            raise ConfigError("epsilon and dt must be positive")
        if self.omega0 < 0:
            raise ConfigError("omega0 must be nonnegative")
        if self.tolerance < 0:
            raise ConfigError("tolerance must be nonnegative")
        if self.max_iter < 1:
            raise ConfigError("max_iter must be at least 1")
        if self.c_value < self.omega0 + 1.0 / self.epsilon - 1e-12:
            raise ConfigError(f"c = {self.c_value} violates the convexity bound "
                              f"omega0 + 1/eps = {self.omega0 + 1.0 / self.epsilon}")

    @property
    def c_value(self):
        return self.omega0 + 3.0 / self.epsilon if self.c is None else self.c


@dataclass
class AllenCahnResult:
    scores: np.ndarray
    iterations: int
    converged: bool


def initial_scores(labels):
    """Labeled rows at their corner, the rest at the barycenter (allencahn.py:157-162)."""
    U = np.full((labels.n, labels.m), 1.0 / labels.m)
    mask = labels.labeled_mask
    U[mask] = labels.F[mask]
    return U


def _dev(x, device):
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return x.to(device=f"cuda:{device}", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=float))).to(f"cuda:{device}")


def allen_cahn_solve(basis, labels, params, callback=None, device=None, return_device=False):
    """Run the convexity-splitting scheme in `basis` (allencahn.py:172-223) on the GPU."""
    torch = _torch()
    if labels.m < 2:
        raise ConfigError("multiclass scheme needs m >= 2")
    phi = basis.vectors
    lam = np.asarray(basis.values, dtype=float)
    if phi.shape[0] != labels.n:
        raise ConfigError("basis and labels disagree on node count")
    if device is None:
        device = phi.device.index if isinstance(phi, torch.Tensor) else torch.cuda.current_device()
    n, k, m = labels.n, int(phi.shape[1]), labels.m
    eps, dt, c = params.epsilon, params.dt, params.c_value
    Phi = _dev(phi, device)
    denom = _dev(1.0 + c * dt + eps * dt * lam, device)
    U = _dev(initial_scores(labels), device)
    Un = torch.empty_like(U)
    F = _dev(labels.F, device)
    fid = _dev(labels.fidelity, device)
    lib = _lib.lib()
    work = torch.empty(int(lib.mlb_ac_work_size(n, k, m)), dtype=torch.float64, device=U.device)
    stats = torch.empty(2, dtype=torch.float64, device=U.device)
    # The device runs one iteration ahead of the host's stopping test (the
    # test of iteration t reads its two maxima from pinned memory while
    # iteration t+1 computes into the other buffer; a stop at t discards
    # t+1).  Iterates are bitwise those of the one-at-a-time loop.
    # MLB_AC_DEPTH=1 (or a callback, which needs every iterate) disables it.
    depth = 1 if callback is not None else max(1, min(2, int(os.environ.get("MLB_AC_DEPTH", "2"))))
    bufs = (U, Un)
    pin = torch.empty((2, 2), dtype=torch.float64, pin_memory=True)
    evs = (torch.cuda.Event(), torch.cuda.Event())
    stream = torch.cuda.current_stream(U.device)

    def launch(it):
        src, dst = bufs[(it - 1) % 2], bufs[it % 2]
        _lib.check(lib.mlb_ac_step2(_lib.ptr(Phi), n, k, m, _lib.ptr(src), _lib.ptr(F), _lib.ptr(fid),
                                    _lib.ptr(denom), 1.0 + c * dt, dt / (2.0 * eps), dt, int(it == 1), _lib.ptr(dst),
                                    _lib.ptr(stats), _lib.ptr(work), _lib.stream_ptr()))
        pin[it % 2].copy_(stats, non_blocking=True)
        evs[it % 2].record(stream)

    converged = False
    iterations = 0
    launch(1)
    for it in range(1, params.max_iter + 1):
        if depth > 1 and it < params.max_iter:
            launch(it + 1)   # speculative: writes the other buffer
        evs[it % 2].synchronize()
        num, den = (float(x) for x in pin[it % 2])
        if den <= 0 or not np.isfinite(num):
            raise NumericalError("Allen-Cahn iterate degenerated")
        U = bufs[it % 2]
        iterations = it
        if callback is not None:
            callback(it, U.cpu().numpy())
        if num / den <= params.tolerance:
            converged = True
            break
        if depth == 1 and it < params.max_iter:
            launch(it + 1)
    stream.synchronize()   # (a discarded speculative step may still run)
    scores = U if return_device else U.cpu().numpy()
    return AllenCahnResult(scores=scores, iterations=iterations, converged=converged)


def predict_labels(scores):
    """Argmax per row, ties to the lowest class (allencahn.py:226-229)."""
    torch = _torch()
    if isinstance(scores, torch.Tensor) and scores.is_cuda:
        s = scores.to(torch.float64).contiguous()
        n, m = s.shape
        out = torch.empty(n, dtype=torch.int32, device=s.device)
        _lib.check(_lib.lib().mlb_argmax_rows(_lib.ptr(s), n, m, _lib.ptr(out), _lib.stream_ptr()))
        return out
    return np.argmax(np.asarray(scores), axis=1)


def simplex_project_rows(U):
    """Row-wise projection onto the probability simplex (allencahn.py:105-124)."""
    U = np.asarray(U, dtype=float)
    squeeze = U.ndim == 1
    if squeeze:
        U = U[None, :]
    n, m = U.shape
    s = -np.sort(-U, axis=1)
    cs = np.cumsum(s, axis=1)
    cond = s + (1.0 - cs) / np.arange(1, m + 1) > 0
    rho = m - np.argmax(cond[:, ::-1], axis=1) - 1
    tau = (1.0 - cs[np.arange(n), rho]) / (rho + 1)
    out = np.maximum(U + tau[:, None], 0.0)
    return out[0] if squeeze else out


def nonlinearity_T(U):
    """Derivative of the multi-well potential, row-wise (allencahn.py:142-154)."""
    U = np.asarray(U, dtype=float)
    aU = np.abs(U)
    A = aU.sum(axis=1, keepdims=True) - aU + np.abs(U - 1.0)
    B = 0.25 * A * A
    n, m = B.shape
    left = np.ones_like(B)
    right = np.ones_like(B)
    np.cumprod(B[:, :-1], axis=1, out=left[:, 1:])
    np.cumprod(B[:, :0:-1], axis=1, out=right[:, -2::-1])
    wt = A * (left * right)
    return 0.5 * wt.sum(axis=1, keepdims=True) - wt


# ------------------------------------------------------- binary scheme ----
@dataclass
class BinaryAllenCahnResult:
    scores: np.ndarray
    iterations: int
    converged: bool


def binary_allen_cahn_solve(basis, f, params, callback=None, device=None, return_device=False):
    """Two-class spectral scheme with the (u^2 - 1)^2 / 4 well (allencahn.py:261-309):

        v+ = [(1 + c dt + dt/eps) v - dt/eps Phi^T u^3 - dt Phi^T (omega (u - f))]
             / (1 + c dt + eps dt lambda),   u = Phi v,

    one mlb_bac_step per iteration (two fixed-order Phi^T reductions, the
    coefficient update, Phi v and the stopping maxima on the device)."""
    torch = _torch()
    phi = basis.vectors
    lam = np.asarray(basis.values, dtype=float)
    f_host = f.cpu().numpy() if isinstance(f, torch.Tensor) else np.asarray(f, dtype=float)
    if f_host.shape != (phi.shape[0],):
        raise ConfigError("labels f must be one value per node")
    if np.any(np.abs(f_host[f_host != 0]) != 1.0):
        raise ConfigError("binary labels must be -1, 0 or +1")
    if device is None:
        device = phi.device.index if isinstance(phi, torch.Tensor) else torch.cuda.current_device()
    n, k = int(phi.shape[0]), int(phi.shape[1])
    eps, dt, c = params.epsilon, params.dt, params.c_value
    Phi = _dev(phi, device)
    fd = _dev(f_host, device)
    fid = _dev(np.where(f_host != 0, params.omega0, 0.0), device)
    denom = _dev(1.0 + c * dt + eps * dt * lam, device)
    lead = 1.0 + c * dt + dt / eps
    lib = _lib.lib()
    from .krylov import gemv_n, gemv_t
    # v = Phi^T f, u = Phi v (Phi row-major n x k == column-major k x n)
    PhiT = Phi.t().contiguous()          # k x n row-major == column-major n x k
    v = torch.empty(k, dtype=torch.float64, device=Phi.device)
    gemv_t(PhiT, n, k, fd, v)
    u = torch.empty(n, dtype=torch.float64, device=Phi.device)
    gemv_n(PhiT, n, k, v, u)
    vn, un = torch.empty_like(v), torch.empty_like(u)
    work = torch.empty(int(lib.mlb_ac_work_size(n, k, 1)), dtype=torch.float64, device=Phi.device)
    stats = torch.empty(2, dtype=torch.float64, device=Phi.device)
    converged = False
    iterations = 0
    for it in range(1, params.max_iter + 1):
        _lib.check(lib.mlb_bac_step(_lib.ptr(Phi), n, k, _lib.ptr(u), _lib.ptr(fd), _lib.ptr(fid), _lib.ptr(v),
                                    _lib.ptr(denom), lead, dt / eps, dt, _lib.ptr(vn), _lib.ptr(un),
                                    _lib.ptr(stats), _lib.ptr(work), _lib.stream_ptr()))
        num, den = stats.cpu().numpy()
        u, un = un, u
        v, vn = vn, v
        iterations = it
        if callback is not None:
            callback(it, u.cpu().numpy())
        if den <= 0:
            converged = True  # the all-zero state is a fixed point
            break
        if not np.isfinite(num):
            raise NumericalError("binary Allen-Cahn iterate degenerated")
        if num / den <= params.tolerance:
            converged = True
            break
    scores = u if return_device else u.cpu().numpy()
    return BinaryAllenCahnResult(scores=scores, iterations=iterations, converged=converged)


def predict_binary(scores):
    """+1 / -1 by sign, an exact zero counts as +1 (allencahn.py:312-314)."""
    torch = _torch()
    if isinstance(scores, torch.Tensor):
        return torch.where(scores >= 0, 1, -1).to(torch.int32)
    return np.where(np.asarray(scores) >= 0, 1, -1)


def ginzburg_landau_energy(scores, operator, labels, epsilon):
    """Diagnostic energy (allencahn.py:232-252): Dirichlet term in the eigenbasis
    (0.5 eps sum_a lambda_a |Phi^T U|_a^2) or with a dense Laplacian
    (0.5 eps sum U * (L U)), the multi-well term and the fidelity term.  The
    row sums run on the device (mlb_gl_energy_partials, fixed partition); the
    host adds the per-block partials in order."""
    torch = _torch()
    U_host = scores.cpu().numpy() if isinstance(scores, torch.Tensor) else np.asarray(scores, dtype=float)
    n, m = U_host.shape
    if labels.F.shape != (n, m):
        raise ConfigError("scores and labels disagree in shape")
    spectral = isinstance(operator, SpectralBasis)
    if spectral:
        phi = operator.vectors
        device = phi.device.index if isinstance(phi, torch.Tensor) else torch.cuda.current_device()
        Phi = _dev(phi, device)
        k = int(Phi.shape[1])
    else:
        device = torch.cuda.current_device()
        Phi, k = None, 0
    U = _dev(U_host, device)
    F = _dev(labels.F, device)
    fid = _dev(labels.fidelity, device)
    lib = _lib.lib()
    part = torch.empty(int(lib.mlb_gl_energy_work_size(max(k, 1), m)), dtype=torch.float64, device=U.device)
    nb = C.c_int(0)
    _lib.check(lib.mlb_gl_energy_partials(_lib.ptr(Phi) if Phi is not None else None, n, k, m, _lib.ptr(U),
                                          _lib.ptr(F), _lib.ptr(fid), _lib.ptr(part), C.byref(nb),
                                          _lib.stream_ptr()))
    width = k * m + 2
    rows = part[: nb.value * width].view(nb.value, width).cpu().numpy()
    tot = np.zeros(width)
    for r in rows:  # fixed block order
        tot += r
    well = tot[k * m] / (2.0 * epsilon)
    fidelity = 0.5 * tot[k * m + 1]
    if spectral:
        Cm = tot[: k * m].reshape(k, m)
        dirichlet = 0.5 * epsilon * float(np.sum(np.asarray(operator.values, dtype=float)[:, None] * Cm * Cm))
    else:
        from .krylov import dot, gemv_n
        L = _dev(np.asarray(operator, dtype=float), device)  # symmetric: row-major == column-major
        LU = torch.empty(n, dtype=torch.float64, device=U.device)
        acc = torch.empty(1, dtype=torch.float64, device=U.device)
        Ut = U.t().contiguous()
        dirichlet = 0.0
        for cidx in range(m):
            gemv_n(L, n, n, Ut[cidx], LU)
            dot(Ut[cidx], LU, acc)
            dirichlet += float(acc.item())
        dirichlet *= 0.5 * epsilon
    return dirichlet + well + fidelity
