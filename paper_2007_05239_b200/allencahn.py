"""Multiclass Allen-Cahn classifier in the eigenbasis -- drop-in for multilap.allencahn.

One convexity-splitting iteration (allencahn.py:172-223):
    R  = (1 + c dt) U - dt/(2 eps) T(U) - dt omega (U - F)
    Vc = Phi^T R / (1 + c dt + eps dt lambda)
    U+ = proj_simplex(Phi Vc)
runs as the libmlb kernel sequence mlb_ac_step (rows of U, F, Phi streamed
once per pass; fixed-order Phi^T R reduction); the host only reads the two
maxima of the stopping rule each iteration.
"""

import ctypes as C
from dataclasses import dataclass

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
    converged = False
    iterations = 0
    for it in range(1, params.max_iter + 1):
        _lib.check(lib.mlb_ac_step(_lib.ptr(Phi), n, k, m, _lib.ptr(U), _lib.ptr(F), _lib.ptr(fid),
                                   _lib.ptr(denom), 1.0 + c * dt, dt / (2.0 * eps), dt, _lib.ptr(Un),
                                   _lib.ptr(stats), _lib.ptr(work), _lib.stream_ptr()))
        num, den = stats.cpu().numpy()
        if den <= 0 or not np.isfinite(num):
            raise NumericalError("Allen-Cahn iterate degenerated")
        U, Un = Un, U
        iterations = it
        if callback is not None:
            callback(it, U.cpu().numpy())
        if num / den <= params.tolerance:
            converged = True
            break
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
