"""Node-range sharded solvers (one large layer split by
node range over the ranks, config 4): PKSM, the outer restarted Lanczos of
power_mean_eigs and the multiclass Allen-Cahn scheme on vectors of which each
rank holds the slice [lo, hi).

Reference: krylov.py:65-71 (CGS2), :74-169 (lanczos_largest_eigs),
:172-216 (lanczos_fn_apply), :219-244 (pksm_apply); powermean.py:64-95,
:130-189; allencahn.py:172-223.

Communication per step (torch.distributed: NCCL on the GPU box, gloo in the
CPU tests), all on the stream, no host round trip inside a reduction:
  * each operator apply: the layers' grid all-reduce (dist.ShardedKernelGraph);
  * each CGS2 (inner PKSM step or outer Lanczos step): TWO all-reduces --
    [h1] (its last entry is the Lanczos alpha), then [h2 | ||w||^2] fused:
    ||w - V h2||^2 = ||w||^2 - ||h2||^2 for orthonormal V, so the norm after
    the second pass needs no third reduction.  When ||h2||^2 is not
    negligible against ||w||^2 (cancellation, e.g. near a breakdown) the
    host falls back to an exact third reduction of the corrected w;
  * each Allen-Cahn iteration: one all-reduce of Phi^T R (k x m) and one
    max-reduction of the two iterate statistics.
Every rank receives identical reduction results, so every host takes the
same decisions (convergence, restarts) and the collectives stay matched.

Vector algebra on the rank's slices: libmlb kernels on the GPU (mlb_gemv_t,
mlb_gemv_n, mlb_dot, mlb_gemm_vs, mlb_ac_rhs_partial / mlb_ac_update_from),
torch on the CPU (the gloo tests, with the oracle as the layer engine).
"""

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, ConvergenceError, NumericalError


def _torch():
    import torch
    return torch


class ShardContext:
    """The rank's node range and the reductions over the ranks.

    comm: dist.Comm or None (one rank); device: CUDA index, or None for CPU
    tensors (torch algebra; the gloo tests)."""

    def __init__(self, comm, n, lo, hi, device=None):
        torch = _torch()
        self.comm, self.n, self.lo, self.hi = comm, int(n), int(lo), int(hi)
        self.gpu = device is not None
        self.device = torch.device("cuda", int(device)) if self.gpu else torch.device("cpu")
        self._work = None

    @property
    def n_local(self):
        return self.hi - self.lo

    # -- reductions ------------------------------------------------------
    def allreduce(self, t):
        if self.comm is not None:
            self.comm.all_reduce_sum(t)
        return t

    def allmax(self, t):
        if self.comm is not None:
            self.comm.dist.all_reduce(t, op=self.comm.dist.ReduceOp.MAX, group=self.comm.group)
        return t

    # -- local algebra ---------------------------------------------------
    def tensor(self, x):
        """This rank's slice of a full-length host vector (or a local tensor as is)."""
        torch = _torch()
        if isinstance(x, torch.Tensor):
            return x.to(self.device, torch.float64)
        x = np.asarray(x, dtype=np.float64)
        if x.shape[0] == self.n and self.n != self.n_local:
            x = x[self.lo:self.hi]
        return torch.from_numpy(np.ascontiguousarray(x)).to(self.device)

    def _w(self, cols):
        torch = _torch()
        need = int(_lib.lib().mlb_krylov_work_size(self.n_local, max(cols, 1)))
        if self._work is None or self._work.numel() < need:
            self._work = torch.empty(need, dtype=torch.float64, device=self.device)
        return self._work

    def gemv_t(self, V, cols, w, out):
        """out[:cols] = V[:cols] w (local rows)."""
        if not self.gpu:
            out[:cols] = V[:cols] @ w
            return out
        _lib.check(_lib.lib().mlb_gemv_t(_lib.ptr(V), self.n_local, self.n_local, cols, _lib.ptr(w), _lib.ptr(out),
                                         _lib.ptr(self._w(cols)), _lib.stream_ptr()))
        return out

    def gemv_n(self, V, cols, c, y, scale=1.0, accumulate=False):
        """y (+)= scale V[:cols]^T c."""
        if not self.gpu:
            r = V[:cols].T @ c[:cols]
            if accumulate:
                y.add_(r, alpha=scale)
            else:
                y.copy_(r).mul_(scale)
            return y
        _lib.check(_lib.lib().mlb_gemv_n(_lib.ptr(V), self.n_local, self.n_local, cols, _lib.ptr(c), _lib.ptr(y),
                                         float(scale), int(accumulate), _lib.stream_ptr()))
        return y

    def dot(self, x, y, out):
        if not self.gpu:
            out.copy_((x * y).sum().reshape(1))
            return out
        _lib.check(_lib.lib().mlb_dot(_lib.ptr(x), _lib.ptr(y), self.n_local, _lib.ptr(out), _lib.ptr(self._w(1)),
                                      _lib.stream_ptr()))
        return out

    def gdot(self, x, y):
        """Global <x, y> (one all-reduce, host value)."""
        torch = _torch()
        t = torch.empty(1, dtype=torch.float64, device=self.device)
        self.dot(x, y, t)
        return float(self.allreduce(t).item())

    def combine(self, V, s, S, k, out):
        """out[:k] = (V[:s]^T S[:s, :k])^T: Ritz / restart vectors (local rows)."""
        torch = _torch()
        if not self.gpu:
            Sk = S[:s, :k] if isinstance(S, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(S[:s, :k]))
            out[:k] = (V[:s].T @ Sk).T
            return out
        Sd = torch.from_numpy(np.asfortranarray(np.asarray(S[:s, :k].cpu() if isinstance(S, torch.Tensor)
                                                           else S[:s, :k])).ravel(order="F")).to(self.device)
        _lib.check(_lib.lib().mlb_gemm_vs(_lib.ptr(V), self.n_local, self.n_local, s, _lib.ptr(Sd), k,
                                          _lib.ptr(out), self.n_local, _lib.stream_ptr()))
        return out

    # -- CGS2 with two reductions ----------------------------------------
    def cgs2(self, V, cols, w, buf):
        """Two-pass classical Gram-Schmidt of the local w against V[:cols]
        (krylov.py:65-71) with global projections.  Returns the host array
        [h1 (cols) | h2 (cols) | ||w_after||^2]."""
        h1, tail = buf[:cols], buf[cols:2 * cols + 1]
        self.gemv_t(V, cols, w, h1)
        self.allreduce(h1)
        self.gemv_n(V, cols, h1, w, -1.0, True)
        self.gemv_t(V, cols, w, tail[:cols])
        self.dot(w, w, tail[cols:cols + 1])          # ||w||^2 before the second update
        self.allreduce(tail)
        self.gemv_n(V, cols, tail[:cols], w, -1.0, True)
        hh = buf[:2 * cols + 1].cpu().numpy().copy()
        h2 = hh[cols:2 * cols]
        ww, hh2 = hh[2 * cols], float(h2 @ h2)
        if hh2 > 1e-8 * max(ww, 1e-300):            # cancellation: measure the corrected w exactly
            ww = self.gdot(w, w)
        else:
            ww = ww - hh2
        hh[2 * cols] = max(ww, 0.0)
        return hh


# ------------------------------------------------------------------ PKSM ----
def _converged(c, c_prev, tol, exact):
    """||y_s - y_{s-1}|| <= tol ||y_s|| on coefficient vectors (V orthonormal:
    the norms are those of the vectors), re-tested on the
    exact vectors within 1e-3 of the threshold (krylov.py:205-211)."""
    diff = c.copy()
    diff[: c.shape[0] - 1] -= c_prev
    lhs, rhs = np.linalg.norm(diff), tol * max(np.linalg.norm(c), 1e-300)
    if rhs > 0 and abs(lhs / rhs - 1.0) < 1e-3:
        lhs, rhs = exact()
    return lhs <= rhs


def sharded_lanczos_fn(ctx, apply, v, fn, krylov_dim=50, tol=1e-8):
    """f(A) v on node-sharded vectors (krylov.py:172-216); `apply(x_local)`
    returns the local rows of A x.  Returns the local rows of y."""
    torch = _torch()
    v = ctx.tensor(v)
    nl = ctx.n_local
    vv = ctx.gdot(v, v)
    if vv == 0.0:
        return torch.zeros_like(v)
    nv = math.sqrt(vv)
    dim = int(min(krylov_dim, ctx.n))
    if dim < 1:
        raise ConfigError(f"krylov_dim must be >= 1, got {krylov_dim}")
    V = torch.empty((dim, nl), dtype=torch.float64, device=ctx.device)
    V[0] = v / nv
    buf = torch.empty(2 * dim + 1, dtype=torch.float64, device=ctx.device)
    alphas, betas = np.empty(dim), np.empty(dim)
    c_prev = None
    s = 0
    while True:
        w = apply(V[s])
        hh = ctx.cgs2(V, s + 1, w, buf)
        alphas[s] = hh[s]                       # first-pass projection on V[s] (krylov.py:198)
        betas[s] = beta = math.sqrt(hh[2 * (s + 1)])
        s += 1
        T = np.diag(alphas[:s])
        if s > 1:
            T += np.diag(betas[: s - 1], 1) + np.diag(betas[: s - 1], -1)
        lam, Q = np.linalg.eigh(T)
        c = nv * (Q @ (fn(lam) * Q[0, :]))

        def exact(c=c, c_prev=c_prev, s=s):
            y = torch.zeros(nl, dtype=torch.float64, device=ctx.device)
            yp = torch.zeros_like(y)
            ctx.gemv_n(V, s, torch.from_numpy(c).to(ctx.device), y)
            ctx.gemv_n(V, s - 1, torch.from_numpy(c_prev).to(ctx.device), yp)
            d = y - yp
            return math.sqrt(ctx.gdot(d, d)), tol * max(math.sqrt(ctx.gdot(y, y)), 1e-300)

        done = c_prev is not None and _converged(c, c_prev, tol, exact)
        happy = beta <= 1e-13 * max(1.0, np.abs(alphas[:s]).max())
        if done or happy or s >= dim:
            y = torch.zeros(nl, dtype=torch.float64, device=ctx.device)
            return ctx.gemv_n(V, s, torch.from_numpy(c).to(ctx.device), y)
        c_prev = c
        V[s] = w / beta


def sharded_pksm(ctx, apply, p, v, krylov_dim=50, tol=1e-8):
    """(L_sym + delta)^p v on node-sharded vectors (krylov.py:219-244)."""
    from .krylov import power_fn
    if p == 0:
        raise ConfigError("p must be nonzero")
    return sharded_lanczos_fn(ctx, apply, v, power_fn(p), krylov_dim, tol)


# ------------------------------------------------------- outer Lanczos ------
@dataclass
class ShardedEigenResult:
    """Largest eigenpairs; `vectors` holds this rank's rows (n_local x k)."""

    values: np.ndarray
    vectors: object
    residuals: np.ndarray
    matvecs: int
    restarts: int


def _symmetry_probe(ctx, apply, name, probes=2, tol=1e-8):
    """<Ax, y> == <x, Ay> on default_rng(0) probe pairs (krylov.py:27-37);
    every rank draws the full probes and keeps its slice."""
    rng = np.random.default_rng(0)
    for _ in range(probes):
        x = ctx.tensor(rng.standard_normal(ctx.n))
        y = ctx.tensor(rng.standard_normal(ctx.n))
        ax, ay = apply(x), apply(y)
        a, b, nax2, ny2 = (ctx.gdot(ax, y), ctx.gdot(x, ay), ctx.gdot(ax, ax), ctx.gdot(y, y))
        scale = max(math.sqrt(nax2) * math.sqrt(ny2), 1e-300)
        if abs(a - b) > tol * scale:
            raise NumericalError(f"{name} fails the symmetry probe")


def sharded_lanczos_largest_eigs(ctx, apply, k, tol=1e-8, max_subspace=None, max_restarts=60, seed=0,
                                 name="operator"):
    """k largest eigenpairs of a symmetric operator on node-sharded vectors
    by thick-restart Lanczos with full CGS2 (krylov.py:74-169)."""
    from .krylov import _start_vector
    torch = _torch()
    n, nl = ctx.n, ctx.n_local
    if not 1 <= k < n:
        raise ConfigError(f"need 1 <= k < n, got k={k}, n={n}")
    _symmetry_probe(ctx, apply, name)
    if max_subspace is None:
        max_subspace = max(2 * k + 10, 20)
    ms = int(min(max_subspace, n))
    if ms < k + 2:
        ms = min(n, k + 2)
    keep = min(ms - 1, k + max(2, k // 2))
    V = torch.empty((ms, nl), dtype=torch.float64, device=ctx.device)
    Vtmp = torch.empty_like(V)
    H = np.zeros((ms, ms))
    u = ctx.tensor(_start_vector(n, seed))
    s, matvecs, beta, best = 0, 0, 0.0, None
    rng_fill = np.random.default_rng(seed + 1)
    buf = torch.empty(2 * ms + 1, dtype=torch.float64, device=ctx.device)
    for restart in range(max_restarts + 1):
        j = s
        while j < ms:
            V[j] = u
            w = apply(u)
            if w.data_ptr() == u.data_ptr():
                w = w.clone()
            matvecs += 1
            hh = ctx.cgs2(V, j + 1, w, buf)
            h = hh[: j + 1] + hh[j + 1:2 * (j + 1)]
            H[: j + 1, j] = h
            H[j, : j + 1] = h
            beta = math.sqrt(hh[2 * (j + 1)])
            j += 1
            if beta <= 1e-13 * max(1.0, np.abs(H[:j, :j]).max()):
                if j >= n:
                    break
                ud = ctx.tensor(rng_fill.standard_normal(n))
                nu = math.sqrt(ctx.cgs2(V, j, ud, buf)[2 * j])
                if nu <= 1e-13:
                    break
                u = ud / nu
                beta = 0.0
            else:
                u = w / beta
        sd = j
        theta, S = np.linalg.eigh(H[:sd, :sd])
        order = np.argsort(theta)[::-1]
        theta, S = theta[order], S[:, order]
        scale = max(abs(theta[0]), abs(theta[-1]), 1e-300)
        res = np.abs(beta * S[sd - 1, :])
        best = res[:k]
        if np.all(res[:k] <= tol * scale) or sd >= n:
            ctx.combine(V, sd, S, k, Vtmp)
            return ShardedEigenResult(values=theta[:k], vectors=Vtmp[:k].T.contiguous(), residuals=res[:k],
                                      matvecs=matvecs, restarts=restart)
        if restart == max_restarts:
            break
        ctx.combine(V, sd, S, keep, Vtmp)
        V[:keep] = Vtmp[:keep]
        H[:, :] = 0.0
        H[:keep, :keep] = np.diag(theta[:keep])
        s = keep   # the Krylov space continues from the last residual direction u
    raise ConvergenceError(
        f"Lanczos did not converge: {matvecs} matvecs, best residuals {np.array2string(best, precision=2)}",
        residuals=best)


def sharded_power_mean_eigs(ctx, layers, config, k, tol=1e-8, max_subspace=None, max_restarts=60, krylov_dim=50,
                            inner_tol=None, seed=0):
    """The k smallest eigenpairs of the power mean Laplacian M_p
    (powermean.py:130-189) on node-sharded vectors.

    layers: per layer t (ascending order), a pair of local-row operators
    (lsym_t(x) = (L_sym,t + delta) x with the configured delta, weighted_t(x) =
    D_t^-1/2 W_t D_t^-1/2 x); p < 0 uses the first, p = 1 the second.
    Returns (values ascending, this rank's rows of the eigenvectors)."""
    p = config.p
    T = len(layers)
    if p == 1:
        def apply(v):
            out = None
            for _, weighted in layers:                      # powermean.py:64-77, layer order
                r = weighted(v)
                out = r.clone() if out is None else out.add_(r)
            return out / T
        res = sharded_lanczos_largest_eigs(ctx, apply, k, tol, max_subspace, max_restarts, seed, "I - L1")
        values = np.maximum(1.0 - res.values, 0.0)
    elif p < 0:
        if config.resolved_delta <= 0:
            raise ConfigError("negative powers require a positive shift delta")
        itol = tol if inner_tol is None else inner_tol

        def apply(v):
            out = None
            for lsym, _ in layers:                          # powermean.py:80-95, layer order
                r = sharded_pksm(ctx, lsym, p, v, krylov_dim, itol)
                out = r if out is None else out.add_(r)
            return out / T
        res = sharded_lanczos_largest_eigs(ctx, apply, k, tol, max_subspace, max_restarts, seed, "Lp^p")
        if res.values.min() <= 0.0:
            raise NumericalError("power mean spectrum is not positive; cannot take the 1/p root")
        values = res.values ** (1.0 / p)
    else:
        raise ConfigError("the sharded eigensolver covers p = 1 and p < 0 (dense p > 0 does not shard)")
    return np.asarray(values), res.vectors


# ------------------------------------------------------------ Allen-Cahn ----
def sharded_allen_cahn(ctx, values, phi_local, labels_local, params, callback=None):
    """The multiclass convexity-splitting scheme (allencahn.py:172-223) with
    this rank's rows of Phi, U, F and the fidelity.  Per iteration: local
    R(U) and Phi^T R partial (mlb_ac_rhs_partial), ONE all-reduce of the
    k x m partial, the local update U <- proj(Phi (Phi^T R / denom))
    (mlb_ac_update_from) and ONE max-reduction of (max |dU|^2, max |U|^2);
    the stopping test (allencahn.py:214-221) sees global maxima, so every
    rank stops at the same iteration.  Returns (local scores, iterations,
    converged)."""
    from .allencahn import initial_scores
    torch = _torch()
    if labels_local.m < 2:
        raise ConfigError("multiclass scheme needs m >= 2")
    lam = np.asarray(values, dtype=float)
    Phi = ctx.tensor(phi_local).contiguous()
    nl, k = Phi.shape
    m = labels_local.m
    eps, dt, c = params.epsilon, params.dt, params.c_value
    dev = ctx.device
    denom = torch.from_numpy(1.0 + c * dt + eps * dt * lam).to(dev)
    U = torch.from_numpy(np.ascontiguousarray(initial_scores(labels_local))).to(dev)
    Un = torch.empty_like(U)
    F = torch.from_numpy(np.ascontiguousarray(labels_local.F, dtype=np.float64)).to(dev)
    fid = torch.from_numpy(np.ascontiguousarray(labels_local.fidelity, dtype=np.float64)).to(dev)
    PtR = torch.empty(k * m, dtype=torch.float64, device=dev)
    stats = torch.empty(2, dtype=torch.float64, device=dev)
    if ctx.gpu:
        lib = _lib.lib()
        work = torch.empty(int(lib.mlb_ac_work_size(nl, k, m)), dtype=torch.float64, device=dev)
    converged, iterations = False, 0
    for it in range(1, params.max_iter + 1):
        if ctx.gpu:
            _lib.check(lib.mlb_ac_rhs_partial(_lib.ptr(Phi), nl, k, m, _lib.ptr(U), _lib.ptr(F), _lib.ptr(fid),
                                              1.0 + c * dt, dt / (2.0 * eps), dt, _lib.ptr(PtR), _lib.ptr(work),
                                              _lib.stream_ptr()))
        else:
            R = _rhs_cpu(U, F, fid, c, dt, eps)
            PtR.copy_((Phi.T @ R).reshape(-1))
        ctx.allreduce(PtR)
        if ctx.gpu:
            _lib.check(lib.mlb_ac_update_from(_lib.ptr(Phi), nl, k, m, _lib.ptr(PtR), _lib.ptr(denom), _lib.ptr(U),
                                              _lib.ptr(Un), _lib.ptr(stats), _lib.ptr(work), _lib.stream_ptr()))
        else:
            from .allencahn import simplex_project_rows
            Vc = PtR.reshape(k, m) / denom[:, None]
            Un.copy_(torch.from_numpy(simplex_project_rows((Phi @ Vc).numpy())))
            d2 = ((Un - U) ** 2).sum(dim=1)
            u2 = (Un ** 2).sum(dim=1)
            stats.copy_(torch.stack([d2.max() if nl else torch.zeros((), dtype=torch.float64),
                                     u2.max() if nl else torch.zeros((), dtype=torch.float64)]))
        ctx.allmax(stats)
        num, den = stats.cpu().numpy()
        if den <= 0 or not np.isfinite(num):
            raise NumericalError("Allen-Cahn iterate degenerated")
        U, Un = Un, U
        iterations = it
        if callback is not None:
            callback(it, U)
        if num / den <= params.tolerance:
            converged = True
            break
    return U, iterations, converged


def _rhs_cpu(U, F, fid, c, dt, eps):
    """R = (1 + c dt) U - dt/(2 eps) T(U) - dt fid (U - F) (allencahn.py:204-210), torch CPU."""
    from .allencahn import nonlinearity_T
    TU = nonlinearity_T(U.numpy())
    import torch
    return (1.0 + c * dt) * U - (dt / (2.0 * eps)) * torch.from_numpy(TU) - dt * fid[:, None] * (U - F)
