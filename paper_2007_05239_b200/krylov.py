"""Device-resident Krylov solvers -- drop-in for multilap.krylov.

* lanczos_largest_eigs: thick-restart Lanczos (krylov.py:74-169)
* lanczos_fn_apply / pksm_apply: Lanczos f(A) v with f = lambda^p (krylov.py:172-244)

The basis V lives on the GPU (column-major: one contiguous row of a torch
(dim, n) tensor per Krylov vector); every O(n) operation -- the operator
apply, the CGS2 reorthogonalisation, norms, the final V c -- runs in
libmlb.so.  Only the O(s^2) projected problems (tridiagonal / small dense
eigh, the stopping logic) run on the host, one small device->host read per
Krylov step.  PKSM keeps the layer's vectors in its binding's cell order so
spread and gather read them coalesced.

PKSM stopping test: the reference forms y_s = |v| V_s Q f(L) Q[0,:] every
step and stops when |y_s - y_{s-1}| <= tol |y_s| (krylov.py:208-211).  With
V orthonormal that equals the same test on the coefficient vectors, so y is
formed once at the end.  Borderline steps (ratio within
1e-3 of the threshold) are re-tested on the exact device y's.
"""

import ctypes as C
import os
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, ConvergenceError, NumericalError


def _torch():
    import torch
    return torch


# ------------------------------------------------------------ device ops ---
class _Work:
    """Per-device scratch for the reduction kernels."""

    _cache = {}

    @classmethod
    def get(cls, device, cols):
        torch = _torch()
        need = int(_lib.lib().mlb_krylov_work_size(0, int(cols) + 2))
        # per (device, stream): chains on concurrent streams keep their own scratch
        key = (int(device), torch.cuda.current_stream(int(device)).cuda_stream)
        buf = cls._cache.get(key)
        if buf is None or buf.numel() < need:
            buf = torch.empty(max(need, 1 << 16), dtype=torch.float64, device=f"cuda:{device}")
            cls._cache[key] = buf
        return buf


def _sp():
    return _lib.stream_ptr()


def gemv_n(V, ld, cols, c, y, scale=1.0, accumulate=False):
    """y (=|+=) scale * V[:, :cols] c   (V column-major with leading dim ld)."""
    n = y.numel()
    _lib.check(_lib.lib().mlb_gemv_n(_lib.ptr(V), ld, n, cols, _lib.ptr(c), _lib.ptr(y), float(scale),
                                     int(accumulate), _sp()))
    return y


def gemv_t(V, ld, cols, w, h):
    n = w.numel()
    work = _Work.get(w.device.index, cols)
    _lib.check(_lib.lib().mlb_gemv_t(_lib.ptr(V), ld, n, cols, _lib.ptr(w), _lib.ptr(h), _lib.ptr(work), _sp()))
    return h


def cgs2(V, cols, w, h_out, h1_out=None, nrm2_out=None):
    """Two-pass classical Gram-Schmidt of w against V[:cols] in place (krylov.py:65-71)."""
    n = w.numel()
    work = _Work.get(w.device.index, cols)
    _lib.check(_lib.lib().mlb_cgs2(_lib.ptr(V), n, n, cols, _lib.ptr(w), _lib.ptr(h_out), _lib.ptr(h1_out),
                                   _lib.ptr(nrm2_out), _lib.ptr(work), _sp()))


def dot(x, y, out):
    work = _Work.get(x.device.index, 1)
    _lib.check(_lib.lib().mlb_dot(_lib.ptr(x), _lib.ptr(y), x.numel(), _lib.ptr(out), _lib.ptr(work), _sp()))
    return out


def axpby(a, x, b, y):
    _lib.check(_lib.lib().mlb_axpby(float(a), _lib.ptr(x), float(b), _lib.ptr(y), y.numel(), _sp()))
    return y


def hadamard(x, y, out=None):
    out = _torch().empty_like(x) if out is None else out
    _lib.check(_lib.lib().mlb_hadamard(_lib.ptr(x), _lib.ptr(y), _lib.ptr(out), x.numel(), _sp()))
    return out


def scale_by(x, y, s_dev, pw):
    _lib.check(_lib.lib().mlb_scale_by(_lib.ptr(x), _lib.ptr(y), x.numel(), _lib.ptr(s_dev), float(pw), _sp()))
    return y


def gemm_vs(V, ld, s, S_dev, k, Out, ldo):
    """Out[:k] = (V[:, :s] S[:s, :k]) column blocks; S column-major s x k on device."""
    n = ld
    _lib.check(_lib.lib().mlb_gemm_vs(_lib.ptr(V), ld, n, s, _lib.ptr(S_dev), k, _lib.ptr(Out), ldo, _sp()))
    return Out


def _to_dev(x, device):
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return x.to(device=f"cuda:{device}", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=float))).to(f"cuda:{device}")


def _host(x):
    torch = _torch()
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


# ------------------------------------------------------------- operators ---
class SymmetricOperator:
    """A symmetric linear map (krylov.py:19-37).

    `apply` keeps the reference meaning (numpy in, numpy out, any callable);
    `apply_dev` (optional) maps a CUDA fp64 tensor to a new CUDA tensor and is
    what the device solvers call -- the GPU layers provide it.
    """

    def __init__(self, n, apply, name="operator", apply_dev=None, device=None):
        self.n = n
        self.apply = apply
        self.name = name
        self._apply_dev = apply_dev
        self.device = _torch().cuda.current_device() if device is None else int(device)

    def apply_dev(self, v):
        if self._apply_dev is not None:
            return self._apply_dev(v)
        return _to_dev(self.apply(v.cpu().numpy()), v.device.index)

    def selftest_symmetry(self, rng=None, probes=2, tol=1e-8):
        """<Ax, y> == <x, Ay> on default_rng(0) probe pairs (krylov.py:27-37)."""
        rng = np.random.default_rng(0) if rng is None else rng
        for _ in range(probes):
            x = rng.standard_normal(self.n)
            y = rng.standard_normal(self.n)
            xd, yd = _to_dev(x, self.device), _to_dev(y, self.device)
            ax, ay = self.apply_dev(xd), self.apply_dev(yd)
            out = _torch().empty(4, dtype=_torch().float64, device=xd.device)
            dot(ax, yd, out[0:1])
            dot(xd, ay, out[1:2])
            dot(ax, ax, out[2:3])
            dot(yd, yd, out[3:4])
            a, b, nax2, ny2 = out.cpu().numpy()
            scale = max(np.sqrt(nax2) * np.sqrt(ny2), 1e-300)
            if abs(a - b) > tol * scale:
                raise NumericalError(f"{self.name} fails the symmetry probe")


def operator_from_layer(layer):
    from .graphs import apply_sym_laplacian, apply_sym_laplacian_dev
    torch = _torch()

    def apply_dev(v):
        y = torch.empty_like(v)
        return apply_sym_laplacian_dev(layer, v, y)

    dev = layer.weights.device if layer.on_device else None
    return SymmetricOperator(layer.n, lambda v: apply_sym_laplacian(layer, v), "sym-laplacian",
                             apply_dev=apply_dev if layer.on_device else None, device=dev)


@dataclass
class EigenResult:
    """Largest eigenpairs: values descending, vectors column-aligned (krylov.py:46-54)."""

    values: np.ndarray
    vectors: np.ndarray
    residuals: np.ndarray
    matvecs: int
    restarts: int


def _start_vector(n, seed):
    rng = np.random.default_rng(seed)                 # krylov.py:57-62
    v = np.ones(n) + 1e-2 * rng.standard_normal(n)
    return v / np.linalg.norm(v)


# ------------------------------------------------------------- Lanczos -----
def lanczos_largest_eigs(op, k, tol=1e-8, max_subspace=None, max_restarts=60, seed=0, return_device=False):
    """k largest eigenpairs of a symmetric operator via restarted Lanczos (krylov.py:74-169)."""
    torch = _torch()
    n = op.n
    if not 1 <= k < n:
        raise ConfigError(f"need 1 <= k < n, got k={k}, n={n}")
    op.selftest_symmetry()
    if max_subspace is None:
        max_subspace = max(2 * k + 10, 20)
    ms = int(min(max_subspace, n))
    if ms < k + 2:
        ms = min(n, k + 2)
    keep = min(ms - 1, k + max(2, k // 2))
    dev = f"cuda:{op.device}"
    V = torch.empty((ms, n), dtype=torch.float64, device=dev)
    Vtmp = torch.empty((ms, n), dtype=torch.float64, device=dev)
    H = np.zeros((ms, ms))
    V[0] = _to_dev(_start_vector(n, seed), op.device)
    u = V[0].clone()
    s = 0
    matvecs = 0
    rng_fill = np.random.default_rng(seed + 1)
    best = None
    hbuf = torch.empty(ms + 2, dtype=torch.float64, device=dev)
    beta = 0.0
    for restart in range(max_restarts + 1):
        j = s
        while j < ms:
            V[j] = u
            w = op.apply_dev(u)
            if w.data_ptr() == u.data_ptr():
                w = w.clone()
            matvecs += 1
            cgs2(V, j + 1, w, hbuf[: j + 1], None, hbuf[ms:ms + 1])
            hh = hbuf.cpu().numpy()
            h = hh[: j + 1]
            H[: j + 1, j] = h
            H[j, : j + 1] = h
            beta = float(np.sqrt(max(hh[ms], 0.0)))
            j += 1
            if beta <= 1e-13 * max(1.0, np.abs(H[:j, :j]).max()):
                if j >= n:
                    break
                ud = _to_dev(rng_fill.standard_normal(n), op.device)
                cgs2(V, j, ud, hbuf[:j], None, hbuf[ms:ms + 1])
                nu = float(np.sqrt(max(hbuf[ms:ms + 1].cpu().item(), 0.0)))
                if nu <= 1e-13:
                    break
                u = axpby(1.0 / nu, ud, 0.0, ud)
                beta = 0.0
            else:
                u = axpby(1.0 / beta, w, 0.0, w)
        sd = j
        theta, S = np.linalg.eigh(H[:sd, :sd])
        order = np.argsort(theta)[::-1]
        theta, S = theta[order], S[:, order]
        scale = max(abs(theta[0]), abs(theta[-1]), 1e-300)
        res = np.abs(beta * S[sd - 1, :])
        best = res[:k]
        if np.all(res[:k] <= tol * scale) or sd >= n:
            Sd = _to_dev(np.asfortranarray(S[:, :k]).ravel(order="F"), op.device)
            gemm_vs(V, n, sd, Sd, k, Vtmp, n)
            vec = Vtmp[:k].T
            vectors = vec if return_device else vec.cpu().numpy()
            return EigenResult(values=theta[:k], vectors=vectors, residuals=res[:k], matvecs=matvecs,
                               restarts=restart)
        if restart == max_restarts:
            break
        Sd = _to_dev(np.asfortranarray(S[:, :keep]).ravel(order="F"), op.device)
        gemm_vs(V, n, sd, Sd, keep, Vtmp, n)
        V[:keep] = Vtmp[:keep]
        H[:, :] = 0.0
        H[:keep, :keep] = np.diag(theta[:keep])
        s = keep
    raise ConvergenceError(
        f"Lanczos did not converge: {matvecs} matvecs, best residuals {np.array2string(best, precision=2)}",
        residuals=best)


# -------------------------------------------------- Lanczos matrix function -
class PksmStats:
    """Counts of the last solves (inner steps / matvecs), for benches."""

    steps = []

    @classmethod
    def reset(cls):
        cls.steps = []


_PINNED = {}


def _pinned_snapshots(shape, device):
    """Reused pinned host buffer for the per-step alpha / beta snapshots (a
    fresh pinned allocation per solve costs far more than the solve's reads).
    Keyed like the Krylov bases by (device, nesting level, shape): a solve
    nested inside an operator of another solve, or a solve on another device
    or thread-stream, never shares the outer solve's rows.  Reuse by the NEXT
    solve at the same level is safe: every read waits for its own step's
    event, which follows any earlier copy into the buffer on the stream."""
    torch = _torch()
    di = int(device.index if hasattr(device, "index") else device)
    key = (di, _VPOOL_DEPTH[0], tuple(shape), torch.cuda.current_stream(di).cuda_stream)
    buf = _PINNED.get(key)
    if buf is None:
        buf = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        _PINNED[key] = buf
    return buf


_VPOOL = {}


class _Depth(threading.local):
    """Nesting level of running solves (an operator may itself run a solve),
    per thread: concurrent per-layer solves (apply_Lp_power_dev) each count
    their own; the pools below are keyed by it and by the current stream."""

    def __init__(self):
        self.v = 0

    def __getitem__(self, i):
        return self.v

    def __setitem__(self, i, x):
        self.v = x


_VPOOL_DEPTH = _Depth()


def _krylov_basis(device, slot, dim, n):
    """Reused (dim, n) Krylov basis buffer number `slot` on `device`: PKSM
    solves run back to back on one stream, so a solve may overwrite the
    previous solve's basis (stream order); allocating ~100 MB per solve made
    the caching allocator release and re-allocate (device syncs)."""
    torch = _torch()
    di = int(device.index if hasattr(device, "index") else device)
    key = (di, _VPOOL_DEPTH[0], slot, torch.cuda.current_stream(di).cuda_stream)
    buf = _VPOOL.get(key)
    if buf is None or buf.numel() < dim * n:
        _VPOOL[key] = buf = torch.empty(dim * n, dtype=torch.float64, device=device)
    return buf[: dim * n].view(dim, n)


def _run_ahead():
    """Krylov steps the device may run ahead of the host's convergence test
    (MLB_PKSM_DEPTH; 1 = lockstep with the host)."""
    try:
        return max(1, int(os.environ.get("MLB_PKSM_DEPTH", "2")))
    except ValueError:
        return 2


def _converged(c, c_prev, tol, exact):
    """The PKSM stopping test on coefficient vectors (krylov.py:205-211),
    re-run on the exact device vectors when within 1e-3 of the threshold."""
    s = c.shape[0]
    diff = c.copy()
    diff[: s - 1] -= c_prev
    lhs = np.linalg.norm(diff)
    rhs = tol * max(np.linalg.norm(c), 1e-300)
    if rhs > 0 and abs(lhs / rhs - 1.0) < 1e-3:
        lhs, rhs = exact()
    return lhs <= rhs


def _exact_test(V, n, c, c_prev, tol, device):
    torch = _torch()
    s = c.shape[0]
    y = torch.zeros(n, dtype=torch.float64, device=device)
    yp = torch.zeros(n, dtype=torch.float64, device=device)
    gemv_n(V, n, s, _to_dev(c, device.index), y)
    gemv_n(V, n, s - 1, _to_dev(c_prev, device.index), yp)
    nb = torch.empty(2, dtype=torch.float64, device=device)
    d = axpby(1.0, y, -1.0, yp)
    dot(d, d, nb[0:1])
    dot(y, y, nb[1:2])
    a2, b2 = nb.cpu().numpy()
    return np.sqrt(a2), tol * max(np.sqrt(b2), 1e-300)


class _Chain:
    """Device side of one Lanczos chain: step j = matvec of V[j], CGS2 against
    V[:j+1] (alpha_j = first-pass coefficient, ||w||^2 into AB), and
    V[j+1] = w / sqrt(||w||^2) computed ON THE DEVICE, so steps can be queued
    ahead of the host's convergence test without changing any value (the
    host's 1 / sqrt is the same correctly rounded operation).

    `fused` = (binding, alpha, beta, gamma, flags): the matvec is one mlb_apply
    into a persistent w; a step is then three C-ABI calls on pointers and a
    stream resolved once per solve (per-call torch stream / pointer lookups
    cost more host time than the device spends on a step).  Otherwise
    `apply_dev(V[j])` is called."""

    def __init__(self, V, ab_row, stream, apply_dev=None, fused=None):
        torch = _torch()
        self.V, self.ab, self.apply_dev, self.fused = V, ab_row, apply_dev, fused
        self.dim, self.n = V.shape
        dev = V.device
        self.h = torch.empty(self.dim + 1, dtype=torch.float64, device=dev)
        self.w = torch.empty(self.n, dtype=torch.float64, device=dev) if fused is not None else None
        self.work = _Work.get(dev.index, self.dim)
        self.sp = C.c_void_p(stream.cuda_stream)
        self.v0 = V.data_ptr()
        self.ab0 = ab_row.data_ptr()
        self.lib = _lib.lib()

    def issue(self, j):
        lib, n, dim, sp = self.lib, self.n, self.dim, self.sp
        row = lambda k: C.c_void_p(self.v0 + 8 * n * k)  # noqa: E731
        if self.fused is not None:
            b, a, bt, g, fl = self.fused
            _lib.check(lib.mlb_apply(b, row(j), C.c_void_p(self.w.data_ptr()), a, bt, g, fl, sp))
            w = self.w
        else:
            w = self.apply_dev(self.V[j])
        wp = C.c_void_p(w.data_ptr())
        nrm = C.c_void_p(self.ab0 + 8 * (dim + j))
        # h1 of this pass lands in ab[0, :j+1]: entry j is alpha_j (earlier
        # entries are stale, the host reads each step's snapshot at column j)
        _lib.check(lib.mlb_cgs2(C.c_void_p(self.v0), n, n, j + 1, wp, C.c_void_p(self.h.data_ptr()),
                                C.c_void_p(self.ab0), nrm, C.c_void_p(self.work.data_ptr()), sp))
        if j + 1 < dim:
            _lib.check(lib.mlb_scale_by(wp, row(j + 1), n, nrm, -0.5, sp))


def lanczos_fn_apply_dev(apply_dev, n, v, fn, krylov_dim=50, tol=1e-8, out=None, out_scale=1.0,
                         accumulate=False, fused=None):
    """Device Lanczos f(A) v (see _lanczos_fn_apply_dev)."""
    _VPOOL_DEPTH[0] += 1
    try:
        return _lanczos_fn_apply_dev(apply_dev, n, v, fn, krylov_dim, tol, out, out_scale, accumulate, fused)
    finally:
        _VPOOL_DEPTH[0] -= 1


def _lanczos_fn_apply_dev(apply_dev, n, v, fn, krylov_dim=50, tol=1e-8, out=None, out_scale=1.0,
                          accumulate=False, fused=None):
    """Device Lanczos f(A) v; v is a CUDA tensor (not modified).

    Returns y (or writes out (=|+=) out_scale * y).  The device runs up to
    MLB_PKSM_DEPTH steps ahead of the host's convergence test (steps past
    the stopping point are computed and discarded; the result only uses
    V[:, :s] and T_s, so it is independent of the depth).
    """
    torch = _torch()
    if tuple(v.shape) != (n,):
        raise ConfigError("v must match the operator dimension")
    dim = int(min(krylov_dim, n))
    if dim < 1:
        raise ConfigError(f"krylov_dim must be >= 1, got {krylov_dim}")
    # AB: h1 row (alpha_j at j) | ||w_j||^2 | <v, v>; V[0] = v / sqrt(<v, v>)
    # on the device (no start-of-solve sync: <v, v> arrives with step 0)
    AB = torch.zeros(2 * dim + 1, dtype=torch.float64, device=v.device)
    vv = AB[2 * dim:2 * dim + 1]
    dot(v, v, vv)
    V = _krylov_basis(v.device, 0, dim, n)
    scale_by(v, V[0], vv, -0.5)
    ABh = _pinned_snapshots((dim, 2 * dim + 1), v.device)
    stream = torch.cuda.current_stream(v.device)
    chain = _Chain(V, AB, stream, apply_dev=apply_dev, fused=fused)
    events = [None] * dim

    def issue(j):
        chain.issue(j)
        ABh[j].copy_(AB, non_blocking=True)
        events[j] = torch.cuda.Event()
        events[j].record(stream)

    alphas = np.empty(dim)
    betas = np.empty(dim)
    depth = _run_ahead()
    issued = 0
    while issued < min(depth, dim):
        issue(issued)
        issued += 1
    c_prev = None
    s = 0
    nv = None
    while True:
        events[s].synchronize()
        snap = ABh[s].numpy()
        if nv is None:
            nv = float(np.sqrt(snap[2 * dim]))
            if nv == 0.0:  # (the queued steps ran on v / 0 and are discarded)
                if out is None:
                    return torch.zeros_like(v)
                if not accumulate:
                    out.zero_()
                return out
        alphas[s] = snap[s]
        beta = float(np.sqrt(max(snap[dim + s], 0.0)))
        betas[s] = beta
        s += 1
        c = _coeffs(alphas[None, :], betas[None, :], s, np.array([nv]), fn)[0]
        stop = False
        if c_prev is not None:
            stop = _converged(c, c_prev, tol, lambda: _exact_test(V, n, c, c_prev, tol, v.device))
        happy = beta <= 1e-13 * max(1.0, np.abs(alphas[:s]).max())
        if stop or happy or s >= dim:
            PksmStats.steps.append(s)
            cd = _to_dev(c, v.device.index)
            if out is None:
                y = torch.empty(n, dtype=torch.float64, device=v.device)
                gemv_n(V, n, s, cd, y)
                return y
            gemv_n(V, n, s, cd, out, out_scale, accumulate)
            return out
        c_prev = c
        if issued < dim:
            issue(issued)
            issued += 1


class _LayerPksm:
    """One layer's state inside the batched PKSM (same arithmetic, in the same
    order, as lanczos_fn_apply_dev on that layer alone)."""

    def __init__(self, layer, v_node, dim, hrow):
        torch = _torch()
        from .graphs import KernelWeights  # noqa: F401  (eligibility checked by the caller)
        w = layer.weights
        self.b = w._bindings[0]
        if w._isd_dev is None:
            w.set_isd(layer.isd_device(w.device))
        self.n = layer.n
        self.K0 = w.kernel.value_at_zero()
        self.a = 1.0 + layer.shift
        self.vs = torch.empty_like(v_node)
        lib = _lib.lib()
        _lib.check(lib.mlb_to_sorted(self.b.ptr, _lib.ptr(v_node), _lib.ptr(self.vs), _sp()))
        self.dim = dim
        self.V = None
        self.h = hrow  # device row: h (dim) | h1 (dim) | nrm2 ...
        self.alphas = np.empty(dim)
        self.betas = np.empty(dim)
        self.c_prev = None
        self.nv = None
        self.w = None
        self.ys = None
        self.done = False

    def apply(self, x):
        y = _torch().empty_like(x)
        _lib.check(_lib.lib().mlb_apply(self.b.ptr, _lib.ptr(x), _lib.ptr(y), self.a, -1.0, self.K0,
                                        _lib.MLB_USE_ISD | _lib.MLB_SORTED, _sp()))
        return y


def pksm_layers_dev(layers, p, v_node, out, out_scale=1.0, krylov_dim=50, tol=1e-8):
    """Lockstep multi-layer PKSM (see _pksm_layers_dev)."""
    _VPOOL_DEPTH[0] += 1
    try:
        return _pksm_layers_dev(layers, p, v_node, out, out_scale, krylov_dim, tol)
    finally:
        _VPOOL_DEPTH[0] -= 1


def _coeffs(alphas, betas, s, nv, fn):
    """c = ||v|| Q f(Lambda) Q[0, :] for a stack of tridiagonal T_s (rows of
    alphas / betas: one Lanczos chain each) -- krylov.py:200-206 -- with one
    batched eigh and one batched product (the stack's entries are independent:
    a one-chain stack gives the bitwise same c)."""
    Ta = alphas.shape[0]
    T = np.zeros((Ta, s, s))
    ix = np.arange(s)
    T[:, ix, ix] = alphas[:, :s]
    if s > 1:
        T[:, ix[:-1], ix[1:]] = betas[:, : s - 1]
        T[:, ix[1:], ix[:-1]] = betas[:, : s - 1]
    lam, Q = np.linalg.eigh(T)
    fl = np.stack([fn(lam[t]) for t in range(Ta)]) if Ta > 1 else fn(lam[0])[None, :]
    return nv[:, None] * np.matmul(Q, (fl * Q[:, 0, :])[:, :, None])[:, :, 0]


_LOCK_POOL = {}
_LOCK_GRAPHS = {}


def _graphs_enabled():
    return os.environ.get("MLB_PKSM_GRAPHS", "1") != "0"


def _lock_buffers(dev, T, dim, n):
    """Per (device, nesting level, T, dim, n): the lockstep solve's device
    buffers at FIXED addresses (AB rows, w, h, reduction scratch per layer;
    the bases come from _krylov_basis), so captured step graphs replay on any
    later solve of the same shape."""
    torch = _torch()
    key = (dev.index, _VPOOL_DEPTH[0], T, dim, n)
    P = _LOCK_POOL.get(key)
    if P is None:
        lib = _lib.lib()
        need = max(int(lib.mlb_krylov_work_size(n, dim + 2)), 1 << 16)
        ld = _ab_ld(dim)
        P = dict(AB=torch.zeros((T, ld), dtype=torch.float64, device=dev),
                 hist=torch.zeros((T, 2 * dim), dtype=torch.float64, device=dev),
                 Cc=torch.zeros((T, dim, dim), dtype=torch.float64, device=dev),
                 w=torch.empty((T, n), dtype=torch.float64, device=dev),
                 h=torch.empty((T, dim + 1), dtype=torch.float64, device=dev),
                 work=torch.empty((T, need), dtype=torch.float64, device=dev),
                 bwork=torch.empty(int(lib.mlb_cgs2_batched_work_size(T)), dtype=torch.float64, device=dev),
                 ABh=torch.empty((dim, T, ld), dtype=torch.float64, pin_memory=True),
                 streams=[torch.cuda.Stream(device=dev)
                          for _ in range(min(T, int(os.environ.get("MLB_PKSM_STREAMS", "8"))))])
        # device pointer arrays of the batched CGS2 (fixed per pool; nrm2 per step j)
        ab0 = P["AB"].data_ptr()
        rows = [ab0 + 8 * ld * t for t in range(T)]
        P["p_w"] = torch.tensor([P["w"][t].data_ptr() for t in range(T)], dtype=torch.int64, device=dev)
        P["p_h"] = torch.tensor([P["h"][t].data_ptr() for t in range(T)], dtype=torch.int64, device=dev)
        P["p_h1"] = torch.tensor(rows, dtype=torch.int64, device=dev)
        P["p_nrm"] = torch.tensor([[r + 8 * (dim + j) for r in rows] for j in range(dim)], dtype=torch.int64,
                                  device=dev)
        _LOCK_POOL[key] = P
    return P


def _ab_ld(dim):
    """Lockstep AB row: h1 (dim) | ||w||^2 (dim) | <v,v> | 4 device-coefficient stats."""
    return 2 * dim + 5


def _device_coeffs_ok(dim, T):
    """Lockstep PKSM coefficients on the device (mlb_tridiag_fn_batched):
    dim <= 64 and at least 2 chains -- one chain's host eigh is cheaper than
    the QL kernel's latency on the step's critical path (config 2's per-layer
    graphs: eigensolve 0.29 -> 0.41 s with it).  MLB_PKSM_DEVICE_COEFFS=0 /
    1 forces the host / device."""
    env = os.environ.get("MLB_PKSM_DEVICE_COEFFS")
    if env is not None:
        return dim <= 64 and env != "0"
    return dim <= 64 and T >= 2


def _issue_coeffs(P, T, j, dim, p, sp):
    """Every chain's step-j coefficients and stop statistics on the device."""
    _lib.check(_lib.lib().mlb_tridiag_fn_batched(T, C.c_void_p(P["AB"].data_ptr()), _ab_ld(dim), dim, j, float(p),
                                                 C.c_void_p(P["hist"].data_ptr()), C.c_void_p(P["Cc"].data_ptr()),
                                                 sp))


def _batched_cgs_ok(dim, n):
    return dim <= 64 and n % 2 == 0 and os.environ.get("MLB_PKSM_BATCHED_CGS", "1") != "0"


def _issue_matvec(x, t, j, P, n, sp):
    """w_t = (L_t + delta) V_t[j] (fused Laplacian, sorted order) on stream sp."""
    v0 = x.V.data_ptr()
    _lib.check(_lib.lib().mlb_apply(x.b.ptr, C.c_void_p(v0 + 8 * n * j), C.c_void_p(P["w"][t].data_ptr()), x.a,
                                    -1.0, x.K0, _lib.MLB_USE_ISD | _lib.MLB_SORTED, sp))


def _issue_cgs_batched(P, p_V, T, j, dim, n, sp):
    """CGS2 of every chain's w against its V[:j+1] in 5 launches, then
    V[j+1] = w / ||w|| (mlb_cgs2_batched: per chain bitwise the single path)."""
    _lib.check(_lib.lib().mlb_cgs2_batched(
        T, C.c_void_p(p_V.data_ptr()), n, n, j + 1, C.c_void_p(P["p_w"].data_ptr()),
        C.c_void_p(P["p_h"].data_ptr()), C.c_void_p(P["p_h1"].data_ptr()), C.c_void_p(P["p_nrm"][j].data_ptr()),
        C.c_void_p(p_V.data_ptr()) if j + 1 < dim else None, C.c_void_p(P["bwork"].data_ptr()), sp))


_MULTI_OK = {}


def _multi_matvec(st, P, dim, n, dev, stream):
    """Whether the lockstep step issues all layers' matvecs with ONE
    mlb_apply_multi per stage (many small layers of one (d, m): config 3's
    52 of 40,000 points, whose per-layer launches are latency-bound).  The
    pointer tables live in the pool; eligibility is probed once per binding
    set by an eager call (it also builds the library's per-set tables outside
    any capture).  MLB_PKSM_MULTI=0 keeps the per-layer launches."""
    if os.environ.get("MLB_PKSM_MULTI", "1") == "0" or len(st) < 2:
        return False
    bkey = tuple(int(x.b.ptr.value) for x in st)
    if len(set(bkey)) != len(bkey):   # a binding twice: its scratch grids would be shared
        return False
    torch = _torch()
    T = len(st)
    if "p_x" not in P:
        rows = [[x.V.data_ptr() + 8 * n * j for x in st] for j in range(dim)]
        P["p_x"] = torch.tensor(rows, dtype=torch.int64, device=dev)
    abg = [x.a for x in st] + [-1.0] * T + [x.K0 for x in st]
    if P.get("abg_key") != abg:
        P["abg"] = torch.tensor(abg, dtype=torch.float64, device=dev)
        P["abg_key"] = abg
    P["b_host"] = (C.c_void_p * T)(*[x.b.ptr.value for x in st])
    ok = _MULTI_OK.get(bkey)
    if ok is None:
        rc = _lib.lib().mlb_apply_multi(P["b_host"], T, C.c_void_p(P["p_x"][0].data_ptr()),
                                        C.c_void_p(P["p_w"].data_ptr()), C.c_void_p(P["abg"].data_ptr()),
                                        _lib.MLB_USE_ISD | _lib.MLB_SORTED, C.c_void_p(stream.cuda_stream))
        ok = _MULTI_OK[bkey] = rc == 0
        for x in st:   # forget the probe result when a binding dies (its address may be reused)
            weakref.finalize(x.b, _MULTI_OK.pop, bkey, None)
    return ok


def _issue_multi(P, T, j, sp):
    """w_t = (L_t + delta) V_t[j] for every chain t: mlb_apply_multi."""
    _lib.check(_lib.lib().mlb_apply_multi(P["b_host"], T, C.c_void_p(P["p_x"][j].data_ptr()),
                                          C.c_void_p(P["p_w"].data_ptr()), C.c_void_p(P["abg"].data_ptr()),
                                          _lib.MLB_USE_ISD | _lib.MLB_SORTED, sp))


def _issue_layer_step(x, t, j, P, dim, n, sp):
    """Step j of layer t's chain on stream `sp`: matvec of V[j] (fused
    Laplacian, sorted order), CGS2 against V[:j+1] (alpha_j and ||w||^2 into
    its AB row), V[j+1] = w / ||w|| on the device."""
    lib = _lib.lib()
    v0 = x.V.data_ptr()
    row = lambda k: C.c_void_p(v0 + 8 * n * k)  # noqa: E731
    w = C.c_void_p(P["w"][t].data_ptr())
    ab0 = P["AB"][t].data_ptr()
    nrm = C.c_void_p(ab0 + 8 * (dim + j))
    _lib.check(lib.mlb_apply(x.b.ptr, row(j), w, x.a, -1.0, x.K0, _lib.MLB_USE_ISD | _lib.MLB_SORTED, sp))
    _lib.check(lib.mlb_cgs2(C.c_void_p(v0), n, n, j + 1, w, C.c_void_p(P["h"][t].data_ptr()), C.c_void_p(ab0),
                            nrm, C.c_void_p(P["work"][t].data_ptr()), sp))
    if j + 1 < dim:
        _lib.check(lib.mlb_scale_by(w, row(j + 1), n, nrm, -0.5, sp))


def _pksm_layers_dev(layers, p, v_node, out, out_scale=1.0, krylov_dim=50, tol=1e-8):
    """out += out_scale * (L_t + delta)^p v for every layer t, summed into out in
    ascending layer order.  The layers' Krylov steps advance in lockstep:

    * device: step j of ALL layers is one replay of a CUDA graph captured
      once per (layer set, j) and cached across solves -- the layers' chains
      on up to 8 forked streams inside the graph, then one D2H snapshot of
      every layer's (alpha_j, ||w_j||^2) -- so a step costs one graph launch
      instead of ~3 C-ABI calls per layer; layers that already stopped keep
      iterating inside the graph (their results were taken at their stop);
    * host: up to MLB_PKSM_DEPTH steps behind the device, one batched eigh
      of every running layer's T_s and the coefficient-space stopping test
      (krylov.py:200-216; exact re-test near the threshold).
    Per layer the arithmetic and its order are those of a one-layer solve, so
    results do not depend on the layer set.  Layers must be single-binding
    fused kernel layers.  MLB_PKSM_GRAPHS=0 issues the steps eagerly."""
    torch = _torch()
    fn = power_fn(p)
    n = v_node.numel()
    dim = int(min(krylov_dim, n))
    if dim < 1:
        raise ConfigError(f"krylov_dim must be >= 1, got {krylov_dim}")
    T = len(layers)
    dev = v_node.device
    st = [_LayerPksm(layer, v_node, dim, None) for layer in layers]
    P = _lock_buffers(dev, T, dim, n)
    AB, ABh = P["AB"], P["ABh"]
    AB.zero_()
    stream = torch.cuda.current_stream(dev)
    for t, x in enumerate(st):
        vv = AB[t, 2 * dim:2 * dim + 1]
        dot(x.vs, x.vs, vv)
        x.V = _krylov_basis(dev, t, dim, n)
        scale_by(x.vs, x.V[0], vv, -0.5)
    use_graphs = _graphs_enabled()
    dev_coeffs = _device_coeffs_ok(dim, T)
    gkey = (dev.index, _VPOOL_DEPTH[0], dim, n, tuple(int(x.b.ptr.value) for x in st),
            tuple((x.a, x.K0) for x in st), tuple(x.V.data_ptr() for x in st), AB.data_ptr(),
            _batched_cgs_ok(dim, n), dev_coeffs, float(p) if dev_coeffs else None,
            os.environ.get("MLB_PKSM_MULTI", "1"))
    graphs = None
    if use_graphs:
        graphs = _LOCK_GRAPHS.get(gkey)
        if graphs is None:
            graphs = _LOCK_GRAPHS[gkey] = {}
            # the graphs bake in the bindings' device pointers: drop them when a binding dies
            for x in st:
                weakref.finalize(x.b, _LOCK_GRAPHS.pop, gkey, None)
    events = [None] * dim
    lib = _lib.lib()

    batched = _batched_cgs_ok(dim, n)
    p_V = None
    if batched:   # the bases' pointer array at a fixed address (captured graphs read it)
        vptrs = [x.V.data_ptr() for x in st]
        if "p_V" not in P:
            P["p_V"] = torch.tensor(vptrs, dtype=torch.int64, device=dev)
            P["p_V_key"] = vptrs
        elif P["p_V_key"] != vptrs:
            P["p_V"].copy_(torch.tensor(vptrs, dtype=torch.int64))
            P["p_V_key"] = vptrs
            P.pop("p_x", None)
        p_V = P["p_V"]
    multi = batched and use_graphs and _multi_matvec(st, P, dim, n, dev, stream)

    def issue(j):
        if not use_graphs:
            for t, x in enumerate(st):
                if not x.done:
                    _issue_layer_step(x, t, j, P, dim, n, C.c_void_p(stream.cuda_stream))
            if dev_coeffs:
                _issue_coeffs(P, T, j, dim, p, C.c_void_p(stream.cuda_stream))
            ABh[j].copy_(AB, non_blocking=True)
        else:
            if j not in graphs:
                if j == 0:  # kernel attributes / first-use setup outside any capture
                    torch.cuda.synchronize(dev)
                g = torch.cuda.CUDAGraph()
                cap = torch.cuda.Stream(device=dev)
                l0 = lib.mlb_launch_count()
                with torch.cuda.graph(g, stream=cap):
                    fork = torch.cuda.Event()
                    fork.record(cap)
                    ss = P["streams"]
                    for s_ in ss:
                        s_.wait_event(fork)
                    # one stream per binding: a binding's scratch grids must not be shared by
                    # concurrent chains (the same layer may appear twice in a layer set)
                    slot = {}
                    if multi:   # every layer's matvec in one launch per stage
                        _issue_multi(P, T, j, C.c_void_p(cap.cuda_stream))
                    for t, x in enumerate(st if not multi else ()):
                        s_ = ss[slot.setdefault(int(x.b.ptr.value), len(slot)) % len(ss)]
                        if batched:    # the layers' matvecs concurrently, then ONE batched CGS2
                            _issue_matvec(x, t, j, P, n, C.c_void_p(s_.cuda_stream))
                        else:
                            _issue_layer_step(x, t, j, P, dim, n, C.c_void_p(s_.cuda_stream))
                    for s_ in ss:
                        e = torch.cuda.Event()
                        e.record(s_)
                        cap.wait_event(e)
                    if batched:
                        _issue_cgs_batched(P, p_V, len(st), j, dim, n, C.c_void_p(cap.cuda_stream))
                    if dev_coeffs:
                        _issue_coeffs(P, T, j, dim, p, C.c_void_p(cap.cuda_stream))
                    ABh[j].copy_(AB, non_blocking=True)
                graphs[j] = (g, int(lib.mlb_launch_count() - l0))
            g, cnt = graphs[j]
            g.replay()
            lib.mlb_note_launches(cnt)
        events[j] = torch.cuda.Event()
        events[j].record(stream)

    if use_graphs and 0 not in graphs:
        # first solve of this layer set: step 0 eagerly once (sets kernel
        # attributes outside capture), then graphs from step 0 on
        for t, x in enumerate(st):
            _issue_layer_step(x, t, 0, P, dim, n, C.c_void_p(stream.cuda_stream))
        if dev_coeffs:
            _issue_coeffs(P, T, 0, dim, p, C.c_void_p(stream.cuda_stream))
        torch.cuda.synchronize(dev)   # (re-running step 0 from the graph recomputes the same values)
    depth = _run_ahead()
    issued = 0
    while issued < min(depth, dim):
        issue(issued)
        issued += 1
    alphas = np.zeros((T, dim))
    betas = np.zeros((T, dim))
    nv = np.full(T, np.nan)
    c_prev = [None] * T
    s = 0
    while any(not x.done for x in st):
        events[s].synchronize()
        snap = ABh[s].numpy()
        ss = s + 1
        for t, x in enumerate(st):
            if x.done or x.nv is not None:
                continue
            x.nv = float(np.sqrt(snap[t, 2 * dim]))
            nv[t] = x.nv
            if x.nv == 0.0:  # zero input: nothing to add (queued steps are discarded)
                x.done = True
                x.ys = None
        act = [t for t, x in enumerate(st) if not x.done]
        if not act:
            break
        alphas[act, s] = snap[act, s]
        betas[act, s] = np.sqrt(np.maximum(snap[act, dim + s], 0.0))
        if dev_coeffs:
            _dev_coeff_step(st, act, snap, s, dim, n, p, fn, tol, alphas, betas, nv, P, dev)
        else:
            cs = _coeffs(alphas[act], betas[act], ss, nv[act], fn)
            for c, t in zip(cs, act):
                x = st[t]
                stop = False
                if c_prev[t] is not None:
                    stop = _converged(c, c_prev[t], tol, lambda: _exact_test(x.V, n, c, c_prev[t], tol, dev))
                happy = betas[t, s] <= 1e-13 * max(1.0, np.abs(alphas[t, :ss]).max())
                if stop or happy or ss >= dim:
                    PksmStats.steps.append(ss)
                    x.ys = torch.empty(n, dtype=torch.float64, device=dev)
                    gemv_n(x.V, n, ss, _to_dev(c, dev.index), x.ys)
                    x.done = True
                else:
                    c_prev[t] = c
        s += 1
        if issued < dim and any(not x.done for x in st):
            issue(issued)
            issued += 1
    for x in st:  # ascending layer order, exactly as the sequential loop
        x.V = None
        if x.ys is None:
            continue
        if out_scale != 1.0:
            x.ys.mul_(out_scale)
        _lib.check(lib.mlb_to_node(x.b.ptr, _lib.ptr(x.ys), _lib.ptr(out), 1, _sp()))
    return out


def _check_spectrum(low, p):
    """power_fn's PSD / positivity checks (krylov.py:230-242) on a minimum eigenvalue."""
    if low < -1e-10:
        raise NumericalError(f"operator is not positive semidefinite (eigenvalue {low:.3e})")
    if p < 0 and max(low, 0.0) <= 0.0:
        raise NumericalError("zero eigenvalue encountered with a negative power; "
                             "a positive shift delta is required")


def _dev_coeff_step(st, act, snap, s, dim, n, p, fn, tol, alphas, betas, nv, P, dev):
    """Host side of one lockstep step with device coefficients: the stop test
    of krylov.py:205-216 on the per-chain statistics the device wrote
    (min eigenvalue, ||c||^2, ||c - c_prev||^2), vectorised over the running
    chains (a Python loop over 52 chains cost about as much as the device
    step); chains near the threshold are re-tested exactly on the device
    vectors, and y = V_s c_s is formed from the device's c."""
    torch = _torch()
    ss = s + 1
    Cc = P["Cc"]
    act = np.asarray(act)
    st4 = snap[act, 2 * dim + 1: 2 * dim + 5]
    low, c2, d2, status = (st4[:, k].copy() for k in range(4))
    for i in np.nonzero(status != 0)[0]:   # QL did not converge: that chain's step on the host
        t = int(act[i])
        c = _coeffs(alphas[t:t + 1], betas[t:t + 1], ss, nv[t:t + 1], fn)[0]
        Cc[t, s, :ss].copy_(_to_dev(c, dev.index))
        diff = c.copy()
        if s > 0:
            diff[:s] -= Cc[t, s - 1, :s].cpu().numpy()
        c2[i], d2[i] = float(c @ c), float(diff @ diff)
        low[i] = np.inf   # (checked by fn inside _coeffs)
    ok = status == 0
    if np.any(ok):   # the errors of the first offending chain, in layer order
        bad = ok & ((low < -1e-10) | ((p < 0) & (np.maximum(low, 0.0) <= 0.0)))
        if np.any(bad):
            _check_spectrum(float(low[np.argmax(bad)]), p)
    stop = np.zeros(len(act), dtype=bool)
    if s > 0:
        lhs = np.sqrt(d2)
        rhs = tol * np.maximum(np.sqrt(c2), 1e-300)
        stop = lhs <= rhs
        near = (rhs > 0) & (np.abs(lhs / rhs - 1.0) < 1e-3)
        for i in np.nonzero(near)[0]:
            t = int(act[i])
            a_, b_ = _exact_test(st[t].V, n, Cc[t, s, :ss], Cc[t, s - 1, :s], tol, dev)
            stop[i] = a_ <= b_
    happy = betas[act, s] <= 1e-13 * np.maximum(1.0, np.abs(alphas[act, :ss]).max(axis=1))
    done = stop | happy | (ss >= dim)
    for i in np.nonzero(done)[0]:
        x = st[int(act[i])]
        PksmStats.steps.append(ss)
        x.ys = torch.empty(n, dtype=torch.float64, device=dev)
        gemv_n(x.V, n, ss, Cc[int(act[i]), s, :ss].contiguous(), x.ys)
        x.done = True


def batchable_layers(layers):
    """True when every layer is a single-binding fused GPU kernel layer."""
    from .graphs import KernelWeights
    return all(isinstance(layer.weights, KernelWeights) and layer.weights.fused
               and layer.weights._bindings is not None and len(layer.weights._bindings) == 1
               for layer in layers)


def lanczos_fn_apply(op, v, fn, krylov_dim=50, tol=1e-8):
    """y ~= f(A) v via the Lanczos relation (krylov.py:172-216)."""
    torch = _torch()
    host = not isinstance(v, torch.Tensor)
    if host:
        v = np.asarray(v, dtype=float)
        if v.shape != (op.n,):
            raise ConfigError("v must match the operator dimension")
    vd = _to_dev(v, op.device)
    y = lanczos_fn_apply_dev(op.apply_dev, op.n, vd, fn, krylov_dim, tol)
    return y.cpu().numpy() if host else y


def power_fn(p):
    """lambda^p with the PSD / positivity checks of pksm_apply (krylov.py:230-242)."""
    def fn(lam):
        low = lam.min()
        if low < -1e-10:
            raise NumericalError(f"operator is not positive semidefinite (eigenvalue {low:.3e})")
        lam = np.maximum(lam, 0.0)
        if p < 0 and lam.min() <= 0.0:
            raise NumericalError("zero eigenvalue encountered with a negative power; "
                                 "a positive shift delta is required")
        return lam ** p
    return fn


def pksm_layer_dev(layer, p, v_node, out, out_scale=1.0, accumulate=True, krylov_dim=50, tol=1e-8):
    """out (+)= out_scale * (L_sym + delta)^p v for a GPU kernel layer.

    Runs in the layer binding's cell order when the layer has one binding
    (vectors coalesced for spread/gather), node order otherwise.
    """
    from .graphs import KernelWeights, apply_sym_laplacian_dev
    torch = _torch()
    fn = power_fn(p)
    w = layer.weights
    if isinstance(w, KernelWeights) and w.fused and len(w._bindings) == 1:
        b = w._bindings[0]
        if w._isd_dev is None:
            w.set_isd(layer.isd_device(w.device))
        lib = _lib.lib()
        vs = torch.empty_like(v_node)
        _lib.check(lib.mlb_to_sorted(b.ptr, _lib.ptr(v_node), _lib.ptr(vs), _sp()))
        K0 = w.kernel.value_at_zero()
        a = 1.0 + layer.shift
        flags = _lib.MLB_USE_ISD | _lib.MLB_SORTED

        def apply_sorted(x):
            y = torch.empty_like(x)
            _lib.check(lib.mlb_apply(b.ptr, _lib.ptr(x), _lib.ptr(y), a, -1.0, K0, flags, _sp()))
            return y

        ys = lanczos_fn_apply_dev(apply_sorted, layer.n, vs, fn, krylov_dim, tol,
                                  fused=(b.ptr, a, -1.0, K0, flags))
        if out_scale != 1.0:
            ys.mul_(out_scale)
        _lib.check(lib.mlb_to_node(b.ptr, _lib.ptr(ys), _lib.ptr(out), int(accumulate), _sp()))
        return out

    def apply_node(x):
        y = torch.empty_like(x)
        return apply_sym_laplacian_dev(layer, x, y)

    return lanczos_fn_apply_dev(apply_node, layer.n, v_node, fn, krylov_dim, tol, out=out, out_scale=out_scale,
                                accumulate=accumulate)


def pksm_apply(target, p, v, krylov_dim=50, tol=1e-8):
    """(L_{sym,delta})^p v, or A^p v for a SymmetricOperator (krylov.py:219-244)."""
    from .graphs import Layer
    torch = _torch()
    if p == 0:
        raise ConfigError("p must be nonzero")
    if isinstance(target, Layer) and target.on_device:
        host = not isinstance(v, torch.Tensor)
        if host:
            v = np.asarray(v, dtype=float)
            if v.shape != (target.n,):
                raise ConfigError("v must match the operator dimension")
        vd = _to_dev(v, target.weights.device)
        out = torch.zeros_like(vd)
        pksm_layer_dev(target, p, vd, out, 1.0, False, krylov_dim, tol)
        return out.cpu().numpy() if host else out
    op = operator_from_layer(target) if isinstance(target, Layer) else target
    return lanczos_fn_apply(op, v, power_fn(p), krylov_dim=krylov_dim, tol=tol)
