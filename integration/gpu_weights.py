"""multilap/gpu_weights.py -- the reference-side binding a `multilap`
maintainer would add, runnable as is.

It talks to libmlb.so through its C ABI only (ctypes declarations below,
mirroring include/multilap_b200.h), and replaces the reference's hot-path
entry points with GPU ones that keep the reference's signatures, return
types and exception classes:

    multilap.fastsum.bind_points     fastsum.py:375-386  -> GpuBinding (mlb_bind)
    multilap.fastsum.fastsum_apply   fastsum.py:475-497  -> mlb_apply (W v, zero diagonal)
    multilap.fastsum.direct_apply    fastsum.py:500-553  -> mlb_direct (exact sums)
    multilap.graphs.KernelWeights    graphs.py:80-144    -> GpuKernelWeights (weights protocol
                                                            {n, matvec, materialize})

`install(multilap)` patches the package (and its re-exports).  The plan
tables (band-limited fused weights, twiddles, window polynomials) come from
paper_2007_05239_b200's plan math, which reproduces the reference's
fused_weights to 1e-13 (tests/test_oracle_golden.py); the plan parameters are
read off the reference's own FastsumPlan.  Vectors cross to the device with
torch (numpy in -> numpy out, the reference convention).
"""

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIBMLB = os.environ.get("LIBMLB", os.path.join(os.path.dirname(_HERE), "paper_2007_05239_b200", "libmlb.so"))

MLB_OK, MLB_ERR_CONFIG, MLB_ERR_NUMERICAL = 0, 1, 2


class PlanDesc(C.Structure):
    """mlb_plan_desc: all 13 fields of include/multilap_b200.h."""
    _fields_ = [("d", C.c_int), ("N", C.c_int), ("m", C.c_int), ("ng", C.c_int),
                ("bin_lo", C.c_int), ("bin_hi", C.c_int), ("win_deg", C.c_int),
                ("K0", C.c_double), ("fused_band", C.c_void_p), ("twiddle", C.c_void_p),
                ("win_coef", C.c_void_p), ("conv_kernel", C.c_void_p), ("sep_kernel", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIBMLB)
        P, I, I64, D, U = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_uint
        L.mlb_last_error.restype = C.c_char_p
        L.mlb_plan_create.argtypes = [C.POINTER(PlanDesc), I, C.POINTER(P)]
        L.mlb_plan_destroy.argtypes = [P]
        L.mlb_bind.argtypes = [P, P, I64, D, P, C.POINTER(P)]
        L.mlb_binding_destroy.argtypes = [P]
        L.mlb_apply.argtypes = [P, P, P, D, D, D, U, P]
        L.mlb_direct.argtypes = [P, I64, I, I, D, P, P, P, D, D, D, I, P]
        L.mlb_launch_count.restype = I64
        _lib = L
    return _lib


def _errors():
    from multilap import errors
    return errors


def _check(rc):
    if rc == MLB_OK:
        return
    msg = (lib().mlb_last_error() or b"").decode(errors="replace")
    errors = _errors()
    if rc == MLB_ERR_CONFIG:
        raise errors.ConfigError(msg)
    if rc == MLB_ERR_NUMERICAL:
        raise errors.NumericalError(msg)
    raise RuntimeError(f"libmlb error {rc}: {msg}")


def _torch():
    import torch
    return torch


def _dev(a):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


# ---------------------------------------------------------------- plans ----
class GpuPlan:
    """libmlb plan of a reference FastsumPlan (one per reference plan object)."""

    def __init__(self, ref_plan):
        import paper_2007_05239_b200 as mb
        ours = mb.build_plan(mb.KernelSpec(ref_plan.kernel.family, ref_plan.kernel.sigma), d=ref_plan.d,
                             N=ref_plan.N, m_nfft=ref_plan.m_nfft, eps_b=ref_plan.eps_b, p_nfft=ref_plan.p_nfft,
                             rho=ref_plan.rho)
        t = ours.device_tables("box")
        self._keep = [t["fused_band"], t["twiddle"], np.ascontiguousarray(ours.win_coef), t["conv_kernel"],
                      t["sep_kernel"]]
        desc = PlanDesc(ours.d, ours.N, ours.m_nfft, ours.n_grid, t["bin_lo"], t["bin_hi"], ours.win_deg,
                        float(ours.K0), self._keep[0].ctypes.data, self._keep[1].ctypes.data,
                        self._keep[2].ctypes.data,
                        None if self._keep[3] is None else self._keep[3].ctypes.data,
                        None if self._keep[4] is None else self._keep[4].ctypes.data)
        self.ptr = C.c_void_p()
        _check(lib().mlb_plan_create(C.byref(desc), _torch().cuda.current_device(), C.byref(self.ptr)))
        self.d, self.K0, self.ball_scale, self.eps_b = ours.d, float(ours.K0), ours.ball_scale, ours.eps_b

    def __del__(self):
        try:
            lib().mlb_plan_destroy(self.ptr)
        except Exception:
            pass


def _gpu_plan(ref_plan):
    gp = getattr(ref_plan, "_gpu_plan", None)
    if gp is None:
        gp = GpuPlan(ref_plan)
        object.__setattr__(ref_plan, "_gpu_plan", gp)
    return gp


class GpuBinding:
    """Replaces PointBinding (fastsum.py:320-330): a libmlb binding handle."""

    def __init__(self, ref_plan, points):
        from multilap import fastsum as F
        pts = F.validate_box(points, ref_plan.eps_b)        # the reference's own box check
        gp = _gpu_plan(ref_plan)
        if pts.shape[1] != gp.d:
            raise _errors().ConfigError(f"points have dimension {pts.shape[1]}, plan expects {gp.d}")
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        self.plan, self.n = gp, pts.shape[0]
        self.ptr = C.c_void_p()
        _check(lib().mlb_bind(gp.ptr, pts.ctypes.data if self.n else None, self.n, gp.ball_scale, None,
                              C.byref(self.ptr)))

    def apply(self, v):
        """W v, zero diagonal: mlb_apply with alpha = -K0, beta = 1, gamma = 0."""
        torch = _torch()
        if self.n == 0:
            return np.zeros(0)
        vd = _dev(v)
        y = torch.empty_like(vd)
        _check(lib().mlb_apply(self.ptr, C.c_void_p(vd.data_ptr()), C.c_void_p(y.data_ptr()), -self.plan.K0, 1.0,
                               0.0, 0, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return y.cpu().numpy()

    def __del__(self):
        try:
            lib().mlb_binding_destroy(self.ptr)
        except Exception:
            pass


# ------------------------------------------------------- module functions ---
def bind_points(plan, points, sort=None):
    return GpuBinding(plan, points)


def fastsum_apply(points, v, plan, binding=None):
    v = np.asarray(v, dtype=float)
    if binding is None:
        binding = GpuBinding(plan, points)
    if v.shape != (binding.n,):
        raise _errors().ConfigError("v must be a real vector matching the number of points")
    return binding.apply(v)


_FAMILY = {"gaussian": 0, "laplacian": 1}
_REF = {}   # the reference objects install() replaced


def direct_apply(points, v, kernel, block_rows=None):
    """Exact W v (zero diagonal) with one device kernel (mlb_direct)."""
    torch = _torch()
    x = np.asarray(points, dtype=float)
    v = np.asarray(v, dtype=float)
    if x.ndim != 2 or v.shape != (x.shape[0],):
        raise _errors().ConfigError("points / v shapes do not match")
    if block_rows is not None and block_rows < 1:
        raise _errors().ConfigError("block_rows must be positive")
    n, d = x.shape
    if n == 0:
        return np.zeros(0)
    Xd, vd = _dev(x), _dev(v)
    y = torch.empty_like(vd)
    _check(lib().mlb_direct(C.c_void_p(Xd.data_ptr()), n, d, _FAMILY[kernel.family], float(kernel.sigma),
                            C.c_void_p(vd.data_ptr()), None, C.c_void_p(y.data_ptr()),
                            -float(kernel.radial(np.array(0.0))), 1.0, 0.0, 0,
                            C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return y.cpu().numpy()


# ---------------------------------------------------------- weights class ---
class GpuKernelWeights:
    """The weights protocol of graphs.py:80-144 ({n, matvec, materialize};
    `points`, `kernel`, `plan` attributes) with every block's matvec on the
    GPU: a libmlb binding per component block when a plan is given, the exact
    device sums otherwise."""

    def __init__(self, points, kernel, plan=None, components=None):
        points = np.asarray(points, dtype=float)
        errors = _errors()
        if points.ndim != 2:
            raise errors.ConfigError(f"points must be a 2-d array, got {points.shape}")
        if not np.all(np.isfinite(points)):
            raise errors.ConfigError("points contain non-finite values")
        self.points, self.kernel, self.plan, self.n = points, kernel, plan, points.shape[0]
        if components is None:
            self._blocks = [np.arange(self.n)]
        else:
            components = np.asarray(components)
            if components.shape != (self.n,):
                raise errors.ConfigError("components must be one label per point")
            self._blocks = [np.flatnonzero(components == c) for c in np.unique(components)]
        if plan is not None:
            if plan.d != points.shape[1]:
                raise errors.ConfigError(f"plan dimension {plan.d} does not match points ({points.shape[1]})")
            self._bindings = [GpuBinding(plan, points[idx]) for idx in self._blocks]
        else:
            self._bindings = None

    def matvec(self, v):
        v = np.asarray(v, dtype=float)
        out = np.zeros(self.n)
        for b, idx in enumerate(self._blocks):
            if self._bindings is not None:
                out[idx] = self._bindings[b].apply(v[idx])
            else:
                out[idx] = direct_apply(self.points[idx], v[idx], self.kernel)
        return out

    def materialize(self):
        """Dense W (the reference's KernelWeights.materialize, graphs.py:131-144)."""
        return _REF["KernelWeights"].materialize(self)


def install(multilap):
    """Route the reference package's hot path through libmlb (idempotent)."""
    import multilap.datapipe as D
    import multilap.fastsum as F
    import multilap.graphs as G
    if getattr(multilap, "_b200_installed", False):
        return
    for mod in (F, multilap):
        for name, fn in (("bind_points", bind_points), ("fastsum_apply", fastsum_apply),
                         ("direct_apply", direct_apply)):
            if hasattr(mod, name):
                setattr(mod, name, fn)
    _REF["KernelWeights"] = G.KernelWeights
    for mod in (G, D, multilap):
        if hasattr(mod, "KernelWeights"):
            mod.KernelWeights = GpuKernelWeights
    multilap._b200_installed = True


def launches():
    return int(lib().mlb_launch_count())
