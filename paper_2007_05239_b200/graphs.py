"""Graph layers and the shifted normalized Laplacian -- drop-in for multilap.graphs.

    L_{sym,delta} v = (1 + delta) v - D^-1/2 W D^-1/2 v      (graphs.py:197-201)

Kernel weights (points + fastsum plan) are bound on the GPU once; each
Laplacian matvec is ONE fused libmlb call: spread of D^-1/2 v, pruned-DFT
convolution, gather with the (1+delta) v - D^-1/2 (.) + K0 D^-1 v epilogue
(the K(0) diagonal removal folded in).

Vectors may be numpy arrays (copied to / from the device -- the reference's
calling convention) or float64 CUDA tensors (stay on the device).
"""

import os
from dataclasses import dataclass, replace

import numpy as np

from . import _lib, fastsum
from .errors import ConfigError, FormatError, NumericalError

_SYM_TOL = 1e-12


def _torch():
    import torch
    return torch


def _is_tensor(v):
    try:
        import torch
        return isinstance(v, torch.Tensor)
    except Exception:
        return False


def _current_device():
    return _torch().cuda.current_device()


def to_device(v, device):
    """fp64 contiguous CUDA tensor view/copy of v."""
    torch = _torch()
    if isinstance(v, torch.Tensor):
        return v.to(device=f"cuda:{device}", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=float))).to(f"cuda:{device}")


class KernelWeights:
    """W_ij = K(x_i - x_j), zero diagonal, from a point cloud (graphs.py:80-144).

    With a plan every component block is bound on the device (one binding per
    block; cross-block weights are zero).  Without a plan the exact O(n^2)
    device kernel (direct.py) is used.
    """

    def __init__(self, points, kernel, plan=None, components=None, device=None, box_map=None, columns=None,
                 host_points=None):
        """`points`: (n, d) box coordinates (the reference's argument), or --
        the feature_group fast path -- a raw feature matrix (host array or
        CUDA tensor) with `columns` naming the group's columns and `box_map`
        (datapipe.BoxMap) the map into the box, applied on the device inside
        the bind; the box coordinates are then materialised on the host only
        if `.points` is read (from `host_points`, the host copy of a device
        feature matrix, when given)."""
        torch = _torch()
        self.kernel = kernel
        self.plan = plan
        self.device = _current_device() if device is None else int(device)
        self._box_map, self._columns = box_map, None if columns is None else tuple(int(c) for c in columns)
        if box_map is None and columns is None and not _is_tensor(points):
            points = np.asarray(points, dtype=float)
            if points.ndim != 2:
                raise ConfigError(f"points must be a 2-d array, got {points.shape}")
            if not np.all(np.isfinite(points)):
                raise ConfigError("points contain non-finite values")
            self._points = points
            self._src = None
        else:
            if tuple(points.shape).__len__() != 2:
                raise ConfigError(f"points must be a 2-d array, got {tuple(points.shape)}")
            self._points = None
            self._src = points          # raw features (host or device), mapped lazily
        self.n = int(points.shape[0])
        d = len(self._columns) if self._columns is not None else int(points.shape[1])
        if components is None:
            self._blocks = [np.arange(self.n)]
        else:
            components = np.asarray(components)
            if components.shape != (self.n,):
                raise ConfigError("components must be one label per point")
            self._blocks = [np.flatnonzero(components == c) for c in np.unique(components)]
        self._isd_dev = None
        if plan is not None:
            if plan.d != d:
                raise ConfigError(f"plan dimension {plan.d} does not match points ({d})")
            if self._src is None:
                self._bindings = [fastsum.bind_points(plan, self._points[idx], device=self.device,
                                                      node_ids=idx.astype(np.int32)) for idx in self._blocks]
            else:
                bm = box_map if (box_map is not None and box_map.half > 0.0) else None
                self._bindings = []
                for idx in self._blocks:
                    if len(self._blocks) == 1:
                        src = self._src
                    elif _is_tensor(self._src):
                        src = self._src[torch.from_numpy(idx).to(self._src.device)]
                    else:
                        src = self._src[idx]
                    if box_map is not None and bm is None:   # constant group: every point at the origin
                        src = np.zeros((len(idx), d))
                        cols = None
                    else:
                        cols = self._columns
                    self._bindings.append(fastsum.PointBinding(plan, src, plan.ball_scale, "box", self.device,
                                                               idx.astype(np.int32), box_map=bm, columns=cols,
                                                               validate=True))
        else:
            self._bindings = None
        if host_points is not None:
            self._src = host_points     # do not keep the device copy alive

    @property
    def points(self):
        """(n, d) box coordinates (graphs.py:89-95): the reference attribute."""
        if self._points is None:
            src = self._src.cpu().numpy() if _is_tensor(self._src) else np.asarray(self._src, dtype=float)
            if self._columns is not None:
                src = src[:, list(self._columns)]
            self._points = self._box_map(src) if self._box_map is not None else np.ascontiguousarray(src)
        return self._points

    # -- device interface ---------------------------------------------------
    @property
    def fused(self):
        """True when matvecs run through libmlb bindings (the NFFT hot path)."""
        return self._bindings is not None

    def set_isd(self, isd_dev):
        self._isd_dev = isd_dev
        if self._bindings is not None:
            for b in self._bindings:
                _lib.check(_lib.lib().mlb_binding_set_isd(b.ptr, _lib.ptr(isd_dev), _lib.stream_ptr()))

    def apply_dev(self, v, y, alpha, beta, gamma, flags=0):
        """y (=|+=) alpha v + s (beta W~(s v) + gamma s v) on device tensors (node order)."""
        if self._bindings is not None:
            for b in self._bindings:
                fastsum.apply_binding(b, v, y, alpha, beta, gamma, flags)
            return y
        from .direct import direct_apply_dev
        s = self._isd_dev if flags & _lib.MLB_USE_ISD else None
        direct_apply_dev(self, v, y, alpha, beta, gamma, s, bool(flags & _lib.MLB_ACCUMULATE))
        return y

    # -- weights protocol (graphs.py:119-144) ---------------------------------
    def matvec(self, v):
        torch = _torch()
        host = not _is_tensor(v)
        vd = to_device(v, self.device)
        if tuple(vd.shape) != (self.n,):
            raise ConfigError("v must be a vector matching the number of points")
        y = torch.empty_like(vd)
        if self.n:
            self.apply_dev(vd, y, -self.kernel.value_at_zero(), 1.0, 0.0, 0)
        return y.cpu().numpy() if host else y

    def materialize(self):
        W = np.zeros((self.n, self.n))
        for idx in self._blocks:
            pts = self.points[idx]
            sq = np.sum(pts ** 2, axis=1)
            d2 = np.maximum(sq[:, None] + sq[None, :] - 2.0 * pts @ pts.T, 0.0)
            blk = self.kernel.of_sqdist(d2)
            np.fill_diagonal(blk, 0.0)
            W[np.ix_(idx, idx)] = blk
        return W


class DenseWeights:
    """Explicit symmetric weights (graphs.py:27-50); matvec on the device GEMV."""

    def __init__(self, W, device=None):
        W = np.asarray(W, dtype=float)
        if W.ndim != 2 or W.shape[0] != W.shape[1]:
            raise ConfigError(f"weight matrix must be square, got {W.shape}")
        if not np.all(np.isfinite(W)):
            raise ConfigError("weight matrix contains non-finite entries")
        scale = max(1.0, np.abs(W).max(initial=0.0))
        if np.abs(W - W.T).max(initial=0.0) > _SYM_TOL * scale:
            raise ConfigError("weight matrix is not symmetric")
        if W.min(initial=0.0) < 0:
            raise ConfigError("weight matrix has negative entries")
        if np.abs(np.diag(W)).max(initial=0.0) > 0:
            raise ConfigError("weight matrix must have a zero diagonal")
        self.W = W
        self.n = W.shape[0]
        self.device = _current_device() if device is None else int(device)
        self._Wd = None

    def _dev(self):
        if self._Wd is None:
            self._Wd = to_device(self.W, self.device)  # symmetric: row-major == column-major
        return self._Wd

    def matvec(self, v):
        from .krylov import gemv_n
        host = not _is_tensor(v)
        vd = to_device(v, self.device)
        y = _torch().empty_like(vd)
        if self.n:
            gemv_n(self._dev(), self.n, self.n, vd, y)
        return y.cpu().numpy() if host else y

    def materialize(self):
        return self.W.copy()


class SparseWeights:
    """CSR weights (graphs.py:53-77).  Not on the NFFT path: kept host-side for
    API compatibility (edge-list graphs have no kernel structure to exploit)."""

    def __init__(self, W):
        import scipy.sparse as sp
        W = sp.csr_array(W, dtype=float)
        if W.shape[0] != W.shape[1]:
            raise ConfigError(f"weight matrix must be square, got {W.shape}")
        if W.nnz and not np.all(np.isfinite(W.data)):
            raise ConfigError("weight matrix contains non-finite entries")
        scale = max(1.0, np.abs(W.data).max(initial=0.0) if W.nnz else 0.0)
        asym = W - W.T
        if asym.nnz and np.abs(asym.data).max() > _SYM_TOL * scale:
            raise ConfigError("weight matrix is not symmetric")
        if W.nnz and W.data.min() < 0:
            raise ConfigError("weight matrix has negative entries")
        if np.abs(W.diagonal()).max(initial=0.0) > 0:
            raise ConfigError("weight matrix must have a zero diagonal")
        self.W = W
        self.n = W.shape[0]

    def matvec(self, v):
        if _is_tensor(v):
            return to_device(self.W @ v.cpu().numpy(), v.device.index)
        return self.W @ np.asarray(v, dtype=float)

    def materialize(self):
        return self.W.toarray()


@dataclass(frozen=True)
class Layer:
    """One graph layer: weights, cached degrees, diagonal shift (graphs.py:147-165)."""

    weights: object
    degrees: np.ndarray
    shift: float = 0.0

    @property
    def n(self):
        return self.weights.n

    @property
    def inv_sqrt_degrees(self):
        isd = self.__dict__.get("_isd")
        if isd is None:
            isd = 1.0 / np.sqrt(self.degrees)
            self.__dict__["_isd"] = isd
        return isd

    def isd_device(self, device):
        key = ("_isd_dev", int(device))
        t = self.__dict__.get(key)
        if t is None:
            t = to_device(self.inv_sqrt_degrees, device)
            self.__dict__[key] = t
        return t

    @property
    def on_device(self):
        return isinstance(self.weights, (KernelWeights, DenseWeights))


def build_layer(weights, shift=0.0):
    """Degrees by one matvec on ones; reject degree <= 1e-300 (graphs.py:168-183)."""
    if shift < 0:
        raise ConfigError(f"shift must be nonnegative, got {shift}")
    degrees = np.asarray(_as_host(weights.matvec(np.ones(weights.n))), dtype=float)
    bad = np.flatnonzero(degrees <= 1e-300)
    if bad.size:
        raise NumericalError(f"node {bad[0]} has zero degree; the normalized Laplacian is undefined")
    layer = Layer(weights=weights, degrees=degrees, shift=float(shift))
    if isinstance(weights, KernelWeights):
        weights.set_isd(layer.isd_device(weights.device))
    return layer


def _as_host(x):
    return x.cpu().numpy() if _is_tensor(x) else x


def with_shift(layer, shift):
    if shift < 0:
        raise ConfigError(f"shift must be nonnegative, got {shift}")
    new = replace(layer, shift=float(shift))
    for k, v in layer.__dict__.items():  # share cached isd
        if isinstance(k, tuple) or k == "_isd":
            new.__dict__[k] = v
    return new


def apply_weight(layer, v):
    return layer.weights.matvec(v if _is_tensor(v) else np.asarray(v, dtype=float))


def apply_sym_laplacian_dev(layer, v, y, accumulate=False, scale=1.0):
    """Device form: y (=|+=) scale * L_{sym,delta} v on CUDA tensors."""
    w = layer.weights
    flags = _lib.MLB_ACCUMULATE if accumulate else 0
    if isinstance(w, KernelWeights):
        if w._isd_dev is None:
            w.set_isd(layer.isd_device(w.device))
        K0 = w.kernel.value_at_zero()
        w.apply_dev(v, y, scale * (1.0 + layer.shift), -scale, scale * K0, flags | _lib.MLB_USE_ISD)
        return y
    from .krylov import axpby, hadamard
    isd = layer.isd_device(v.device.index)
    t = hadamard(isd, v)
    Wt = w.matvec(t)
    Wt = to_device(Wt, v.device.index)
    r = hadamard(isd, Wt)
    # y = scale*((1+shift) v - r) (+ y)
    if accumulate:
        axpby(scale * (1.0 + layer.shift), v, 1.0, y)
    else:
        y.copy_(v).mul_(scale * (1.0 + layer.shift))
    axpby(-scale, r, 1.0, y)
    return y


def apply_sym_laplacian(layer, v):
    """(1 + shift) v - D^-1/2 W D^-1/2 v (graphs.py:197-201)."""
    if not layer.on_device:
        v = np.asarray(_as_host(v), dtype=float)
        isd = layer.inv_sqrt_degrees
        return (1.0 + layer.shift) * v - isd * np.asarray(_as_host(layer.weights.matvec(isd * v)))
    torch = _torch()
    dev = layer.weights.device
    if _is_tensor(v) and not v.is_cuda:
        # host tensor (e.g. pinned): async copy in, compute, copy back to host
        vd = v.to(device=f"cuda:{dev}", dtype=torch.float64, non_blocking=True)
        if tuple(vd.shape) != (layer.n,):
            raise ConfigError("v must match the layer size")
        y = torch.empty_like(vd)
        apply_sym_laplacian_dev(layer, vd, y)
        out = torch.empty(y.shape, dtype=torch.float64, pin_memory=v.is_pinned())
        out.copy_(y)
        return out
    host = not _is_tensor(v)
    vd = to_device(v, dev)
    if tuple(vd.shape) != (layer.n,):
        raise ConfigError("v must match the layer size")
    y = torch.empty_like(vd)
    apply_sym_laplacian_dev(layer, vd, y)
    return y.cpu().numpy() if host else y


def materialize_sym_laplacian(layer):
    W = layer.weights.materialize()
    isd = layer.inv_sqrt_degrees
    L = -(isd[:, None] * W * isd[None, :])
    L[np.diag_indices_from(L)] += 1.0 + layer.shift
    return L


@dataclass(frozen=True)
class MultilayerGraph:
    """Layers over one node set (graphs.py:213-238)."""

    layers: tuple

    def __post_init__(self):
        if not self.layers:
            raise ConfigError("a multilayer graph needs at least one layer")
        sizes = {layer.n for layer in self.layers}
        if len(sizes) != 1:
            raise ConfigError(f"layers disagree on node count: {sorted(sizes)}")

    @property
    def n(self):
        return self.layers[0].n

    @property
    def T(self):
        return len(self.layers)

    def with_shift(self, shift):
        return MultilayerGraph(tuple(with_shift(s, shift) for s in self.layers))

    def subgraph(self, layer_indices):
        return MultilayerGraph(tuple(self.layers[i] for i in layer_indices))


def _fills_sms(layer):
    """Do the layer's spread / gather run one CTA per SM for a whole wave?"""
    plan = getattr(layer.weights, "plan", None)
    return plan is not None and plan.d == 3 and plan.m_nfft >= 5


def _layer_cost(layer):
    """Relative cost of one L_sym apply of a layer: n (2m+1)^d for NFFT layers."""
    w = layer.weights
    plan = getattr(w, "plan", None)
    if plan is not None:
        return layer.n * (2 * plan.m_nfft + 1) ** plan.d
    return layer.n


class LaplacianBatch:
    """Every layer's normalized Laplacian applied to one vector: the
    independent layers run on their own CUDA streams (fork / join on the
    caller's stream), each replayed from its own captured CUDA graph (one
    launch per layer instead of ~8).  Host input: one pinned host->device
    copy of v; each layer's result is copied to pinned host memory on its own
    stream as soon as that layer finishes.

        batch = LaplacianBatch(graph)
        Y = batch.apply(v)            # (T, n) host results; v host or device
    """

    def __init__(self, graph, use_graph=True):
        torch = _torch()
        if not all(layer.on_device for layer in graph.layers):
            raise ConfigError("LaplacianBatch needs device-resident layers")
        self.graph = graph
        self.device = graph.layers[0].weights.device
        self.n, self.T = graph.n, graph.T
        dev = torch.device("cuda", self.device)
        with torch.cuda.device(dev):
            self._v = torch.empty(self.n, dtype=torch.float64, device=dev)
            self._y = torch.empty((self.T, self.n), dtype=torch.float64, device=dev)
            # the costliest layer (the step's critical path) gets the highest
            # stream priority; cheaper layers fill the SMs it leaves idle
            cost = [_layer_cost(layer) for layer in graph.layers]
            # Stream priorities.  Results that stay on the device (`_run()`,
            # `apply_dev`): the costliest layer -- the step's critical path -- first
            # in line for free SMs.  Results copied to the host (`apply` with host
            # buffers, `apply_many`): when the costliest layer's kernels hold every
            # SM for their whole run (d = 3, m >= 5: one CTA per SM, one wave) the
            # CHEAP layer gets the priority instead, so its result -- and its
            # device->host copy -- comes first and overlaps the long layer
            # (config 4, same box: device step 3.08 ms with the costly priority vs
            # 3.12; streamed e2e 5.5 -> 5.7e9, synchronous 2.69 -> 3.29e9 with the
            # cheap one).  Every step issues the layers cheapest first (`_order`;
            # apply_many's copy-out stream then gets results in finishing order).
            # MLB_PRIO_LAYER=costly / cheap forces one rule for both.
            costly = max(range(len(cost)), key=lambda i: cost[i])
            cheap = min(range(len(cost)), key=lambda i: cost[i])
            pl = os.environ.get("MLB_PRIO_LAYER", "auto")
            top_dev = cheap if pl == "cheap" else costly
            top_host = cheap if (pl == "cheap" or (pl == "auto" and _fills_sms(graph.layers[costly]))) else costly
            self._order = sorted(range(len(cost)), key=lambda i: cost[i])
            prio = os.environ.get("MLB_NO_STREAM_PRIORITY") is None
            hi = int(os.environ.get("MLB_STREAM_PRIORITY", "-1"))  # torch range on B200: 0 (low) .. -3 (high)

            def stream_set(top):
                # one stream per weights object: a binding's scratch grids must not be
                # shared by concurrent layers (a graph may hold the same weights twice)
                by_w, out = {}, []
                for i, layer in enumerate(graph.layers):
                    key = id(layer.weights)
                    if key not in by_w:
                        by_w[key] = torch.cuda.Stream(device=dev, priority=(hi if (prio and i == top) else 0))
                    out.append(by_w[key])
                return out

            self._streams = stream_set(top_host)
            self._streams_dev = self._streams if top_dev == top_host else stream_set(top_dev)
            self._fork = torch.cuda.Event()
            self._joins = [torch.cuda.Event() for _ in graph.layers]
        self._pin_in = None
        self._use_graph = use_graph
        self._graphs = None
        self._graph_launches = []
        self._full = {}   # (host src, host out) pointers -> whole-step graph
        self._seen = {}

    def _capture(self):
        torch = _torch()
        for t, layer in enumerate(self.graph.layers):  # warm-up: kernel attributes, D^-1/2
            apply_sym_laplacian_dev(layer, self._v, self._y[t])
        torch.cuda.synchronize(self.device)
        def capture(streams):
            graphs, counts = [], []
            for t, layer in enumerate(self.graph.layers):
                l0 = _lib.lib().mlb_launch_count()
                g = torch.cuda.CUDAGraph()
                # (a captured kernel keeps the priority of its capture stream)
                with torch.cuda.graph(g, stream=streams[t]):
                    apply_sym_laplacian_dev(layer, self._v, self._y[t])
                counts.append(int(_lib.lib().mlb_launch_count() - l0))
                graphs.append(g)
            return graphs, counts

        self._graphs, self._graph_launches = capture(self._streams)
        self._graphs_dev = (self._graphs if self._streams_dev is self._streams
                            else capture(self._streams_dev)[0])
        torch.cuda.synchronize(self.device)

    def _layer(self, t, dev=False):
        if self._use_graph:
            (self._graphs_dev if dev else self._graphs)[t].replay()
            _lib.lib().mlb_note_launches(self._graph_launches[t])
        else:
            apply_sym_laplacian_dev(self.graph.layers[t], self._v, self._y[t])

    def _run(self, out=None):
        """Y = L_t v for every layer on the caller's stream (device buffers);
        with `out` (pinned (T, n)) each layer's row is copied out on its stream."""
        torch = _torch()
        if self._use_graph and self._graphs is None:
            self._capture()
        main = torch.cuda.current_stream(self.device)
        self._fork.record(main)
        streams = self._streams if out is not None else self._streams_dev
        for t in self._order:   # cheapest layer issued first
            s, j = streams[t], self._joins[t]
            s.wait_event(self._fork)
            with torch.cuda.stream(s):
                self._layer(t, dev=out is None)
                if out is not None:
                    out[t].copy_(self._y[t], non_blocking=True)
            j.record(s)
        for j in self._joins:
            main.wait_event(j)

    def apply_dev(self, v):
        """(T, n) device tensor of L_t v (a view of the batch's buffer)."""
        self._v.copy_(v)
        self._run()
        return self._y

    def apply(self, v, out=None):
        """(T, n) results for a host (numpy / pinned tensor) or device vector v;
        `out`: optional pinned (T, n) float64 tensor to receive them (no allocation)."""
        torch = _torch()
        if _is_tensor(v) and v.is_cuda:
            return self.apply_dev(v).clone()
        if _is_tensor(v) and v.is_pinned() and v.dtype == torch.float64 and v.is_contiguous():
            src = v
        else:
            if self._pin_in is None:
                self._pin_in = torch.empty(self.n, dtype=torch.float64, pin_memory=True)
            self._pin_in.copy_(torch.as_tensor(np.asarray(v, dtype=float)) if not _is_tensor(v) else v)
            src = self._pin_in
        if tuple(src.shape) != (self.n,):
            raise ConfigError("v must match the graph size")
        if out is None:
            out = torch.empty((self.T, self.n), dtype=torch.float64, pin_memory=True)
        elif not (_is_tensor(out) and out.is_pinned() and out.dtype == torch.float64
                  and tuple(out.shape) == (self.T, self.n) and out.is_contiguous()):
            raise ConfigError("out must be a contiguous pinned float64 tensor of shape (T, n)")
        main = torch.cuda.current_stream(self.device)
        key = (src.data_ptr(), out.data_ptr())
        if self._use_graph and key in self._full:
            # persistent host buffers: the whole step (H2D, every layer, D2H)
            # is one captured graph
            g, cnt = self._full[key]
            g.replay()
            _lib.lib().mlb_note_launches(cnt)
        elif self._use_graph and self._seen.get(key, 0) >= 1 and len(self._full) < 4:
            self._run(out)  # (graphs of the layers exist after the first call)
            torch.cuda.synchronize(self.device)
            l0 = _lib.lib().mlb_launch_count()
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(device=self.device)
            with torch.cuda.graph(g, stream=cap):
                self._v.copy_(src, non_blocking=True)
                self._step_direct(cap, out)
            self._full[key] = (g, int(_lib.lib().mlb_launch_count() - l0))
            g.replay()
            _lib.lib().mlb_note_launches(self._full[key][1])
        else:
            self._seen[key] = self._seen.get(key, 0) + 1
            self._v.copy_(src, non_blocking=True)
            self._run(out)
        main.synchronize()
        return out.numpy() if not _is_tensor(v) else out

    def _ensure_stream_buffers(self):
        """Second device buffer set + its layer graphs, and per-layer copy-out
        streams, for the double-buffered `apply_many` pipeline."""
        torch = _torch()
        if getattr(self, "_vb", None) is not None:
            return
        if self._use_graph and self._graphs is None:
            self._capture()
        dev = torch.device("cuda", self.device)
        with torch.cuda.device(dev):
            v2 = torch.empty_like(self._v)
            y2 = torch.empty_like(self._y)
            # one copy-out stream (MLB_COUT=layer: one per layer): device->host
            # copies queue in finishing order, so the D2H engine never idles
            # behind a layer still computing while another's result waits
            if os.environ.get("MLB_COUT", "one") == "layer":
                self._couts = [torch.cuda.Stream(device=dev) for _ in self.graph.layers]
            else:
                self._couts = [torch.cuda.Stream(device=dev)] * len(self.graph.layers)
            self._cin = torch.cuda.Stream(device=dev)
        graphs2 = None
        if self._use_graph:
            for t, layer in enumerate(self.graph.layers):  # warm-up on the new buffers
                apply_sym_laplacian_dev(layer, v2, y2[t])
            torch.cuda.synchronize(self.device)
            graphs2 = []
            for t, layer in enumerate(self.graph.layers):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self._streams[t]):
                    apply_sym_laplacian_dev(layer, v2, y2[t])
                graphs2.append(g)
            torch.cuda.synchronize(self.device)
        self._vb, self._yb = [self._v, v2], [self._y, y2]
        self._graphs_b = [self._graphs, graphs2]

    def apply_many(self, V, out=None):
        """(k, T, n): every layer's L_sym of k host vectors (rows of V), streamed.

        Vector i+1's host->device copy and vector i-1's device->host copies
        run on copy streams while vector i computes (two device buffer sets,
        one captured graph per layer and buffer), so at steady state a
        vector costs max(H2D, compute, D2H) instead of their sum.  V: pinned
        (k, n) float64 tensor or array (staged once into pinned memory);
        `out`: optional pinned (k, T, n) float64 tensor.  Returns after the
        last result has landed in host memory.
        """
        torch = _torch()
        if _is_tensor(V) and V.is_pinned() and V.dtype == torch.float64 and V.is_contiguous() and V.dim() == 2:
            src = V
        else:
            arr = V.cpu().numpy() if _is_tensor(V) else np.asarray(V, dtype=float)
            if arr.ndim != 2:
                raise ConfigError("V must be a (k, n) matrix of vectors")
            src = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).pin_memory()
        k = int(src.shape[0])
        if tuple(src.shape) != (k, self.n):
            raise ConfigError("V must have one row of length n per vector")
        if out is None:
            out = torch.empty((k, self.T, self.n), dtype=torch.float64, pin_memory=True)
        elif not (_is_tensor(out) and out.is_pinned() and out.dtype == torch.float64
                  and tuple(out.shape) == (k, self.T, self.n) and out.is_contiguous()):
            raise ConfigError("out must be a contiguous pinned float64 tensor of shape (k, T, n)")
        self._ensure_stream_buffers()
        T = self.T
        main = torch.cuda.current_stream(self.device)
        start = torch.cuda.Event()
        start.record(main)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [[torch.cuda.Event() for _ in range(T)] for _ in range(2)]
        ev_out = [[torch.cuda.Event() for _ in range(T)] for _ in range(2)]
        self._cin.wait_event(start)
        for s in self._streams + self._couts:
            s.wait_event(start)
        for i in range(k):
            b = i & 1
            if i >= 2:  # buffer b's input is free once vector i-2's layers have read it
                for t in range(T):
                    self._cin.wait_event(ev_done[b][t])
            with torch.cuda.stream(self._cin):
                self._vb[b].copy_(src[i], non_blocking=True)
            ev_in[b].record(self._cin)
            for t in self._order:
                s = self._streams[t]
                s.wait_event(ev_in[b])
                if i >= 2:  # buffer b's output row is free once vector i-2's copy-out is done
                    s.wait_event(ev_out[b][t])
                with torch.cuda.stream(s):
                    if self._use_graph:
                        self._graphs_b[b][t].replay()
                        _lib.lib().mlb_note_launches(self._graph_launches[t])
                    else:
                        apply_sym_laplacian_dev(self.graph.layers[t], self._vb[b], self._yb[b][t])
                ev_done[b][t].record(s)
                co = self._couts[t]
                co.wait_event(ev_done[b][t])
                with torch.cuda.stream(co):
                    out[i, t].copy_(self._yb[b][t], non_blocking=True)
                ev_out[b][t].record(co)
        for s in list(dict.fromkeys(self._couts + self._streams + [self._cin])):
            main.wait_stream(s)
        main.synchronize()
        return out

    def _step_direct(self, main, out):
        """Kernel-by-kernel step with per-layer D2H (for whole-step capture)."""
        torch = _torch()
        self._fork.record(main)
        for t in self._order:   # cheapest layer issued first
            layer, s, j = self.graph.layers[t], self._streams[t], self._joins[t]
            s.wait_event(self._fork)
            with torch.cuda.stream(s):
                apply_sym_laplacian_dev(layer, self._v, self._y[t])
                out[t].copy_(self._y[t], non_blocking=True)
            j.record(s)
        for j in self._joins:
            main.wait_event(j)


def apply_sym_laplacians(graph, v, use_graph=True):
    """(T, n): every layer's L_{sym} applied to v (host or device vector)."""
    if not all(layer.on_device for layer in graph.layers):
        return np.stack([apply_sym_laplacian(layer, v) for layer in graph.layers])
    cache = graph.__dict__.setdefault("_batch_cache", {})
    key = bool(use_graph)
    if key not in cache:
        cache[key] = LaplacianBatch(graph, use_graph=use_graph)
    return cache[key].apply(v)


def load_edge_list(path, n=None):
    """`i j w` edge list -> SparseWeights (graphs.py:241-279)."""
    import scipy.sparse as sp
    rows, cols, vals = [], [], []
    with open(path) as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            parts = line.split()
            if len(parts) != 3:
                raise FormatError(f"{path}:{lineno}: expected 'i j w', got {raw.strip()!r}")
            try:
                i, j, w = int(parts[0]), int(parts[1]), float(parts[2])
            except ValueError as exc:
                raise FormatError(f"{path}:{lineno}: {exc}") from exc
            if i < 0 or j < 0:
                raise FormatError(f"{path}:{lineno}: node ids must be >= 0")
            if not np.isfinite(w) or w < 0:
                raise FormatError(f"{path}:{lineno}: weight must be finite and >= 0")
            if i != j:
                rows.append(i)
                cols.append(j)
                vals.append(w)
    if n is None:
        if not rows:
            raise FormatError(f"{path}: empty edge list and no node count given")
        n = max(max(rows), max(cols)) + 1
    elif rows and max(max(rows), max(cols)) >= n:
        raise FormatError(f"{path}: node id exceeds declared node count {n}")
    W = sp.coo_array((vals, (rows, cols)), shape=(n, n)).tocsr()
    return SparseWeights(W.maximum(W.T))
