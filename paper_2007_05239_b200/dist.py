"""Multi-GPU partitioning of the NFFT Laplacian path.

Two partitionings, one process per GPU, torch.distributed for the plumbing
(NCCL over NVLink on the B200 box, gloo in the CPU tests):

1. Layer round-robin -- `LayerParallelGraph`.  Layers are independent until
   the layer sum of apply_Lp_power (powermean.py:80-95) / apply_one_minus_L1
   (powermean.py:64-77); rank r owns layers t = r, r+W, ...  Each operator
   apply gathers the per-layer results and every rank sums them in layer
   order, so all ranks hold bitwise-identical vectors and the outer Lanczos
   runs replicated with no further communication.

2. Node-range sharding of one large layer -- `ShardedLayer`.  Spreading is
   additive over point subsets: each rank spreads its node range into a
   private grid, the grids are summed over the ranks (all-reduce of the
   active sub-box only), each rank convolves redundantly and gathers its own
   nodes.  Krylov vectors are sharded by the same ranges; dot products are
   all-reduced (`sharded_pksm`).

The per-rank compute is an `engine` (spread / convolve / gather on the
local points): `BindingEngine` runs libmlb on the GPU; the CPU tests plug in
an engine built from the numpy oracle, which is how the partitioning logic
is verified with gloo at world_size 2 without GPUs.
"""

import ctypes
import math
import os

import numpy as np

from . import _lib
from .errors import ConfigError, NumericalError


def _torch():
    import torch
    return torch


# ------------------------------------------------------------------ comm ----
class Comm:
    """Thin wrapper over a torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_reduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def all_gather(self, t):
        out = [_torch().empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return out

    def ordered_sum(self, t):
        """Sum over ranks in rank order (deterministic, unlike a tree all-reduce)."""
        parts = self.all_gather(t)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        t.copy_(acc)
        return t


def shard_range(n, rank, world):
    """Contiguous node range [lo, hi) of `rank` (balanced)."""
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return lo, hi


# ------------------------------------------------ 1. layer round-robin ------
class LayerParallelGraph:
    """A MultilayerGraph whose layers are owned round-robin by the ranks.

    `local_layers[t]` is this rank's Layer for global layer t (None if owned
    elsewhere).  `pksm(layer, p, v)` / `weighted(layer, v)` compute one
    layer's contribution; by default the GPU ones.
    """

    def __init__(self, T, n, local_layers, comm, pksm=None, weighted=None):
        self.T, self.n, self.comm = T, n, comm
        self.local_layers = local_layers
        self._pksm = pksm
        self._weighted = weighted

    def owner(self, t):
        return t % self.comm.world

    def _layer_sum(self, contrib, v):
        """(1/T) sum_t contrib(layer_t, v), summed in layer order on every rank."""
        torch = _torch()
        mine = [t for t in range(self.T) if self.owner(t) == self.comm.rank]
        slots = int(math.ceil(self.T / self.comm.world))
        buf = torch.zeros((slots, self.n), dtype=torch.float64, device=v.device)
        for i, t in enumerate(mine):
            buf[i] = contrib(self.local_layers[t], v)
        gathered = self.comm.all_gather(buf)
        out = torch.zeros_like(v)
        for t in range(self.T):                     # fixed layer order
            out += gathered[self.owner(t)][t // self.comm.world]
        return out / self.T

    def apply_Lp_power(self, p, v, krylov_dim=50, tol=1e-8):
        if self._pksm is None:
            from .krylov import pksm_layer_dev

            def contrib(layer, x):
                out = _torch().zeros_like(x)
                return pksm_layer_dev(layer, p, x, out, 1.0, False, krylov_dim, tol)
        else:
            def contrib(layer, x):
                return self._pksm(layer, p, x)
        return self._layer_sum(contrib, v)

    def apply_one_minus_L1(self, v):
        if self._weighted is None:
            from .graphs import KernelWeights

            def contrib(layer, x):
                out = _torch().zeros_like(x)
                w = layer.weights
                if not isinstance(w, KernelWeights):
                    raise ConfigError("layer-parallel p=1 path needs GPU kernel layers")
                w.apply_dev(x, out, 0.0, 1.0, -w.kernel.value_at_zero(), _lib.MLB_USE_ISD)
                return out
        else:
            contrib = self._weighted
        return self._layer_sum(contrib, v)


def power_mean_eigs_layer_parallel(lpg, config, k, tol=1e-8, max_subspace=None, max_restarts=60, krylov_dim=50,
                                   inner_tol=None, seed=0, device=None):
    """power_mean_eigs (powermean.py:130-189) with the layer sum distributed.

    Every rank runs the same outer Lanczos on identical vectors; only the
    operator apply communicates.  Returns (values ascending, vectors n x k).
    """
    from .krylov import SymmetricOperator, lanczos_largest_eigs
    p = config.p
    itol = tol if inner_tol is None else inner_tol
    if p == 1:
        apply_dev = lpg.apply_one_minus_L1
    elif p < 0:
        apply_dev = lambda v: lpg.apply_Lp_power(p, v, krylov_dim, itol)  # noqa: E731
    else:
        raise ConfigError("layer-parallel eigensolver covers p = 1 and p < 0")
    op = SymmetricOperator(lpg.n, None, "layer-parallel", apply_dev=apply_dev, device=device)
    res = lanczos_largest_eigs(op, k, tol=tol, max_subspace=max_subspace, max_restarts=max_restarts, seed=seed)
    if p == 1:
        values = np.maximum(1.0 - res.values, 0.0)
    else:
        if res.values.min() <= 0.0:
            raise NumericalError("power mean spectrum is not positive; cannot take the 1/p root")
        values = res.values ** (1.0 / p)
    return values, res.vectors


# ------------------------------------------------ 2. node-range sharding ----
class BindingEngine:
    """libmlb spread / convolve / gather on this rank's points (GPU)."""

    def __init__(self, plan, points_local, device=None):
        from . import fastsum
        torch = _torch()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.binding = fastsum.bind_points(plan, points_local, device=self.device)
        self.cells = self.binding.stats()["grid_cells"]

    def new_grid(self):
        torch = _torch()
        return torch.zeros(self.cells, dtype=torch.float64, device=f"cuda:{self.device}")

    def ones(self, n):
        torch = _torch()
        return torch.ones(n, dtype=torch.float64, device=f"cuda:{self.device}")

    def spread(self, x):
        g = self.new_grid()
        _lib.check(_lib.lib().mlb_spread(self.binding.ptr, _lib.ptr(x), _lib.ptr(g), 0, _lib.stream_ptr()))
        return g

    def enable_peer_exchange(self, comm):
        """Use the fused NVLink peer exchange for the grid sum (PeerGridExchange)."""
        self.exchange = PeerGridExchange(comm, self.cells, self.device)
        return self

    def spread_summed(self, x):
        """The spread grid summed over the ranks through the peer exchange."""
        return self.exchange.spread_sum(self.binding, x, self.new_grid())

    def convolve(self, g):
        out = _torch().empty_like(g)
        _lib.check(_lib.lib().mlb_convolve(self.binding.ptr, _lib.ptr(g), _lib.ptr(out), _lib.stream_ptr()))
        return out

    def gather(self, g):
        y = _torch().empty(self.binding.n, dtype=_torch().float64, device=g.device)
        _lib.check(_lib.lib().mlb_gather(self.binding.ptr, _lib.ptr(g), _lib.ptr(y), 0, _lib.stream_ptr()))
        return y


class PeerGridExchange:
    """The per-matvec sum of the ranks' sub-box grids over NVLink peer memory.

    Every rank owns a receive buffer of `world` grid slots; the buffers are
    mapped into every peer with CUDA IPC once.  Each matvec the final spread
    reduction kernel of rank r stores its grid straight into slot r of every
    rank's buffer (mlb_spread_peers: the exchange is fused into the kernel
    that produces the grid, P2P stores), a one-element NCCL all-reduce on
    the stream orders those stores before any reader, and each rank sums its
    slots in rank order (mlb_grid_sum_slots) -- bitwise the same grid
    everywhere, with no all-gather of the grids through NCCL.

    `slots` may be supplied directly (single-process tests emulate ranks with
    local buffers); otherwise they are built from IPC handles exchanged over
    the process group.  Not available (ValueError) for world > 8 or when
    peer mapping fails; callers then use the NCCL path.
    """

    def __init__(self, comm, cells, device, recv=None, slots=None):
        torch = _torch()
        self.comm, self.cells, self.device = comm, int(cells), int(device)
        world = 1 if comm is None else comm.world
        rank = 0 if comm is None else comm.rank
        if world > 8:
            raise ValueError("peer grid exchange supports at most 8 ranks")
        self.world, self.rank = world, rank
        # two receive buffers, alternated per call (write-after-read safety:
        # rank r's stores of call k+2 into buffer (k mod 2) follow call k+1's
        # barrier, which every peer reaches only after its slot sum of call k)
        if recv is None:
            recv = [torch.zeros(world * self.cells, dtype=torch.float64, device=f"cuda:{self.device}")
                    for _ in range(2)]
        elif not isinstance(recv, (list, tuple)):
            recv = [recv]
        self.recv = list(recv)
        self._opened = []
        if slots is None:
            lib = _lib.lib()
            slots = []
            for buf_local in self.recv:
                h = (ctypes.c_ubyte * 64)()
                _lib.check(lib.mlb_ipc_handle(_lib.ptr(buf_local), h))
                handles = [None] * world
                comm.dist.all_gather_object(handles, bytes(h), group=comm.group)
                bases = []
                for q in range(world):
                    if q == rank:
                        bases.append(buf_local.data_ptr())
                        continue
                    ptr = ctypes.c_void_p()
                    buf = (ctypes.c_ubyte * 64).from_buffer_copy(handles[q])
                    _lib.check(lib.mlb_ipc_open(buf, self.device, ctypes.byref(ptr)))
                    self._opened.append(ptr)
                    bases.append(ptr.value)
                slots.append([b + 8 * rank * self.cells for b in bases])
        elif slots and not isinstance(slots[0], (list, tuple)):
            slots = [slots]
        if len(slots) != len(self.recv):
            raise ValueError("one slot list per receive buffer")
        self.slots = [(ctypes.c_void_p * len(sl))(*sl) for sl in slots]
        self._calls = 0
        self._flag = torch.zeros(1, dtype=torch.float64, device=f"cuda:{self.device}")

    def spread_sum(self, binding, x, grid, flags=0):
        """grid = sum over ranks of their spreads (this rank spreads x)."""
        lib = _lib.lib()
        sp = _lib.stream_ptr()
        k = self._calls % len(self.recv)
        self._calls += 1
        _lib.check(lib.mlb_spread_peers(binding.ptr, _lib.ptr(x), self.slots[k], self.world, int(flags), sp))
        if self.world > 1:  # every rank's peer stores precede every rank's reads
            self.comm.dist.all_reduce(self._flag, group=self.comm.group)
        _lib.check(lib.mlb_grid_sum_slots(_lib.ptr(self.recv[k]), self.world, self.cells, _lib.ptr(grid), sp))
        return grid

    def close(self):
        lib = _lib.lib()
        for ptr in self._opened:
            lib.mlb_ipc_close(ptr)
        self._opened = []


class ShardedLayer:
    """One kernel layer split by node range over the ranks.

    Vectors are this rank's slice [lo, hi).  Every Laplacian apply performs
    exactly one collective: the sum of the spread grids (active sub-box).
    """

    def __init__(self, engine, n_global, lo, hi, comm, K0=1.0, shift=0.0, deterministic=True):
        self.engine, self.n, self.lo, self.hi, self.comm = engine, n_global, lo, hi, comm
        self.K0, self.shift, self.deterministic = float(K0), float(shift), deterministic
        self.degrees = None
        self.isd = None

    @property
    def n_local(self):
        return self.hi - self.lo

    def w_tilde(self, x):
        """(W~ x)_local: spread local charges, sum grids over ranks, convolve, gather."""
        if getattr(self.engine, "exchange", None) is not None:
            g = self.engine.spread_summed(x)  # fused P2P exchange, rank-order sum
        else:
            g = self.engine.spread(x)
            if self.deterministic:
                self.comm.ordered_sum(g)
            else:
                self.comm.all_reduce_sum(g)
        return self.engine.gather(self.engine.convolve(g))

    def matvec(self, x):
        """(W x)_local with zero diagonal (fastsum_apply, fastsum.py:475-497)."""
        return self.w_tilde(x) - self.K0 * x

    def build(self):
        """Degrees W 1 and D^-1/2 (graphs.py:168-183); zero degree on any rank raises."""
        torch = _torch()
        ones = self._ones()
        deg = self.matvec(ones)
        host = deg.cpu().numpy() if isinstance(deg, torch.Tensor) else np.asarray(deg)
        bad = np.flatnonzero(host <= 1e-300)
        first = torch.tensor([float(self.lo + bad[0]) if bad.size else float(self.n)], dtype=torch.float64)
        if isinstance(deg, torch.Tensor) and deg.is_cuda:
            first = first.to(deg.device)
        self.comm.dist.all_reduce(first, op=self.comm.dist.ReduceOp.MIN, group=self.comm.group)
        if int(first.item()) < self.n:
            raise NumericalError(f"node {int(first.item())} has zero degree; the normalized Laplacian is undefined")
        self.degrees = deg
        self.isd = 1.0 / (deg ** 0.5) if isinstance(deg, torch.Tensor) else 1.0 / np.sqrt(deg)
        return self

    def _ones(self):
        return self.engine.ones(self.n_local)

    def apply_lsym(self, x):
        """((1+shift) I - D^-1/2 W D^-1/2) x, local rows (graphs.py:197-201)."""
        return (1.0 + self.shift) * x - self.isd * self.matvec(self.isd * x)

    def dot(self, a, b):
        torch = _torch()
        if isinstance(a, torch.Tensor):
            t = (a * b).sum().reshape(1).to(torch.float64)
        else:
            t = torch.tensor([float(np.dot(a, b))], dtype=torch.float64)
        parts = self.comm.all_gather(t)
        return float(sum(float(p.item()) for p in parts))   # rank order: deterministic


def sharded_pksm(layer, p, v, krylov_dim=50, tol=1e-8):
    """(L_sym + delta)^p v on node-sharded vectors (krylov.py:219-244) for a
    ShardedLayer: the solver of sharded.py (two fused reductions per step)
    with this layer's Laplacian; numpy in -> numpy out (CPU engines), CUDA
    tensor in -> CUDA tensor out."""
    from .sharded import ShardContext
    from .sharded import sharded_pksm as _pksm
    torch = _torch()
    is_t = isinstance(v, torch.Tensor)
    dev = v.device.index if is_t and v.is_cuda else None
    ctx = ShardContext(layer.comm, layer.n, layer.lo, layer.hi, dev)

    def apply(x):
        if dev is None:
            return torch.from_numpy(np.ascontiguousarray(layer.apply_lsym(x.numpy()), dtype=np.float64))
        return layer.apply_lsym(x)
    x = v if is_t else torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
    y = _pksm(ctx, apply, p, x, krylov_dim, tol)
    return y if is_t else y.numpy()


# ------------------------------- 2b. node-range sharded multilayer graph ----
class ShardedKernelGraph:
    """Every layer of a multilayer kernel graph split by the SAME node range
    over the ranks: rank r owns nodes [lo, hi)
    of every layer and binds only those points (the active sub-box of a
    plan is fixed by the plan's admissible box, so every rank's grid has the
    same layout).

    One normalized-Laplacian step (every layer's L_sym + delta of one vector),
    per layer on its own stream (cheapest layer issued first):
      mlb_spread of the rank's nodes (D^-1/2 folded in) into that layer's
                  slice of one buffer holding all layers' sub-box grids;
      all-reduce (sum) of that slice over the ranks -- the layer's only
                  collective (NCCL over NVLink on the box; the cheap layers'
                  collectives overlap the costly layer's spread);
      mlb_convolve (redundant on every rank: the band-limited
                  convolution of a <= 700 KB sub-box) and mlb_gather_apply,
                  the gather with the fused epilogue
                  y = (1+delta) v - D^-1/2 W~ D^-1/2 v + K0 D^-1 v on the
                  rank's nodes (fastsum.py:475-497, graphs.py:197-201).
    With one rank it is the single-GPU matvec (no collective).

    layer_points: per layer the (n_local x d_t) box-unit points of this
    rank's nodes; kernels / plans: per layer KernelSpec (box units) and
    FastsumPlan.  Build the pieces with `shard_feature_groups`.
    """

    def __init__(self, layer_points, kernels, plans, n_global, lo, hi, comm=None, shift=0.0, device=None):
        from .graphs import KernelWeights
        torch = _torch()
        self.comm = comm
        self.world = 1 if comm is None else comm.world
        self.n, self.lo, self.hi = int(n_global), int(lo), int(hi)
        self.shift = float(shift)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.dev = torch.device("cuda", self.device)
        self.weights = [KernelWeights(pts, k, plan=pl, device=self.device)
                        for pts, k, pl in zip(layer_points, kernels, plans)]
        for w in self.weights:
            if w.n != self.n_local:
                raise ConfigError("every layer must hold this rank's node range")
        self.T = len(self.weights)
        self.K0 = [w.kernel.value_at_zero() for w in self.weights]
        cells = [w._bindings[0].stats()["grid_cells"] for w in self.weights]
        self.offsets = np.concatenate([[0], np.cumsum(cells)]).astype(np.int64)
        self.grids = torch.zeros(int(self.offsets[-1]), dtype=torch.float64, device=self.dev)
        self.conv = torch.zeros_like(self.grids)
        self.degrees = None
        self.isd = None

    @property
    def n_local(self):
        return self.hi - self.lo

    def _grid(self, buf, t):
        return buf[int(self.offsets[t]):int(self.offsets[t + 1])]

    def _all_reduce(self):
        if self.comm is not None:   # (a world-size-1 group still runs the collective)
            self.comm.all_reduce_sum(self.grids)

    def _layer_streams(self):
        """One stream per layer, the costliest layer's at high priority (as in
        LaplacianBatch), and the issue order: cheapest layer first, so that the
        collectives, which one communicator runs in issue order, come in the
        order the layers' spreads finish."""
        torch = _torch()
        if getattr(self, "_streams", None) is None:
            cost = [w.n * (2 * w.plan.m_nfft + 1) ** w.plan.d for w in self.weights]
            top = int(np.argmax(cost))
            prio = os.environ.get("MLB_NO_STREAM_PRIORITY") != "1"
            self._streams = [torch.cuda.Stream(self.dev, priority=-1 if (prio and t == top) else 0)
                             for t in range(self.T)]
            self._order = [int(t) for t in np.argsort(cost, kind="stable")]
            self._fork_ev = torch.cuda.Event()
            self._join_ev = [torch.cuda.Event() for _ in range(self.T)]
        return self._streams

    def _per_layer(self, fn):
        """fn(t, stream_ptr) for every layer on its own stream (the current
        torch stream inside fn, so collectives issued there order against the
        layer's kernels), forked from and joined back into the caller's stream.
        MLB_SHARD_ONE_STREAM=1: every layer in order on the caller's stream."""
        torch = _torch()
        if self.T == 1 or os.environ.get("MLB_SHARD_ONE_STREAM") == "1":
            sp = _lib.stream_ptr()
            for t in range(self.T):
                fn(t, sp)
            return
        streams = self._layer_streams()
        main = torch.cuda.current_stream(self.dev)
        self._fork_ev.record(main)
        for t in self._order:
            s = streams[t]
            s.wait_event(self._fork_ev)
            with torch.cuda.stream(s):
                fn(t, s.cuda_stream)
            self._join_ev[t].record(s)
        for t in self._order:
            main.wait_event(self._join_ev[t])

    def spread_local(self, v, flags):
        """Every layer's spread of this rank's nodes into self.grids."""
        lib = _lib.lib()
        spread_flags = int(flags) & (_lib.MLB_USE_ISD | _lib.MLB_SORTED)

        def spread(t, sp):
            _lib.check(lib.mlb_spread(self.weights[t]._bindings[0].ptr, _lib.ptr(v),
                                      _lib.ptr(self._grid(self.grids, t)), spread_flags, sp))
        self._per_layer(spread)

    def _finish_layer(self, t, v, y, coef, flags, sp):
        lib = _lib.lib()
        b = self.weights[t]._bindings[0].ptr
        g_in, g_out = self._grid(self.grids, t), self._grid(self.conv, t)
        _lib.check(lib.mlb_convolve(b, _lib.ptr(g_in), _lib.ptr(g_out), sp))
        a, be, ga = coef
        _lib.check(lib.mlb_gather_apply(b, _lib.ptr(g_out), _lib.ptr(v), _lib.ptr(y), float(a), float(be),
                                        float(ga), int(flags), sp))

    def _step(self, v, ys, coef, flags):
        """ys[t] (=|+=) coef[t] combination for every layer.

        Default: every layer's chain -- spread, all-reduce of ITS grid slice,
        convolution, fused gather -- on its own stream, so a cheap layer's
        whole chain (and its collective) runs under the costly layer's spread
        and fills the costly layer's merge / all-reduce gaps.
        MLB_SHARD_JOINED=1 (or one stream): both spreads, ONE all-reduce of all
        layers' grids, then the convolutions and gathers."""
        if self.T > 1 and os.environ.get("MLB_SHARD_JOINED") != "1" and \
                os.environ.get("MLB_SHARD_ONE_STREAM") != "1":
            lib = _lib.lib()
            spread_flags = int(flags) & (_lib.MLB_USE_ISD | _lib.MLB_SORTED)

            def chain(t, sp):
                g_in = self._grid(self.grids, t)
                _lib.check(lib.mlb_spread(self.weights[t]._bindings[0].ptr, _lib.ptr(v), _lib.ptr(g_in),
                                          spread_flags, sp))
                if self.comm is not None:
                    self.comm.all_reduce_sum(g_in)
                self._finish_layer(t, v, ys[t], coef[t], flags, sp)
            self._per_layer(chain)
            return ys
        self.spread_local(v, flags)
        self._all_reduce()
        return self.finish(v, ys, coef, flags)

    def finish(self, v, ys, coef, flags):
        """Convolve the summed grids and gather this rank's nodes (fused epilogue)."""
        self._per_layer(lambda t, sp: self._finish_layer(t, v, ys[t], coef[t], flags, sp))
        return ys

    def build(self):
        """Degrees W 1 of every layer (graphs.py:168-183) through the sharded
        matvec; a zero degree on any rank raises NumericalError naming the
        first global node; then D^-1/2 is stored in every binding."""
        torch = _torch()
        ones = torch.ones(self.n_local, dtype=torch.float64, device=self.dev)
        degs = [torch.empty_like(ones) for _ in range(self.T)]
        self._step(ones, degs, [(-k0, 1.0, 0.0) for k0 in self.K0], 0)
        first = torch.tensor([float(self.n)], dtype=torch.float64, device=self.dev)
        for d in degs:
            bad = torch.nonzero(d <= 1e-300)
            if bad.numel():
                first = torch.minimum(first, (bad[0].to(torch.float64) + self.lo).reshape(1))
        if self.world > 1:
            self.comm.dist.all_reduce(first, op=self.comm.dist.ReduceOp.MIN, group=self.comm.group)
        if int(first.item()) < self.n:
            raise NumericalError(f"node {int(first.item())} has zero degree; the normalized Laplacian is undefined")
        return self.set_degrees(degs)

    def set_degrees(self, degs):
        """Store this rank's degrees and D^-1/2 (1 / sqrt, as graphs.py:159-165)."""
        torch = _torch()
        self.degrees = degs
        self.isd = [1.0 / torch.sqrt(d) for d in degs]
        for w, s in zip(self.weights, self.isd):
            w.set_isd(s)
        return self

    def _step_layer(self, t, v, y, coef, flags):
        """One layer alone: its spread, the all-reduce of ITS grid slice only,
        convolution and fused gather (the per-layer operator of PKSM)."""
        lib = _lib.lib()
        sp = _lib.stream_ptr()
        g_in = self._grid(self.grids, t)
        _lib.check(lib.mlb_spread(self.weights[t]._bindings[0].ptr, _lib.ptr(v), _lib.ptr(g_in),
                                  int(flags) & (_lib.MLB_USE_ISD | _lib.MLB_SORTED), sp))
        if self.comm is not None:
            self.comm.all_reduce_sum(g_in)
        self._finish_layer(t, v, y, coef, flags, sp)
        return y

    def layer_ops(self):
        """Per layer (ascending): (x -> (L_sym,t + shift) x, x -> D^-1/2 W D^-1/2 x)
        on this rank's rows, each a new tensor -- the operators of
        sharded.sharded_power_mean_eigs."""
        torch = _torch()
        ops = []
        for t, k0 in enumerate(self.K0):
            def lsym(x, t=t, k0=k0):
                return self._step_layer(t, x, torch.empty_like(x), (1.0 + self.shift, -1.0, k0), _lib.MLB_USE_ISD)

            def weighted(x, t=t, k0=k0):
                return self._step_layer(t, x, torch.empty_like(x), (0.0, 1.0, -k0), _lib.MLB_USE_ISD)
            ops.append((lsym, weighted))
        return ops

    def lsym(self, v, ys, accumulate=False):
        """ys[t] = (L_sym,t + shift) v for every layer t (local rows)."""
        flags = _lib.MLB_USE_ISD | (_lib.MLB_ACCUMULATE if accumulate else 0)
        return self._step(v, ys, [(1.0 + self.shift, -1.0, k0) for k0 in self.K0], flags)

    def weighted(self, v, ys):
        """ys[t] = D^-1/2 W D^-1/2 v (the apply_one_minus_L1 term, powermean.py:75-76)."""
        return self._step(v, ys, [(0.0, 1.0, -k0) for k0 in self.K0], _lib.MLB_USE_ISD)

    def lsym_graph(self, v, ys):
        """`lsym` replayed from a CUDA graph captured once per (v, ys) buffer
        set: the per-layer streams, the NCCL all-reduces (NCCL supports stream
        capture; the communicator is warmed up by one eager step on a side
        stream first) and every kernel, with no host issue gaps (projected
        per-rank step at N = 8: 0.57 -> 0.53 ms).  Falls back to the eager
        step (and remembers it) if the capture fails."""
        torch = _torch()
        if getattr(self, "_graphs", None) is None:
            self._graphs = {}
        key = (v.data_ptr(), tuple(y.data_ptr() for y in ys))
        ent = self._graphs.get(key)
        if ent is None:
            lib = _lib.lib()
            main = torch.cuda.current_stream(self.dev)
            side = torch.cuda.Stream(self.dev)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                self.lsym(v, ys)
            main.wait_stream(side)
            torch.cuda.synchronize(self.dev)
            try:
                g = torch.cuda.CUDAGraph()
                l0 = lib.mlb_launch_count()
                with torch.cuda.graph(g):
                    self.lsym(v, ys)
                ent = (g, int(lib.mlb_launch_count() - l0))
            except Exception:   # capture unsupported here: eager from now on
                torch.cuda.synchronize(self.dev)
                ent = (None, 0)
            if len(self._graphs) >= 4:   # a few buffer sets at most (each graph pins its buffers' addresses)
                self._graphs.pop(next(iter(self._graphs)))
            self._graphs[key] = ent
        g, cnt = ent
        if g is None:
            return self.lsym(v, ys)
        g.replay()
        _lib.lib().mlb_note_launches(cnt)
        return ys

    def lsym_many(self, V, out=None):
        """(k, T, n_local): `lsym` of k host vectors (rows of V, this rank's
        slices), streamed like LaplacianBatch.apply_many: vector i+1's H2D and
        vector i-1's D2H run on copy streams while vector i's sharded step
        (spreads, the all-reduce, convolutions, gathers) runs on the current
        stream, with two device buffer sets.  V: pinned contiguous (k,
        n_local) float64 tensor; out: optional pinned (k, T, n_local).
        Returns after the last result has landed in host memory."""
        torch = _torch()
        if not (torch.is_tensor(V) and V.is_pinned() and V.dtype == torch.float64 and V.is_contiguous()
                and V.dim() == 2 and V.shape[1] == self.n_local):
            raise ConfigError("V must be a contiguous pinned float64 (k, n_local) tensor")
        k, T = int(V.shape[0]), self.T
        if out is None:
            out = torch.empty((k, T, self.n_local), dtype=torch.float64, pin_memory=True)
        elif not (torch.is_tensor(out) and out.is_pinned() and out.dtype == torch.float64 and out.is_contiguous()
                  and tuple(out.shape) == (k, T, self.n_local)):
            raise ConfigError("out must be a contiguous pinned float64 tensor of shape (k, T, n_local)")
        if getattr(self, "_many", None) is None:
            self._many = (torch.cuda.Stream(self.dev), torch.cuda.Stream(self.dev),
                          [torch.empty(self.n_local, dtype=torch.float64, device=self.dev) for _ in range(2)],
                          [[torch.empty(self.n_local, dtype=torch.float64, device=self.dev) for _ in range(T)]
                           for _ in range(2)])
        cin, cout, vb, yb = self._many
        main = torch.cuda.current_stream(self.dev)
        start = torch.cuda.Event()
        start.record(main)
        cin.wait_event(start)
        cout.wait_event(start)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        for i in range(k):
            b = i & 1
            if i >= 2:          # vb[b] is free once vector i-2's step has read it
                cin.wait_event(ev_done[b])
            with torch.cuda.stream(cin):
                vb[b].copy_(V[i], non_blocking=True)
            ev_in[b].record(cin)
            main.wait_event(ev_in[b])
            if i >= 2:          # yb[b] is free once vector i-2's results are copied out
                main.wait_event(ev_out[b])
            self.lsym(vb[b], yb[b])
            ev_done[b].record(main)
            cout.wait_event(ev_done[b])
            with torch.cuda.stream(cout):
                for t in range(T):
                    out[i, t].copy_(yb[b][t], non_blocking=True)
            ev_out[b].record(cout)
        main.wait_stream(cin)
        main.wait_stream(cout)
        main.synchronize()
        return out


def shard_feature_groups(X, groups, rank, world, eps_b=None):
    """Box-scaled points of this rank's node range for every column group.

    groups: [(columns, KernelSpec in feature units, fastsum params dict)].
    The box scaling uses the WHOLE feature matrix (every rank holds X), so
    each rank's points and kernel widths are those of the unsharded layer
    (datapipe.feature_group's scaling).  Returns (lo, hi, points, kernels, plans).
    """
    from . import datapipe, fastsum
    n = X.shape[0]
    lo, hi = shard_range(n, rank, world)
    pts, kerns, plans = [], [], []
    for columns, kernel, params in groups:
        params = dict(params or {})
        eb = params.get("eps_b", fastsum.DEFAULT_EPS_B) if eps_b is None else eps_b
        Xb, kb = datapipe.box_points(X[:, list(columns)], kernel, "fastsum-box", eb)
        pts.append(np.ascontiguousarray(Xb[lo:hi]))
        kerns.append(kb)
        plans.append(fastsum.build_plan(kb, d=len(columns), **params))
    return lo, hi, pts, kerns, plans
