"""Feature grouping into GPU kernel layers -- drop-in for the hot-path part of
multilap.datapipe (datapipe.py:32-170, :367-385).

Each column group is centred and scaled isotropically into the fastsum box,
its bandwidth converted to box units, a plan attached when the group has at
most 3 columns, and the layer built with GPU-bound KernelWeights.
"""

import logging
import math
from dataclasses import dataclass

import numpy as np

from . import fastsum
from .allencahn import LabelData
from .errors import ConfigError, FormatError
from .graphs import KernelWeights, MultilayerGraph, build_layer
from .kernels import KernelSpec

log = logging.getLogger(__name__)

SCALING_MODES = ("fastsum-box", "unit-box", "none")


@dataclass(frozen=True)
class GroupSpec:
    """One layer: column subset, kernel, scaling mode (datapipe.py:32-65)."""

    columns: tuple
    kernel: KernelSpec
    mode: str = "fastsum-box"
    per_component: bool = False

    def __post_init__(self):
        object.__setattr__(self, "columns", tuple(int(c) for c in self.columns))
        if len(self.columns) == 0:
            raise ConfigError("feature group must select at least one column")
        if len(set(self.columns)) != len(self.columns):
            raise ConfigError(f"duplicate column in group {self.columns}")
        if self.mode not in SCALING_MODES:
            raise ConfigError(f"unknown scaling mode {self.mode!r}, expected one of {SCALING_MODES}")
        if self.mode == "fastsum-box" and len(self.columns) > 3:
            raise ConfigError(f"group of width {len(self.columns)} cannot use mode 'fastsum-box' (limit 3); "
                              "use 'unit-box' or 'none'")


@dataclass(frozen=True)
class GroupingSpec:
    groups: tuple

    def __post_init__(self):
        object.__setattr__(self, "groups", tuple(self.groups))
        if not self.groups:
            raise ConfigError("grouping needs at least one group")
        seen = set()
        for g in self.groups:
            dup = seen.intersection(g.columns)
            if dup:
                raise ConfigError(f"column(s) {sorted(dup)} appear in more than one group")
            seen.update(g.columns)

    @property
    def used_columns(self):
        return sorted(c for g in self.groups for c in g.columns)


@dataclass(frozen=True)
class ScalingInfo:
    midpoints: np.ndarray
    factor: float
    mode: str


def scale_for_fastsum(X, eps_b=fastsum.DEFAULT_EPS_B):
    """Centre at column midpoints, one isotropic factor into the box (datapipe.py:100-123)."""
    X = np.asarray(X, dtype=float)
    if X.ndim != 2:
        raise ConfigError("expected a 2-d feature block")
    if not np.all(np.isfinite(X)):
        raise FormatError("non-finite feature values")
    s = fastsum.box_halfwidth(eps_b)
    lo, hi = X.min(axis=0), X.max(axis=0)
    mid = 0.5 * (lo + hi)
    half = float(np.max(hi - lo)) / 2.0
    if half == 0.0:
        return np.zeros_like(X), ScalingInfo(midpoints=mid, factor=1.0, mode="fastsum-box")
    unit = np.clip((X - mid) / half, -1.0, 1.0)
    return unit * s, ScalingInfo(midpoints=mid, factor=half / s, mode="fastsum-box")


def _scaled_group(Xg, g, eps_b):
    Xb, info = scale_for_fastsum(Xg, eps_b)
    if g.mode == "fastsum-box":
        sigma_box = g.kernel.sigma / info.factor
    else:
        sigma_box = g.kernel.sigma * fastsum.box_halfwidth(eps_b)
    return Xb, KernelSpec(family=g.kernel.family, sigma=sigma_box), info


def feature_group(X, spec, components=None, fastsum_params=None, device=None):
    """One GPU graph layer per column group (datapipe.py:136-170)."""
    X = np.asarray(X, dtype=float)
    if X.ndim != 2:
        raise ConfigError("feature matrix must be 2-d")
    n, d = X.shape
    for g in spec.groups:
        bad = [c for c in g.columns if c < 0 or c >= d]
        if bad:
            raise ConfigError(f"column index {bad[0]} out of range for {d} feature columns")
    unused = sorted(set(range(d)) - set(spec.used_columns))
    if unused:
        log.info("dropping %d unused feature column(s): %s", len(unused), unused)
    params = dict(fastsum_params or {})
    eps_b = params.get("eps_b", fastsum.DEFAULT_EPS_B)
    layers = []
    for g in spec.groups:
        Xg = X[:, list(g.columns)]
        comp = components if g.per_component else None
        if g.mode == "none":
            weights = KernelWeights(Xg, g.kernel, plan=None, components=comp, device=device)
        else:
            Xb, kern_box, _ = _scaled_group(Xg, g, eps_b)
            plan = fastsum.build_plan(kern_box, d=len(g.columns), **params) if len(g.columns) <= 3 else None
            weights = KernelWeights(Xb, kern_box, plan=plan, components=comp, device=device)
        layers.append(build_layer(weights))
    return MultilayerGraph(tuple(layers))


def sample_labels(truth, fraction, seed, omega0=1000.0):
    """Per class ceil(fraction * size) labelled nodes, default_rng(seed) (datapipe.py:367-385)."""
    truth = np.asarray(truth)
    if not 0.0 < fraction <= 1.0:
        raise ConfigError(f"label fraction {fraction} outside (0, 1]")
    m = int(truth.max()) + 1
    if truth.min() < 0:
        raise ConfigError("ground truth must label every node (no negatives)")
    rng = np.random.default_rng(seed)
    ids = np.full(truth.shape[0], -1)
    for c in range(m):
        members = np.flatnonzero(truth == c)
        if members.size == 0:
            raise ConfigError(f"class {c} absent from ground truth")
        count = max(1, math.ceil(fraction * members.size))
        ids[rng.choice(members, size=count, replace=False)] = c
    return LabelData.from_class_ids(ids, m, omega0)
