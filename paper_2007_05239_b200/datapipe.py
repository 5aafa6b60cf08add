"""Column groups -> GPU kernel layers: the hot-path part of multilap.datapipe
(reference datapipe.py:32-170 feature grouping, :367-385 label sampling).

The unit that does the work here is `BoxMap`: the affine map of one column
group into the fastsum box (centre = per-column midpoint of the data range,
ONE isotropic factor, so kernel distances only change by that factor).  A
group becomes a layer in three steps -- fit the map, express the kernel
width in box units (mode "fastsum-box": sigma / factor; "unit-box": sigma
times the box half-width), bind the mapped points on the device with a plan
when the group has <= 3 columns -- and the exact O(n^2) device path
otherwise.  `feature_group` accepts a `weights_factory` so callers can plug
other weights objects (the reference hard-codes KernelWeights,
datapipe.py:162-168); the node-range sharded path (dist.shard_feature_groups)
uses `box_points` directly so every rank maps its nodes with the map fitted
on the whole matrix.

API names, fields and error messages are the reference's (drop-in).
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
_BOX_LIMIT = 3   # widest group a fastsum plan (and "fastsum-box" mode) accepts


# ------------------------------------------------------------ spec types ---
def _group_problem(columns, mode):
    """The first reason a (columns, mode) pair is not a valid group, or None."""
    if not columns:
        return "feature group must select at least one column"
    if len(set(columns)) < len(columns):
        return f"duplicate column in group {columns}"
    if mode not in SCALING_MODES:
        return f"unknown scaling mode {mode!r}, expected one of {SCALING_MODES}"
    if mode == "fastsum-box" and len(columns) > _BOX_LIMIT:
        return (f"group of width {len(columns)} cannot use mode 'fastsum-box' (limit {_BOX_LIMIT}); "
                "use 'unit-box' or 'none'")
    return None


@dataclass(frozen=True)
class GroupSpec:
    """One layer: a column subset, its kernel and scaling mode (datapipe.py:32-65).
    kernel.sigma is in the columns' own units for "fastsum-box" / "none" and
    in [-1, 1]-scaled units for "unit-box"; `per_component` keeps the
    kernel block-diagonal over the component labels."""

    columns: tuple
    kernel: KernelSpec
    mode: str = "fastsum-box"
    per_component: bool = False

    def __post_init__(self):
        cols = tuple(int(c) for c in self.columns)
        object.__setattr__(self, "columns", cols)
        problem = _group_problem(cols, self.mode)
        if problem:
            raise ConfigError(problem)


@dataclass(frozen=True)
class GroupingSpec:
    """Disjoint column groups, one layer each (datapipe.py:68-83)."""

    groups: tuple

    def __post_init__(self):
        groups = tuple(self.groups)
        object.__setattr__(self, "groups", groups)
        if not groups:
            raise ConfigError("grouping needs at least one group")
        owner = {}
        for gi, g in enumerate(groups):
            shared = sorted(c for c in g.columns if owner.get(c, gi) != gi)
            if shared:
                raise ConfigError(f"column(s) {shared} appear in more than one group")
            owner.update((c, gi) for c in g.columns)

    @property
    def used_columns(self):
        return sorted(c for g in self.groups for c in g.columns)


@dataclass(frozen=True)
class ScalingInfo:
    """x_box = (x - midpoints) / factor (datapipe.py:86-97)."""

    midpoints: np.ndarray
    factor: float
    mode: str


# ------------------------------------------------------------ box map ------
@dataclass(frozen=True)
class BoxMap:
    """Affine map of a column group into [-s, s]^d, s = 1/4 - eps_b/2
    (datapipe.py:100-123): x -> clip((x - mid) / half, -1, 1) * s, with
    `half` the largest half-range over the columns.  A constant group maps
    to the origin with factor 1."""

    mid: np.ndarray
    half: float
    s: float

    @classmethod
    def fit(cls, X, eps_b=fastsum.DEFAULT_EPS_B, columns=None, X_dev=None):
        """Fit on a feature block, or on `columns` of a wider matrix.  With
        `X_dev` (the device copy of X) the column ranges are reduced on the
        GPU (min / max are exact: the same map as the host reduction)."""
        if X_dev is not None:
            import torch
            cols = range(X_dev.shape[1]) if columns is None else columns
            sub = X_dev[:, list(cols)]
            if not bool(torch.isfinite(sub).all()):
                raise FormatError("non-finite feature values")
            lo_t, hi_t = torch.aminmax(sub, dim=0)
            lo, hi = lo_t.cpu().numpy(), hi_t.cpu().numpy()
        else:
            X = np.asarray(X, dtype=float)
            if X.ndim != 2:
                raise ConfigError("expected a 2-d feature block")
            Xg = X if columns is None else X[:, list(columns)]
            if not np.isfinite(Xg).all():
                raise FormatError("non-finite feature values")
            lo, hi = Xg.min(axis=0), Xg.max(axis=0)
        return cls(mid=0.5 * (lo + hi), half=float((hi - lo).max()) / 2.0, s=fastsum.box_halfwidth(eps_b))

    @property
    def factor(self):
        """Original units per box unit (1 for a constant group)."""
        return 1.0 if self.half == 0.0 else self.half / self.s

    def __call__(self, X):
        X = np.asarray(X, dtype=float)
        if self.half == 0.0:
            return np.zeros_like(X)
        # the clip absorbs the one-ulp overshoot at the extremes; with a
        # dyadic s the product then stays inside the box
        return np.clip((X - self.mid) / self.half, -1.0, 1.0) * self.s

    def info(self):
        return ScalingInfo(midpoints=self.mid, factor=self.factor, mode="fastsum-box")

    def kernel_in_box(self, kernel, mode):
        """The group's kernel with sigma in box units (datapipe.py:126-133)."""
        sigma = kernel.sigma / self.factor if mode == "fastsum-box" else kernel.sigma * self.s
        return KernelSpec(family=kernel.family, sigma=sigma)


def scale_for_fastsum(X, eps_b=fastsum.DEFAULT_EPS_B):
    """(box coordinates, ScalingInfo) of one column group (datapipe.py:100-123)."""
    bm = BoxMap.fit(X, eps_b)
    return bm(X), bm.info()


def box_points(Xg, kernel, mode="fastsum-box", eps_b=fastsum.DEFAULT_EPS_B):
    """(box coordinates, box-unit kernel) of one column group."""
    bm = BoxMap.fit(Xg, eps_b)
    return bm(Xg), bm.kernel_in_box(kernel, mode)


# ------------------------------------------------------------ layers -------
def _checked_matrix(X, spec):
    X = np.asarray(X, dtype=float)
    if X.ndim != 2:
        raise ConfigError("feature matrix must be 2-d")
    d = X.shape[1]
    out_of_range = [c for g in spec.groups for c in g.columns if not 0 <= c < d]
    if out_of_range:
        raise ConfigError(f"column index {out_of_range[0]} out of range for {d} feature columns")
    unused = sorted(set(range(d)).difference(spec.used_columns))
    if unused:
        log.info("dropping %d unused feature column(s): %s", len(unused), unused)
    return X


def _group_weights(X, X_dev, g, components, params, device, factory):
    comp = components if g.per_component else None
    eps_b = params.get("eps_b", fastsum.DEFAULT_EPS_B)
    if g.mode == "none":          # original units, exact sums
        return factory(X[:, list(g.columns)], g.kernel, plan=None, components=comp, device=device)
    planned = len(g.columns) <= _BOX_LIMIT
    if planned and factory is KernelWeights:
        # the box map runs on the device inside the bind, reading the group's
        # columns straight from the (device copy of the) feature matrix
        bm = BoxMap.fit(X, eps_b, columns=g.columns, X_dev=X_dev)
        kernel_box = bm.kernel_in_box(g.kernel, g.mode)
        plan = fastsum.build_plan(kernel_box, d=len(g.columns), **params)
        return KernelWeights(X if X_dev is None else X_dev, kernel_box, plan=plan, components=comp, device=device,
                             box_map=bm, columns=g.columns, host_points=X)
    Xb, kernel_box = box_points(X[:, list(g.columns)], g.kernel, g.mode, eps_b)
    plan = fastsum.build_plan(kernel_box, d=len(g.columns), **params) if planned else None
    return factory(Xb, kernel_box, plan=plan, components=comp, device=device)


def feature_group(X, spec, components=None, fastsum_params=None, device=None, weights_factory=None):
    """One graph layer per column group (datapipe.py:136-170), bound on the GPU.

    The feature matrix goes to the device once; every planned group binds
    from that copy (box map, box check, cells and sort on the GPU).
    `weights_factory(points, kernel, plan=, components=, device=)` replaces
    KernelWeights for every group (it receives box coordinates)."""
    X = _checked_matrix(X, spec)
    params = dict(fastsum_params or {})
    factory = KernelWeights if weights_factory is None else weights_factory
    X_dev = None
    if factory is KernelWeights and any(g.mode != "none" and len(g.columns) <= _BOX_LIMIT for g in spec.groups):
        import torch
        dev = torch.cuda.current_device() if device is None else int(device)
        X_dev = torch.from_numpy(np.ascontiguousarray(X)).to(f"cuda:{dev}")
    return MultilayerGraph(tuple(build_layer(_group_weights(X, X_dev, g, components, params, device, factory))
                                 for g in spec.groups))


# ------------------------------------------------------------ labels -------
def sample_labels(truth, fraction, seed, omega0=1000.0):
    """Known labels: per class c = 0..m-1 in order, ceil(fraction * |c|)
    members (at least one) drawn without replacement by one
    default_rng(seed) stream (datapipe.py:367-385)."""
    truth = np.asarray(truth)
    if not 0.0 < fraction <= 1.0:
        raise ConfigError(f"label fraction {fraction} outside (0, 1]")
    m = int(truth.max()) + 1
    if truth.min() < 0:
        raise ConfigError("ground truth must label every node (no negatives)")
    sizes = np.bincount(truth.astype(np.int64), minlength=m)
    if (sizes == 0).any():
        raise ConfigError(f"class {int(np.argmin(sizes > 0))} absent from ground truth")
    by_class = np.argsort(truth, kind="stable")        # members of class c, ascending node index
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    rng = np.random.default_rng(seed)
    ids = np.full(truth.shape[0], -1)
    for c in range(m):
        members = by_class[bounds[c]:bounds[c + 1]]
        ids[rng.choice(members, size=max(1, math.ceil(fraction * sizes[c])), replace=False)] = c
    return LabelData.from_class_ids(ids, m, omega0)


# ------------------------------------------------------------ images -------
@dataclass(frozen=True)
class ImageStack:
    """Vectorised images (datapipe.py:285-297): rgb (n x 3), xy (n x 2: column,
    row), component id per pixel, (h, w) per image."""

    rgb: np.ndarray
    xy: np.ndarray
    components: np.ndarray
    shapes: tuple

    @property
    def n(self):
        return self.rgb.shape[0]


def image_to_features(images):
    """One image or a list of 8-bit RGB images, pixels row-major (datapipe.py:300-325)."""
    X, comps, shapes = image_features(images)
    return ImageStack(rgb=X[:, :3], xy=X[:, 3:], components=comps, shapes=shapes)


def load_image(path):
    """8-bit RGB PNG -> (h, w, 3) uint8 (datapipe.py:341-352)."""
    from PIL import Image
    try:
        with Image.open(path) as img:
            if img.mode != "RGB":
                raise FormatError(f"{path}: expected an 8-bit RGB image, got mode {img.mode!r}")
            return np.asarray(img, dtype=np.uint8)
    except (FileNotFoundError, FormatError):
        raise
    except Exception as exc:
        raise FormatError(f"{path}: cannot decode image ({exc})") from exc


def save_image(path, array):
    from PIL import Image
    a = np.asarray(array).astype(np.uint8)
    Image.fromarray(a, mode="L" if a.ndim == 2 else "RGB").save(path)


def image_features(images):
    """Row-major pixel features of a list of RGB images (datapipe.py:300-325):
    (n x 5 [r, g, b, col, row], component id per pixel, shapes)."""
    if isinstance(images, np.ndarray):
        images = [images]
    if not images:
        raise ConfigError("need at least one image")
    feats, comps, shapes = [], [], []
    for k, img in enumerate(images):
        img = np.asarray(img)
        if img.ndim != 3 or img.shape[2] != 3 or img.dtype != np.uint8:
            raise FormatError(f"image {k}: expected 8-bit RGB of shape (h, w, 3), got {img.dtype} {img.shape}")
        h, w = img.shape[:2]
        rows, cols = np.divmod(np.arange(h * w), w)
        feats.append(np.column_stack([img.reshape(-1, 3).astype(float), cols.astype(float), rows.astype(float)]))
        comps.append(np.full(h * w, k))
        shapes.append((h, w))
    return np.vstack(feats), np.concatenate(comps), tuple(shapes)


def masks_from_labels(labels, shapes):
    """Per image (h, w) label arrays (datapipe.py:328-338)."""
    labels = np.asarray(labels)
    ends = np.cumsum([h * w for h, w in shapes])
    if (ends[-1] if len(ends) else 0) != labels.shape[0]:
        raise ConfigError(f"label vector length {labels.shape[0]} does not match shapes {shapes}")
    starts = np.concatenate([[0], ends[:-1]])
    return [labels[a:b].reshape(h, w) for a, b, (h, w) in zip(starts, ends, shapes)]


# ------------------------------------------------------------- file formats --
# The reference keeps its CSV readers / writers in datapipe (datapipe.py:392-
# 470); here they live in csvio and are re-exported under the same names.
from .csvio import load_features_csv, load_labels_csv, write_predictions_csv  # noqa: E402
from .csvio import write_matrix_csv as write_scores_csv  # noqa: E402
from .csvio import write_matrix_csv as write_values_csv  # noqa: E402


# ------------------------------------------------- out of scope --
# Stochastic block models (datapipe.py:178-279) build edge-list layers with no
# NFFT kernel path; the names exist so a drop-in `from multilap.datapipe
# import ...` resolves, and using them raises ConfigError.
def _sbm_unsupported(*_args, **_kwargs):
    raise ConfigError("stochastic block models are not part of the B200 backend "
                      "(edge-list layers have no NFFT kernel path; use the reference package)")


class SbmLayerSpec:
    def __init__(self, *args, **kwargs):
        _sbm_unsupported()


class SbmSpec:
    def __init__(self, *args, **kwargs):
        _sbm_unsupported()


sbm_generate = noisy_pair_sbm = complementary_sbm = _sbm_unsupported
