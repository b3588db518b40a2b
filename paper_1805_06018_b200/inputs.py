"""Operator inputs for the BASELINE.json configurations (harness, not the apply path).

The apply path consumes an already-constructed operator: sample points p_k,
weights w_k and extended impulses phi_k^E (pc_operator.hpp:20-22).  This module
builds those inputs for the benchmark configurations exactly the way the
reference's construction code would for a tensor lattice of sample points:

* node lattice per axis, ``llround(j/m * ext)`` (pc_operator.cpp:187-194);
* multilinear tent weights on the footprint box [node_{j-1}, node_{j+1}]
  (pc_operator.cpp:211-248), evaluated with the same floating-point operation
  order so the values are bitwise those of the reference rule;
* impulses phi_k[z] = (A delta_{p_k})[z + p_k] on Omega - p_k (impulse.cpp:5-15)
  for the config blur A[y,x] = exp(-|y-x|^2 / (2 sigma(x)^2)) / Z(x), truncated
  at 4 sigma (Euclidean ball, ellipse for c3), Z(x) = full-lattice sum over the
  truncated ball;
* boundary extension phi_k^E (impulse.cpp:17-89): c_k counts the neighbour
  windows Omega - p_j covering z, 1 on Omega - p_k; outside Omega - p_k the
  neighbours' impulses are averaged, summed in ascending neighbour id.  The
  neighbour set of a lattice node is its 3^d lattice neighbourhood (the points
  sharing a lattice cell, grid.hpp:52-53).  tests/test_inputs.py pins this
  against the reference's own ``extend_impulse`` compiled in oracle/_ref.

Because every phi_j vanishes outside its truncation ball, phi_k^E is exactly
zero outside ``[-R, R]^d`` (R = the largest neighbour radius); by default the
extended impulse is returned on that box intersected with the counting box
(``full_box=False``), which is the same grid function under the reference's
zero-outside convention (grid_function.hpp:41-43).  ``full_box=True`` returns
it on the reference's counting box (impulse.cpp:25-27,74).

Vectors follow the reference idiom ``std::mt19937_64(seed)`` +
``std::normal_distribution<double>`` with vector b = draws [bN, (b+1)N)
(adaptivity.cpp:19-23); they are drawn by the library's host helper
``pcb_normal_fill`` so the stream is libstdc++'s.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np


@dataclass
class Field:
    """A dense fp64 grid function on an inclusive integer box (last axis fastest)."""

    lo: Tuple[int, ...]
    values: np.ndarray

    @property
    def hi(self) -> Tuple[int, ...]:
        return tuple(l + s - 1 for l, s in zip(self.lo, self.values.shape))

    @property
    def dim(self) -> int:
        return len(self.lo)


@dataclass
class OperatorInputs:
    """Everything pcb_create needs: domain, sample points, weights, extended impulses."""

    name: str
    dom_lo: Tuple[int, ...]
    dom_hi: Tuple[int, ...]
    points: List[Tuple[int, ...]]
    weights: List[Field]
    impulses: List[Field]
    meta: dict = field(default_factory=dict)

    @property
    def dim(self) -> int:
        return len(self.dom_lo)

    @property
    def shape(self) -> Tuple[int, ...]:
        return tuple(h - l + 1 for l, h in zip(self.dom_lo, self.dom_hi))

    @property
    def n_points(self) -> int:
        return int(np.prod(self.shape))

    @property
    def rank(self) -> int:
        return len(self.weights)

    def checksum(self) -> str:
        """sha256 over the domain, boxes and values (pins golden fixtures to their inputs)."""
        import hashlib

        h = hashlib.sha256()
        h.update(repr((tuple(self.dom_lo), tuple(self.dom_hi))).encode())
        for w, e in zip(self.weights, self.impulses):
            h.update(repr(tuple(w.lo)).encode())
            h.update(np.ascontiguousarray(w.values).tobytes())
            h.update(repr(tuple(e.lo)).encode())
            h.update(np.ascontiguousarray(e.values).tobytes())
        return h.hexdigest()

    def subset(self, ks: Sequence[int]) -> "OperatorInputs":
        return OperatorInputs(self.name, self.dom_lo, self.dom_hi, [self.points[k] for k in ks],
                              [self.weights[k] for k in ks], [self.impulses[k] for k in ks],
                              dict(self.meta))


# ---------------------------------------------------------------------------
# lattice + tents (pc_operator.cpp:179-248)


def uniform_nodes(n: int, m: int, lo: int = 0) -> List[int]:
    """Node coordinates ``lo + llround(j/m * (n-1))`` (pc_operator.cpp:187-194)."""
    ext = n - 1
    out = []
    for j in range(m + 1):
        t = j / m
        v = t * float(ext)
        out.append(lo + int(math.floor(v + 0.5)) if v >= 0 else lo - int(math.floor(-v + 0.5)))
    return out


def graded_nodes(n: int, fine: int, coarse: int) -> List[int]:
    """Per-axis nodes with one extra refinement level on the low half (config 3, D4 option A).

    ``fine`` equal intervals on [0, n/2] and ``coarse`` on [n/2, n-1]; with fine = 2*coarse the
    low half carries twice the density, the tensor analogue of one more quadtree level in the
    largest-gradient quadrant.
    """
    half = n // 2
    nodes = [int(math.floor(j * half / fine + 0.5)) for j in range(fine + 1)]
    nodes += [half + int(math.floor(j * (n - 1 - half) / coarse + 0.5)) for j in range(1, coarse + 1)]
    return nodes


def lattice_points(nodes: Sequence[Sequence[int]]) -> List[Tuple[int, ...]]:
    """Lexicographic node lattice (pc_operator.cpp:197-215)."""
    grids = np.meshgrid(*[np.asarray(a, dtype=np.int64) for a in nodes], indexing="ij")
    return [tuple(int(g.flat[i]) for g in grids) for i in range(grids[0].size)]


def lattice_index(nodes: Sequence[Sequence[int]], flat: int) -> Tuple[int, ...]:
    sizes = [len(a) for a in nodes]
    return tuple(int(v) for v in np.unravel_index(flat, sizes))


def tent_weight(nodes: Sequence[Sequence[int]], idx: Tuple[int, ...]) -> Field:
    """Multilinear hat of node ``idx`` on [node_{j-1}, node_{j+1}] (pc_operator.cpp:217-248).

    Same operation order as the reference: v = 1.0, then per axis v *= factor, where the
    factor is skipped when x_a == p_a, (x-l)/(p-l) below and 1 - (x-p)/(h-p) above.
    """
    d = len(nodes)
    lo, hi, p = [], [], []
    for a in range(d):
        ns = nodes[a]
        j = idx[a]
        p.append(ns[j])
        lo.append(ns[j - 1] if j > 0 else ns[j])
        hi.append(ns[j + 1] if j + 1 < len(ns) else ns[j])
    shape = tuple(h - l + 1 for l, h in zip(lo, hi))
    v = np.ones(shape, dtype=np.float64)
    for a in range(d):
        xa = np.arange(lo[a], hi[a] + 1, dtype=np.int64)
        fa = np.ones(xa.shape, dtype=np.float64)
        below = xa < p[a]
        above = xa > p[a]
        if below.any():
            fa[below] = (xa[below] - lo[a]).astype(np.float64) / float(p[a] - lo[a])
        if above.any():
            fa[above] = 1.0 - (xa[above] - p[a]).astype(np.float64) / float(hi[a] - p[a])
        bshape = [1] * d
        bshape[a] = -1
        fb = fa.reshape(bshape)
        eq = (xa == p[a]).reshape(bshape)
        v = np.where(eq, v, v * fb)
    return Field(tuple(lo), v)


# ---------------------------------------------------------------------------
# config blurs


@dataclass
class BlurSpec:
    """Kernel of A at source x: exp(-sum_a z_a^2 / (2 s_a(x)^2)) / Z(x), on sum (z_a/s_a)^2 <= 16."""

    n: int
    dim: int
    sigma: Callable[[Tuple[int, ...]], Tuple[float, ...]]  # per-axis widths at source x

    def radius(self, x: Tuple[int, ...]) -> Tuple[int, ...]:
        return tuple(int(math.floor(4.0 * s)) for s in self.sigma(x))

    def sigma_field(self) -> np.ndarray:
        """Per-source widths on the whole lattice, shape (n^dim, dim), lexicographic (last axis fastest)."""
        return np.array([self.sigma(x) for x in np.ndindex(*([self.n] * self.dim))], dtype=np.float64)

    def kernel(self, x: Tuple[int, ...]) -> Tuple[Tuple[int, ...], np.ndarray]:
        """Normalised truncated kernel on its support box [-R, R]; returns (lo, values)."""
        s = self.sigma(x)
        R = self.radius(x)
        axes = [np.arange(-r, r + 1, dtype=np.float64) for r in R]
        grids = np.meshgrid(*axes, indexing="ij")
        q = np.zeros(grids[0].shape)
        e = np.zeros(grids[0].shape)
        for g, sa in zip(grids, s):
            q = q + (g / sa) ** 2
            e = e + g * g / (2.0 * sa * sa)
        vals = np.where(q <= 16.0, np.exp(-e), 0.0)
        vals = vals / vals.sum()
        return tuple(-r for r in R), vals


def blur_c1(n: int = 128, s0: float = 3.0) -> BlurSpec:
    def sig(x):
        s = s0 * (1.0 + 0.5 * math.sin(2.0 * math.pi * x[0] / n)) * (1.0 + 0.3 * math.cos(2.0 * math.pi * x[1] / n))
        return (s, s)

    return BlurSpec(n, 2, sig)


def blur_c3(n: int = 1024) -> BlurSpec:
    def sig(x):
        return (8.0 + 4.0 * math.sin(2.0 * math.pi * x[0] / n), 5.0 + 3.0 * math.cos(2.0 * math.pi * x[1] / n))

    return BlurSpec(n, 2, sig)


def blur_c4(n: int = 128) -> BlurSpec:
    def sig(x):
        s = 2.0 * (1.0 + 0.5 * math.sin(2.0 * math.pi * x[0] / n) * math.sin(2.0 * math.pi * x[2] / n))
        return (s, s, s)

    return BlurSpec(n, 3, sig)


def blur_const(n: int, dim: int, s: float) -> BlurSpec:
    return BlurSpec(n, dim, lambda x: (s,) * dim)


# ---------------------------------------------------------------------------
# impulses and extension (impulse.cpp:5-89)


def _box_inter(alo, ahi, blo, bhi):
    lo = tuple(max(a, b) for a, b in zip(alo, blo))
    hi = tuple(min(a, b) for a, b in zip(ahi, bhi))
    return (lo, hi) if all(l <= h for l, h in zip(lo, hi)) else None


def _slices(sub_lo, sub_hi, box_lo):
    return tuple(slice(l - b, h - b + 1) for l, h, b in zip(sub_lo, sub_hi, box_lo))


def impulse_on(blur: BlurSpec, dom_lo, dom_hi, p, box_lo, box_hi) -> np.ndarray:
    """phi_p[z] = (A delta_p)[z + p] for z in the given box, zero off Omega - p and off the ball."""
    shape = tuple(h - l + 1 for l, h in zip(box_lo, box_hi))
    out = np.zeros(shape)
    klo, kv = blur.kernel(p)
    khi = tuple(l + s - 1 for l, s in zip(klo, kv.shape))
    win_lo = tuple(l - q for l, q in zip(dom_lo, p))
    win_hi = tuple(h - q for h, q in zip(dom_hi, p))
    ov = _box_inter(klo, khi, win_lo, win_hi)
    if ov is None:
        return out
    ov = _box_inter(ov[0], ov[1], box_lo, box_hi)
    if ov is None:
        return out
    out[_slices(ov[0], ov[1], box_lo)] = kv[_slices(ov[0], ov[1], klo)]
    return out


def extend_lattice_impulse(blur: BlurSpec, dom_lo, dom_hi, nodes, k: int, full_box: bool = False) -> Field:
    """phi_k^E for lattice node k (impulse.cpp:17-41 counting, :61-89 stitching)."""
    d = len(dom_lo)
    sizes = [len(a) for a in nodes]
    idx = lattice_index(nodes, k)
    nb_idx = []
    for off in np.ndindex(*([3] * d)):
        j = tuple(i + o - 1 for i, o in zip(idx, off))
        if all(0 <= j[a] < sizes[a] for a in range(d)):
            nb_idx.append(j)
    nbrs = sorted(int(np.ravel_multi_index(j, sizes)) for j in nb_idx)
    pts = [tuple(nodes[a][lattice_index(nodes, j)[a]] for a in range(d)) for j in nbrs]
    p_k = tuple(nodes[a][idx[a]] for a in range(d))
    # counting box = bounding box of Omega - p_j over neighbours (impulse.cpp:25-27)
    c_lo = tuple(min(dom_lo[a] - q[a] for q in pts) for a in range(d))
    c_hi = tuple(max(dom_hi[a] - q[a] for q in pts) for a in range(d))
    if full_box:
        b_lo, b_hi = c_lo, c_hi
    else:
        R = [max(blur.radius(q)[a] for q in pts) for a in range(d)]
        ov = _box_inter(tuple(-r for r in R), tuple(R), c_lo, c_hi)
        b_lo, b_hi = ov
    shape = tuple(h - l + 1 for l, h in zip(b_lo, b_hi))
    # c_k on the evaluation box
    count = np.zeros(shape)
    for j, q in zip(nbrs, pts):
        if j == k:
            continue
        ov = _box_inter(tuple(dom_lo[a] - q[a] for a in range(d)), tuple(dom_hi[a] - q[a] for a in range(d)), b_lo, b_hi)
        if ov is not None:
            count[_slices(ov[0], ov[1], b_lo)] += 1.0
    self_lo = tuple(dom_lo[a] - p_k[a] for a in range(d))
    self_hi = tuple(dom_hi[a] - p_k[a] for a in range(d))
    self_ov = _box_inter(self_lo, self_hi, b_lo, b_hi)
    in_self = np.zeros(shape, dtype=bool)
    if self_ov is not None:
        in_self[_slices(self_ov[0], self_ov[1], b_lo)] = True
    count[in_self] = 1.0
    out = np.zeros(shape)
    # step 1: exact copy of phi_k on Omega - p_k
    phik = impulse_on(blur, dom_lo, dom_hi, p_k, b_lo, b_hi)
    out[in_self] = phik[in_self]
    # step 2: neighbours averaged outside the self window, ascending neighbour id
    for j, q in zip(nbrs, pts):
        if j == k:
            continue
        win_lo = tuple(dom_lo[a] - q[a] for a in range(d))
        win_hi = tuple(dom_hi[a] - q[a] for a in range(d))
        ov = _box_inter(win_lo, win_hi, b_lo, b_hi)
        if ov is None:
            continue
        phij = impulse_on(blur, dom_lo, dom_hi, q, b_lo, b_hi)
        sl = _slices(ov[0], ov[1], b_lo)
        region = np.zeros(shape, dtype=bool)
        region[sl] = True
        region &= ~in_self
        out[region] = out[region] + phij[region] / count[region]
    return Field(b_lo, out)


def lattice_operator(name: str, blur: BlurSpec, nodes: Sequence[Sequence[int]], full_box: bool = False,
                     extend: bool = True, ks: Optional[Sequence[int]] = None) -> OperatorInputs:
    d = blur.dim
    n = blur.n
    dom_lo = (0,) * d
    dom_hi = (n - 1,) * d
    pts = lattice_points(nodes)
    sizes = [len(a) for a in nodes]
    weights, imps = [], []
    for k in (range(len(pts)) if ks is None else ks):
        idx = lattice_index(nodes, k)
        weights.append(tent_weight(nodes, idx))
        if extend:
            imps.append(extend_lattice_impulse(blur, dom_lo, dom_hi, nodes, k, full_box))
        else:  # zero extension (impulse.cpp:91-93): the raw impulse on its natural box
            p = pts[k]
            lo = tuple(dom_lo[a] - p[a] for a in range(d))
            hi = tuple(dom_hi[a] - p[a] for a in range(d))
            imps.append(Field(lo, impulse_on(blur, dom_lo, dom_hi, p, lo, hi)))
    if ks is not None:
        pts = [pts[k] for k in ks]
    return OperatorInputs(name, dom_lo, dom_hi, pts, weights, imps,
                          {"nodes": [list(a) for a in nodes], "lattice": sizes})


# ---------------------------------------------------------------------------
# the BASELINE.json configurations


CONFIGS = {
    "c1": dict(desc="2D 128^2, r=16 (4x4 tents), sigma=3(1+.5 sin)(1+.3 cos), B=1, seed 0", B=1, seed=0),
    "c2": dict(desc="2D 512^2, r=64 (8x8 tents), sigma0=6, B=16, seed 1", B=16, seed=1),
    "c3": dict(desc="2D 1024^2, r=256 (graded 16x16 tents), anisotropic sigma, B=64 probes, seed 2", B=64, seed=2),
    "c4": dict(desc="3D 128^3, r=512 (8x8x8 tents), sigma=2(1+.5 sin sin), B=8, seed 4", B=8, seed=4),
    "c5": dict(desc="c2 operator, 4096 dense 8x8-patch blocks (64x64), origins mt19937_64(3) in [0,504]", B=0, seed=3),
}


def config_spec(name: str):
    """(blur, nodes) of a BASELINE.json configuration."""
    if name in ("c1",):
        return blur_c1(128, 3.0), [uniform_nodes(128, 3)] * 2
    if name in ("c2", "c5"):
        return blur_c1(512, 6.0), [uniform_nodes(512, 7)] * 2
    if name == "c3":
        return blur_c3(1024), [graded_nodes(1024, 10, 5)] * 2
    if name == "c4":
        return blur_c4(128), [uniform_nodes(128, 7)] * 3
    raise ValueError(f"unknown config {name!r}")


def make_config(name: str, full_box: bool = False, ks: Optional[Sequence[int]] = None) -> OperatorInputs:
    blur, nodes = config_spec(name)
    op = lattice_operator(name, blur, nodes, full_box, ks=ks)
    op.meta.update(CONFIGS[name])
    return op


def small_lattice(n: int = 24, dim: int = 2, m: int = 3, sigma: float = 1.7, varying: bool = True,
                  full_box: bool = False, extend: bool = True) -> OperatorInputs:
    """Small test operators (c1 family shrunk) for fast parity cases."""
    if varying:
        if dim == 2:
            blur = blur_c1(n, sigma)
        else:
            def sig(x):
                s = sigma * (1.0 + 0.5 * math.sin(2.0 * math.pi * x[0] / n) * math.sin(2.0 * math.pi * x[-1] / n))
                return (s,) * dim
            blur = BlurSpec(n, dim, sig)
    else:
        blur = blur_const(n, dim, sigma)
    nodes = [uniform_nodes(n, m)] * dim
    return lattice_operator(f"small{dim}d_n{n}_m{m}", blur, nodes, full_box, extend)


def apply_true_blur(blur: BlurSpec, f: np.ndarray) -> np.ndarray:
    """(A f)[y] = sum_x A[y,x] f[x] with the truncated config kernel (direct stencil; small n)."""
    n, d = blur.n, blur.dim
    g = np.zeros_like(f)
    for x in np.ndindex(*f.shape):
        v = f[x]
        if v == 0.0:
            continue
        klo, kv = blur.kernel(x)
        lo = [x[a] + klo[a] for a in range(d)]
        sl_out, sl_k = [], []
        for a in range(d):
            a0 = max(lo[a], 0)
            a1 = min(lo[a] + kv.shape[a] - 1, n - 1)
            sl_out.append(slice(a0, a1 + 1))
            sl_k.append(slice(a0 - lo[a], a1 - lo[a] + 1))
        g[tuple(sl_out)] += v * kv[tuple(sl_k)]
    return g
