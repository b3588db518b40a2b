"""ORACLE — TEST INFRASTRUCTURE ONLY.  Never imported by the product path.

A numpy restatement of the reference's apply path (arXiv 1805.06018, `pcop`),
used by tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg as
the checker.  Every function cites the reference lines it restates
(paths relative to /root/reference/proj/core).

Parity pin: tests/test_oracle.py checks this module against (a) the
reference's own known-answer tests (test_fft.cpp, test_pc_operator.cpp,
acceptance.cpp criterion 10) and (b) the reference library itself compiled
verbatim from its sources (oracle/Makefile -> oracle/_ref/libpcopref.so) and
the golden vectors that build generated (tests/golden/, made by
tests/golden/make_golden.py).

FFT: the reference calls FFTW (version unpinned, fft.cpp:21-22,47); this
restatement uses numpy.fft on the same zero-padded power-of-two shapes.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

Box = Tuple[Tuple[int, ...], Tuple[int, ...]]


# --- L0: boxes (box.hpp:22-70, box.cpp:5-108) ------------------------------

def box_of(lo, values) -> Box:
    lo = tuple(int(v) for v in lo)
    return lo, tuple(l + s - 1 for l, s in zip(lo, values.shape))


def minkowski_sum(a: Box, b: Box) -> Box:  # box.cpp:5-13
    return tuple(x + y for x, y in zip(a[0], b[0])), tuple(x + y for x, y in zip(a[1], b[1]))


def minkowski_diff(a: Box, b: Box) -> Box:  # box.cpp:15-23
    return tuple(x - y for x, y in zip(a[0], b[1])), tuple(x - y for x, y in zip(a[1], b[0]))


def intersect(a: Box, b: Box) -> Optional[Box]:  # box.cpp:66-75
    lo = tuple(max(x, y) for x, y in zip(a[0], b[0]))
    hi = tuple(min(x, y) for x, y in zip(a[1], b[1]))
    return (lo, hi) if all(l <= h for l, h in zip(lo, hi)) else None


def contains(b: Box, p) -> bool:  # box.hpp:49-53
    return all(l <= v <= h for l, v, h in zip(b[0], p, b[1]))


def _sl(sub: Box, base_lo) -> tuple:
    return tuple(slice(l - b, h - b + 1) for l, h, b in zip(sub[0], sub[1], base_lo))


class GF:
    """GridFunction: dense fp64 on an inclusive box, zero outside (grid_function.hpp:14-67)."""

    def __init__(self, lo, values):
        self.lo = tuple(int(v) for v in lo)
        self.values = np.asarray(values, dtype=np.float64)

    @property
    def box(self) -> Box:
        return box_of(self.lo, self.values)

    def value_or_zero(self, p) -> float:  # grid_function.hpp:41-43
        b = self.box
        if not contains(b, p):
            return 0.0
        return float(self.values[tuple(v - l for v, l in zip(p, self.lo))])


def restrict_to(f: GF, box: Box) -> GF:  # grid_function.cpp:62-70
    out = np.zeros(tuple(h - l + 1 for l, h in zip(*box)))
    ov = intersect(f.box, box)
    if ov is not None:
        out[_sl(ov, box[0])] = f.values[_sl(ov, f.lo)]
    return GF(box[0], out)


def accumulate(dst: GF, src: GF, scale: float = 1.0) -> None:  # grid_function.cpp:41-52
    ov = intersect(dst.box, src.box)
    if ov is not None:
        dst.values[_sl(ov, dst.lo)] += scale * src.values[_sl(ov, src.lo)]


def flip(f: GF) -> GF:  # grid_function.cpp:72-81
    lo = tuple(-h for h in f.box[1])
    return GF(lo, f.values[tuple(slice(None, None, -1) for _ in f.lo)].copy())


# --- L1: FFT convolution (fft.cpp:58-162) ----------------------------------

def next_pow2(n: int) -> int:  # fft.cpp:58-62
    p = 1
    while p < n:
        p <<= 1
    return p


def conv_padded_shape(a: Box, b: Box) -> List[int]:  # fft.cpp:64-70
    return [next_pow2((ah - al) + (bh - bl) + 1) for al, ah, bl, bh in zip(a[0], a[1], b[0], b[1])]


def fft_convolve(psi: GF, f: GF) -> GF:
    """(psi * f)[y] = sum_x f[x] psi[y - x] on [psi.lo + f.lo, psi.hi + f.hi] (fft.cpp:145-162)."""
    if psi.values.size == 0 or f.values.size == 0:
        raise ValueError("fft_convolve: empty input")  # fft.cpp:146
    shape = conv_padded_shape(psi.box, f.box)
    axes = list(range(len(shape)))
    A = np.fft.fftn(psi.values, s=shape, axes=axes)
    B = np.fft.fftn(f.values, s=shape, axes=axes)
    out_box = minkowski_sum(psi.box, f.box)
    full = np.fft.ifftn(A * B, axes=axes).real
    return GF(out_box[0], full[tuple(slice(0, h - l + 1) for l, h in zip(*out_box))].copy())


def direct_convolve(psi: GF, f: GF) -> GF:
    """Brute-force double sum (tests/test_helpers.hpp:28-40)."""
    ob = minkowski_sum(psi.box, f.box)
    out = np.zeros(tuple(h - l + 1 for l, h in zip(*ob)))
    for x in np.ndindex(*f.values.shape):
        v = f.values[x]
        sl = tuple(slice(xi, xi + s) for xi, s in zip(x, psi.values.shape))
        out[sl] += v * psi.values
    return GF(ob[0], out)


# --- L4: the assembled operator (pc_operator.cpp:26-148) --------------------

class PCOperator:
    """ProductConvolutionOperator restated (pc_operator.hpp:17-66); grid = null (terms_at scans)."""

    def __init__(self, dom_lo, dom_hi, weights: Sequence[GF], impulses: Sequence[GF]):
        if len(weights) != len(impulses):
            raise ValueError("PCOp: one weight per impulse required")  # pc_operator.cpp:34-35
        self.domain: Box = (tuple(dom_lo), tuple(dom_hi))
        self.weights = list(weights)
        self.impulses = list(impulses)

    @classmethod
    def from_inputs(cls, inp) -> "PCOperator":
        return cls(inp.dom_lo, inp.dom_hi, [GF(w.lo, w.values) for w in inp.weights],
                   [GF(e.lo, e.values) for e in inp.impulses])

    @property
    def shape(self):
        return tuple(h - l + 1 for l, h in zip(*self.domain))

    @property
    def rank(self) -> int:
        return len(self.weights)

    def apply(self, f: np.ndarray, ks: Optional[Sequence[int]] = None) -> np.ndarray:
        """g = sum_k crop_Omega(phi_k^E * (w_k . f)), k ascending (pc_operator.cpp:45-56)."""
        f = np.asarray(f, dtype=np.float64)
        if f.size != int(np.prod(self.shape)):
            raise ValueError("PCOp::apply: shape mismatch")
        fg = GF(self.domain[0], f.reshape(self.shape))
        out = GF(self.domain[0], np.zeros(self.shape))
        for k in (range(self.rank) if ks is None else ks):
            w = self.weights[k]
            wf = restrict_to(fg, w.box)  # :51
            wf.values *= w.values  # multiply_into :52 (footprint == w box)
            accumulate(out, fft_convolve(self.impulses[k], wf))  # :53
        return out.values.reshape(-1)

    def apply_adjoint(self, f: np.ndarray, ks: Optional[Sequence[int]] = None) -> np.ndarray:
        """sum_k w_k . (flip(phi_k^E) * f) on Omega cap box(w_k) (pc_operator.cpp:58-69)."""
        f = np.asarray(f, dtype=np.float64)
        if f.size != int(np.prod(self.shape)):
            raise ValueError("PCOp::apply_adjoint: shape mismatch")
        fg = GF(self.domain[0], f.reshape(self.shape))
        out = GF(self.domain[0], np.zeros(self.shape))
        for k in (range(self.rank) if ks is None else ks):
            conv = fft_convolve(flip(self.impulses[k]), fg)
            w = self.weights[k]
            ov = intersect(w.box, conv.box)
            ov = intersect(ov, out.box) if ov is not None else None
            if ov is not None:  # accumulate_product :15-22
                out.values[_sl(ov, out.lo)] += w.values[_sl(ov, w.lo)] * conv.values[_sl(ov, conv.lo)]
        return out.values.reshape(-1)

    def terms_at(self, x) -> List[int]:  # pc_operator.cpp:78-81 (no grid: footprint scan)
        return [k for k in range(self.rank) if contains(self.weights[k].box, x)]

    def entry(self, y, x) -> float:
        """sum_{k: x in U_k} w_k(x) phi_k^E(y - x), k ascending (pc_operator.cpp:84-96)."""
        if not contains(self.domain, y) or not contains(self.domain, x):
            raise ValueError("PCOp::entry: index outside the domain")
        z = tuple(a - b for a, b in zip(y, x))
        s = 0.0
        for k in self.terms_at(x):
            wx = self.weights[k].value_or_zero(x)
            if wx == 0.0:
                continue
            s += wx * self.impulses[k].value_or_zero(z)
        return s

    def apply_block(self, T: Box, S: Box, f: GF, adjoint: bool = False) -> GF:
        """g on T from f on S via G = T - S kernel slices (pc_operator.cpp:98-130)."""
        if intersect(self.domain, T) != (tuple(T[0]), tuple(T[1])) or intersect(self.domain, S) != (tuple(S[0]), tuple(S[1])):
            raise ValueError("PCOp::apply_block: boxes must lie inside the domain")
        out = GF(T[0], np.zeros(tuple(h - l + 1 for l, h in zip(*T))))
        G = minkowski_diff(T, S)
        for k in range(self.rank):
            w, phi = self.weights[k], self.impulses[k]
            if not adjoint:
                if intersect(w.box, S) is None:
                    continue
                wf = restrict_to(f, S)  # overwrite into S (zeros outside f's box)
                wf.values = wf.values * restrict_to(w, S).values  # multiply_into
                sb = intersect(phi.box, G)
                if sb is None:
                    continue
                accumulate(out, fft_convolve(restrict_to(phi, sb), wf))
            else:
                if intersect(w.box, T) is None:
                    continue
                sb = intersect(phi.box, minkowski_diff(S, T))
                if sb is None:
                    continue
                conv = fft_convolve(flip(restrict_to(phi, sb)), restrict_to(f, S))
                ov = intersect(w.box, conv.box)
                ov = intersect(ov, out.box) if ov is not None else None
                if ov is not None:
                    out.values[_sl(ov, out.lo)] += w.values[_sl(ov, w.lo)] * conv.values[_sl(ov, conv.lo)]
        return out

    def dense(self) -> np.ndarray:
        """Dense matrix via apply of basis vectors (verification.cpp:21-33); small N only."""
        N = int(np.prod(self.shape))
        A = np.zeros((N, N))
        for j in range(N):
            e = np.zeros(N)
            e[j] = 1.0
            A[:, j] = self.apply(e)
        return A


# --- estimator (adaptivity.cpp:14-121) -------------------------------------

def estimate(op: PCOperator, Z: np.ndarray, Y: np.ndarray, leaves: Sequence[Box]):
    """Ytilde_i = Atilde* zeta_i (update_samples :75-100), eta_abs/eta_rel (:101-111),
    eta_C per leaf box (eta_for_cells :114-121)."""
    q = Z.shape[0]
    Yt = np.stack([op.apply_adjoint(Z[i]) for i in range(q)])
    D = Yt - Y
    d2 = float(np.sum(D * D))
    y_norm = math.sqrt(float(np.sum(Y * Y)))
    eta_abs = math.sqrt(d2 / q)
    eta_rel = math.sqrt(d2) / y_norm if y_norm > 0 else 0.0
    Dg = D.reshape((q,) + op.shape)
    cells = []
    for lo, hi in leaves:
        ov = intersect(op.domain, (tuple(lo), tuple(hi)))
        s = 0.0 if ov is None else float(np.sum(Dg[(slice(None),) + _sl(ov, op.domain[0])] ** 2))
        cells.append(math.sqrt(s / q))
    return Yt, np.array(cells), eta_abs, eta_rel
