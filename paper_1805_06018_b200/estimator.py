"""GPU-resident a-posteriori estimator, mirroring adaptivity.hpp:14-56.

    est = Estimator(op.domain, q=5, seed=0)        # make_probes' Z (adaptivity.cpp:14-28), on the device
    est.set_y(Y) / est.set_y_from(blur)            # Y = A^* Z; ||Y||_F (make_estimator_state, :30-37)
    eta_abs, eta_rel = est.update(op, changed_ks)  # update_samples (:75-112), same changed_ks checks
    eta_c = est.cells(leaves)                      # eta_for_cells (:114-121)

Z, Y and Ytilde stay in HBM across iterations; only the eta values come back.  Errors carry the
reference's messages (ValueError for std::invalid_argument / std::logic_error).
"""
from __future__ import annotations

import ctypes
from typing import Iterable, Sequence, Tuple

import numpy as np

from . import lib as _L


def _rc(rc: int) -> None:
    if rc == 1:
        raise ValueError(_L.load().pcb_last_error().decode())
    _L.check(rc)


class Estimator:
    def __init__(self, domain: Tuple[Sequence[int], Sequence[int]], q: int, seed: int, device: int = -1,
                 generator: str = "mt19937"):
        """generator: "mt19937" = the reference's probe stream (adaptivity.cpp:19-23, host-drawn);
        "philox" = counter-based Philox normals drawn on the device (throughput runs)."""
        lo, hi = [int(v) for v in domain[0]], [int(v) for v in domain[1]]
        self.dim = len(lo)
        self.domain = (tuple(lo), tuple(hi))
        self.shape = tuple(h - l + 1 for l, h in zip(lo, hi))
        self.n_points = int(np.prod(self.shape))
        self.q = int(q)
        self.seed = int(seed)
        h = _L.vp()
        A = ctypes.c_int64 * self.dim
        _rc(_L.load().pcb_estimator_create_ex(self.dim, A(*lo), A(*hi), self.q, ctypes.c_uint64(self.seed),
                                              int(device), _L.RNG[generator], ctypes.byref(h)))
        self._h = h
        self.eta_abs = None
        self.eta_rel = None

    def close(self) -> None:
        if getattr(self, "_h", None):
            _L.load().pcb_estimator_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def device_pointers(self) -> Tuple[int, int, int]:
        """(Z, Y, Ytilde) device pointers, q x N fp64 each."""
        z, y, t = _L.vp(), _L.vp(), _L.vp()
        _rc(_L.load().pcb_estimator_probes(self._h, ctypes.byref(z), ctypes.byref(y), ctypes.byref(t)))
        return z.value, y.value, t.value

    def set_y(self, Y: np.ndarray) -> None:
        Y = np.ascontiguousarray(Y, dtype=np.float64).reshape(self.q, self.n_points)
        _rc(_L.load().pcb_estimator_set_y(self._h, Y.ctypes.data, 0))

    def set_y_dev(self, dY: int) -> None:
        _rc(_L.load().pcb_estimator_set_y(self._h, dY, 1))

    def set_y_from(self, blur) -> None:
        """Y = A^* Z on the device with a true operator (``true_operator.BlurOperator``)."""
        _rc(_L.load().pcb_estimator_set_y_blur(self._h, blur._h))

    def update(self, op, changed_ks: Iterable[int]) -> Tuple[float, float]:
        ks = np.ascontiguousarray(list(changed_ks), dtype=np.int32)
        ea, er = _L.dbl(), _L.dbl()
        _rc(_L.load().pcb_estimator_update(self._h, op._h, len(ks), ks.ctypes.data if len(ks) else None,
                                           ctypes.byref(ea), ctypes.byref(er)))
        self.eta_abs, self.eta_rel = ea.value, er.value
        return self.eta_abs, self.eta_rel

    def cells(self, leaves: Iterable) -> np.ndarray:
        leaves = list(leaves)
        lo = np.ascontiguousarray([l for l, _ in leaves], dtype=np.int64).reshape(-1)
        hi = np.ascontiguousarray([h for _, h in leaves], dtype=np.int64).reshape(-1)
        out = np.zeros(max(1, len(leaves)))
        _rc(_L.load().pcb_estimator_cells(self._h, len(leaves), lo.ctypes.data if len(leaves) else None,
                                          hi.ctypes.data if len(leaves) else None, out.ctypes.data))
        return out[: len(leaves)]

    def read(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        Z, Y, T = (np.empty((self.q, self.n_points)) for _ in range(3))
        _rc(_L.load().pcb_estimator_read(self._h, Z.ctypes.data, Y.ctypes.data, T.ctypes.data))
        return Z, Y, T
