"""The true operator A of the benchmark configurations on the GPU.

``BlurOperator`` wraps ``pcb_blur_*`` (include/pcb/pcb.h): the direct fp64 stencil of the
truncated, spatially varying Gaussian blur the configurations define (inputs.py ``BlurSpec``).
It plays the reference's ``OperatorHandle`` role for the true operator (operators.hpp:20-51):
``compute_impulse`` needs ``A delta_p`` (impulse.cpp:5-15) and ``make_probes`` needs
``Y = A^* Z`` (adaptivity.cpp:14-28).  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from . import lib as _L


class BlurOperator:
    def __init__(self, shape: Sequence[int], sigma: np.ndarray):
        self.shape = tuple(int(v) for v in shape)
        self.dim = len(self.shape)
        self.N = int(np.prod(self.shape))
        sig = np.ascontiguousarray(sigma, dtype=np.float64).reshape(self.N, self.dim)
        L = _L.load()
        h = ctypes.c_void_p()
        _L.check_blur(L.pcb_blur_create(self.dim, (ctypes.c_int64 * self.dim)(*self.shape),
                                        sig.ctypes.data, ctypes.byref(h)))
        self._h = h

    @classmethod
    def from_spec(cls, blur) -> "BlurOperator":
        return cls((blur.n,) * blur.dim, blur.sigma_field())

    def close(self) -> None:
        if getattr(self, "_h", None):
            _L.load().pcb_blur_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _run(self, F: np.ndarray, adjoint: bool) -> np.ndarray:
        single = F.ndim == self.dim or (F.ndim == 1 and F.size == self.N)
        X = np.ascontiguousarray(F, dtype=np.float64).reshape(-1, self.N)
        G = np.empty_like(X)
        _L.check_blur(_L.load().pcb_blur_apply(self._h, X.shape[0], X.ctypes.data, G.ctypes.data, int(adjoint), 0,
                                               None))
        return G.reshape(F.shape) if single else G.reshape((X.shape[0],) + self.shape)

    def apply(self, F: np.ndarray) -> np.ndarray:
        """A f for one field (shape = lattice) or a batch (B, *lattice)."""
        return self._run(F, False)

    def apply_adjoint(self, F: np.ndarray) -> np.ndarray:
        return self._run(F, True)

    def apply_dev(self, B: int, F_ptr: int, G_ptr: int, adjoint: bool = False, stream: int = 0) -> None:
        """Device pointers (B x N fp64), ordered on ``stream``."""
        _L.check_blur(_L.load().pcb_blur_apply(self._h, B, F_ptr, G_ptr, int(adjoint), 1, stream or None))
