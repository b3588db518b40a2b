"""H-matrix assembly over the GPU operator and the PCHM container.

Mirrors the reference's ``hmatrix.hpp`` (ClusterTree, admissible, compress_block, HMatrix,
assemble_hmatrix, save_hmatrix / load_hmatrix) over ``pcb_cluster_tree`` / ``pcb_hmatrix_*``
(include/pcb/pcb.h; native C++ in csrc/hmatrix.cpp).  Entry and block-apply evaluations run on the
GPU, batched across blocks; the cluster tree, the partition, the factor algebra and the container
are host code, as in the reference.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import lib as _L

METHODS = {"randomized": 0, "cur": 1}


def _rc(rc: int) -> None:
    if rc == 1:
        raise ValueError(_L.load().pcb_last_error().decode())
    _L.check(rc)


@dataclass
class ClusterNode:
    begin: int
    end: int
    split_axis: int
    child_lo: int
    child_hi: int
    lo: Tuple[int, ...]
    hi: Tuple[int, ...]

    def is_leaf(self) -> bool:
        return self.child_lo < 0

    def size(self) -> int:
        return self.end - self.begin


@dataclass
class Block:
    t_node: int
    s_node: int
    low_rank: bool
    B: Optional[np.ndarray] = None
    C: Optional[np.ndarray] = None
    dense: Optional[np.ndarray] = None

    @property
    def rank(self) -> int:
        return 0 if self.B is None else self.B.shape[1]


class HMatrix:
    def __init__(self, handle):
        self._h = handle
        info = _L.HMatrixInfo()
        _rc(_L.load().pcb_hmatrix_get_info(self._h, ctypes.byref(info)))
        self.info = info.as_dict()
        self.dim = self.info["dim"]
        self.n_points = self.info["n_points"]

    # --- construction ---------------------------------------------------------------------
    @classmethod
    def cluster_tree(cls, domain, leaf_cap: int) -> "HMatrix":
        """ClusterTree::build (hmatrix.cpp:40-76): the tree alone, no blocks."""
        lo, hi = [int(v) for v in domain[0]], [int(v) for v in domain[1]]
        A = ctypes.c_int64 * len(lo)
        h = _L.vp()
        _rc(_L.load().pcb_cluster_tree(len(lo), A(*lo), A(*hi), int(leaf_cap), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def assemble(cls, op, tol: float, leaf_cap: int, method: str = "randomized", fixed_rank: int = 0) -> "HMatrix":
        """assemble_hmatrix (hmatrix.cpp:338-377) of a ``ProductConvolutionOperator``."""
        h = _L.vp()
        _rc(_L.load().pcb_hmatrix_assemble(op._h, float(tol), int(leaf_cap), METHODS[method], int(fixed_rank),
                                           ctypes.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path: str) -> "HMatrix":
        h = _L.vp()
        _rc(_L.load().pcb_hmatrix_load(str(path).encode(), ctypes.byref(h)))
        return cls(h)

    def save(self, path: str) -> None:
        _rc(_L.load().pcb_hmatrix_save(self._h, str(path).encode()))

    def compress(self, op, pairs: Sequence[Tuple[int, int]], method: str = "randomized", tol: float = 1e-8,
                 fixed_rank: int = 0) -> List[Block]:
        """compress_block (hmatrix.cpp:320-336) for (t, s) node pairs; returns the new blocks."""
        t = np.ascontiguousarray([p[0] for p in pairs], dtype=np.int32)
        s = np.ascontiguousarray([p[1] for p in pairs], dtype=np.int32)
        n0 = self._refresh()["n_blocks"]
        _rc(_L.load().pcb_hmatrix_compress(op._h, self._h, len(t), t.ctypes.data if len(t) else None,
                                           s.ctypes.data if len(s) else None, METHODS[method], float(tol),
                                           int(fixed_rank)))
        n1 = self._refresh()["n_blocks"]
        return [self.block(i) for i in range(n0, n1)]

    def _refresh(self) -> dict:
        info = _L.HMatrixInfo()
        _rc(_L.load().pcb_hmatrix_get_info(self._h, ctypes.byref(info)))
        self.info = info.as_dict()
        return self.info

    def close(self) -> None:
        if getattr(self, "_h", None):
            _L.load().pcb_hmatrix_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- inspection -------------------------------------------------------------------------
    def perm(self) -> np.ndarray:
        p = np.empty(self.n_points, dtype=np.int64)
        _rc(_L.load().pcb_hmatrix_tree(self._h, p.ctypes.data, None, None, None))
        return p

    def nodes(self) -> List[ClusterNode]:
        n = self._refresh()["n_nodes"]
        rng = np.empty((n, 2), dtype=np.int64)
        links = np.empty((n, 3), dtype=np.int32)
        bbox = np.empty((n, 2 * self.dim), dtype=np.int64)
        _rc(_L.load().pcb_hmatrix_tree(self._h, None, rng.ctypes.data, links.ctypes.data, bbox.ctypes.data))
        d = self.dim
        return [ClusterNode(int(rng[i, 0]), int(rng[i, 1]), int(links[i, 0]), int(links[i, 1]), int(links[i, 2]),
                            tuple(int(v) for v in bbox[i, :d]), tuple(int(v) for v in bbox[i, d:])) for i in range(n)]

    def admissible(self, t: int, s: int) -> Tuple[bool, float, float, float]:
        adm = ctypes.c_int32()
        dist, dt, ds = _L.dbl(), _L.dbl(), _L.dbl()
        _rc(_L.load().pcb_hmatrix_admissible(self._h, int(t), int(s), ctypes.byref(adm), ctypes.byref(dist),
                                             ctypes.byref(dt), ctypes.byref(ds)))
        return bool(adm.value), dist.value, dt.value, ds.value

    def block(self, i: int) -> Block:
        tsk = np.empty(3, dtype=np.int32)
        rcr = np.empty(3, dtype=np.int64)
        _rc(_L.load().pcb_hmatrix_block(self._h, int(i), tsk.ctypes.data, rcr.ctypes.data, None, None, None))
        rows, cols, rank = (int(v) for v in rcr)
        if tsk[2] == 0:
            B = np.empty((rows, rank))
            C = np.empty((rank, cols))
            _rc(_L.load().pcb_hmatrix_block(self._h, int(i), None, None, B.ctypes.data, C.ctypes.data, None))
            return Block(int(tsk[0]), int(tsk[1]), True, B=B, C=C)
        D = np.empty((rows, cols))
        _rc(_L.load().pcb_hmatrix_block(self._h, int(i), None, None, None, None, D.ctypes.data))
        return Block(int(tsk[0]), int(tsk[1]), False, dense=D)

    def blocks(self) -> List[Block]:
        return [self.block(i) for i in range(self._refresh()["n_blocks"])]

    def matvec(self, f: np.ndarray) -> np.ndarray:
        f = np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
        if f.size != self.n_points:
            raise ValueError("HMatrix::matvec: size mismatch")
        g = np.empty_like(f)
        _rc(_L.load().pcb_hmatrix_matvec(self._h, f.ctypes.data, g.ctypes.data))
        return g

    def matvec_batch(self, F: np.ndarray, device: int = 0) -> np.ndarray:
        """B products at once on the GPU (pcb_hmatrix_matvec_batch): bit-identical to matvec per vector."""
        F = np.ascontiguousarray(F, dtype=np.float64)
        if F.ndim != 2 or F.shape[1] != self.n_points:
            raise ValueError("HMatrix::matvec: size mismatch")
        G = np.empty_like(F)
        _rc(_L.load().pcb_hmatrix_matvec_batch(self._h, int(device), F.shape[0], F.ctypes.data, G.ctypes.data))
        return G
