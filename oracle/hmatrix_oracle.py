"""ORACLE — TEST INFRASTRUCTURE ONLY.  Never imported by the product path.

Pure-Python / numpy restatement of the reference's H-matrix layer (paths relative to
/root/reference/proj/core/src/hmatrix.cpp): the cluster tree, admissibility, the block partition,
the CUR (adaptive cross approximation) compression, the matvec and the PCHM v1 container.  Used by
tests/test_hmatrix_cpu.py and tests/test_gpu_hmatrix.py to check paper_1805_06018_b200/hmatrix.py
(csrc/hmatrix.cpp).

Parity pin: the reference's own known-answer tests for this layer (test_hmatrix.cpp:22-53 tree
shapes, :56-98 admissibility vs brute force, :100-115 partition cover) are re-asserted against this
module in tests/test_hmatrix_cpu.py.  hmatrix.cpp itself is not compiled into oracle/_ref: it needs
Eigen's HouseholderQR / JacobiSVD, which the shim does not provide.
"""
from __future__ import annotations

import math
import struct
from typing import Callable, List, Sequence, Tuple

import numpy as np


def delinearize(lo, hi, lin: int) -> Tuple[int, ...]:
    """hmatrix.cpp:13-22 (last axis fastest)."""
    d = len(lo)
    p = [0] * d
    for i in range(d - 1, -1, -1):
        w = hi[i] - lo[i] + 1
        p[i] = lo[i] + lin % w
        lin //= w
    return tuple(p)


def points_bbox(lo, hi, perm, b, e):
    """hmatrix.cpp:24-36."""
    pts = [delinearize(lo, hi, perm[i]) for i in range(b, e)]
    return tuple(min(p[a] for p in pts) for a in range(len(lo))), tuple(max(p[a] for p in pts) for a in range(len(lo)))


class Tree:
    """ClusterTree::build (hmatrix.cpp:40-76)."""

    def __init__(self, lo, hi, leaf_cap: int):
        if leaf_cap < 1:
            raise ValueError("ClusterTree: leaf_cap >= 1 required")
        self.lo, self.hi, self.leaf_cap = tuple(lo), tuple(hi), leaf_cap
        self.N = int(np.prod([h - l + 1 for l, h in zip(lo, hi)]))
        self.perm = list(range(self.N))
        self.nodes: List[dict] = []
        self._rec(0, self.N)

    def _rec(self, b, e):
        nid = len(self.nodes)
        self.nodes.append(dict(begin=b, end=e, child_lo=-1, child_hi=-1, split_axis=-1,
                               bbox=points_bbox(self.lo, self.hi, self.perm, b, e)))
        if e - b > self.leaf_cap:
            blo, bhi = self.nodes[nid]["bbox"]
            axis = 0
            for a in range(1, len(self.lo)):
                if bhi[a] - blo[a] > bhi[axis] - blo[axis]:
                    axis = a
            seg = self.perm[b:e]
            seg.sort(key=lambda x: (delinearize(self.lo, self.hi, x)[axis], x))
            self.perm[b:e] = seg
            mid = b + (e - b + 1) // 2
            lo_id = self._rec(b, mid)
            hi_id = self._rec(mid, e)
            self.nodes[nid].update(child_lo=lo_id, child_hi=hi_id, split_axis=axis)
        return nid

    def is_leaf(self, i):
        return self.nodes[i]["child_lo"] < 0

    def size(self, i):
        return self.nodes[i]["end"] - self.nodes[i]["begin"]

    def point_at(self, pos):
        return delinearize(self.lo, self.hi, self.perm[pos])

    def diameter(self, i):
        """hmatrix.cpp:90-95 (extent = hi - lo)."""
        lo, hi = self.nodes[i]["bbox"]
        return math.sqrt(sum(float((h - l) * (h - l)) for l, h in zip(lo, hi)))

    @staticmethod
    def distance(a, b):
        """hmatrix.cpp:97-104."""
        s = 0.0
        for i in range(len(a[0])):
            gap = max(0, max(a[0][i] - b[1][i], b[0][i] - a[1][i]))
            s += float(gap * gap)
        return math.sqrt(s)

    def admissible(self, t, s):
        """hmatrix.cpp:106-110."""
        return self.distance(self.nodes[t]["bbox"], self.nodes[s]["bbox"]) >= min(self.diameter(t), self.diameter(s))


def partition(tree: Tree) -> List[Tuple[int, int, bool]]:
    """The block recursion of assemble_hmatrix (hmatrix.cpp:345-375), preorder: (t, s, low_rank)."""
    out = []

    def rec(t, s):
        if tree.admissible(t, s):
            out.append((t, s, True))
            return
        if tree.is_leaf(t) and tree.is_leaf(s):
            out.append((t, s, False))
            return
        ts = [t] if tree.is_leaf(t) else [tree.nodes[t]["child_lo"], tree.nodes[t]["child_hi"]]
        ss = [s] if tree.is_leaf(s) else [tree.nodes[s]["child_lo"], tree.nodes[s]["child_hi"]]
        for tc in ts:
            for sc in ss:
                rec(tc, sc)

    rec(0, 0)
    return out


def dense_block(entry: Callable, tree: Tree, t, s) -> np.ndarray:
    """hmatrix.cpp:138-150."""
    tn, sn = tree.nodes[t], tree.nodes[s]
    out = np.zeros((tree.size(t), tree.size(s)))
    for j in range(tree.size(s)):
        x = tree.point_at(sn["begin"] + j)
        for i in range(tree.size(t)):
            out[i, j] = entry(tree.point_at(tn["begin"] + i), x)
    return out


def compress_cur(entry: Callable, tree: Tree, t, s, tol: float, fixed_rank: int = 0):
    """Partially pivoted ACA (hmatrix.cpp:236-318); returns (B, C, capped)."""
    tn, sn = tree.nodes[t], tree.nodes[s]
    nt, ns = tree.size(t), tree.size(s)
    max_rank = min(fixed_rank, min(nt, ns)) if fixed_rank > 0 else min(nt, ns)
    row_of = lambda i: np.array([entry(tree.point_at(tn["begin"] + i), tree.point_at(sn["begin"] + j)) for j in range(ns)])
    col_of = lambda j: np.array([entry(tree.point_at(tn["begin"] + i), tree.point_at(sn["begin"] + j)) for i in range(nt)])
    us, vs = [], []
    used = [False] * nt
    fro2 = 0.0
    next_row = 0
    while len(us) < max_rank:
        r = row_of(next_row)
        for k in range(len(us)):
            r = r - us[k][next_row] * vs[k]
        used[next_row] = True
        jpiv = int(np.argmax(np.abs(r)))
        rmax = abs(r[jpiv])
        if rmax == 0.0:
            cand = next((i for i in range(nt) if not used[i]), -1)
            if cand < 0:
                break
            next_row = cand
            continue
        v = r / r[jpiv]
        u = col_of(jpiv)
        for k in range(len(us)):
            u = u - vs[k][jpiv] * us[k]
        cross = sum(float(us[k] @ u) * float(vs[k] @ v) for k in range(len(us)))
        fro2 += 2.0 * cross + float(u @ u) * float(v @ v)
        us.append(u)
        vs.append(v)
        if np.linalg.norm(u) * np.linalg.norm(v) <= tol * math.sqrt(max(fro2, 1e-300)):
            break
        next_row, best = -1, -1.0
        for i in range(nt):
            if not used[i] and abs(u[i]) > best:
                best, next_row = abs(u[i]), i
        if next_row < 0:
            break
    capped = len(us) >= max_rank and fixed_rank > 0
    B = np.stack(us, 1) if us else np.zeros((nt, 0))
    C = np.stack(vs, 0) if vs else np.zeros((0, ns))
    return B, C, capped


def matvec(tree: Tree, blocks, f: np.ndarray) -> np.ndarray:
    """HMatrix::matvec (hmatrix.cpp:379-400); blocks: (t, s, low_rank, B, C, dense)."""
    out = np.zeros(tree.N)
    perm = np.asarray(tree.perm)
    for t, s, lr, B, C, D in blocks:
        tn, sn = tree.nodes[t], tree.nodes[s]
        x = f[perm[sn["begin"]:sn["end"]]]
        y = B @ (C @ x) if lr else D @ x
        np.add.at(out, perm[tn["begin"]:tn["end"]], y)
    return out


# --- PCHM v1 (hmatrix.cpp:402-526) -------------------------------------------------------------

def write_pchm(path, lo, hi, leaf_cap, perm, nodes, blocks) -> None:
    """save_hmatrix (hmatrix.cpp:433-471); nodes: dicts with begin/end/split_axis/child_lo/child_hi;
    blocks: (t, s, low_rank, B, C, dense)."""
    with open(path, "wb") as fp:
        fp.write(b"PCHM")
        fp.write(struct.pack("<IIQI", 1, len(lo), len(perm), leaf_cap))
        for l, h in zip(lo, hi):
            fp.write(struct.pack("<qq", l, h))
        fp.write(np.asarray(perm, dtype="<i8").tobytes())
        fp.write(struct.pack("<Q", len(nodes)))
        for n in nodes:
            fp.write(struct.pack("<qqiii", n["begin"], n["end"], n["split_axis"], n["child_lo"], n["child_hi"]))
        fp.write(struct.pack("<Q", len(blocks)))

        def mat(m):
            m = np.ascontiguousarray(m, dtype="<f8")
            fp.write(struct.pack("<QQ", m.shape[0], m.shape[1]))
            fp.write(m.tobytes())

        for t, s, lr, B, C, D in blocks:
            fp.write(struct.pack("<iiB", t, s, 0 if lr else 1))
            if lr:
                fp.write(struct.pack("<I", B.shape[1]))
                mat(B)
                mat(C)
            else:
                fp.write(struct.pack("<I", 0))
                mat(D)


def read_pchm(path):
    """load_hmatrix (hmatrix.cpp:473-526) -> dict(lo, hi, N, leaf_cap, perm, nodes, blocks)."""
    with open(path, "rb") as fp:
        buf = fp.read()
    if buf[:4] != b"PCHM":
        raise ValueError("load_hmatrix: bad magic")
    off = 4
    ver, d, N, cap = struct.unpack_from("<IIQI", buf, off)
    off += 20
    if ver != 1:
        raise ValueError("load_hmatrix: unsupported version")
    lo, hi = [], []
    for _ in range(d):
        l, h = struct.unpack_from("<qq", buf, off)
        off += 16
        lo.append(l)
        hi.append(h)
    n = int(np.prod([h - l + 1 for l, h in zip(lo, hi)]))
    perm = np.frombuffer(buf, dtype="<i8", count=n, offset=off).copy()
    off += 8 * n
    (nn,) = struct.unpack_from("<Q", buf, off)
    off += 8
    nodes = []
    for _ in range(nn):
        b, e, ax, cl, ch = struct.unpack_from("<qqiii", buf, off)
        off += 28
        nodes.append(dict(begin=b, end=e, split_axis=ax, child_lo=cl, child_hi=ch))
    (nb,) = struct.unpack_from("<Q", buf, off)
    off += 8

    def mat():
        nonlocal off
        r, c = struct.unpack_from("<QQ", buf, off)
        off += 16
        m = np.frombuffer(buf, dtype="<f8", count=r * c, offset=off).reshape(r, c).copy()
        off += 8 * r * c
        return m

    blocks = []
    for _ in range(nb):
        t, s, kind = struct.unpack_from("<iiB", buf, off)
        off += 9
        (rank,) = struct.unpack_from("<I", buf, off)
        off += 4
        if kind == 0:
            B, C = mat(), mat()
            blocks.append((t, s, True, B, C, None))
        else:
            blocks.append((t, s, False, None, None, mat()))
    if off != len(buf):
        raise ValueError("load_hmatrix: trailing bytes")
    return dict(lo=tuple(lo), hi=tuple(hi), N=N, leaf_cap=cap, perm=perm, nodes=nodes, blocks=blocks)
