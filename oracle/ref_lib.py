"""ORACLE — TEST INFRASTRUCTURE ONLY.  ctypes binding of oracle/_ref/libpcopref.so.

That library is the reference's own apply path (pc_operator.cpp, fft.cpp,
grid_function.cpp, box.cpp, impulse.cpp, adaptivity.cpp) compiled verbatim
from /root/reference/proj/core/src against the shims in oracle/shim/ (see
oracle/Makefile).  Used by tests/ as the parity pin and by bench.py
``--impl reference`` / ``cpu_baseline`` as the reference CPU implementation.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libpcopref.so")

_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle)")
        L = ctypes.CDLL(LIB_PATH)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_create.restype = ctypes.c_void_p
        L.ref_destroy.argtypes = [ctypes.c_void_p]
        for name in ("ref_apply", "ref_apply_adjoint"):
            getattr(L, name).argtypes = [ctypes.c_void_p, _dp, _dp]
        L.ref_apply_batch_threads.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _dp, _dp, ctypes.c_int]
        L.ref_entries.argtypes = [ctypes.c_void_p, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64), _dp]
        L.ref_apply_block.argtypes = [ctypes.c_void_p] + [ctypes.POINTER(_i64)] * 4 + [_dp, ctypes.c_int, _dp]
        L.ref_normal_fill.argtypes = [ctypes.c_uint64, _i64, _dp]
        L.ref_hmatrix_assemble.restype = ctypes.c_void_p
        L.ref_hmatrix_assemble.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.ref_hmatrix_destroy.argtypes = [ctypes.c_void_p]
        L.ref_hmatrix_save.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.ref_hmatrix_load.restype = ctypes.c_void_p
        L.ref_hmatrix_load.argtypes = [ctypes.c_char_p]
        L.ref_hmatrix_matvec.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.ref_hmatrix_info.argtypes = [ctypes.c_void_p, ctypes.POINTER(_i64)]
        L.ref_hmatrix_block.argtypes = [ctypes.c_void_p, _i64, ctypes.POINTER(_i64), _dp, _dp, _dp]
        L.ref_estimate.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp, ctypes.c_int, ctypes.POINTER(_i64),
                                   ctypes.POINTER(_i64), _dp, _dp, _dp, _dp]
        _lib = L
    return _lib


def _arr(seq, ct):
    seq = list(seq)
    return (ct * max(1, len(seq)))(*seq)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _check(rc: int):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib().ref_last_error().decode()}")


class RefOperator:
    """The reference ProductConvolutionOperator built from explicit inputs (grid = null)."""

    def __init__(self, inp, ks: Optional[Sequence[int]] = None):
        L = lib()
        ks = list(range(inp.rank)) if ks is None else list(ks)
        d = inp.dim
        self.dim = d
        self.N = inp.n_points
        self._keep = []
        w_lo, w_hi, p_lo, p_hi, w_ptr, p_ptr = [], [], [], [], [], []
        for k in ks:
            w = inp.weights[k]
            e = inp.impulses[k]
            wv = np.ascontiguousarray(w.values, dtype=np.float64)
            ev = np.ascontiguousarray(e.values, dtype=np.float64)
            self._keep += [wv, ev]
            w_lo += list(w.lo)
            w_hi += list(w.hi)
            p_lo += list(e.lo)
            p_hi += list(e.hi)
            w_ptr.append(wv.ctypes.data)
            p_ptr.append(ev.ctypes.data)
        PP = ctypes.c_void_p * max(1, len(ks))
        self.h = L.ref_create(ctypes.c_int(d), _arr(inp.dom_lo, _i64), _arr(inp.dom_hi, _i64), ctypes.c_int(len(ks)),
                              _arr(w_lo, _i64), _arr(w_hi, _i64), PP(*w_ptr), _arr(p_lo, _i64), _arr(p_hi, _i64),
                              PP(*p_ptr))
        if not self.h:
            raise RuntimeError(f"ref_create failed: {L.ref_last_error().decode()}")

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ref_destroy(self.h)
                self.h = None
        except Exception:  # interpreter shutdown
            pass

    def apply(self, f: np.ndarray, adjoint: bool = False) -> np.ndarray:
        f = np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
        g = np.zeros(self.N)
        fn = lib().ref_apply_adjoint if adjoint else lib().ref_apply
        _check(fn(self.h, _dptr(f), _dptr(g)))
        return g

    def apply_batch(self, F: np.ndarray, adjoint: bool = False, threads: int = 1) -> np.ndarray:
        F = np.ascontiguousarray(F, dtype=np.float64)
        B = F.shape[0]
        G = np.zeros((B, self.N))
        _check(lib().ref_apply_batch_threads(self.h, int(adjoint), B, _dptr(F), _dptr(G), threads))
        return G

    def entries(self, y: np.ndarray, x: np.ndarray) -> np.ndarray:
        y = np.ascontiguousarray(y, dtype=np.int64).reshape(-1, self.dim)
        x = np.ascontiguousarray(x, dtype=np.int64).reshape(-1, self.dim)
        out = np.zeros(y.shape[0])
        _check(lib().ref_entries(self.h, y.shape[0], y.ctypes.data_as(ctypes.POINTER(_i64)),
                                 x.ctypes.data_as(ctypes.POINTER(_i64)), _dptr(out)))
        return out

    def apply_block(self, T, S, f: np.ndarray, adjoint: bool = False) -> np.ndarray:
        """Reference apply_block (pc_operator.cpp:98-130): f on box S -> g on box T."""
        f = np.ascontiguousarray(f, dtype=np.float64)
        shape = tuple(h - l + 1 for l, h in zip(T[0], T[1]))
        out = np.zeros(int(np.prod(shape)))
        L = lib()
        _check(L.ref_apply_block(self.h, _arr(T[0], _i64), _arr(T[1], _i64), _arr(S[0], _i64), _arr(S[1], _i64),
                                 _dptr(f), int(adjoint), _dptr(out)))
        return out.reshape(shape)

    def estimate(self, Z: np.ndarray, Y: np.ndarray, leaves):
        Z = np.ascontiguousarray(Z, dtype=np.float64)
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        q = Z.shape[0]
        lo = np.ascontiguousarray([l for l, _ in leaves], dtype=np.int64).reshape(-1)
        hi = np.ascontiguousarray([h for _, h in leaves], dtype=np.int64).reshape(-1)
        yt = np.zeros_like(Z)
        cells = np.zeros(len(leaves))
        ea, er = ctypes.c_double(), ctypes.c_double()
        _check(lib().ref_estimate(self.h, q, _dptr(Z), _dptr(Y), len(leaves), lo.ctypes.data_as(ctypes.POINTER(_i64)),
                                  hi.ctypes.data_as(ctypes.POINTER(_i64)), _dptr(yt), _dptr(cells),
                                  ctypes.byref(ea), ctypes.byref(er)))
        return yt, cells, ea.value, er.value


class RefHMatrix:
    """The reference's assemble_hmatrix / HMatrix / PCHM container (hmatrix.cpp:338-526), compiled
    verbatim against oracle/shim/Eigen (Householder QR, one-sided Jacobi SVD)."""

    def __init__(self, handle, N: int):
        if not handle:
            raise RuntimeError(f"reference H-matrix failed: {lib().ref_last_error().decode()}")
        self.h = handle
        self.N = N

    @classmethod
    def assemble(cls, op: "RefOperator", tol: float, leaf_cap: int, method: str = "randomized",
                 fixed_rank: int = 0) -> "RefHMatrix":
        m = {"randomized": 0, "cur": 1}[method]
        return cls(lib().ref_hmatrix_assemble(op.h, float(tol), int(leaf_cap), m, int(fixed_rank)), op.N)

    @classmethod
    def load(cls, path: str, N: int) -> "RefHMatrix":
        return cls(lib().ref_hmatrix_load(str(path).encode()), N)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ref_hmatrix_destroy(self.h)
                self.h = None
        except Exception:  # interpreter shutdown
            pass

    def save(self, path: str) -> None:
        _check(lib().ref_hmatrix_save(self.h, str(path).encode()))

    def matvec(self, f: np.ndarray) -> np.ndarray:
        f = np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
        g = np.zeros(self.N)
        _check(lib().ref_hmatrix_matvec(self.h, _dptr(f), _dptr(g)))
        return g

    def info(self) -> dict:
        c = (_i64 * 5)()
        _check(lib().ref_hmatrix_info(self.h, c))
        return {"n_blocks": c[0], "n_low_rank": c[1], "max_rank": c[2], "any_rank_capped": bool(c[3]),
                "n_nodes": c[4]}

    def block(self, i: int):
        """(t_node, s_node, low_rank, B, C, dense) of block i."""
        meta = (_i64 * 6)()
        _check(lib().ref_hmatrix_block(self.h, int(i), meta, None, None, None))
        t, s, lr, rows, cols, rank = (int(v) for v in meta)
        if lr:
            B, C = np.zeros((rows, rank)), np.zeros((rank, cols))
            _check(lib().ref_hmatrix_block(self.h, int(i), meta, _dptr(B), _dptr(C), None))
            return t, s, True, B, C, None
        D = np.zeros((rows, cols))
        _check(lib().ref_hmatrix_block(self.h, int(i), meta, None, None, _dptr(D)))
        return t, s, False, None, None, D


def normal_vectors(seed: int, count: int, n: int) -> np.ndarray:
    """count x n draws of std::mt19937_64(seed) + std::normal_distribution<double>
    (adaptivity.cpp:19-23), drawn inside the reference build (no product library loaded)."""
    out = np.empty(count * n)
    _check(lib().ref_normal_fill(ctypes.c_uint64(seed), count * n, _dptr(out)))
    return out.reshape(count, n)


def apply_split(inp, F: np.ndarray, adjoint: bool = False, threads: int = 0) -> np.ndarray:
    """The reference apply / apply_adjoint (pc_operator.cpp:45-69) of the FULL operator, with its
    serial k-loop split across host threads: thread t owns the terms k = t, t+T, t+2T, ... as its
    own reference ProductConvolutionOperator and the partial outputs are summed (linearity of the
    k-sum).  Each thread runs the unmodified reference routine; only the order of the final sum
    over threads differs from the reference's single ascending-k accumulation (rounding ~1e-16).
    ctypes releases the GIL during the calls, so the threads run concurrently."""
    from concurrent.futures import ThreadPoolExecutor

    F = np.atleast_2d(np.ascontiguousarray(F, dtype=np.float64))
    T = max(1, min(threads or (os.cpu_count() or 1), inp.rank))
    parts = [list(range(t, inp.rank, T)) for t in range(T)]
    ops = [RefOperator(inp, ks=p) for p in parts]
    out = np.zeros_like(F)
    for b in range(F.shape[0]):
        with ThreadPoolExecutor(T) as ex:
            res = list(ex.map(lambda o: o.apply(F[b], adjoint=adjoint), ops))
        for r in res:  # fixed thread order: deterministic
            out[b] += r
    return out


def entries_split(op: "RefOperator", y: np.ndarray, x: np.ndarray, threads: int = 0) -> np.ndarray:
    """Reference entry (pc_operator.cpp:84-96) for many (y, x) pairs, chunked across host threads
    (entry is pure and thread-safe, pc_operator.hpp:15-16).  Every value is the reference's own."""
    from concurrent.futures import ThreadPoolExecutor

    y = np.ascontiguousarray(y, dtype=np.int64).reshape(-1, op.dim)
    x = np.ascontiguousarray(x, dtype=np.int64).reshape(-1, op.dim)
    T = max(1, threads or (os.cpu_count() or 1))
    cuts = np.linspace(0, y.shape[0], T + 1).astype(np.int64)
    with ThreadPoolExecutor(T) as ex:
        res = list(ex.map(lambda i: op.entries(y[cuts[i]:cuts[i + 1]], x[cuts[i]:cuts[i + 1]]), range(T)))
    return np.concatenate(res) if res else np.zeros(0)


def fft_convolve(psi_lo, psi, f_lo, f):
    """Reference fft_convolve (fft.cpp:145-151); psi=None exercises the empty-input check."""
    L = lib()
    d = len(f_lo)
    f = np.ascontiguousarray(f, dtype=np.float64)
    f_hi = [l + s - 1 for l, s in zip(f_lo, f.shape)]
    if psi is not None:
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        p_hi = [l + s - 1 for l, s in zip(psi_lo, psi.shape)]
        shape = [a + b - 1 for a, b in zip(psi.shape, f.shape)]
    else:
        p_hi = list(psi_lo)
        shape = list(f.shape)
    cap = int(np.prod(shape))
    out = np.zeros(cap)
    olo, ohi = (_i64 * d)(), (_i64 * d)()
    rc = L.ref_fft_convolve(ctypes.c_int(d), _arr(psi_lo, _i64), _arr(p_hi, _i64),
                            _dptr(psi) if psi is not None else None, _arr(f_lo, _i64), _arr(f_hi, _i64),
                            _dptr(f), olo, ohi, _dptr(out), _i64(cap))
    _check(rc)
    lo = tuple(olo[i] for i in range(d))
    hi = tuple(ohi[i] for i in range(d))
    return lo, out[: int(np.prod([h - l + 1 for l, h in zip(lo, hi)]))].reshape([h - l + 1 for l, h in zip(lo, hi)])


def conv_padded_shape(a_lo, a_hi, b_lo, b_hi):
    d = len(a_lo)
    shape = (ctypes.c_int * d)()
    _check(lib().ref_conv_padded_shape(ctypes.c_int(d), _arr(a_lo, _i64), _arr(a_hi, _i64), _arr(b_lo, _i64),
                                       _arr(b_hi, _i64), shape))
    return [shape[i] for i in range(d)]


def extend_impulse(dom_lo, dom_hi, k, nbr_ids, nbr_pts, nbr_phis):
    """Reference extend_impulse (impulse.cpp:61-89) with c_k as build_extension_weights fills it."""
    L = lib()
    d = len(dom_lo)
    keep = [np.ascontiguousarray(p.values, dtype=np.float64) for p in nbr_phis]
    plo = [v for p in nbr_phis for v in p.lo]
    phi = [v for p in nbr_phis for v in p.hi]
    PP = ctypes.c_void_p * len(keep)
    olo, ohi = (_i64 * d)(), (_i64 * d)()
    args = [ctypes.c_int(d), _arr(dom_lo, _i64), _arr(dom_hi, _i64), ctypes.c_int(k), ctypes.c_int(len(nbr_ids)),
            _arr(nbr_ids, ctypes.c_int), _arr([v for p in nbr_pts for v in p], _i64), _arr(plo, _i64), _arr(phi, _i64),
            PP(*[a.ctypes.data for a in keep]), olo, ohi]
    _check(L.ref_extend_impulse(*args, None, _i64(0)))
    shape = [ohi[i] - olo[i] + 1 for i in range(d)]
    out = np.zeros(int(np.prod(shape)))
    _check(L.ref_extend_impulse(*args, _dptr(out), _i64(out.size)))
    return tuple(olo[i] for i in range(d)), out.reshape(shape)
