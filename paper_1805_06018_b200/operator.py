"""Python mirror of ``pcop::ProductConvolutionOperator`` over the C ABI.

Same names, argument meaning and error behaviour as the reference
(proj/core/include/pcop/pc_operator.hpp:17-66):

* ``ProductConvolutionOperator(domain, weights, impulses)`` — pc_operator.cpp:26-38
  (``ValueError`` for a weight/impulse count mismatch, like std::invalid_argument);
* ``apply(f)`` / ``apply_adjoint(f)`` — pc_operator.cpp:45-69 (``ValueError`` "shape mismatch");
* ``entry(y, x)`` — pc_operator.cpp:84-96 (``ValueError`` "index outside the domain");
* ``apply_batch`` / ``apply_adjoint_batch`` — batched forms (fft_convolve_batch analogue, fft.cpp:164-181);
* ``entries`` / ``blocks`` — vectorised entry gather for H-matrix conversion (hmatrix.cpp:138-150);
* ``probe_estimate`` — the randomized estimator's adjoint samples and eta (adaptivity.cpp:75-121).

All compute runs in the sm_100a kernels of ``lib/libpcop_b200.so``; numpy arrays are host
buffers, and the ``*_dev`` methods take device pointers (e.g. ``torch.Tensor.data_ptr()``).
"""
from __future__ import annotations

import ctypes
from typing import Iterable, Optional, Sequence, Tuple

import numpy as np

from . import lib as _L


def _i64arr(vals) -> ctypes.Array:
    vals = [int(v) for v in vals]
    return (_L.i64 * max(1, len(vals)))(*vals)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class ProductConvolutionOperator:
    """Immutable assembled operator; kernels, spectra and scratch live on one B200."""

    def __init__(self, domain: Tuple[Sequence[int], Sequence[int]], weights: Sequence, impulses: Sequence,
                 points: Optional[Sequence[Sequence[int]]] = None, mode: str = "auto", max_batch: int = 16,
                 shard: Tuple[int, int] = (0, 1), device: int = -1, scratch_bytes: int = 0,
                 nccl_id: Optional[bytes] = None, reduce: str = "all", partition: str = "cost",
                 host_sub_mb: int = 0, devices: Optional[Sequence[int]] = None):
        """domain = (lo, hi) inclusive; weights / impulses: objects with ``.lo`` and ``.values``
        (``inputs.Field``) or (lo, values) pairs.

        Shard-by-k: ``shard = (rank, count)`` keeps this rank's cost-balanced block
        of terms (``partition``); with ``nccl_id`` (``lib.comm_unique_id()`` on one rank, sent to the
        others) construction joins an NCCL communicator and every apply sums the shards' partials
        inside the library (``reduce``: "all" = every rank gets the full result, "root" = rank 0,
        "none" = partial).  Without it, apply returns this shard's partial sum.

        Single-process multi-GPU: ``devices = [d0, d1, ...]`` builds one handle whose shard s runs
        on devices[s] (pcb_create_multi); buffers of the ``*_dev`` calls live on devices[0]."""
        if len(weights) != len(impulses):
            raise ValueError("PCOp: one weight per impulse required")
        L = _L.load()
        lo, hi = [int(v) for v in domain[0]], [int(v) for v in domain[1]]
        self.dim = len(lo)
        self.domain = (tuple(lo), tuple(hi))
        self.shape = tuple(h - l + 1 for l, h in zip(lo, hi))
        self.n_points = int(np.prod(self.shape))
        r = len(weights)
        self.rank = r

        def unpack(f):
            if hasattr(f, "values"):
                return tuple(int(v) for v in f.lo), np.ascontiguousarray(f.values, dtype=np.float64)
            return tuple(int(v) for v in f[0]), np.ascontiguousarray(f[1], dtype=np.float64)

        keep = []
        w_lo, w_hi, p_lo, p_hi, w_ptr, p_ptr = [], [], [], [], [], []
        for w, e in zip(weights, impulses):
            wl, wv = unpack(w)
            el, ev = unpack(e)
            if wv.ndim != self.dim or ev.ndim != self.dim:
                raise ValueError("IndexBox: dim mismatch")
            keep += [wv, ev]
            w_lo += wl
            w_hi += [l + s - 1 for l, s in zip(wl, wv.shape)]
            p_lo += el
            p_hi += [l + s - 1 for l, s in zip(el, ev.shape)]
            w_ptr.append(wv.ctypes.data)
            p_ptr.append(ev.ctypes.data)
        pts = None
        if points is not None:
            pts = _i64arr([c for p in points for c in p])
        opt = _L.default_options()
        opt.mode = _L.MODES[mode]
        opt.max_batch = int(max_batch)
        opt.shard_rank, opt.shard_count = int(shard[0]), int(shard[1])
        opt.device = int(device)
        opt.scratch_bytes = int(scratch_bytes)
        opt.partition = _L.PARTITION[partition]
        opt.host_sub_mb = int(host_sub_mb)
        id_buf = None
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id must be 128 bytes (pcb_comm_unique_id)")
            id_buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            opt.nccl_id = ctypes.cast(id_buf, _L.vp)
            opt.reduce = _L.REDUCE[reduce]
        PP = _L.vp * max(1, r)
        h = _L.vp()
        if devices is not None:
            devs = (_L.i32 * max(1, len(devices)))(*[int(d) for d in devices])
            rc = L.pcb_create_multi(self.dim, _i64arr(lo), _i64arr(hi), r, pts, _i64arr(w_lo), _i64arr(w_hi),
                                    PP(*w_ptr), _i64arr(p_lo), _i64arr(p_hi), PP(*p_ptr), ctypes.byref(opt), devs,
                                    len(devices), ctypes.byref(h))
        else:
            rc = L.pcb_create(self.dim, _i64arr(lo), _i64arr(hi), r, pts, _i64arr(w_lo), _i64arr(w_hi),
                              PP(*w_ptr), _i64arr(p_lo), _i64arr(p_hi), PP(*p_ptr), ctypes.byref(opt), ctypes.byref(h))
        if rc == 1:
            raise ValueError(L.pcb_last_error().decode())
        _L.check(rc)
        self._h = h
        info = _L.Info()
        _L.check(L.pcb_get_info(self._h, ctypes.byref(info)))
        self.info = info.as_dict()

    @classmethod
    def from_inputs(cls, inp, **kw) -> "ProductConvolutionOperator":
        return cls((inp.dom_lo, inp.dom_hi), inp.weights, inp.impulses, points=inp.points, **kw)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _L.load().pcb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- apply -------------------------------------------------------------
    def _vecs(self, F, what: str) -> np.ndarray:
        F = np.ascontiguousarray(F, dtype=np.float64)
        if F.ndim == 1:
            if F.size != self.n_points:
                raise ValueError(f"PCOp::{what}: shape mismatch")
            return F.reshape(1, -1)
        F = F.reshape(F.shape[0], -1) if F.shape[0] > 0 else F.reshape(0, int(np.prod(F.shape[1:])))
        if F.shape[1] != self.n_points:
            raise ValueError(f"PCOp::{what}: shape mismatch")
        return F

    def apply_batch(self, F: np.ndarray) -> np.ndarray:
        F = self._vecs(F, "apply")
        G = np.empty_like(F)
        self._rc(_L.load().pcb_apply_batch(self._h, F.shape[0], _ptr(F), _ptr(G)))
        return G

    def apply_adjoint_batch(self, F: np.ndarray) -> np.ndarray:
        F = self._vecs(F, "apply_adjoint")
        G = np.empty_like(F)
        self._rc(_L.load().pcb_apply_adjoint_batch(self._h, F.shape[0], _ptr(F), _ptr(G)))
        return G

    def apply(self, f: np.ndarray) -> np.ndarray:
        f = np.asarray(f, dtype=np.float64)
        if f.size != self.n_points:
            raise ValueError("PCOp::apply: shape mismatch")
        return self.apply_batch(f.reshape(1, -1))[0]

    def apply_adjoint(self, f: np.ndarray) -> np.ndarray:
        f = np.asarray(f, dtype=np.float64)
        if f.size != self.n_points:
            raise ValueError("PCOp::apply_adjoint: shape mismatch")
        return self.apply_adjoint_batch(f.reshape(1, -1))[0]

    def apply_batch_dev(self, B: int, dF: int, dG: int, stream: int = 0, adjoint: bool = False) -> None:
        fn = _L.load().pcb_apply_adjoint_batch_dev if adjoint else _L.load().pcb_apply_batch_dev
        self._rc(fn(self._h, int(B), dF, dG, stream or None))

    # --- entries -----------------------------------------------------------
    def entry(self, y: Sequence[int], x: Sequence[int]) -> float:
        return float(self.entries(np.asarray([y]), np.asarray([x]))[0])

    def entries(self, y: np.ndarray, x: np.ndarray) -> np.ndarray:
        y = np.ascontiguousarray(y, dtype=np.int64).reshape(-1, self.dim)
        x = np.ascontiguousarray(x, dtype=np.int64).reshape(-1, self.dim)
        if y.shape != x.shape:
            raise ValueError("entries: y and x must have the same count")
        out = np.empty(y.shape[0])
        self._rc(_L.load().pcb_entries(self._h, y.shape[0], _ptr(y), _ptr(x), _ptr(out)))
        return out

    def blocks(self, t_origin: np.ndarray, s_origin: np.ndarray, block_shape: Sequence[int]) -> np.ndarray:
        t = np.ascontiguousarray(t_origin, dtype=np.int64).reshape(-1, self.dim)
        s = np.ascontiguousarray(s_origin, dtype=np.int64).reshape(-1, self.dim)
        bs = int(np.prod(block_shape))
        out = np.empty((t.shape[0], bs, bs))
        self._rc(_L.load().pcb_blocks(self._h, t.shape[0], _ptr(t), _ptr(s), _i64arr(block_shape), _ptr(out)))
        return out

    def blocks_dev(self, nblk: int, d_t: int, d_s: int, block_shape: Sequence[int], d_out: int, stream: int = 0):
        self._rc(_L.load().pcb_blocks_dev(self._h, int(nblk), d_t, d_s, _i64arr(block_shape), d_out, stream or None))

    # --- block apply (pc_operator.cpp:98-130) ------------------------------
    def apply_block(self, T, S, f, adjoint: bool = False) -> np.ndarray:
        """g on box T from f on box S (boxes (lo, hi) inclusive, inside the domain); one block."""
        return self.apply_blocks([T], [S], [f], adjoint)[0]

    def apply_blocks(self, Ts, Ss, fs, adjoint: bool = False):
        """Batched block apply: returns [g_b on T_b]; f_b given on S_b (arrays of the box shape)."""
        nb = len(Ts)
        tl = np.ascontiguousarray([t[0] for t in Ts], dtype=np.int64).reshape(-1)
        th = np.ascontiguousarray([t[1] for t in Ts], dtype=np.int64).reshape(-1)
        sl = np.ascontiguousarray([s[0] for s in Ss], dtype=np.int64).reshape(-1)
        sh = np.ascontiguousarray([s[1] for s in Ss], dtype=np.int64).reshape(-1)
        shapes_t = [tuple(h - l + 1 for l, h in zip(t[0], t[1])) for t in Ts]
        flat = np.ascontiguousarray(np.concatenate([np.asarray(f, dtype=np.float64).reshape(-1) for f in fs])
                                    if nb else np.zeros(0))
        out = np.empty(int(sum(int(np.prod(s)) for s in shapes_t)))
        self._rc(_L.load().pcb_apply_block(self._h, nb, _ptr(tl), _ptr(th), _ptr(sl), _ptr(sh), _ptr(flat),
                                           _ptr(out), int(adjoint)))
        res, o = [], 0
        for s in shapes_t:
            n = int(np.prod(s))
            res.append(out[o:o + n].reshape(s))
            o += n
        return res

    # --- estimator ---------------------------------------------------------
    def probe_estimate(self, Z: np.ndarray, Y: np.ndarray, leaves: Iterable = (), want_ytilde: bool = False):
        Z = self._vecs(Z, "apply_adjoint")
        Y = self._vecs(Y, "apply_adjoint")
        leaves = list(leaves)
        lo = np.ascontiguousarray([l for l, _ in leaves], dtype=np.int64).reshape(-1)
        hi = np.ascontiguousarray([h for _, h in leaves], dtype=np.int64).reshape(-1)
        cells = np.zeros(max(1, len(leaves)))
        yt = np.empty_like(Z) if want_ytilde else None
        ea, er = _L.dbl(), _L.dbl()
        self._rc(_L.load().pcb_probe_estimate(self._h, Z.shape[0], _ptr(Z), _ptr(Y), len(leaves),
                                              _ptr(lo) if len(leaves) else None, _ptr(hi) if len(leaves) else None,
                                              _ptr(yt) if yt is not None else None, _ptr(cells),
                                              ctypes.byref(ea), ctypes.byref(er)))
        return yt, cells[: len(leaves)], ea.value, er.value

    def probe_estimate_dev(self, q: int, dZ: int, dY: int, dYt: int, leaves: Iterable = (), stream: int = 0):
        leaves = list(leaves)
        lo = np.ascontiguousarray([l for l, _ in leaves], dtype=np.int64).reshape(-1)
        hi = np.ascontiguousarray([h for _, h in leaves], dtype=np.int64).reshape(-1)
        cells = np.zeros(max(1, len(leaves)))
        ea, er = _L.dbl(), _L.dbl()
        self._rc(_L.load().pcb_probe_estimate_dev(self._h, int(q), dZ, dY, dYt, len(leaves),
                                                  _ptr(lo) if len(leaves) else None,
                                                  _ptr(hi) if len(leaves) else None, _ptr(cells),
                                                  ctypes.byref(ea), ctypes.byref(er), stream or None))
        return cells[: len(leaves)], ea.value, er.value

    # --- per-kernel profile ------------------------------------------------
    def profile_begin(self) -> None:
        _L.check(_L.load().pcb_profile_begin(self._h))

    def profile_end(self) -> dict:
        """{kernel name: (total ms, launches)} for launches since profile_begin (CUDA events)."""
        mx = 64
        names = ctypes.create_string_buffer(32 * mx)
        ms = np.zeros(mx)
        cnt = np.zeros(mx, dtype=np.int32)
        n = _L.i32()
        _L.check(_L.load().pcb_profile_end(self._h, mx, names, _ptr(ms), _ptr(cnt), ctypes.byref(n)))
        out = {}
        for i in range(min(n.value, mx)):
            nm = names.raw[32 * i: 32 * (i + 1)].split(b"\0", 1)[0].decode()
            out[nm] = (float(ms[i]), int(cnt[i]))
        return out

    # --- errors ------------------------------------------------------------
    @staticmethod
    def _rc(rc: int) -> None:
        if rc == 1:
            raise ValueError(_L.load().pcb_last_error().decode())
        _L.check(rc)


def normal_vectors(seed: int, count: int, n: int) -> np.ndarray:
    """count x n draws of std::mt19937_64(seed) + std::normal_distribution<double> (adaptivity.cpp:19-23)."""
    out = np.empty(count * n)
    _L.check(_L.load().pcb_normal_fill(ctypes.c_uint64(seed), count * n, _ptr(out)))
    return out.reshape(count, n)


def uniform_ints(seed: int, lo: int, hi: int, count: int) -> np.ndarray:
    """std::mt19937_64(seed) + std::uniform_int_distribution<int64_t>(lo, hi)."""
    out = np.empty(count, dtype=np.int64)
    _L.check(_L.load().pcb_uniform_int_fill(ctypes.c_uint64(seed), lo, hi, count, _ptr(out)))
    return out


def plan_shards(inp, shard_count: int, partition: str = "cost"):
    """The C planner's shard partition (pcb_plan_shards, host only): (owner[k], cost[k]) per term;
    owner -1 = inactive term.  pcb_create with shard_rank s keeps exactly the terms owned by s."""
    L = _L.load()
    r = inp.rank
    keep, w_lo, w_hi, p_lo, p_hi, w_ptr, p_ptr = [], [], [], [], [], [], []
    for w, e in zip(inp.weights, inp.impulses):
        wv = np.ascontiguousarray(w.values, dtype=np.float64)
        ev = np.ascontiguousarray(e.values, dtype=np.float64)
        keep += [wv, ev]
        w_lo += list(w.lo)
        w_hi += [l + s - 1 for l, s in zip(w.lo, wv.shape)]
        p_lo += list(e.lo)
        p_hi += [l + s - 1 for l, s in zip(e.lo, ev.shape)]
        w_ptr.append(wv.ctypes.data)
        p_ptr.append(ev.ctypes.data)
    PP = _L.vp * max(1, r)
    owner = np.zeros(max(1, r), dtype=np.int32)
    cost = np.zeros(max(1, r))
    _L.check(L.pcb_plan_shards(inp.dim, _i64arr(inp.dom_lo), _i64arr(inp.dom_hi), r, _i64arr(w_lo), _i64arr(w_hi),
                               PP(*w_ptr), _i64arr(p_lo), _i64arr(p_hi), PP(*p_ptr), int(shard_count),
                               _L.PARTITION[partition], _ptr(owner), _ptr(cost)))
    return owner[:r], cost[:r]
