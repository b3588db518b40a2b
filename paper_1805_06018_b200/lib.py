"""ctypes binding of the C ABI (include/pcb/pcb.h) — the only way Python reaches the kernels.

The product path has no fallback: if ``lib/libpcop_b200.so`` is missing, ``load()`` raises; if no
sm_100 device is present, ``pcb_create`` fails with PCB_ECUDA.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCB_LIB_PATH") or os.path.join(PKG, "lib", "libpcop_b200.so")  # PCB_LIB_PATH: A/B builds

i32 = ctypes.c_int32
i64 = ctypes.c_int64
dbl = ctypes.c_double
vp = ctypes.c_void_p
P_i64 = ctypes.POINTER(i64)
P_dbl = ctypes.POINTER(dbl)

STATUS = {0: "PCB_OK", 1: "PCB_EINVAL", 2: "PCB_ENOMEM", 3: "PCB_ECUDA", 4: "PCB_ENCCL", 5: "PCB_EINTERNAL"}
MODES = {"auto": 0, "global": 1, "local": 2}
MODE_NAMES = {v: k for k, v in MODES.items()}
KERNEL_FAMILIES = ("rows_fwd", "mid", "cols", "rows_inv")

# every symbol include/pcb/pcb.h declares
EXPORTS = ["pcb_default_options", "pcb_last_error", "pcb_create", "pcb_destroy", "pcb_get_info", "pcb_apply_batch",
           "pcb_apply_adjoint_batch", "pcb_apply_batch_dev", "pcb_apply_adjoint_batch_dev", "pcb_entries",
           "pcb_blocks", "pcb_blocks_dev", "pcb_probe_estimate", "pcb_probe_estimate_dev", "pcb_launch_count",
           "pcb_normal_fill", "pcb_uniform_int_fill", "pcb_profile_begin", "pcb_profile_end", "pcb_apply_block",
           "pcb_blur_create", "pcb_blur_destroy", "pcb_blur_apply", "pcb_blur_last_error",
           "pcb_estimator_create", "pcb_estimator_destroy", "pcb_estimator_probes", "pcb_estimator_set_y",
           "pcb_estimator_set_y_blur", "pcb_estimator_update", "pcb_estimator_cells", "pcb_estimator_read",
           "pcb_get_domain", "pcb_cluster_tree", "pcb_hmatrix_assemble", "pcb_hmatrix_compress",
           "pcb_hmatrix_destroy", "pcb_hmatrix_get_info", "pcb_hmatrix_tree", "pcb_hmatrix_block",
           "pcb_hmatrix_admissible", "pcb_hmatrix_matvec", "pcb_hmatrix_save", "pcb_hmatrix_load",
           "pcb_comm_unique_id", "pcb_plan_shards", "pcb_debug_guard_check", "pcb_estimator_create_ex",
           "pcb_host_alloc", "pcb_host_free", "pcb_create_multi", "pcb_host_register", "pcb_host_unregister", "pcb_hmatrix_matvec_batch"]
RNG = {"mt19937": 0, "philox": 1}
REDUCE = {"none": 0, "all": 1, "root": 2}
PARTITION = {"cost": 0, "count": 1}


class Options(ctypes.Structure):
    _fields_ = [("device", i32), ("mode", i32), ("max_batch", i32), ("shard_rank", i32), ("shard_count", i32),
                ("reduce", i32), ("scratch_bytes", i64), ("nccl_id", vp), ("partition", i32), ("host_sub_mb", i32)]


class Info(ctypes.Structure):
    _fields_ = [("dim", i32), ("rank", i32), ("rank_active", i32), ("mode", i32), ("n_groups", i32),
                ("fft_size", i32 * 3), ("n_points", i64), ("spectra_bytes", i64), ("device_bytes", i64),
                ("bytes_per_vector", dbl), ("flops_per_vector", dbl), ("launches_per_batch", i32),
                ("n_row_families", i32), ("kernel_bytes", dbl * 4), ("kernel_flops", dbl * 4),
                ("n_column_chains", i32), ("n_chained_terms", i32), ("shard_rank", i32), ("shard_count", i32),
                ("comm_nranks", i32), ("comm_version", i32), ("term_lo", i32), ("term_hi", i32),
                ("shard_cost", dbl), ("total_cost", dbl), ("model_ms_local", dbl), ("model_ms_global", dbl),
                ("plan_terms", i32), ("split_terms", i32)]

    def as_dict(self) -> dict:
        return {"dim": self.dim, "rank": self.rank, "rank_active": self.rank_active,
                "mode": MODE_NAMES.get(self.mode, self.mode), "n_groups": self.n_groups,
                "fft_size": [self.fft_size[i] for i in range(self.dim)], "n_points": self.n_points,
                "spectra_bytes": self.spectra_bytes, "device_bytes": self.device_bytes,
                "bytes_per_vector": self.bytes_per_vector, "flops_per_vector": self.flops_per_vector,
                "launches_per_batch": self.launches_per_batch, "n_row_families": self.n_row_families,
                "n_column_chains": self.n_column_chains, "n_chained_terms": self.n_chained_terms,
                "kernel_bytes": dict(zip(KERNEL_FAMILIES, list(self.kernel_bytes))),
                "kernel_flops": dict(zip(KERNEL_FAMILIES, list(self.kernel_flops))),
                "shard_rank": self.shard_rank, "shard_count": self.shard_count, "comm_nranks": self.comm_nranks,
                "comm_version": self.comm_version, "term_lo": self.term_lo, "term_hi": self.term_hi,
                "shard_cost": self.shard_cost, "total_cost": self.total_cost,
                "model_ms_local": self.model_ms_local, "model_ms_global": self.model_ms_global,
                "plan_terms": self.plan_terms, "split_terms": self.split_terms}


class HMatrixInfo(ctypes.Structure):
    _fields_ = [("dim", i32), ("leaf_cap", i32), ("n_points", i64), ("n_nodes", i64), ("n_blocks", i64),
                ("n_low_rank", i64), ("n_dense", i64), ("max_rank", i64), ("stored_doubles", i64),
                ("any_rank_capped", i32), ("method", i32), ("tol", dbl), ("fixed_rank", i32), ("reserved", i32)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "reserved"}


class PcbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


_lib = None


def load():
    """Load the in-tree library (built by ``__graft_entry__.build()`` / ``python -m paper_1805_06018_b200.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(f"{LIB_PATH} is not built; run `python -m paper_1805_06018_b200.build` "
                                "(there is no CPU fallback for the apply path)")
    L = ctypes.CDLL(LIB_PATH)
    L.pcb_default_options.argtypes = [ctypes.POINTER(Options)]
    L.pcb_default_options.restype = None
    L.pcb_last_error.restype = ctypes.c_char_p
    L.pcb_create.argtypes = [i32, P_i64, P_i64, i32, P_i64, P_i64, P_i64, ctypes.POINTER(vp), P_i64, P_i64,
                             ctypes.POINTER(vp), ctypes.POINTER(Options), ctypes.POINTER(vp)]
    L.pcb_create_multi.argtypes = [i32, P_i64, P_i64, i32, P_i64, P_i64, P_i64, ctypes.POINTER(vp), P_i64, P_i64,
                                   ctypes.POINTER(vp), ctypes.POINTER(Options), ctypes.POINTER(i32), i32,
                                   ctypes.POINTER(vp)]
    L.pcb_destroy.argtypes = [vp]
    L.pcb_get_info.argtypes = [vp, ctypes.POINTER(Info)]
    for n in ("pcb_apply_batch", "pcb_apply_adjoint_batch"):
        getattr(L, n).argtypes = [vp, i32, vp, vp]
    for n in ("pcb_apply_batch_dev", "pcb_apply_adjoint_batch_dev"):
        getattr(L, n).argtypes = [vp, i32, vp, vp, vp]
    L.pcb_entries.argtypes = [vp, i64, vp, vp, vp]
    L.pcb_blocks.argtypes = [vp, i32, vp, vp, P_i64, vp]
    L.pcb_blocks_dev.argtypes = [vp, i32, vp, vp, P_i64, vp, vp]
    L.pcb_apply_block.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, i32]
    L.pcb_probe_estimate.argtypes = [vp, i32, vp, vp, i32, vp, vp, vp, vp, P_dbl, P_dbl]
    L.pcb_probe_estimate_dev.argtypes = [vp, i32, vp, vp, vp, i32, vp, vp, vp, P_dbl, P_dbl, vp]
    L.pcb_launch_count.restype = ctypes.c_longlong
    L.pcb_profile_begin.argtypes = [vp]
    L.pcb_profile_end.argtypes = [vp, i32, vp, vp, vp, ctypes.POINTER(i32)]
    L.pcb_normal_fill.argtypes = [ctypes.c_uint64, i64, vp]
    L.pcb_uniform_int_fill.argtypes = [ctypes.c_uint64, i64, i64, i64, vp]
    L.pcb_blur_create.argtypes = [i32, P_i64, vp, ctypes.POINTER(vp)]
    L.pcb_blur_destroy.argtypes = [vp]
    L.pcb_blur_apply.argtypes = [vp, i32, vp, vp, i32, i32, vp]
    L.pcb_blur_last_error.restype = ctypes.c_char_p
    L.pcb_estimator_create.argtypes = [i32, P_i64, P_i64, i32, ctypes.c_uint64, i32, ctypes.POINTER(vp)]
    L.pcb_estimator_create_ex.argtypes = [i32, P_i64, P_i64, i32, ctypes.c_uint64, i32, i32, ctypes.POINTER(vp)]
    L.pcb_estimator_destroy.argtypes = [vp]
    L.pcb_estimator_probes.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp)]
    L.pcb_estimator_set_y.argtypes = [vp, vp, i32]
    L.pcb_estimator_set_y_blur.argtypes = [vp, vp]
    L.pcb_estimator_update.argtypes = [vp, vp, i32, vp, P_dbl, P_dbl]
    L.pcb_estimator_cells.argtypes = [vp, i32, vp, vp, vp]
    L.pcb_estimator_read.argtypes = [vp, vp, vp, vp]
    L.pcb_get_domain.argtypes = [vp, P_i64, P_i64]
    L.pcb_cluster_tree.argtypes = [i32, P_i64, P_i64, i32, ctypes.POINTER(vp)]
    L.pcb_hmatrix_assemble.argtypes = [vp, dbl, i32, i32, i32, ctypes.POINTER(vp)]
    L.pcb_hmatrix_compress.argtypes = [vp, vp, i32, vp, vp, i32, dbl, i32]
    L.pcb_hmatrix_destroy.argtypes = [vp]
    L.pcb_hmatrix_get_info.argtypes = [vp, ctypes.POINTER(HMatrixInfo)]
    L.pcb_hmatrix_tree.argtypes = [vp, vp, vp, vp, vp]
    L.pcb_hmatrix_block.argtypes = [vp, i64, vp, vp, vp, vp, vp]
    L.pcb_hmatrix_admissible.argtypes = [vp, i32, i32, vp, vp, vp, vp]
    L.pcb_hmatrix_matvec.argtypes = [vp, vp, vp]
    L.pcb_hmatrix_matvec_batch.argtypes = [vp, i32, i32, vp, vp]
    L.pcb_hmatrix_save.argtypes = [vp, ctypes.c_char_p]
    L.pcb_hmatrix_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    L.pcb_comm_unique_id.argtypes = [vp]
    L.pcb_debug_guard_check.argtypes = [P_i64, P_i64]
    L.pcb_host_alloc.argtypes = [ctypes.c_uint64, ctypes.POINTER(vp)]
    L.pcb_host_free.argtypes = [vp]
    L.pcb_host_register.argtypes = [vp, ctypes.c_uint64]
    L.pcb_host_unregister.argtypes = [vp]
    L.pcb_plan_shards.argtypes = [i32, P_i64, P_i64, i32, P_i64, P_i64, ctypes.POINTER(vp), P_i64, P_i64,
                                  ctypes.POINTER(vp), i32, i32, vp, vp]
    for n in EXPORTS:
        if n not in ("pcb_default_options", "pcb_last_error", "pcb_launch_count", "pcb_blur_last_error"):
            getattr(L, n).restype = ctypes.c_int
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        raise PcbError(rc, load().pcb_last_error().decode())


def check_blur(rc: int) -> None:
    if rc != 0:
        raise PcbError(rc, load().pcb_blur_last_error().decode())


def default_options() -> Options:
    o = Options()
    load().pcb_default_options(ctypes.byref(o))
    return o


def launch_count() -> int:
    return int(load().pcb_launch_count())


def comm_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (pcb_comm_unique_id) for pcb_options.nccl_id."""
    buf = ctypes.create_string_buffer(128)
    check(load().pcb_comm_unique_id(buf))
    return buf.raw


class host_registered:
    """Context manager: page-lock numpy arrays the caller owns (pcb_host_register) so the host-buffer
    calls on them take the copy-engine path; unregistered on exit."""

    def __init__(self, *arrays):
        self._arrays = [a for a in arrays if a.size]
        self._done = []

    def __enter__(self):
        for a in self._arrays:
            check(load().pcb_host_register(a.ctypes.data, a.nbytes))
            self._done.append(a)
        return self

    def __exit__(self, *exc):
        for a in reversed(self._done):
            load().pcb_host_unregister(a.ctypes.data)
        self._done = []
        return False


def guard_check():
    """(guarded allocations, overwritten canary bytes) -- PCB_GUARD=1 debug mode (pcb_debug_guard_check)."""
    a, b = i64(), i64()
    check(load().pcb_debug_guard_check(ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value
