"""Pageable host path (pcb_apply_batch on plain numpy buffers) at c3: sub-batch size sweep for one
PCB_HOST_THREADS setting (the pool is created once per process).  usage: pageable_sweep.py [cfg]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06018_b200 import inputs, lib  # noqa: E402
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
B = {"c3": 64, "c4": 8, "c2": 16}[cfg]
inp = inputs.make_config(cfg)
F = normal_vectors(2, B, inp.n_points)
G = np.empty_like(F)
for sub in (8, 16, 32, 64, 128, 256):
    op = ProductConvolutionOperator.from_inputs(inp, host_sub_mb=sub, max_batch=B)
    fn = lib.load().pcb_apply_batch
    lib.check(fn(op._h, B, F.ctypes.data, G.ctypes.data))
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        lib.check(fn(op._h, B, F.ctypes.data, G.ctypes.data))
    dt = (time.perf_counter() - t0) / reps
    print(f"{cfg} threads={os.environ.get('PCB_HOST_THREADS', 'default')} sub_mb={sub}: {dt * 1e3:.1f} ms, {B / dt:.0f} vec/s", flush=True)
    op.close()
