import os, sys, time, numpy as np
sys.path.insert(0, '.')
from paper_1805_06018_b200 import inputs, lib
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors
for cfg, B in (("c4", 8), ("c2", 16), ("c3", 64)):
    inp = inputs.make_config(cfg)
    F = normal_vectors(2, B, inp.n_points); G = np.empty_like(F)
    op = ProductConvolutionOperator.from_inputs(inp, max_batch=B)
    fn = lib.load().pcb_apply_batch
    lib.check(fn(op._h, B, F.ctypes.data, G.ctypes.data))
    t0 = time.perf_counter()
    for _ in range(4): lib.check(fn(op._h, B, F.ctypes.data, G.ctypes.data))
    dt = (time.perf_counter() - t0) / 4
    print(f"{cfg} sub_pg={os.environ.get('PCB_SUB_MB_PAGEABLE')}: {dt*1e3:.1f} ms, {B/dt:.0f} vec/s", flush=True)
    op.close()
