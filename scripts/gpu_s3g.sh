#!/bin/bash
# pageable host path: sub-batch size for pageable buffers (default 128 MiB) and non-temporal bounce copies
echo "== host pipeline tests: $(timeout 900 python -m pytest tests/test_gpu_tools.py -q -x -k 'host_pipeline or multi_device' 2>&1 | tail -1)"
for nt in 1 0; do for t in 16 8; do
PCB_HOST_NT=$nt PCB_HOST_THREADS=$t python - <<'PY'
import os, sys, time, numpy as np
sys.path.insert(0, '.')
from paper_1805_06018_b200 import inputs, lib
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors
for cfg, B in (("c3", 64), ("c4", 8), ("c2", 16)):
    inp = inputs.make_config(cfg)
    F = normal_vectors(2, B, inp.n_points); G = np.empty_like(F)
    op = ProductConvolutionOperator.from_inputs(inp, max_batch=B)
    fn = lib.load().pcb_apply_batch
    lib.check(fn(op._h, B, F.ctypes.data, G.ctypes.data)); G0 = G.copy()
    t0 = time.perf_counter()
    for _ in range(4): lib.check(fn(op._h, B, F.ctypes.data, G.ctypes.data))
    dt = (time.perf_counter() - t0) / 4
    assert np.array_equal(G, G0)
    print(f"{cfg} nt={os.environ['PCB_HOST_NT']} threads={os.environ['PCB_HOST_THREADS']}: {dt*1e3:.1f} ms, {B/dt:.0f} vec/s", flush=True)
    op.close()
PY
done; done
