"""Single-process multi-device handle (pcb_create_multi) vs the single handle at c3, device-timed,
on one GPU (every shard on GPU 0): the overhead of the shard partials and the reduction kernel.
usage: python scripts/multi_time.py [ndev] [device list...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06018_b200 import inputs  # noqa: E402
from paper_1805_06018_b200.operator import ProductConvolutionOperator  # noqa: E402

ndev = int(sys.argv[1]) if len(sys.argv) > 1 else 2
devs = [int(v) for v in sys.argv[2:]] or [0] * ndev
inp = inputs.make_config("c3")
B = 64
F = torch.randn(B, inp.n_points, dtype=torch.float64, device="cuda")
G = torch.empty_like(F)
s = torch.cuda.current_stream().cuda_stream
res = {}
for name, kw in (("single", {}), (f"multi{devs}", {"devices": devs})):
    op = ProductConvolutionOperator.from_inputs(inp, max_batch=B, **kw)
    for _ in range(3):
        op.apply_batch_dev(B, F.data_ptr(), G.data_ptr(), s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        op.apply_batch_dev(B, F.data_ptr(), G.data_ptr(), s)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    res[name] = {"ms_per_step": ms, "vectors_per_s": B / (ms * 1e-3)}
    op.close()
print(json.dumps(res))
