"""Time the GPU true-operator stencils (pcb_blur_apply) at the config sizes."""
import json
import sys
import time

import torch

from paper_1805_06018_b200 import inputs
from paper_1805_06018_b200.true_operator import BlurOperator

out = {}
for name in sys.argv[1:] or ["c1", "c3", "c4"]:
    blur, _ = inputs.config_spec(name)
    t0 = time.time()
    A = BlurOperator.from_spec(blur)
    torch.cuda.synchronize()
    t_create = time.time() - t0
    N = blur.n ** blur.dim
    B = 64 if N <= 2 ** 20 else 16
    F = torch.randn(B, N, dtype=torch.float64, device="cuda")
    G = torch.empty_like(F)
    res = {"create_s": t_create}
    for adj in (0, 1):
        A.apply_dev(B, F.data_ptr(), G.data_ptr(), bool(adj), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        A.apply_dev(B, F.data_ptr(), G.data_ptr(), bool(adj), torch.cuda.current_stream().cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        res["adjoint_ms_per_vec" if adj else "apply_ms_per_vec"] = e0.elapsed_time(e1) / B
    out[name] = res
    print(name, res, flush=True)
json.dump(out, open("gpurun_out/blur_time.json", "w"), indent=1)
