"""Where does c3 e2e time go?  The library's sub-batch pipeline restated with torch streams:
copies only, kernels only (per sub-batch), and both, for several sub-batch sizes."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1805_06018_b200 import inputs  # noqa: E402
from paper_1805_06018_b200.operator import ProductConvolutionOperator  # noqa: E402

B = 64
inp = inputs.make_config("c3")
N = inp.n_points
op = ProductConvolutionOperator.from_inputs(inp, mode="local", max_batch=64)
hF = torch.randn(B, N, dtype=torch.float64).pin_memory()
hG = torch.empty(B, N, dtype=torch.float64).pin_memory()
dF = torch.empty(B, N, dtype=torch.float64, device="cuda")
dG = torch.empty(B, N, dtype=torch.float64, device="cuda")
sh, sc, sd = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def run(sizes, copies=True, compute=True):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sh)
    sc.wait_stream(sh)
    sd.wait_stream(sh)
    b0 = 0
    for s in sizes:
        b1 = b0 + s
        if copies:
            with torch.cuda.stream(sh):
                dF[b0:b1].copy_(hF[b0:b1], non_blocking=True)
            sc.wait_stream(sh)
        if compute:
            op.apply_batch_dev(s, dF[b0:b1].data_ptr(), dG[b0:b1].data_ptr(), stream=sc.cuda_stream)
        sd.wait_stream(sc)
        if copies:
            with torch.cuda.stream(sd):
                hG[b0:b1].copy_(dG[b0:b1], non_blocking=True)
        b0 = b1
    sh.wait_stream(sd)
    e1.record(sh)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


res = {}
for name, sizes in {"3+6x9+4+3": [3] + [6] * 9 + [4, 3], "4+8x7+4": [4] + [8] * 7 + [4], "64": [64]}.items():
    for mode, kw in {"copies": dict(compute=False), "kernels": dict(copies=False), "both": {}}.items():
        run(sizes, **kw)
        t = min(run(sizes, **kw) for _ in range(3))
        res[f"{name} {mode}"] = round(t, 3)
        print(name, mode, round(t, 3), flush=True)
json.dump(res, open("gpurun_out/e2e_probe.json", "w"), indent=1)
