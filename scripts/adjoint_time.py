"""Device-timed apply vs adjoint throughput (vectors/s) at a config, per-kernel profile of both."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1805_06018_b200 import inputs  # noqa: E402
from paper_1805_06018_b200.operator import ProductConvolutionOperator  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
inp = inputs.make_config(cfg)
op = ProductConvolutionOperator.from_inputs(inp, max_batch=B)
F = torch.randn(B, inp.n_points, dtype=torch.float64, device="cuda")
G = torch.empty_like(F)
s = torch.cuda.current_stream().cuda_stream
out = {}
for adj in (False, True):
    for _ in range(3):
        op.apply_batch_dev(B, F.data_ptr(), G.data_ptr(), s, adjoint=adj)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        op.apply_batch_dev(B, F.data_ptr(), G.data_ptr(), s, adjoint=adj)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    op.profile_begin()
    op.apply_batch_dev(B, F.data_ptr(), G.data_ptr(), s, adjoint=adj)
    torch.cuda.synchronize()
    prof = {k: round(v[0], 3) for k, v in op.profile_end().items()}
    out["adjoint" if adj else "apply"] = {"vec_per_s": B / (ms * 1e-3), "ms": ms, "kernels_ms": prof}
    print(cfg, "adjoint" if adj else "apply", round(B / (ms * 1e-3)), prof, flush=True)
json.dump(out, open(f"gpurun_out/adjoint_{cfg}.json", "w"), indent=1)
