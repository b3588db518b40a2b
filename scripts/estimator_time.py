"""c3 randomized a-posteriori estimator: q = 64 Gaussian probes, Ytilde = Atilde^* Z and eta over a
16 x 16 grid of leaf cells (adaptivity.cpp:75-121), device-resident Z / Y (probe_estimate_dev) and
through the host C-ABI (probe_estimate, Z and Y copied in, eta out).  Writes gpurun_out/estimator_c3.json."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06018_b200 import inputs  # noqa: E402
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors  # noqa: E402

q = 64
inp = inputs.make_config("c3")
n = inp.shape[0]
op = ProductConvolutionOperator.from_inputs(inp, max_batch=q)
Zh = normal_vectors(2, q, inp.n_points)
Yh = normal_vectors(3, q, inp.n_points)
leaves = [((i * 64, j * 64), (i * 64 + 63, j * 64 + 63)) for i in range(n // 64) for j in range(n // 64)]
Z, Y = torch.from_numpy(Zh).cuda(), torch.from_numpy(Yh).cuda()
Yt = torch.empty_like(Z)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    op.probe_estimate_dev(q, Z.data_ptr(), Y.data_ptr(), Yt.data_ptr(), leaves, s)
torch.cuda.synchronize()
reps = 5
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    cells, ea, er = op.probe_estimate_dev(q, Z.data_ptr(), Y.data_ptr(), Yt.data_ptr(), leaves, s)
b.record()
torch.cuda.synchronize()
dev_ms = a.elapsed_time(b) / reps
Zp, Yp = torch.from_numpy(Zh).pin_memory().numpy(), torch.from_numpy(Yh).pin_memory().numpy()
op.probe_estimate(Zp, Yp, leaves)
t0 = time.perf_counter()
for _ in range(reps):
    yt, cells_h, ea_h, er_h = op.probe_estimate(Zp, Yp, leaves)
host_ms = (time.perf_counter() - t0) / reps * 1e3
# probe creation: the reference's mt19937_64 stream (host) vs Philox on the device
from paper_1805_06018_b200.estimator import Estimator  # noqa: E402

create_s = {}
for gen in ("mt19937", "philox"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    est = Estimator((inp.dom_lo, inp.dom_hi), q=q, seed=2, generator=gen)
    torch.cuda.synchronize()
    create_s[gen] = time.perf_counter() - t0
    est.close()
res = {"config": "c3", "probes": q, "probe_creation_s": create_s, "leaves": len(leaves), "device_ms": dev_ms, "probes_per_s_device": q / (dev_ms * 1e-3),
       "host_ms": host_ms, "probes_per_s_host": q / (host_ms * 1e-3), "eta_abs": ea, "eta_rel": er,
       "host_equals_device": bool(np.isclose(ea, ea_h, rtol=1e-12) and np.isclose(er, er_h, rtol=1e-12))}
print(json.dumps(res))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/estimator_c3.json", "w"), indent=1)
