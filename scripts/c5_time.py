"""Config 5 throughput: 4096 dense 64x64 blocks (8x8-point patches) of the c2 operator by the K6
block gather (pcb_blocks_dev), device-timed, against HBM (the 134 MB output written once), and the
reference's own entry() (oracle/_ref, pc_operator.cpp:84-96) on a bounded sample of blocks, one
host thread.  Writes gpurun_out/c5_time.json."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06018_b200 import inputs  # noqa: E402
from paper_1805_06018_b200.operator import ProductConvolutionOperator, uniform_ints  # noqa: E402

inp = inputs.make_config("c2")
op = ProductConvolutionOperator.from_inputs(inp)
nblk = 4096
org = uniform_ints(3, 0, 504, 4 * nblk).reshape(nblk, 4)
d_t = torch.from_numpy(np.ascontiguousarray(org[:, :2])).cuda()
d_s = torch.from_numpy(np.ascontiguousarray(org[:, 2:])).cuda()
out = torch.empty((nblk, 64, 64), dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    op.blocks_dev(nblk, d_t.data_ptr(), d_s.data_ptr(), (8, 8), out.data_ptr(), s)
torch.cuda.synchronize()
reps = 20
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    op.blocks_dev(nblk, d_t.data_ptr(), d_s.data_ptr(), (8, 8), out.data_ptr(), s)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
op.profile_begin()  # the kernel alone (CUDA events around the launch on its stream)
for _ in range(reps):
    op.blocks_dev(nblk, d_t.data_ptr(), d_s.data_ptr(), (8, 8), out.data_ptr(), s)
torch.cuda.synchronize()
prof = op.profile_end()
kernel_ms = sum(v[0] for v in prof.values()) / reps
split_ms = {k: v[0] / reps for k, v in prof.items()}
hbm = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6552.0
gbs = out.numel() * 8 / (ms * 1e-3) / 1e9
kgbs = out.numel() * 8 / (kernel_ms * 1e-3) / 1e9
res = {"blocks": nblk, "ms_per_call": ms, "kernel_ms": kernel_ms, "split_ms": split_ms,
       "zero_mode": os.environ.get("PCB_C5_ZERO", "default"), "kernel_GBs": kgbs, "kernel_frac_hbm": kgbs / hbm,
       "ms_per_launch": ms, "blocks_per_s": nblk / (ms * 1e-3),
       "entries_per_s": out.numel() / (ms * 1e-3), "output_GBs": gbs, "frac_hbm": gbs / hbm,
       "bound": "hbm (output written once; the gathers read ~KB per block, L2-resident)"}
try:
    from oracle import ref_lib  # reported baseline only
    if ref_lib.available():
        ref = ref_lib.RefOperator(inp)
        nb = 16
        off = np.array([(i, j) for i in range(8) for j in range(8)])
        yy = np.concatenate([np.repeat(org[k, :2] + off, 64, axis=0) for k in range(nb)])
        xx = np.concatenate([np.tile(org[k, 2:] + off, (64, 1)) for k in range(nb)])
        t0 = time.perf_counter()
        e = ref.entries(yy, xx)
        wall = time.perf_counter() - t0
        assert np.array_equal(e.reshape(nb, 64, 64), out[:nb].cpu().numpy())
        res["reference"] = {"entries_per_s": e.size / wall, "threads": 1,
                            "sample": f"{nb} blocks ({e.size} entries) through the reference entry()"}
        res["speedup_vs_reference_1core"] = res["entries_per_s"] / res["reference"]["entries_per_s"]
except Exception as ex:  # reported, never fatal
    res["reference"] = {"unavailable": str(ex)[:200]}
print(json.dumps(res))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/c5_time.json", "w"), indent=1)
