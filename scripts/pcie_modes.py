"""PCIe experiment: H2D/D2H of 512 MiB each by copy engines (1 or 2 streams per direction) and by
SM-driven copies through mapped pinned memory.  Prints ms and GB/s per mode."""
import ctypes
import json
import os

import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "pcie_sm.so"))
n = 64 << 20
h_in = torch.randn(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.randn(n, dtype=torch.float64, device="cuda")
S = [torch.cuda.Stream() for _ in range(4)]


def ce(dst, src, parts, streams):
    k = n // parts
    for p in range(parts):
        with torch.cuda.stream(streams[p]):
            dst[p * k:(p + 1) * k].copy_(src[p * k:(p + 1) * k], non_blocking=True)


def sm(dst, src, blocks, stream):
    rc = lib.pcie_sm_copy(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()), ctypes.c_longlong(n * 8),
                          blocks, ctypes.c_void_p(stream.cuda_stream))
    assert rc == 0, rc


modes = {
    "h2d_ce1": lambda: ce(d_in, h_in, 1, S[:1]),
    "h2d_ce2": lambda: ce(d_in, h_in, 2, S[:2]),
    "d2h_ce1": lambda: ce(h_out, d_out, 1, S[:1]),
    "both_ce1": lambda: (ce(d_in, h_in, 1, S[:1]), ce(h_out, d_out, 1, S[1:2])),
    "both_ce2": lambda: (ce(d_in, h_in, 2, S[:2]), ce(h_out, d_out, 2, S[2:4])),
    "h2d_sm148": lambda: sm(d_in, h_in, 148, S[0]),
    "h2d_sm592": lambda: sm(d_in, h_in, 592, S[0]),
    "d2h_sm592": lambda: sm(h_out, d_out, 592, S[0]),
    "both_sm": lambda: (sm(d_in, h_in, 296, S[0]), sm(h_out, d_out, 296, S[1])),
    "both_smh2d_ced2h": lambda: (sm(d_in, h_in, 296, S[0]), ce(h_out, d_out, 1, S[1:2])),
    "both_ceh2d_smd2h": lambda: (ce(d_in, h_in, 1, S[:1]), sm(h_out, d_out, 296, S[1])),
}
res = {}
for name, fn in modes.items():
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for s in S:
            s.wait_stream(torch.cuda.current_stream())
        fn()
        for s in S:
            torch.cuda.current_stream().wait_stream(s)
        t1.record()
        torch.cuda.synchronize()
        best = min(best, t0.elapsed_time(t1))
    gb = (2 if name.startswith("both") else 1) * n * 8 / 1e9
    res[name] = {"ms": round(best, 2), "GB/s": round(gb / (best * 1e-3), 1)}
    print(name, res[name], flush=True)
assert torch.equal(d_in.cpu(), h_in)
json.dump(res, open("gpurun_out/pcie_modes.json", "w"), indent=1)
