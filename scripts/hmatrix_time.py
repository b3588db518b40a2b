"""H-matrix conversion timed end to end: the GPU-driven assembly
(pcb_hmatrix_assemble: batched entry gathers, lockstep ACA / batched block applies on the device,
QR / SVD on the host) against the reference's own assemble_hmatrix (hmatrix.cpp:338-431, compiled
into oracle/_ref, one host thread -- the reference has no parallel path), same operator, tolerance
and leaf size; the two results are compared through a matvec.  Writes gpurun_out/hmatrix_time.json."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06018_b200 import inputs  # noqa: E402
from paper_1805_06018_b200.hmatrix import HMatrix  # noqa: E402
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors  # noqa: E402

CASES = [dict(n=64, dim=2, m=4, sigma=2.5, leaf=64), dict(n=96, dim=2, m=4, sigma=3.0, leaf=64)]
res = {"tol": 1e-8, "cases": []}
for case in CASES:
    leaf = case.pop("leaf")
    inp = inputs.small_lattice(**case)
    op = ProductConvolutionOperator.from_inputs(inp)
    f = normal_vectors(5, 1, inp.n_points)[0]
    g_op = op.apply(f)
    row = {"operator": inp.name, "N": inp.n_points, "rank": inp.rank, "leaf_cap": leaf}
    for method in ("cur", "randomized"):
        HMatrix.assemble(op, 1e-8, leaf, method)  # warm-up (allocations, kernel load)
        t0 = time.perf_counter()
        h = HMatrix.assemble(op, 1e-8, leaf, method)
        t_gpu = time.perf_counter() - t0
        t0 = time.perf_counter()
        g = h.matvec(f)
        t_host_mv = time.perf_counter() - t0
        Fb = normal_vectors(6, 32, inp.n_points)
        h.matvec_batch(Fb)  # first call copies the blocks to the device
        t0 = time.perf_counter()
        Gb = h.matvec_batch(Fb)
        t_gpu_mv = time.perf_counter() - t0
        r = {"gpu_assemble_s": t_gpu, "blocks": len(h.blocks()),
             "matvec_vs_apply_rel": float(np.linalg.norm(g - g_op) / np.linalg.norm(g_op)),
             "host_matvec_ms_per_vector": t_host_mv * 1e3, "gpu_matvec_batch32_ms": t_gpu_mv * 1e3,
             "gpu_matvec_equals_host": bool(np.array_equal(Gb[0], h.matvec(Fb[0])))}
        try:
            from oracle import ref_lib  # reported baseline only
            if ref_lib.available():
                rop = ref_lib.RefOperator(inp)
                t0 = time.perf_counter()
                hr = ref_lib.RefHMatrix.assemble(rop, 1e-8, leaf, method)
                r["reference_assemble_s"] = time.perf_counter() - t0
                r["reference_threads"] = 1
                t0 = time.perf_counter()
                gr = hr.matvec(f)
                r["reference_matvec_ms_per_vector"] = (time.perf_counter() - t0) * 1e3
                r["matvec_vs_reference_rel"] = float(np.linalg.norm(g - gr) / np.linalg.norm(gr))
                r["speedup"] = r["reference_assemble_s"] / t_gpu
        except Exception as ex:  # reported, never fatal
            r["reference"] = {"unavailable": str(ex)[:200]}
        row[method] = r
        print(inp.name, method, r, flush=True)
    res["cases"].append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/hmatrix_time.json", "w"), indent=1)
print(json.dumps(res))
