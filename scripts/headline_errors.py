"""Measured parity at the headline configurations (the numbers behind tests/test_gpu_headline.py):
relative l2 errors of the GPU apply / adjoint against the reference's own outputs (committed
fingerprints, and the live reference build where it is shipped), both plans at c3, and the c5
block hash.  Writes gpurun_out/headline_parity.json."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from headline_common import c5_origins, compare, rel, sha256_f64  # noqa: E402
from paper_1805_06018_b200 import inputs  # noqa: E402
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors  # noqa: E402

out = {}
for cfg, seed in (("c3", 2), ("c4", 4)):
    inp = inputs.make_config(cfg)
    gold = np.load(os.path.join(ROOT, "tests", "golden", f"headline_{cfg}.npz"))
    F = normal_vectors(seed, 2, inp.n_points)
    for mode in (("local", "global") if cfg == "c3" else ("local",)):
        op = ProductConvolutionOperator.from_inputs(inp, mode=mode)
        G = op.apply_batch(F)
        GA = op.apply_adjoint_batch(F[:1])
        fp = lambda pre: {k: gold[f"{pre}_{k}"] for k in ("samples", "tiles", "norm")}  # noqa: E731
        out[f"{cfg}_{mode}"] = {"apply0": compare(G[0], inp.shape, fp("apply0")),
                                "apply1": compare(G[1], inp.shape, fp("apply1")),
                                "adjoint0": compare(GA[0], inp.shape, fp("adjoint0"))}
        if mode == "local":
            try:
                from oracle import ref_lib

                if ref_lib.available():
                    R = ref_lib.apply_split(inp, F)
                    out[f"{cfg}_{mode}"]["live_apply_full_vector"] = [rel(G[b], R[b]) for b in range(2)]
                    if cfg == "c3":
                        RA = ref_lib.apply_split(inp, F[:1], adjoint=True)
                        out[f"{cfg}_{mode}"]["live_adjoint_full_vector"] = rel(GA[0], RA[0])
            except Exception as e:  # reported, not fatal
                out[f"{cfg}_{mode}"]["live_error"] = str(e)[:200]
        op.close()
gold = np.load(os.path.join(ROOT, "tests", "golden", "headline_c5.npz"))
op = ProductConvolutionOperator.from_inputs(inputs.make_config("c2"))
org = c5_origins()
B = op.blocks(org[:, :2], org[:, 2:], (8, 8))
out["c5"] = {"sha256_equal": sha256_f64(B) == str(gold["sha256"]), "blocks": int(B.shape[0]),
             "nonzero_blocks": int((np.abs(B).reshape(4096, -1).max(axis=1) > 0).sum())}
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/headline_parity.json", "w"), indent=1)
