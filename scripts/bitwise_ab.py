"""Bitwise comparison of apply / adjoint outputs between the in-tree library and another build
(argv[1] = path of the other .so) on c1, c3 (4 vectors) and c4 (2 vectors)."""
import os
import subprocess
import sys

import numpy as np

if len(sys.argv) > 2:  # child: run one library, dump outputs
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1805_06018_b200 import inputs
    from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors
    out = {}
    for cfg, B in (("c1", 2), ("c3", 4), ("c4", 2)):
        inp = inputs.make_config(cfg)
        op = ProductConvolutionOperator.from_inputs(inp, mode="local")
        F = normal_vectors(21, B, inp.n_points)
        out[cfg] = op.apply_batch(F)
        out[cfg + "_adj"] = op.apply_adjoint_batch(F)
    np.savez(sys.argv[2], **out)
    sys.exit(0)
other = sys.argv[1]
env = dict(os.environ)
subprocess.run([sys.executable, __file__, "x", "/tmp/bw_new.npz"], check=True, env=env)
env["PCB_LIB_PATH"] = other
subprocess.run([sys.executable, __file__, "x", "/tmp/bw_old.npz"], check=True, env=env)
a, b = np.load("/tmp/bw_new.npz"), np.load("/tmp/bw_old.npz")
for k in a.files:
    d = np.abs(a[k] - b[k]).max()
    print(k, "bitwise" if np.array_equal(a[k], b[k]) else f"max|diff| {d:.3e} rel {d / np.abs(b[k]).max():.2e}")
