"""Target program for the compute-sanitizer runs in tests/test_gpu_tools.py: every
entry point of the library on small operators -- c1 (128^2, r = 16) and a 3-D lattice, both plans:
apply / adjoint (device and host buffers), entries, blocks, apply_block, probe estimate.  It exits
non-zero if a result is off; the sanitizer reports memory errors / shared-memory races itself."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1805_06018_b200 import inputs  # noqa: E402
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors  # noqa: E402


def main():
    gold = np.load(os.path.join(ROOT, "tests", "golden", "c1.npz"))
    cases = [("c1", inputs.make_config("c1")), ("3d", inputs.small_lattice(n=12, dim=3, m=2, sigma=1.1))]
    for name, inp in cases:
        for mode in ("local", "global"):
            op = ProductConvolutionOperator.from_inputs(inp, mode=mode)
            F = normal_vectors(3, 3, inp.n_points)
            G = op.apply_batch(F)
            GA = op.apply_adjoint_batch(F)
            # adjoint identity as a cheap correctness check under the sanitizer
            lhs, rhs = float(G[0] @ F[1]), float(F[0] @ GA[1])
            assert abs(lhs - rhs) <= 1e-11 * max(1.0, abs(lhs)), (name, mode, lhs, rhs)
            if name == "c1":
                g = op.apply(gold["f"])
                assert np.linalg.norm(g - gold["g"]) <= 1e-11 * np.linalg.norm(gold["g"])
                assert np.array_equal(op.entries(gold["y"], gold["x"]), gold["E"])
                org = np.array([[0, 0, 3, 5], [60, 60, 64, 58], [120, 120, 100, 110]])
                op.blocks(org[:, :2], org[:, 2:], (8, 8))
                T = ((10, 10), (30, 40))
                S = ((5, 12), (40, 33))
                op.apply_block(T, S, np.ones((36, 22)))
            Z = normal_vectors(5, 2, inp.n_points)
            lo = tuple(inp.dom_lo)
            hi = tuple(inp.dom_hi)
            op.probe_estimate(Z, Z * 0.5, [(lo, hi)])
            op.close()
    print("SANITIZE TARGET OK", flush=True)


if __name__ == "__main__":
    main()
