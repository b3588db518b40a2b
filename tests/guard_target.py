"""Target program of the guard-band test (tests/test_gpu_tools.py::test_guard_bands, run with
PCB_GUARD=1): every entry point of the library -- apply / adjoint on host and device buffers, both
plans, entries, blocks, apply_block, the probe estimator, split long-line terms -- on c1, c3 and c4
(full size, a few vectors) and small 1-D / 3-D lattices; after each case the 64 KiB canary bands
around every device allocation must be intact (pcb_debug_guard_check), i.e. no kernel wrote out of
bounds.  (compute-sanitizer is disabled on this GPU pool.)"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1805_06018_b200 import inputs  # noqa: E402
from paper_1805_06018_b200 import lib  # noqa: E402
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors  # noqa: E402


def guards_ok(tag, expect_regions=True):
    regions, bad = lib.guard_check()
    assert regions > 0 or not expect_regions, "PCB_GUARD=1 not in effect"
    assert bad == 0, (tag, bad)
    print(f"{tag}: {regions} guarded allocations, canaries intact", flush=True)


def main():
    gold = np.load(os.path.join(ROOT, "tests", "golden", "c1.npz"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_long_lines import CASES as LONG

    cases = [("c1", inputs.make_config("c1")), ("3d", inputs.small_lattice(n=12, dim=3, m=2, sigma=1.1)),
             ("1d", inputs.small_lattice(n=50, dim=1, m=5, sigma=2.0)), ("c3", inputs.make_config("c3")),
             ("c4", inputs.make_config("c4")), ("long1d", LONG["1d_n12000"]())]
    for name, inp in cases:
        for mode in ("local", "global"):
            if name == "long1d" and mode == "global":
                continue
            if name in ("c3", "c4") and mode == "global":
                continue
            op = ProductConvolutionOperator.from_inputs(inp, mode=mode, host_sub_mb=1)
            F = normal_vectors(3, 3, inp.n_points)
            G = op.apply_batch(F)
            GA = op.apply_adjoint_batch(F)
            # adjoint identity as a cheap correctness check
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
            guards_ok(f"{name}/{mode}")
            op.close()
    # the single-process multi-device handle (every shard on GPU 0): partials + reduction kernel
    inp = inputs.make_config("c2")
    op = ProductConvolutionOperator.from_inputs(inp, devices=[0, 0, 0])
    F = normal_vectors(4, 3, inp.n_points)
    op.apply_batch(F)
    op.apply_adjoint_batch(F)
    guards_ok("c2/multi")
    op.close()
    # config 5: the tiled dense-block gather and its zero-block path, all 4096 blocks
    from headline_common import c5_origins

    op = ProductConvolutionOperator.from_inputs(inputs.make_config("c2"))
    org = c5_origins()
    op.blocks(org[:, :2], org[:, 2:], (8, 8))
    guards_ok("c5")
    op.close()
    guards_ok("end", expect_regions=False)
    print("GUARD TARGET OK", flush=True)


if __name__ == "__main__":
    main()
