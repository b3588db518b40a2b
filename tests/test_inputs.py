"""Input generator (harness) vs the reference's construction rules."""
import os

import numpy as np
import pytest

from paper_1805_06018_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_node_rule():  # pc_operator.cpp:187-194
    assert inputs.uniform_nodes(128, 3) == [0, 42, 85, 127]
    assert inputs.uniform_nodes(512, 7) == [0, 73, 146, 219, 292, 365, 438, 511]
    assert inputs.uniform_nodes(128, 7) == [0, 18, 36, 54, 73, 91, 109, 127]


def test_graded_nodes_c3():
    nodes = inputs.graded_nodes(1024, 10, 5)
    assert len(nodes) == 16 and nodes[0] == 0 and nodes[-1] == 1023
    assert all(b > a for a, b in zip(nodes, nodes[1:]))


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_tents_partition_of_unity(cfg):  # test_pc_operator.cpp:243-249
    inp = inputs.make_config(cfg)
    s = np.zeros(inp.shape)
    for w in inp.weights:
        sl = tuple(slice(l, l + n) for l, n in zip(w.lo, w.values.shape))
        s[sl] += w.values
    assert np.allclose(s, 1.0, rtol=1e-12, atol=0)


def test_tent_is_kronecker_at_nodes():
    inp = inputs.make_config("c1")
    for k, w in enumerate(inp.weights):
        for j, p in enumerate(inp.points):
            if all(l <= c < l + n for c, l, n in zip(p, w.lo, w.values.shape)):
                v = w.values[tuple(c - l for c, l in zip(p, w.lo))]
                assert v == (1.0 if j == k else 0.0)


def test_extension_matches_reference_golden():  # impulse.cpp:61-89 outputs from the reference build
    d = np.load(os.path.join(GOLD, "c1.npz"))
    full = inputs.make_config("c1", full_box=True)
    trimmed = inputs.make_config("c1")
    for k in (0, 5, 6, 15):
        assert tuple(d[f"ext{k}_lo"]) == full.impulses[k].lo
        assert np.array_equal(d[f"ext{k}"], full.impulses[k].values)  # bitwise
        # the trimmed box is the same grid function (zero outside, grid_function.hpp:41-43)
        t, f = trimmed.impulses[k], full.impulses[k]
        sl = tuple(slice(a - b, a - b + s) for a, b, s in zip(t.lo, f.lo, t.values.shape))
        assert np.array_equal(f.values[sl], t.values)
        outside = f.values.copy()
        outside[sl] = 0.0
        assert not outside.any()


@pytest.mark.skipif(not __import__("oracle.ref_lib", fromlist=["x"]).available(),
                    reason="oracle/_ref not built here")
@pytest.mark.parametrize("k", [0, 3, 9, 12])
def test_extension_vs_reference_extend_impulse_3d(k):
    from oracle import ref_lib

    n, m = 10, 2
    blur = inputs.blur_c4(n)
    nodes = [inputs.uniform_nodes(n, m)] * 3
    full = inputs.lattice_operator("x", blur, nodes, full_box=True, ks=[k])
    sizes = [len(a) for a in nodes]
    idx = inputs.lattice_index(nodes, k)
    nb = sorted(int(np.ravel_multi_index(tuple(i + o - 1 for i, o in zip(idx, off)), sizes))
                for off in np.ndindex(3, 3, 3)
                if all(0 <= i + o - 1 < s for i, o, s in zip(idx, off, sizes)))
    pts = [tuple(nodes[a][inputs.lattice_index(nodes, j)[a]] for a in range(3)) for j in nb]
    phis = []
    for q in pts:
        lo = tuple(-v for v in q)
        hi = tuple(n - 1 - v for v in q)
        phis.append(inputs.Field(lo, inputs.impulse_on(blur, (0,) * 3, (n - 1,) * 3, q, lo, hi)))
    lo, vals = ref_lib.extend_impulse((0,) * 3, (n - 1,) * 3, k, nb, pts, phis)
    assert lo == full.impulses[0].lo
    assert np.array_equal(vals, full.impulses[0].values)
