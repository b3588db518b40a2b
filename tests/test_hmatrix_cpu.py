"""Host-side H-matrix layer (no GPU): cluster tree, admissibility, PCHM container.

The library's ClusterTree (csrc/hmatrix.cpp via pcb_cluster_tree) vs the oracle restatement
(oracle/hmatrix_oracle.py), both vs the reference's known answers (test_hmatrix.cpp:22-98), and the
PCHM v1 byte format in both directions (hmatrix.cpp:433-526).
"""
import itertools
import math
import os

import numpy as np
import pytest

from oracle import hmatrix_oracle as HO
from paper_1805_06018_b200 import lib
from paper_1805_06018_b200.hmatrix import HMatrix

pytestmark = pytest.mark.skipif(not os.path.exists(lib.LIB_PATH), reason="library not built")


def test_reference_tree_kats():
    """test_hmatrix.cpp:22-53."""
    for impl in ("lib", "oracle"):
        def tree(lo, hi, cap):
            if impl == "lib":
                return [(n.size(), n.lo, n.hi, n.split_axis, n.child_lo) for n in HMatrix.cluster_tree((lo, hi), cap).nodes()]
            t = HO.Tree(lo, hi, cap)
            return [(t.size(i), n["bbox"][0], n["bbox"][1], n["split_axis"], n["child_lo"]) for i, n in enumerate(t.nodes)]
        t = tree((0,), (7,), 2)
        assert len(t) == 7 and all(n[0] == 2 for n in t if n[4] < 0)
        t = tree((0, 0), (7, 7), 32)
        assert [n[0] for n in t] == [64, 32, 32] and t[1][4] < 0 and t[0][3] == 0
        assert (t[1][1], t[1][2]) == ((0, 0), (3, 7)) and (t[2][1], t[2][2]) == ((4, 0), (7, 7))
        t = tree((0, 0), (1, 1), 8)
        assert len(t) == 1 and t[0][4] < 0
        t = tree((0,), (6,), 4)
        assert t[0][4] >= 0 and t[t[0][4]][0] == 4 and t[0][0] - t[t[0][4]][0] == 3


@pytest.mark.parametrize("lo,hi,cap", [((0,), (40,), 3), ((0, 0), (12, 9), 7), ((-3, 2), (9, 20), 16),
                                       ((0, 0, 0), (5, 6, 4), 9), ((2,), (2,), 1), ((0, 0), (8, 8), 8)])
def test_tree_matches_oracle(lo, hi, cap):
    h = HMatrix.cluster_tree((lo, hi), cap)
    o = HO.Tree(lo, hi, cap)
    assert list(h.perm()) == o.perm
    for n, m in zip(h.nodes(), o.nodes):
        assert (n.begin, n.end, n.split_axis, n.child_lo, n.child_hi) == \
            (m["begin"], m["end"], m["split_axis"], m["child_lo"], m["child_hi"])
        assert (n.lo, n.hi) == m["bbox"]
    assert len(h.nodes()) == len(o.nodes)


def test_admissibility_brute_force():
    """test_hmatrix.cpp:56-98: bboxes, diameters, distances and admissibility vs brute force."""
    lo, hi = (0, 0), (10, 13)
    h = HMatrix.cluster_tree((lo, hi), 6)
    o = HO.Tree(lo, hi, 6)
    nodes = h.nodes()
    perm = h.perm()
    rng = np.random.default_rng(0)
    for _ in range(200):
        a, b = (int(v) for v in rng.integers(0, len(nodes), 2))
        pa = [HO.delinearize(lo, hi, p) for p in perm[nodes[a].begin:nodes[a].end]]
        pb = [HO.delinearize(lo, hi, p) for p in perm[nodes[b].begin:nodes[b].end]]
        bb = lambda ps: (tuple(min(p[i] for p in ps) for i in range(2)), tuple(max(p[i] for p in ps) for i in range(2)))
        ba, bbx = bb(pa), bb(pb)
        assert (nodes[a].lo, nodes[a].hi) == ba
        diam = lambda x: math.sqrt(sum((x[1][i] - x[0][i]) ** 2 for i in range(2)))
        gap = lambda x, y: math.sqrt(sum(max(0, x[0][i] - y[1][i], y[0][i] - x[1][i]) ** 2 for i in range(2)))
        adm, dist, da, db = h.admissible(a, b)
        assert abs(da - diam(ba)) <= 1e-12 * max(1, diam(ba)) and abs(dist - gap(ba, bbx)) <= 1e-12 * max(1, dist)
        assert adm == (gap(ba, bbx) >= min(diam(ba), diam(bbx))) == o.admissible(a, b)
        assert adm == h.admissible(b, a)[0]


def test_partition_covers_product_once():
    """test_hmatrix.cpp:100-115 on the oracle partition (the library's is checked on the GPU)."""
    o = HO.Tree((0, 0), (8, 8), 8)
    cover = np.zeros((o.N, o.N), dtype=int)
    for t, s, _ in HO.partition(o):
        for i in range(o.nodes[t]["begin"], o.nodes[t]["end"]):
            for j in range(o.nodes[s]["begin"], o.nodes[s]["end"]):
                cover[o.perm[i], o.perm[j]] += 1
    assert (cover == 1).all()


def test_pchm_both_directions(tmp_path):
    lo, hi = (0, 0), (6, 9)
    h = HMatrix.cluster_tree((lo, hi), 5)
    p1 = str(tmp_path / "lib.pchm")
    h.save(p1)
    d = HO.read_pchm(p1)
    o = HO.Tree(lo, hi, 5)
    assert d["lo"] == lo and d["hi"] == hi and d["leaf_cap"] == 5 and list(d["perm"]) == o.perm
    assert [tuple(n.values()) for n in d["nodes"]] == \
        [(n["begin"], n["end"], n["split_axis"], n["child_lo"], n["child_hi"]) for n in o.nodes]
    # an oracle-written file with blocks loads, inspects and multiplies in the library
    rng = np.random.default_rng(1)
    blocks = []
    for t, s, lr in HO.partition(o):
        nt, ns = o.size(t), o.size(s)
        if lr:
            k = int(rng.integers(0, 3))
            blocks.append((t, s, True, rng.standard_normal((nt, k)), rng.standard_normal((k, ns)), None))
        else:
            blocks.append((t, s, False, None, None, rng.standard_normal((nt, ns))))
    p2 = str(tmp_path / "oracle.pchm")
    HO.write_pchm(p2, lo, hi, 5, o.perm, o.nodes, blocks)
    g = HMatrix.load(p2)
    f = rng.standard_normal(o.N)
    assert np.allclose(g.matvec(f), HO.matvec(o, blocks, f), rtol=1e-13, atol=1e-13)
    for i, b in enumerate(g.blocks()):
        ref = blocks[i]
        assert (b.t_node, b.s_node, b.low_rank) == ref[:3]
        if b.low_rank:
            assert np.array_equal(b.B, ref[3]) and np.array_equal(b.C, ref[4])
        else:
            assert np.array_equal(b.dense, ref[5])
    p3 = str(tmp_path / "again.pchm")
    g.save(p3)
    assert open(p2, "rb").read() == open(p3, "rb").read()


def test_pchm_errors(tmp_path):
    p = tmp_path / "bad.pchm"
    p.write_bytes(b"XXXX" + bytes(40))
    with pytest.raises(ValueError, match="bad magic"):
        HMatrix.load(str(p))
    h = HMatrix.cluster_tree(((0,), (9,)), 3)
    h.save(str(p))
    data = p.read_bytes()
    p.write_bytes(data[:4] + b"\x02\x00\x00\x00" + data[8:])
    with pytest.raises(ValueError, match="unsupported version"):
        HMatrix.load(str(p))
    p.write_bytes(data[:-10])
    with pytest.raises(ValueError, match="truncated"):
        HMatrix.load(str(p))
    with pytest.raises(ValueError, match="cannot open"):
        HMatrix.load(str(tmp_path / "missing.pchm"))
    with pytest.raises(ValueError, match="leaf_cap >= 1"):
        HMatrix.cluster_tree(((0,), (9,)), 0)
    with pytest.raises(ValueError, match="size mismatch"):
        h.matvec(np.zeros(3))


def test_oracle_tree_and_partition_vs_reference_pchm(tmp_path):
    """The numpy restatement (oracle/hmatrix_oracle.py) against the reference's own PCHM files
    (tests/golden/hmatrix_ref_*.pchm.gz, assemble_hmatrix + save_hmatrix compiled verbatim)."""
    import gzip
    import os

    from oracle import hmatrix_oracle as HO
    from paper_1805_06018_b200 import inputs

    inp = inputs.small_lattice(n=12, dim=2, m=2, sigma=3.0)
    gold = os.path.join(os.path.dirname(__file__), "golden")
    for method in ("randomized", "cur"):
        p = tmp_path / f"{method}.pchm"
        p.write_bytes(gzip.decompress((open(os.path.join(gold, f"hmatrix_ref_{method}.pchm.gz"), "rb").read())))
        d = HO.read_pchm(str(p))
        o = HO.Tree(inp.dom_lo, inp.dom_hi, 16)
        assert list(d["perm"]) == o.perm
        assert [(n["begin"], n["end"], n["split_axis"], n["child_lo"], n["child_hi"]) for n in d["nodes"]] == \
            [(n["begin"], n["end"], n["split_axis"], n["child_lo"], n["child_hi"]) for n in o.nodes]
        assert [(t, s, lr) for t, s, lr, *_ in d["blocks"]] == HO.partition(o)
