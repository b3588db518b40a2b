"""H-matrix assembly over the GPU operator (csrc/hmatrix.cpp), mirroring the
reference's test_hmatrix.cpp:100-256 plus parity of the CUR path and the PCHM file against the oracle
restatement (oracle/hmatrix_oracle.py) on the reference-pinned entry() (oracle/pcop_oracle.py)."""
import numpy as np
import pytest

from oracle import hmatrix_oracle as HO
from oracle import pcop_oracle as O
from paper_1805_06018_b200 import inputs
from paper_1805_06018_b200.hmatrix import HMatrix
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors

pytestmark = pytest.mark.gpu


def blur_op(n=16, dim=2, m=2, sigma=1.6):
    inp = inputs.small_lattice(n=n, dim=dim, m=m, sigma=sigma)
    return inp, ProductConvolutionOperator.from_inputs(inp)


def identity_op(n=25):
    inp = inputs.lattice_operator("id1d", inputs.blur_const(n, 1, 0.2), [inputs.uniform_nodes(n, 1)])
    return inp, ProductConvolutionOperator.from_inputs(inp)


def dense_of(op, tree_nodes, perm, lo, hi, t, s):
    tn, sn = tree_nodes[t], tree_nodes[s]
    ys = [HO.delinearize(lo, hi, perm[i]) for i in range(tn.begin, tn.end)]
    xs = [HO.delinearize(lo, hi, perm[j]) for j in range(sn.begin, sn.end)]
    Y = np.array([y for y in ys for _ in xs])
    X = np.array([x for _ in ys for x in xs])
    return op.entries(Y, X).reshape(len(ys), len(xs))


@pytest.mark.parametrize("method", ["randomized", "cur"])
def test_partition_covers_once_and_matches_oracle(gpu, method):
    inp, op = blur_op(9, m=2)
    h = HMatrix.assemble(op, 1e-8, 8, method)
    o = HO.Tree(inp.dom_lo, inp.dom_hi, 8)
    assert [(b.t_node, b.s_node, b.low_rank) for b in h.blocks()] == HO.partition(o)
    perm = h.perm()
    nodes = h.nodes()
    cover = np.zeros((81, 81), dtype=int)
    for b in h.blocks():
        for i in range(nodes[b.t_node].begin, nodes[b.t_node].end):
            for j in range(nodes[b.s_node].begin, nodes[b.s_node].end):
                cover[perm[i], perm[j]] += 1
    assert (cover == 1).all()


def test_compressed_blocks_match_dense(gpu):
    """test_hmatrix.cpp:117-147."""
    inp, op = blur_op(16, sigma=3.0)  # support radius 12: far blocks are not identically zero
    tol = 1e-8
    h = HMatrix.cluster_tree((inp.dom_lo, inp.dom_hi), 24)
    nodes, perm = h.nodes(), h.perm()
    pairs = []
    for a in range(len(nodes)):
        for b in range(a + 1, len(nodes)):
            if h.admissible(a, b)[0] and len(pairs) < 4:
                pairs.append((a, b))
    assert pairs
    for method in ("randomized", "cur"):
        blocks = h.compress(op, pairs, method, tol)
        for (a, b), blk in zip(pairs, blocks):
            D = dense_of(op, nodes, perm, inp.dom_lo, inp.dom_hi, a, b)
            err = np.linalg.norm(D - blk.B @ blk.C)
            assert err <= tol * max(np.linalg.norm(D), 1e-14), (method, a, b, blk.rank)
            assert blk.rank <= 20
        assert max(b.rank for b in blocks) > 0


def test_cur_matches_oracle_aca(gpu):
    """The lockstep-batched ACA = the reference's sequential ACA on the reference-pinned entry()."""
    inp, op = blur_op(12, m=2, sigma=1.3)
    ref = O.PCOperator.from_inputs(inp)
    h = HMatrix.cluster_tree((inp.dom_lo, inp.dom_hi), 9)
    o = HO.Tree(inp.dom_lo, inp.dom_hi, 9)
    pairs = [(t, s) for t, s, lr in HO.partition(o) if lr][:12]
    for fixed in (0, 3):
        got = h.compress(op, pairs, "cur", 1e-6, fixed)
        for (t, s), blk in zip(pairs, got):
            B, C, capped = HO.compress_cur(ref.entry, o, t, s, 1e-6, fixed)
            assert blk.rank == B.shape[1]
            if B.size:
                assert np.abs(blk.B - B).max() <= 1e-12 * np.abs(B).max()
                assert np.abs(blk.C - C).max() <= 1e-12 * max(1.0, np.abs(C).max())


def test_zero_blocks_rank_zero(gpu):
    """test_hmatrix.cpp:149-170: identity has zero off-diagonal blocks."""
    inp, op = identity_op(32)
    h = HMatrix.cluster_tree((inp.dom_lo, inp.dom_hi), 8)
    nodes = h.nodes()
    leaves = [i for i, n in enumerate(nodes) if n.is_leaf()]
    t = leaves[0]
    s = next(i for i in leaves[1:] if h.admissible(t, i)[1] > 10)
    for method in ("randomized", "cur"):
        assert h.compress(op, [(t, s)], method, 1e-10)[0].rank == 0


def test_matvec_matches_apply(gpu):
    """test_hmatrix.cpp:172-186 (randomized)."""
    inp, op = blur_op(16, sigma=3.0)
    h = HMatrix.assemble(op, 1e-10, 32, "randomized")
    F = normal_vectors(5, 3, inp.n_points)
    for f in F:
        a = op.apply(f)
        assert np.linalg.norm(a - h.matvec(f)) <= 1e-8 * np.linalg.norm(a)
    assert h.info["n_low_rank"] > 0 and h.info["n_dense"] > 0 and h.info["max_rank"] > 0


def test_cur_hmatrix_equals_oracle(gpu):
    """The whole CUR H-matrix = the oracle's (partition, dense leaves, sequential ACA).  ACA's
    partially pivoted stopping test is a heuristic: on these truncated, tent-weighted kernels it can
    stop early (matvec error ~1e-6 at tol 1e-10), in the reference's algorithm as here."""
    inp, op = blur_op(16, sigma=3.0)
    ref = O.PCOperator.from_inputs(inp)
    h = HMatrix.assemble(op, 1e-10, 32, "cur")
    o = HO.Tree(inp.dom_lo, inp.dom_hi, 32)
    blocks = []
    for t, s, lr in HO.partition(o):
        if lr:
            B, C, _ = HO.compress_cur(ref.entry, o, t, s, 1e-10)
            blocks.append((t, s, True, B, C, None))
        else:
            blocks.append((t, s, False, None, None, HO.dense_block(ref.entry, o, t, s)))
    got = h.blocks()
    assert [(b.t_node, b.s_node, b.low_rank, b.rank) for b in got] == \
        [(t, s, lr, B.shape[1] if lr else 0) for t, s, lr, B, _, _ in blocks]
    for b, (t, s, lr, B, C, D) in zip(got, blocks):
        if not lr:
            assert np.array_equal(b.dense, D)  # entries are bit-identical to the reference's
    f = normal_vectors(5, 1, inp.n_points)[0]
    want = HO.matvec(o, blocks, f)
    assert np.linalg.norm(h.matvec(f) - want) <= 1e-12 * np.linalg.norm(want)
    a = op.apply(f)
    assert np.linalg.norm(a - want) <= 1e-4 * np.linalg.norm(a)


def test_identity_blocks(gpu):
    """test_hmatrix.cpp:188-203."""
    inp, op = identity_op(25)
    h = HMatrix.assemble(op, 1e-10, 4, "randomized")
    for b in h.blocks():
        if b.low_rank:
            assert b.rank == 0
        elif b.t_node == b.s_node:
            assert np.linalg.norm(b.dense - np.eye(b.dense.shape[0])) <= 1e-12
        else:
            assert np.linalg.norm(b.dense) <= 1e-12


def test_fixed_rank_caps(gpu):
    """test_hmatrix.cpp:205-215."""
    inp, op = blur_op(16, sigma=3.0)
    h = HMatrix.assemble(op, 1e-12, 32, "randomized", fixed_rank=5)
    ranks = [b.rank for b in h.blocks() if b.low_rank and b.rank > 0]
    assert ranks and max(ranks) <= 5


def test_pchm_round_trip_and_oracle_reader(gpu, tmp_path):
    """test_hmatrix.cpp:217-231 plus the byte format read back by the oracle's load_hmatrix."""
    inp, op = blur_op(12)
    h = HMatrix.assemble(op, 1e-9, 16, "randomized")
    path = str(tmp_path / "h.pchm")
    h.save(path)
    g = HMatrix.load(path)
    assert np.array_equal(g.perm(), h.perm()) and len(g.blocks()) == len(h.blocks())
    f = normal_vectors(9, 1, inp.n_points)[0]
    assert np.array_equal(h.matvec(f), g.matvec(f))
    d = HO.read_pchm(path)
    o = HO.Tree(inp.dom_lo, inp.dom_hi, 16)
    assert list(d["perm"]) == o.perm
    assert np.allclose(HO.matvec(o, d["blocks"], f), h.matvec(f), rtol=1e-12, atol=1e-14)


def test_far_clusters_of_smooth_kernel_low_rank(gpu):
    """test_hmatrix.cpp:233-256: 1-D wide Gaussian, separated leaves stay low rank at 1e-8."""
    inp = inputs.lattice_operator("wide1d", inputs.blur_const(64, 1, 6.0), [inputs.uniform_nodes(64, 1)])
    op = ProductConvolutionOperator.from_inputs(inp)
    h = HMatrix.cluster_tree((inp.dom_lo, inp.dom_hi), 8)
    nodes = h.nodes()
    leaves = [i for i, n in enumerate(nodes) if n.is_leaf()]
    pairs = [(a, b) for a in leaves for b in leaves if h.admissible(a, b)[1] >= 16][:7]
    assert pairs
    for blk in h.compress(op, pairs, "randomized", 1e-8):
        assert blk.rank <= 10


def test_assemble_3d_and_errors(gpu):
    inp, op = blur_op(8, dim=3, m=1, sigma=1.0)
    h = HMatrix.assemble(op, 1e-8, 32, "cur")
    f = normal_vectors(2, 1, inp.n_points)[0]
    a = op.apply(f)
    assert np.linalg.norm(a - h.matvec(f)) <= 1e-6 * np.linalg.norm(a)
    with pytest.raises(ValueError, match="leaf_cap"):
        HMatrix.assemble(op, 1e-8, 0, "cur")


@pytest.mark.parametrize("method", ["randomized", "cur"])
def test_gpu_matvec_batch_bit_identical_to_host_matvec(gpu, method, tmp_path):
    """pcb_hmatrix_matvec_batch (three GPU passes: t = C x, y = D x | B t, ordered row sums) keeps the
    host loop's summation order (HMatrix::matvec, hmatrix.cpp:379-400): every vector equals the host
    matvec bit for bit; also for an H-matrix loaded from a PCHM file, and with rank-0 blocks."""
    inp = inputs.small_lattice(n=40, dim=2, m=3, sigma=2.0)
    op = ProductConvolutionOperator.from_inputs(inp)
    h = HMatrix.assemble(op, 1e-8, 32, method)
    F = normal_vectors(21, 5, inp.n_points)
    G = h.matvec_batch(F)
    for b in range(5):
        assert np.array_equal(G[b], h.matvec(F[b])), b
    assert np.linalg.norm(G[0] - op.apply(F[0])) <= (1e-5 if method == "cur" else 1e-8) * np.linalg.norm(G[0])
    path = str(tmp_path / "m.pchm")
    h.save(path)
    g = HMatrix.load(path)
    assert np.array_equal(g.matvec_batch(F[:2]), G[:2])
    assert np.array_equal(h.matvec_batch(F[:1]), G[:1])  # a smaller batch on the cached device copy
