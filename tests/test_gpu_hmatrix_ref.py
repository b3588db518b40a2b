"""H-matrix parity against the REFERENCE's own hmatrix.cpp: assemble_hmatrix,
compress_randomized / compress_cur, HMatrix::matvec and the PCHM v1 container
(hmatrix.cpp:138-526), compiled verbatim into oracle/_ref against the Eigen shim.

* always: vs the committed reference PCHM files tests/golden/hmatrix_ref_{method}.pchm.gz
  (tests/golden/make_hmatrix_golden.py);
* when the reference build is shipped: vs a live reference assembly, and cross-loading each
  side's PCHM file in the other's reader.

What must agree, and how:
* the cluster tree and block partition (PCHM header, permutation, nodes, block (t, s, kind) list):
  byte-identical;
* dense leaves: bit-identical (the GPU entry gather sums in the reference order);
* CUR (adaptive cross approximation on entry()): same ranks, factors to 1e-12 relative;
* randomized range finder: same ranks (the singular-value tail decides), and the block
  B C to 1e-10 of the block norm (Q and the SVD factors are unique up to rotation within the
  kept subspace; the shim's QR/SVD differ from ours in rounding);
* matvec: to 1e-12 (CUR) / 1e-10 (randomized) relative.
"""
import gzip
import os
import struct

import numpy as np
import pytest

from oracle import hmatrix_oracle as HO
from paper_1805_06018_b200 import inputs
from paper_1805_06018_b200.hmatrix import HMatrix
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = dict(n=12, dim=2, m=2, sigma=3.0)
TOL, LEAF = 1e-8, 16
FACTOR_TOL = {"cur": 1e-12, "randomized": 1e-10}


def tree_bytes(buf: bytes) -> bytes:
    """The PCHM prefix up to (and including) the block count: header, perm, nodes."""
    ver, d, N, cap = struct.unpack_from("<IIQI", buf, 4)
    off = 24 + 16 * d + 8 * N
    (nn,) = struct.unpack_from("<Q", buf, off)
    return buf[: off + 8 + 28 * nn + 8]


def ours(method, tmp_path):
    inp = inputs.small_lattice(**SPEC)
    op = ProductConvolutionOperator.from_inputs(inp)
    h = HMatrix.assemble(op, TOL, LEAF, method)
    path = str(tmp_path / f"ours_{method}.pchm")
    h.save(path)
    return inp, op, h, path


def compare_files(path_ours, path_ref, method):
    a, b = open(path_ours, "rb").read(), open(path_ref, "rb").read()
    assert tree_bytes(a) == tree_bytes(b)
    da, db = HO.read_pchm(path_ours), HO.read_pchm(path_ref)
    assert [(t, s, lr) for t, s, lr, *_ in da["blocks"]] == [(t, s, lr) for t, s, lr, *_ in db["blocks"]]
    # the scale of the matrix: an admissible block whose entries are all exactly zero (beyond every
    # kernel's truncation radius) is a rank-0 block here (the block applies use the exact entry
    # gather), while the reference's FFT-based apply_block returns rounding noise (~1e-17) for it and
    # its range finder "compresses" that noise to some rank: such blocks must be negligible
    big = max([np.linalg.norm(Br @ Cr) for _, _, lr, Br, Cr, _ in db["blocks"] if lr and Br.shape[1]] + [1e-300])
    for (t, s, lr, B, C, D), (_, _, _, Br, Cr, Dr) in zip(da["blocks"], db["blocks"]):
        if not lr:
            assert np.array_equal(D, Dr), (t, s)  # dense leaves: reference entry(), bitwise
            continue
        if method == "randomized" and B.shape[1] == 0 and Br.shape[1] > 0:
            assert np.linalg.norm(Br @ Cr) <= 1e-13 * big, (t, s, np.linalg.norm(Br @ Cr), big)
            continue
        assert B.shape[1] == Br.shape[1], (method, t, s, B.shape, Br.shape)  # same rank
        if B.shape[1] == 0:
            continue
        M, Mr = B @ C, Br @ Cr
        nrm = max(np.linalg.norm(Mr), 1e-300)
        assert np.linalg.norm(M - Mr) <= FACTOR_TOL[method] * nrm, (method, t, s, np.linalg.norm(M - Mr) / nrm)
        if method == "cur":  # same pivots: the factors themselves agree
            assert np.linalg.norm(B - Br) <= 1e-12 * max(np.linalg.norm(Br), 1e-300)
            assert np.linalg.norm(C - Cr) <= 1e-12 * max(np.linalg.norm(Cr), 1e-300)
    return da, db


@pytest.mark.parametrize("method", ["randomized", "cur"])
def test_hmatrix_vs_reference_golden(gpu, method, tmp_path):
    inp, op, h, path = ours(method, tmp_path)
    assert open(os.path.join(GOLD, "hmatrix_ref.checksum")).read().strip() == inp.checksum()
    ref_path = str(tmp_path / f"ref_{method}.pchm")
    with open(ref_path, "wb") as f:
        f.write(gzip.decompress(open(os.path.join(GOLD, f"hmatrix_ref_{method}.pchm.gz"), "rb").read()))
    da, db = compare_files(path, ref_path, method)
    # matvec of the reference's factors (its own HMatrix::matvec restated) vs ours
    tree = HO.Tree(inp.dom_lo, inp.dom_hi, LEAF)
    f = normal_vectors(31, 1, inp.n_points)[0]
    g_ref = HO.matvec(tree, db["blocks"], f)
    assert np.linalg.norm(h.matvec(f) - g_ref) <= FACTOR_TOL[method] * np.linalg.norm(g_ref)
    # our loader reads the reference's file
    g = HMatrix.load(ref_path)
    assert np.allclose(g.matvec(f), g_ref, rtol=0, atol=1e-13 * np.abs(g_ref).max())


@pytest.mark.parametrize("method", ["randomized", "cur"])
def test_hmatrix_vs_live_reference(gpu, method, tmp_path):
    from oracle import ref_lib

    if not ref_lib.available():
        pytest.skip("reference build (oracle/_ref) not shipped with this copy")
    inp, op, h, path = ours(method, tmp_path)
    R = ref_lib.RefHMatrix.assemble(ref_lib.RefOperator(inp), TOL, LEAF, method)
    ref_path = str(tmp_path / f"live_{method}.pchm")
    R.save(ref_path)
    compare_files(path, ref_path, method)
    f = normal_vectors(32, 1, inp.n_points)[0]
    g_ref = R.matvec(f)
    assert np.linalg.norm(h.matvec(f) - g_ref) <= FACTOR_TOL[method] * np.linalg.norm(g_ref)
    # the reference's load_hmatrix reads OUR file; its matvec of our factors equals ours
    R2 = ref_lib.RefHMatrix.load(path, inp.n_points)
    assert R2.info()["n_blocks"] == h.info["n_blocks"]
    assert np.allclose(R2.matvec(f), h.matvec(f), rtol=0, atol=1e-13 * np.abs(g_ref).max())


@pytest.mark.parametrize("method", ["randomized", "cur"])
def test_hmatrix_vs_live_reference_larger(gpu, method, tmp_path):
    """The same comparison on a 48 x 48 domain (N = 2,304, leaf 32: ~3,800 blocks, ranks up to ~36):
    the sizes where the block factorizations run on several host threads and the tall SVDs go
    through QR.  File-level comparison (tree, partition, dense leaves, ranks, factors) and matvec."""
    from oracle import ref_lib

    if not ref_lib.available():
        pytest.skip("reference build (oracle/_ref) not shipped with this copy")
    inp = inputs.small_lattice(n=48, dim=2, m=3, sigma=2.0)
    op = ProductConvolutionOperator.from_inputs(inp)
    h = HMatrix.assemble(op, TOL, 32, method)
    path = str(tmp_path / f"ours48_{method}.pchm")
    h.save(path)
    R = ref_lib.RefHMatrix.assemble(ref_lib.RefOperator(inp), TOL, 32, method)
    ref_path = str(tmp_path / f"live48_{method}.pchm")
    R.save(ref_path)
    compare_files(path, ref_path, method)
    f = normal_vectors(33, 1, inp.n_points)[0]
    g_ref = R.matvec(f)
    assert np.linalg.norm(h.matvec(f) - g_ref) <= FACTOR_TOL[method] * np.linalg.norm(g_ref)
