"""The numpy oracle vs the reference's known answers and the reference build's golden vectors.

Pins oracle/pcop_oracle.py (the checker of every GPU parity test) against:
* the reference's own known-answer tests (test_fft.cpp, test_pc_operator.cpp, acceptance.cpp),
  re-expressed here;
* golden outputs of the reference library compiled from its sources (tests/golden, made by
  tests/golden/make_golden.py);
* when oracle/_ref is built in this container, the reference library directly.
"""
import os

import numpy as np
import pytest

from oracle import pcop_oracle as O
from paper_1805_06018_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# --- FFT engine known answers (test_fft.cpp) -------------------------------

def test_delta_kernel_is_identity():  # test_fft.cpp:10-18
    f = O.GF((2,), np.arange(1, 6, dtype=float))
    g = O.fft_convolve(O.GF((0,), np.ones(1)), f)
    assert g.box == f.box
    assert np.allclose(g.values, f.values, rtol=1e-13, atol=0)


def test_hand_convolution():  # test_fft.cpp:20-32
    g = O.fft_convolve(O.GF((0,), np.ones(2)), O.GF((0,), np.array([1.0, 2, 3])))
    assert g.box == ((0,), (3,))
    assert np.allclose(g.values, [1, 3, 5, 3], rtol=1e-13)


def test_offsets_add():  # test_fft.cpp:34-39
    g = O.fft_convolve(O.GF((-2,), np.ones(2)), O.GF((5,), np.full(3, 2.0)))
    assert g.box == ((3,), (6,))


def test_matches_direct_sum_random():  # test_fft.cpp:41-68
    rng = np.random.default_rng(123)
    for d in (1, 2):
        for _ in range(40):
            a_shape = tuple(int(v) for v in rng.integers(0, 9, d) + 1)
            b_shape = tuple(int(v) for v in rng.integers(0, 9, d) + 1)
            psi = O.GF(tuple(rng.integers(-5, 6, d)), rng.uniform(-1, 1, a_shape))
            f = O.GF(tuple(rng.integers(-5, 6, d)), rng.uniform(-1, 1, b_shape))
            fast, slow = O.fft_convolve(psi, f), O.direct_convolve(psi, f)
            assert fast.box == slow.box
            assert np.linalg.norm(fast.values - slow.values) <= 1e-10 * max(1.0, np.linalg.norm(slow.values))


def test_empty_input_rejected():  # test_fft.cpp:70-73
    with pytest.raises(ValueError):
        O.fft_convolve(O.GF((0,), np.zeros(0)), O.GF((0,), np.ones(4)))


def test_padded_shape():  # test_fft.cpp:75-80
    assert O.conv_padded_shape(((0, 0), (4, 9)), ((0, 0), (4, 2))) == [16, 16]


def test_fft_golden_exhaustive():  # acceptance.cpp:459-500 shapes, reference fft_convolve outputs
    d = np.load(os.path.join(GOLD, "fft_kats.npz"))
    assert np.allclose(d["hand"], [1, 3, 5, 3]) and list(d["hand_lo"]) == [0]
    assert list(d["offsets_lo"]) == [3] and d["offsets"].shape == (4,)
    assert list(d["padded_shape"]) == [16, 16]
    worst = 0.0
    for i in range(int(d["n_ex1"])):
        g = O.fft_convolve(O.GF((-2,), d[f"ex1_{i}_psi"]), O.GF((1,), d[f"ex1_{i}_f"]))
        ref = d[f"ex1_{i}_g"]
        worst = max(worst, np.linalg.norm(g.values - ref) / max(1.0, np.linalg.norm(ref)))
        slow = O.direct_convolve(O.GF((-2,), d[f"ex1_{i}_psi"]), O.GF((1,), d[f"ex1_{i}_f"]))
        assert np.linalg.norm(slow.values - ref) <= 1e-10 * max(1.0, np.linalg.norm(ref))
    for i in range(int(d["n_ex2"])):
        g = O.fft_convolve(O.GF((0, -1), d[f"ex2_{i}_psi"]), O.GF((-3, 2), d[f"ex2_{i}_f"]))
        assert list(g.box[0]) == list(d[f"ex2_{i}_lo"])
        ref = d[f"ex2_{i}_g"]
        worst = max(worst, np.linalg.norm(g.values - ref) / max(1.0, np.linalg.norm(ref)))
    assert worst <= 1e-13


# --- the assembled operator (test_pc_operator.cpp) -------------------------

SMALL = {
    "small2d": dict(n=24, dim=2, m=3, sigma=1.7),
    "small3d": dict(n=12, dim=3, m=2, sigma=1.1),
    "small1d": dict(n=50, dim=1, m=5, sigma=2.0),
    "small2d_zeroext": dict(n=20, dim=2, m=2, sigma=1.5, extend=False),
}


@pytest.mark.parametrize("name", list(SMALL))
def test_oracle_vs_reference_golden(name):
    d = np.load(os.path.join(GOLD, f"{name}.npz"))
    inp = inputs.small_lattice(**SMALL[name])
    assert str(d["checksum"]) == inp.checksum(), "input generator changed since the fixtures were made"
    op = O.PCOperator.from_inputs(inp)
    for b in range(d["F"].shape[0]):
        assert rel(op.apply(d["F"][b]), d["G"][b]) <= 1e-13
        assert rel(op.apply_adjoint(d["F"][b]), d["GA"][b]) <= 1e-13
    E = np.array([op.entry(tuple(y), tuple(x)) for y, x in zip(d["y"], d["x"])])
    assert np.array_equal(E, d["E"])  # same summation order as pc_operator.cpp:90-94


def test_oracle_c1_vs_reference_golden():
    d = np.load(os.path.join(GOLD, "c1.npz"))
    inp = inputs.make_config("c1")
    op = O.PCOperator.from_inputs(inp)
    assert rel(op.apply(d["f"]), d["g"]) <= 1e-13
    assert rel(op.apply_adjoint(d["f"]), d["ga"]) <= 1e-13
    E = np.array([op.entry(tuple(y), tuple(x)) for y, x in zip(d["y"], d["x"])])
    assert np.array_equal(E, d["E"])


def _small_op(seed=0):
    return O.PCOperator.from_inputs(inputs.small_lattice(n=14, dim=2, m=2, sigma=1.3))


def test_zero_in_zero_out():  # test_pc_operator.cpp:54-59
    op = _small_op()
    assert np.linalg.norm(op.apply(np.zeros(int(np.prod(op.shape))))) == 0.0


def test_adjoint_is_transpose():  # test_pc_operator.cpp:61-73
    op = _small_op()
    A = op.dense()
    N = A.shape[0]
    At = np.stack([op.apply_adjoint(np.eye(N)[j]) for j in range(N)], 1)
    assert np.linalg.norm(At - A.T) <= 1e-12 * np.linalg.norm(A)


def test_inner_product_identity_and_linearity():  # test_pc_operator.cpp:75-95
    op = _small_op()
    rng = np.random.default_rng(5)
    N = int(np.prod(op.shape))
    for _ in range(10):
        f, h = rng.standard_normal(N), rng.standard_normal(N)
        lhs, rhs = op.apply(f) @ h, f @ op.apply_adjoint(h)
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))
    f, h = rng.standard_normal(N), rng.standard_normal(N)
    assert rel(op.apply(2.5 * f - 0.75 * h), 2.5 * op.apply(f) - 0.75 * op.apply(h)) <= 1e-13


def test_entry_column_equals_apply_of_basis_vector():  # test_pc_operator.cpp:97-116
    op = _small_op()
    n0, n1 = op.shape
    for x in [(0, 0), (3, 7), (13, 13), (6, 0)]:
        e = np.zeros(n0 * n1)
        e[x[0] * n1 + x[1]] = 1.0
        col = op.apply(e)
        via = np.array([op.entry((i, j), x) for i in range(n0) for j in range(n1)])
        assert np.max(np.abs(via - col)) <= 1e-12 * max(1.0, np.linalg.norm(col))


def test_entry_at_sample_point_is_exact_column():  # test_pc_operator.cpp:118-132
    inp = inputs.small_lattice(n=14, dim=2, m=2, sigma=1.3)
    op = O.PCOperator.from_inputs(inp)
    blur = inputs.blur_c1(14, 1.3)
    for p in inp.points:
        e = np.zeros(14 * 14)
        e[p[0] * 14 + p[1]] = 1.0
        true_col = inputs.apply_true_blur(blur, e.reshape(14, 14)).reshape(-1)
        via = np.array([op.entry((i, j), p) for i in range(14) for j in range(14)])
        assert np.max(np.abs(via - true_col)) <= 1e-12


def test_out_of_domain_entry_rejected():  # test_pc_operator.cpp:208-214
    op = _small_op()
    with pytest.raises(ValueError):
        op.entry((-1, 0), (0, 0))


def test_extension_vs_zero_extension_exactness():  # test_pc_operator.cpp:216-227, acceptance criterion 1
    n = 16
    blur = inputs.blur_const(n, 2, 1.4)
    nodes = [inputs.uniform_nodes(n, 2)] * 2
    A = np.stack([inputs.apply_true_blur(blur, np.eye(n * n)[j].reshape(n, n)).reshape(-1) for j in range(n * n)], 1)
    with_ext = O.PCOperator.from_inputs(inputs.lattice_operator("x", blur, nodes)).dense()
    without = O.PCOperator.from_inputs(inputs.lattice_operator("x", blur, nodes, extend=False)).dense()
    assert np.linalg.norm(with_ext - A) / np.linalg.norm(A) <= 1e-12
    assert np.linalg.norm(without - A) / np.linalg.norm(A) >= 1e-3


def test_estimator_vs_reference_golden():  # adaptivity.cpp:75-121
    d = np.load(os.path.join(GOLD, "estimator.npz"))
    inp = inputs.small_lattice(**SMALL["small2d"])
    op = O.PCOperator.from_inputs(inp)
    leaves = [(tuple(l), tuple(h)) for l, h in zip(d["leaf_lo"], d["leaf_hi"])]
    yt, cells, ea, er = O.estimate(op, d["Z"], d["Y"], leaves)
    assert rel(yt, d["ytilde"]) <= 1e-13
    assert np.allclose(cells, d["cells"], rtol=1e-12, atol=0)
    assert abs(ea - float(d["eta_abs"])) <= 1e-12 * float(d["eta_abs"])
    assert abs(er - float(d["eta_rel"])) <= 1e-12 * float(d["eta_rel"])


@pytest.mark.skipif(not __import__("oracle.ref_lib", fromlist=["x"]).available(),
                    reason="oracle/_ref not built here")
def test_oracle_vs_reference_library_random():
    """Direct check against the reference build on random small operators (varying sigma, zero-ext)."""
    from oracle import ref_lib

    for n, dim, m, s, ext in [(18, 2, 2, 1.4, True), (26, 2, 4, 2.1, True), (10, 3, 2, 0.9, True),
                              (30, 1, 4, 1.7, False)]:
        inp = inputs.small_lattice(n=n, dim=dim, m=m, sigma=s, extend=ext)
        ref = ref_lib.RefOperator(inp)
        op = O.PCOperator.from_inputs(inp)
        rng = np.random.default_rng(n)
        f = rng.standard_normal(inp.n_points)
        assert rel(op.apply(f), ref.apply(f)) <= 1e-13
        assert rel(op.apply_adjoint(f), ref.apply(f, adjoint=True)) <= 1e-13


def test_oracle_apply_block_vs_reference_golden():  # pc_operator.cpp:98-130 via the reference build
    d = np.load(os.path.join(GOLD, "apply_block.npz"))
    inp = inputs.small_lattice(**SMALL["small2d"])
    assert str(d["checksum"]) == inp.checksum()
    op = O.PCOperator.from_inputs(inp)
    for i in range(int(d["n"])):
        T = tuple(map(tuple, d[f"b{i}_T"]))
        S = tuple(map(tuple, d[f"b{i}_S"]))
        f = O.GF(S[0], d[f"b{i}_f"])
        for adj in (0, 1):
            g = op.apply_block(T, S, f, bool(adj))
            ref = d[f"b{i}_{adj}"]
            assert np.max(np.abs(g.values - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_oracle_apply_block_is_apply_then_restrict():  # test_pc_operator.cpp:153-183
    inp = inputs.small_lattice(n=14, dim=2, m=2, sigma=1.3)
    op = O.PCOperator.from_inputs(inp)
    rng = np.random.default_rng(10)
    for _ in range(6):
        slo = np.minimum(rng.integers(0, 14, 2), rng.integers(0, 14, 2))
        shi = np.maximum(slo, rng.integers(0, 14, 2))
        tlo = np.minimum(rng.integers(0, 14, 2), rng.integers(0, 14, 2))
        thi = np.maximum(tlo, rng.integers(0, 14, 2))
        T, S = (tuple(tlo), tuple(thi)), (tuple(slo), tuple(shi))
        f = O.GF(S[0], rng.uniform(-1, 1, tuple(shi - slo + 1)))
        full = np.zeros((14, 14))
        full[slo[0]:shi[0] + 1, slo[1]:shi[1] + 1] = f.values
        for adj in (False, True):
            g = (op.apply_adjoint if adj else op.apply)(full.reshape(-1)).reshape(14, 14)
            blk = op.apply_block(T, S, f, adj)
            assert np.max(np.abs(blk.values - g[tlo[0]:thi[0] + 1, tlo[1]:thi[1] + 1])) <= 1e-12


@pytest.mark.parametrize("cfg,seed", [("c3", 2)])
def test_oracle_vs_reference_headline_fingerprint(cfg, seed):
    """The numpy restatement at the FULL c3 size against the reference's own apply
    (tests/golden/headline_c3.npz, made by tests/golden/make_headline_golden.py)."""
    import os

    from headline_common import compare
    from paper_1805_06018_b200.operator import normal_vectors

    inp = inputs.make_config(cfg)
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", f"headline_{cfg}.npz"))
    assert str(gold["checksum"]) == inp.checksum()
    f = normal_vectors(seed, 1, inp.n_points)[0]
    err = compare(O.PCOperator.from_inputs(inp).apply(f), inp.shape,
                  {k: gold[f"apply0_{k}"] for k in ("samples", "tiles", "norm")})
    assert max(err.values()) <= 1e-12, err
