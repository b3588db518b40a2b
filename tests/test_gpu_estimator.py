"""GPU-resident estimator state (``pcb_estimator_*``; adaptivity.cpp:14-121).

* probes = the reference's draws (mt19937_64 + normal_distribution, probe i = draws [iN,(i+1)N));
* one update with every k = the reference golden (tests/golden/estimator.npz) and pcb_probe_estimate;
* incremental = scratch (test_adaptivity.cpp:77-119): grow the operator, pass only the new ks;
* the reference's changed_ks checks (adaptivity.cpp:79-88) raise with the reference's messages;
* Y = A^* Z on the device through the true operator equals the host route.
"""
import os

import numpy as np
import pytest

from paper_1805_06018_b200 import inputs
from paper_1805_06018_b200.estimator import Estimator
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors
from paper_1805_06018_b200.true_operator import BlurOperator

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
SMALL2D = dict(n=24, dim=2, m=3, sigma=1.7)


def test_probes_are_reference_draws(gpu):
    est = Estimator(((0, 0), (23, 23)), q=3, seed=7)
    Z, _, _ = est.read()
    assert np.array_equal(Z, normal_vectors(7, 3, 576))


@pytest.mark.parametrize("mode", ["global", "local"])
def test_update_matches_reference_golden(gpu, mode):
    d = np.load(os.path.join(GOLD, "estimator.npz"))
    inp = inputs.small_lattice(**SMALL2D)
    op = ProductConvolutionOperator.from_inputs(inp, mode=mode)
    est = Estimator((inp.dom_lo, inp.dom_hi), q=4, seed=5)
    Z, _, _ = est.read()
    assert np.array_equal(Z, d["Z"])  # the golden probes are seed-5 draws
    est.set_y(d["Y"])
    ea, er = est.update(op, range(op.rank))
    assert abs(ea - float(d["eta_abs"])) <= 1e-11 * float(d["eta_abs"])
    assert abs(er - float(d["eta_rel"])) <= 1e-11 * float(d["eta_rel"])
    leaves = [(tuple(l), tuple(h)) for l, h in zip(d["leaf_lo"], d["leaf_hi"])]
    assert np.allclose(est.cells(leaves), d["cells"], rtol=1e-11, atol=0)
    _, _, yt = est.read()
    assert np.linalg.norm(yt - d["ytilde"]) <= 1e-11 * np.linalg.norm(d["ytilde"])


def test_incremental_equals_scratch(gpu):
    """Grow the expansion r1 -> r (new terms appended, as build_adaptive's append_pair does) and
    pass only the new ks: eta equals a from-scratch estimate on the grown operator."""
    inp = inputs.small_lattice(n=40, dim=2, m=4, sigma=2.3)
    blur = inputs.blur_c1(40, 2.3)
    r = inp.rank
    r1 = r // 2
    A = BlurOperator.from_spec(blur)
    est = Estimator((inp.dom_lo, inp.dom_hi), q=5, seed=3)
    est.set_y_from(A)
    op1 = ProductConvolutionOperator.from_inputs(inp.subset(range(r1)))
    e1 = est.update(op1, range(r1))
    op2 = ProductConvolutionOperator.from_inputs(inp)
    e2 = est.update(op2, range(r1, r))
    scratch = Estimator((inp.dom_lo, inp.dom_hi), q=5, seed=3)
    scratch.set_y_from(A)
    s2 = scratch.update(op2, range(r))
    assert e1[1] > e2[1]
    assert abs(e2[0] - s2[0]) <= 1e-12 * s2[0] and abs(e2[1] - s2[1]) <= 1e-12 * s2[1]
    Z, Y, _ = est.read()
    _, cells, ea, er = op2.probe_estimate(Z, Y, [((0, 0), (39, 39))])
    assert abs(er - e2[1]) <= 1e-12 * er and abs(cells[0] - ea) <= 1e-12 * ea


def test_changed_ks_checks(gpu):
    inp = inputs.small_lattice(**SMALL2D)
    op = ProductConvolutionOperator.from_inputs(inp)
    est = Estimator((inp.dom_lo, inp.dom_hi), q=2, seed=1)
    with pytest.raises(ValueError, match="Y = A"):
        est.update(op, range(op.rank))
    est.set_y(np.zeros((2, inp.n_points)))
    with pytest.raises(ValueError, match="eta_for_cells"):
        est.cells([((0, 0), (1, 1))])
    with pytest.raises(ValueError, match="bad changed id"):
        est.update(op, [op.rank])
    with pytest.raises(ValueError, match="uncached sample point not marked changed"):
        est.update(op, range(op.rank - 1))
    est.update(op, range(op.rank))
    assert est.eta_rel == 0.0  # ||Y|| = 0 -> eta_rel = 0 (adaptivity.cpp:111)
    small = ProductConvolutionOperator.from_inputs(inp.subset(range(op.rank - 1)))
    with pytest.raises(ValueError, match="stale cache"):
        est.update(small, [])
    with pytest.raises(ValueError, match="leaf box outside"):
        est.cells([((0, 0), (24, 3))])
    with pytest.raises(ValueError, match="q >= 1"):
        Estimator((inp.dom_lo, inp.dom_hi), q=0, seed=1)


def test_y_from_true_operator_c3(gpu):
    blur = inputs.blur_c3(1024)
    A = BlurOperator.from_spec(blur)
    est = Estimator(((0, 0), (1023, 1023)), q=2, seed=2)
    est.set_y_from(A)
    Z, Y, _ = est.read()
    H = A.apply_adjoint(Z.reshape(2, 1024, 1024)).reshape(2, -1)
    assert np.array_equal(Y, H)


def test_one_dimensional_domain(gpu):
    inp = inputs.small_lattice(n=50, dim=1, m=5, sigma=2.0)
    op = ProductConvolutionOperator.from_inputs(inp)
    est = Estimator((inp.dom_lo, inp.dom_hi), q=3, seed=4)
    Z, _, _ = est.read()
    Y = Z * 0.5
    est.set_y(Y)
    ea, er = est.update(op, range(op.rank))
    leaves = [((0,), (24,)), ((25,), (49,))]
    yt, cells, ea2, er2 = op.probe_estimate(Z, Y, leaves, want_ytilde=True)
    assert abs(ea - ea2) <= 1e-13 * ea2 and abs(er - er2) <= 1e-13 * er2
    assert np.allclose(est.cells(leaves), cells, rtol=1e-13, atol=0)


def _philox_ref(seed, count):
    """numpy restatement of Philox4x32-10 + Box-Muller (the device generator's definition)."""
    M0, M1, W0, W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85
    pairs = (count + 1) // 2
    i = np.arange(pairs, dtype=np.uint64)
    c = [(i & 0xFFFFFFFF).astype(np.uint64), (i >> np.uint64(32)).astype(np.uint64), np.zeros_like(i), np.zeros_like(i)]
    k0, k1 = np.uint64(seed & 0xFFFFFFFF), np.uint64(seed >> 32)
    mask = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = np.uint64(M0) * c[0]
        p1 = np.uint64(M1) * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & mask
        hi1, lo1 = p1 >> np.uint64(32), p1 & mask
        c = [(hi1 ^ c[1] ^ k0) & mask, lo1, (hi0 ^ c[3] ^ k1) & mask, lo0]
        k0 = (k0 + np.uint64(W0)) & mask
        k1 = (k1 + np.uint64(W1)) & mask
    a = (c[0] << np.uint64(32)) | c[1]
    b = (c[2] << np.uint64(32)) | c[3]
    u1 = ((a >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = (b >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    out = np.empty(2 * pairs)
    out[0::2] = r * np.cos(2 * np.pi * u2)
    out[1::2] = r * np.sin(2 * np.pi * u2)
    return out[:count]


def test_philox_probes_and_parity(gpu):
    """Device-drawn Philox probes (throughput runs): the documented generator (numpy restatement,
    bits of the uniforms exact, normals to 1e-13), N(0,1) moments, and the estimator on those
    probes equals pcb_probe_estimate fed the same Z read back."""
    inp = inputs.small_lattice(**SMALL2D)
    N = inp.n_points
    est = Estimator((inp.dom_lo, inp.dom_hi), q=6, seed=2024, generator="philox")
    Z, _, _ = est.read()
    ref = _philox_ref(2024, 6 * N).reshape(6, N)
    assert np.allclose(Z, ref, rtol=0, atol=1e-13 * np.abs(ref).max())
    big = Estimator((inp.dom_lo, inp.dom_hi), q=400, seed=5, generator="philox").read()[0].reshape(-1)
    assert abs(big.mean()) < 0.01 and abs(big.var() - 1.0) < 0.01
    op = ProductConvolutionOperator.from_inputs(inp)
    Y = 0.5 * normal_vectors(4, 6, N)
    est.set_y(Y)
    ea, er = est.update(op, range(op.rank))
    _, _, ea2, er2 = op.probe_estimate(Z, Y, [])
    assert abs(ea - ea2) <= 1e-12 * ea2 and abs(er - er2) <= 1e-12 * er2
