"""Operators whose per-term linear convolution exceeds one 4096-point FFT line.

The reference pads every term to next_pow2(ext phi + ext F + 1) of any size (fft.cpp:58-70); the
engine's lines stop at 4096, so pcb_create splits such a term into exact pieces (sub-windows of
X_k, sub-boxes of K_k; pcop_b200.cpp "Terms too large for one FFT line").  Checked against the
numpy oracle (pinned to the reference build) and, when shipped, the reference build itself:
* 1-D n = 12,000 with kernels of global support (random phi^E over [-(n-1), n-1]);
* 2-D 2,200 x 48 with kernels global along axis 0 (only that axis splits);
* both directions; entries stay bit-identical (the entry gather uses the unsplit terms).
"""
import numpy as np
import pytest

from oracle import pcop_oracle as O
from paper_1805_06018_b200 import inputs
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors

pytestmark = pytest.mark.gpu
TOL = 1e-11


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def global_kernel_operator(shape, lattice, seed):
    """Tent weights on a uniform lattice; phi_k^E = smooth random field over the full window
    Omega - Omega (every offset reachable), so nothing can be trimmed."""
    rng = np.random.default_rng(seed)
    d = len(shape)
    nodes = [inputs.uniform_nodes(n, m) for n, m in zip(shape, lattice)]
    pts = inputs.lattice_points(nodes)
    weights, imps = [], []
    for k in range(len(pts)):
        weights.append(inputs.tent_weight(nodes, inputs.lattice_index(nodes, k)))
        lo = tuple(-(n - 1) for n in shape)
        ext = tuple(2 * n - 1 for n in shape)
        v = rng.standard_normal(ext)
        for a in range(d):  # smooth it a little (decay away from 0)
            z = np.arange(ext[a]) - (shape[a] - 1)
            v = v * np.exp(-np.abs(z) / (0.5 * shape[a])).reshape([-1 if b == a else 1 for b in range(d)])
        imps.append(inputs.Field(lo, v))
    return inputs.OperatorInputs("global%dd" % d, (0,) * d, tuple(n - 1 for n in shape), pts, weights, imps,
                                 {"nodes": nodes})


CASES = {
    "1d_n12000": lambda: global_kernel_operator((12000,), (3,), 0),
    "2d_2200x48": lambda: global_kernel_operator((2200, 48), (2, 2), 1),
}


@pytest.mark.parametrize("name", list(CASES))
def test_split_terms_vs_oracle(gpu, name):
    inp = CASES[name]()
    op = ProductConvolutionOperator.from_inputs(inp)
    info = op.info
    assert info["mode"] == "local" and info["split_terms"] > 0, info
    assert info["plan_terms"] > info["rank_active"]
    ref = O.PCOperator.from_inputs(inp)
    F = normal_vectors(21, 2, inp.n_points)
    G = op.apply_batch(F)
    GA = op.apply_adjoint_batch(F)
    for b in range(2):
        assert rel(G[b], ref.apply(F[b])) <= TOL, (b, rel(G[b], ref.apply(F[b])))
        assert rel(GA[b], ref.apply_adjoint(F[b])) <= TOL
    # entries: the unsplit terms, bit-identical to the oracle's reference-order sum
    rng = np.random.default_rng(5)
    y = np.stack([rng.integers(0, n, 300) for n in inp.shape], 1)
    x = np.stack([rng.integers(0, n, 300) for n in inp.shape], 1)
    e = op.entries(y, x)
    er = np.array([ref.entry(tuple(a), tuple(c)) for a, c in zip(y, x)])
    assert np.array_equal(e, er)


def test_split_terms_vs_reference_build(gpu):
    from oracle import ref_lib

    if not ref_lib.available():
        pytest.skip("reference build (oracle/_ref) not shipped with this copy")
    inp = CASES["1d_n12000"]()
    op = ProductConvolutionOperator.from_inputs(inp)
    F = normal_vectors(22, 1, inp.n_points)
    R = ref_lib.RefOperator(inp)
    assert rel(op.apply(F[0]), R.apply(F[0])) <= TOL
    assert rel(op.apply_adjoint(F[0]), R.apply(F[0], adjoint=True)) <= TOL


def test_global_plan_rejects_long_lines(gpu):
    inp = CASES["1d_n12000"]()
    with pytest.raises(ValueError, match="exceeds 4096"):
        ProductConvolutionOperator.from_inputs(inp, mode="global")
