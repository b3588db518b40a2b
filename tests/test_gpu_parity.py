"""GPU parity: the sm_100a apply path vs the oracle on seeded inputs."""
import numpy as np
import pytest

from paper_1805_06018_b200 import inputs
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors
from oracle import pcop_oracle as O

pytestmark = pytest.mark.gpu

APPLY_TOL = 1e-11  # north_star: relative l2 <= 1e-11 in fp64


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


CASES = [
    ("2d_n24", lambda: inputs.small_lattice(n=24, dim=2, m=3, sigma=1.7)),
    ("2d_n40_m4", lambda: inputs.small_lattice(n=40, dim=2, m=4, sigma=2.3)),
    ("3d_n12", lambda: inputs.small_lattice(n=12, dim=3, m=2, sigma=1.1)),
    ("1d_n50", lambda: inputs.small_lattice(n=50, dim=1, m=5, sigma=2.0)),
]


@pytest.mark.parametrize("mode", ["global", "local"])
@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_apply_adjoint_vs_oracle(gpu, name, make, mode):
    inp = make()
    op = ProductConvolutionOperator.from_inputs(inp, mode=mode)
    ref = O.PCOperator.from_inputs(inp)
    F = normal_vectors(11, 3, inp.n_points)
    G = op.apply_batch(F)
    for b in range(3):
        assert rel(G[b], ref.apply(F[b])) <= APPLY_TOL
    GA = op.apply_adjoint_batch(F)
    for b in range(3):
        assert rel(GA[b], ref.apply_adjoint(F[b])) <= APPLY_TOL
