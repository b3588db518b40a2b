import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_1805_06018_b200 import inputs
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors
from oracle import pcop_oracle as O
def rel(a,b): return np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-300)
for name, inp in [("2d", inputs.small_lattice(n=24, dim=2, m=3, sigma=1.7)), ("3d", inputs.small_lattice(n=12, dim=3, m=2, sigma=1.1)), ("1d", inputs.small_lattice(n=50, dim=1, m=5, sigma=2.0)), ("c1", inputs.make_config("c1"))]:
    ref = O.PCOperator.from_inputs(inp)
    F = normal_vectors(11, 2, inp.n_points)
    for mode in ["global", "local"]:
        try:
            op = ProductConvolutionOperator.from_inputs(inp, mode=mode)
            G = op.apply_batch(F); GA = op.apply_adjoint_batch(F)
            print(name, mode, op.info["fft_size"], op.info["n_groups"], "apply", [rel(G[b], ref.apply(F[b])) for b in range(2)], "adj", [rel(GA[b], ref.apply_adjoint(F[b])) for b in range(2)], flush=True)
        except Exception as e:
            print(name, mode, "ERR", e, flush=True)
    # entries
    rng = np.random.default_rng(0)
    y = np.stack([rng.integers(l, h+1, 50) for l,h in zip(inp.dom_lo, inp.dom_hi)], 1)
    x = np.stack([rng.integers(l, h+1, 50) for l,h in zip(inp.dom_lo, inp.dom_hi)], 1)
    e = op.entries(y, x); er = np.array([ref.entry(tuple(a), tuple(b)) for a,b in zip(y,x)])
    print(name, "entries maxdiff", np.abs(e-er).max(), "bitexact", np.array_equal(e, er), flush=True)
