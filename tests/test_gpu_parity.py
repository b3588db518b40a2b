"""GPU parity of the sm_100a apply path.

* vs golden outputs of the reference library (tests/golden): apply / adjoint <= 1e-11 relative l2
  (north_star tolerance), entry / block evaluation bit-identical (reference summation order);
* vs the numpy oracle on seeded inputs, both plans (global / local), 1-D, 2-D, 3-D, edge cases;
* at the full BASELINE sizes through size-independent properties (linearity, the adjoint
  identity, plan agreement, batch consistency, determinism, exactness for a single kernel).
"""
import os

import numpy as np
import pytest

from oracle import pcop_oracle as O
from paper_1805_06018_b200 import inputs
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors, uniform_ints

pytestmark = pytest.mark.gpu

APPLY_TOL = 1e-11  # north_star: relative l2 <= 1e-11 in fp64
GOLD = os.path.join(os.path.dirname(__file__), "golden")
MODES = ["global", "local"]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


SMALL = {
    "small2d": dict(n=24, dim=2, m=3, sigma=1.7),
    "small3d": dict(n=12, dim=3, m=2, sigma=1.1),
    "small1d": dict(n=50, dim=1, m=5, sigma=2.0),
    "small2d_zeroext": dict(n=20, dim=2, m=2, sigma=1.5, extend=False),
}


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("name", list(SMALL))
def test_vs_reference_golden_small(gpu, name, mode):
    d = np.load(os.path.join(GOLD, f"{name}.npz"))
    inp = inputs.small_lattice(**SMALL[name])
    assert str(d["checksum"]) == inp.checksum()
    op = ProductConvolutionOperator.from_inputs(inp, mode=mode)
    G = op.apply_batch(d["F"])
    GA = op.apply_adjoint_batch(d["F"])
    for b in range(d["F"].shape[0]):
        assert rel(G[b], d["G"][b]) <= APPLY_TOL
        assert rel(GA[b], d["GA"][b]) <= APPLY_TOL
    assert np.array_equal(op.entries(d["y"], d["x"]), d["E"])  # bit-identical to pc_operator.cpp:84-96


@pytest.mark.parametrize("mode", MODES)
def test_c1_vs_reference_golden(gpu, mode):
    d = np.load(os.path.join(GOLD, "c1.npz"))
    inp = inputs.make_config("c1")
    assert str(d["checksum"]) == inp.checksum()
    op = ProductConvolutionOperator.from_inputs(inp, mode=mode)
    assert rel(op.apply(d["f"]), d["g"]) <= APPLY_TOL
    assert rel(op.apply_adjoint(d["f"]), d["ga"]) <= APPLY_TOL
    assert np.array_equal(op.entries(d["y"], d["x"]), d["E"])
    # the reference's own full-box extended impulses give the same operator
    opF = ProductConvolutionOperator.from_inputs(inputs.make_config("c1", full_box=True), mode=mode)
    assert rel(opF.apply(d["f"]), d["g"]) <= APPLY_TOL


def test_c5_blocks_vs_reference_golden(gpu):
    d = np.load(os.path.join(GOLD, "c5_blocks.npz"))
    inp = inputs.make_config("c2")
    assert str(d["checksum"]) == inp.checksum()
    op = ProductConvolutionOperator.from_inputs(inp)
    org = d["origins"]
    out = op.blocks(org[:, :2], org[:, 2:], (8, 8))
    assert np.array_equal(out, d["blocks"])  # entry-wise <= 1e-12 required; the gather is exact


def test_c5_full_4096_blocks(gpu):
    """Config 5: 4096 64x64 blocks (8x8 patches), origins mt19937_64(3) in [0, 504]."""
    op = ProductConvolutionOperator.from_inputs(inputs.make_config("c2"))
    org = uniform_ints(3, 0, 504, 4 * 4096).reshape(4096, 4)
    out = op.blocks(org[:, :2], org[:, 2:], (8, 8))
    assert out.shape == (4096, 64, 64)
    off = np.array([(i, j) for i in range(8) for j in range(8)])
    for b in (0, 17, 4095):
        yy = np.repeat(org[b, :2] + off, 64, axis=0)
        xx = np.tile(org[b, 2:] + off, (64, 1))
        assert np.array_equal(op.entries(yy, xx).reshape(64, 64), out[b])


def test_estimator_vs_reference_golden(gpu):
    d = np.load(os.path.join(GOLD, "estimator.npz"))
    inp = inputs.small_lattice(**SMALL["small2d"])
    leaves = [(tuple(l), tuple(h)) for l, h in zip(d["leaf_lo"], d["leaf_hi"])]
    for mode in MODES:
        op = ProductConvolutionOperator.from_inputs(inp, mode=mode)
        yt, cells, ea, er = op.probe_estimate(d["Z"], d["Y"], leaves, want_ytilde=True)
        assert rel(yt, d["ytilde"]) <= APPLY_TOL
        assert np.allclose(cells, d["cells"], rtol=1e-11, atol=0)
        assert abs(ea - float(d["eta_abs"])) <= 1e-11 * float(d["eta_abs"])
        assert abs(er - float(d["eta_rel"])) <= 1e-11 * float(d["eta_rel"])


CASES = {
    "2d_n40_m4": lambda: inputs.small_lattice(n=40, dim=2, m=4, sigma=2.3),
    "2d_const": lambda: inputs.small_lattice(n=33, dim=2, m=3, sigma=2.0, varying=False),
    "3d_n16_m3": lambda: inputs.small_lattice(n=16, dim=3, m=3, sigma=1.2),
    "1d_zeroext": lambda: inputs.small_lattice(n=70, dim=1, m=6, sigma=3.0, extend=False),
}


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("name", list(CASES))
def test_vs_oracle(gpu, name, mode):
    inp = CASES[name]()
    op = ProductConvolutionOperator.from_inputs(inp, mode=mode)
    ref = O.PCOperator.from_inputs(inp)
    F = normal_vectors(11, 3, inp.n_points)
    G, GA = op.apply_batch(F), op.apply_adjoint_batch(F)
    for b in range(3):
        assert rel(G[b], ref.apply(F[b])) <= APPLY_TOL
        assert rel(GA[b], ref.apply_adjoint(F[b])) <= APPLY_TOL


def _random_operator(n, dim, r, seed, spill=False):
    """Dense random phi^E on full windows (nothing to trim) and random weights; with spill,
    footprints stick out of Omega and kernel boxes do not cover the window."""
    rng = np.random.default_rng(seed)
    ws, es = [], []
    for k in range(r):
        lo = tuple(int(v) for v in rng.integers(-3 if spill else 0, n - 4, dim))
        ext = tuple(int(v) for v in rng.integers(1, 8, dim))
        ws.append(inputs.Field(lo, rng.uniform(-1, 1, tuple(e + 1 for e in ext))))
        if spill:
            klo = tuple(int(v) for v in rng.integers(-n // 2, 0, dim))
            kext = tuple(int(v) for v in rng.integers(1, n, dim))
        else:
            klo = tuple(-(n - 1) for _ in range(dim))
            kext = tuple(2 * n - 2 for _ in range(dim))
        es.append(inputs.Field(klo, rng.uniform(-1, 1, tuple(e + 1 for e in kext))))
    return inputs.OperatorInputs("random", (0,) * dim, (n - 1,) * dim, [(0,) * dim] * r, ws, es)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("dim,n,r,spill", [(2, 21, 7, False), (2, 17, 9, True), (3, 9, 5, True), (1, 40, 6, True)])
def test_random_dense_kernels_vs_oracle(gpu, mode, dim, n, r, spill):
    inp = _random_operator(n, dim, r, seed=dim * 100 + n, spill=spill)
    op = ProductConvolutionOperator.from_inputs(inp, mode=mode)
    ref = O.PCOperator.from_inputs(inp)
    F = normal_vectors(3, 2, inp.n_points)
    for b in range(2):
        assert rel(op.apply(F[b]), ref.apply(F[b])) <= APPLY_TOL
        assert rel(op.apply_adjoint(F[b]), ref.apply_adjoint(F[b])) <= APPLY_TOL
    rng = np.random.default_rng(1)
    y = rng.integers(0, n, (300, dim))
    x = rng.integers(0, n, (300, dim))
    E = np.array([ref.entry(tuple(a), tuple(b)) for a, b in zip(y, x)])
    assert np.array_equal(op.entries(y, x), E)


def test_edge_cases(gpu):
    # rank 0 operator: Atilde = 0
    op0 = ProductConvolutionOperator(((0, 0), (9, 9)), [], [])
    f = np.ones(100)
    assert not op0.apply(f).any() and not op0.apply_adjoint(f).any()
    # all-zero kernel and a footprint outside Omega: both contribute nothing
    inp = inputs.small_lattice(n=16, dim=2, m=2, sigma=1.3)
    ws = list(inp.weights) + [inputs.Field((40, 40), np.ones((3, 3))), inputs.Field((2, 2), np.ones((4, 4)))]
    es = list(inp.impulses) + [inputs.Field((-1, -1), np.ones((3, 3))), inputs.Field((-2, -2), np.zeros((5, 5)))]
    op = ProductConvolutionOperator((inp.dom_lo, inp.dom_hi), ws, es)
    ref = O.PCOperator(inp.dom_lo, inp.dom_hi, [O.GF(w.lo, w.values) for w in ws], [O.GF(e.lo, e.values) for e in es])
    F = normal_vectors(9, 2, 256)
    assert rel(op.apply(F[0]), ref.apply(F[0])) <= APPLY_TOL
    assert rel(op.apply_adjoint(F[1]), ref.apply_adjoint(F[1])) <= APPLY_TOL
    assert op.info["rank_active"] == inp.rank
    # zero input -> exactly zero output; empty batch is a no-op
    assert not op.apply(np.zeros(256)).any()
    assert op.apply_batch(np.zeros((0, 256))).shape == (0, 256)


BLOCK_CASES = {
    "1d": (lambda: inputs.small_lattice(n=50, dim=1, m=5, sigma=2.0), (5,)),
    "2d_rect": (lambda: inputs.small_lattice(n=24, dim=2, m=3, sigma=1.7), (3, 5)),
    "3d": (lambda: inputs.small_lattice(n=12, dim=3, m=2, sigma=1.1), (2, 3, 2)),
    "2d_odd": (lambda: inputs.small_lattice(n=24, dim=2, m=3, sigma=1.7), (3, 3)),  # 81 entries: odd block size
    "c1_large": (lambda: inputs.make_config("c1"), (16, 16)),  # 256 points: the staged path's upper end
    "c1_huge": (lambda: inputs.make_config("c1"), (20, 20)),   # too large to stage: the per-entry kernel
}


@pytest.mark.parametrize("name", list(BLOCK_CASES))
@pytest.mark.parametrize("streams", ["2", "1"])
def test_blocks_match_entries(gpu, name, streams, monkeypatch):
    """Dense blocks of every dimension and shape -- near-diagonal ones (terms contribute), far ones
    (the zero test / zero fill), coincident origins, blocks at the domain edge -- equal the per-entry
    gather bit for bit (entry() is pinned to the reference), on two streams and on one."""
    monkeypatch.setenv("PCB_BLOCKS_STREAMS", streams)
    make, bs = BLOCK_CASES[name]
    inp = make()
    op = ProductConvolutionOperator.from_inputs(inp)
    d = inp.dim
    n = np.array(inp.shape)
    bsz = np.array(bs)
    rng = np.random.default_rng(7)
    nb = 40 if name.startswith("c1") else 150
    t = np.stack([rng.integers(0, n[a] - bsz[a] + 1, nb) for a in range(d)], 1)
    s = t + rng.integers(-4, 5, (nb, d))  # near the diagonal
    far = rng.random(nb) < 0.4
    s[far] = np.stack([rng.integers(0, n[a] - bsz[a] + 1, int(far.sum())) for a in range(d)], 1)
    s = np.clip(s, 0, n - bsz)
    t[0] = 0  # corners of the domain
    s[0] = 0
    t[1] = n - bsz
    s[1] = n - bsz
    out = op.blocks(t, s, bs)
    off = np.array(list(np.ndindex(*bs)))
    npx = len(off)
    for b in range(nb):
        yy = np.repeat(t[b] + off, npx, axis=0)
        xx = np.tile(s[b] + off, (npx, 1))
        assert np.array_equal(op.entries(yy, xx).reshape(npx, npx), out[b]), (name, b)
    assert any(out[b].any() for b in range(nb)) and any(not out[b].any() for b in range(nb))
    bad_t = t.copy()
    bad_t[3] = n - bsz + 1  # one block leaves the domain
    with pytest.raises(ValueError, match="index outside the domain"):
        op.blocks(bad_t, s, bs)


def test_errors_mirror_reference(gpu):
    op = ProductConvolutionOperator.from_inputs(inputs.small_lattice(n=12, dim=2, m=2, sigma=1.0))
    with pytest.raises(ValueError, match="PCOp::apply: shape mismatch"):
        op.apply(np.zeros(10))
    with pytest.raises(ValueError, match="PCOp::apply_adjoint: shape mismatch"):
        op.apply_adjoint(np.zeros(10))
    with pytest.raises(ValueError, match="PCOp::entry: index outside the domain"):
        op.entry((-1, 0), (0, 0))
    with pytest.raises(ValueError, match="index outside the domain"):
        op.blocks(np.array([[10, 10]]), np.array([[0, 0]]), (4, 4))
    with pytest.raises(ValueError, match="lo > hi"):
        ProductConvolutionOperator(((0, 0), (5, -1)), [], [])


def test_device_pointer_api_and_determinism(gpu):
    import torch

    inp = inputs.make_config("c1")
    op = ProductConvolutionOperator.from_inputs(inp)
    F = torch.from_numpy(normal_vectors(0, 4, inp.n_points)).cuda()
    G1 = torch.empty_like(F)
    G2 = torch.empty_like(F)
    s = torch.cuda.current_stream().cuda_stream
    op.apply_batch_dev(4, F.data_ptr(), G1.data_ptr(), s)
    op.apply_batch_dev(4, F.data_ptr(), G2.data_ptr(), s)
    torch.cuda.synchronize()
    assert torch.equal(G1, G2)  # deterministic: fixed-order gather, no atomics
    ref = O.PCOperator.from_inputs(inp)
    assert rel(G1[2].cpu().numpy(), ref.apply(F[2].cpu().numpy())) <= APPLY_TOL
    # batch of one == row of a batch, bitwise
    g = op.apply(F[3].cpu().numpy())
    assert np.array_equal(g, G1[3].cpu().numpy())


@pytest.mark.parametrize("mode", MODES)
def test_k_shards_sum_to_full_apply(gpu, mode):
    """Shard-by-k (pcb_options.shard_rank/shard_count): partial outputs sum to the full apply."""
    inp = inputs.make_config("c1")
    F = normal_vectors(1, 2, inp.n_points)
    full = ProductConvolutionOperator.from_inputs(inp, mode=mode).apply_batch(F)
    for world in (2, 3):
        parts = [ProductConvolutionOperator.from_inputs(inp, mode=mode, shard=(r, world)).apply_batch(F)
                 for r in range(world)]
        assert rel(sum(parts), full) <= 1e-14
        adj = [ProductConvolutionOperator.from_inputs(inp, mode=mode, shard=(r, world)).apply_adjoint_batch(F)
               for r in range(world)]
        full_adj = ProductConvolutionOperator.from_inputs(inp, mode=mode).apply_adjoint_batch(F)
        assert rel(sum(adj), full_adj) <= 1e-14


# --- full BASELINE sizes: size-independent properties ----------------------

def test_c2_full_vs_oracle(gpu):
    inp = inputs.make_config("c2")
    op = ProductConvolutionOperator.from_inputs(inp)
    ref = O.PCOperator.from_inputs(inp)
    F = normal_vectors(1, 2, inp.n_points)
    G = op.apply_batch(F)
    assert rel(G[0], ref.apply(F[0])) <= APPLY_TOL
    assert rel(op.apply_adjoint(F[1]), ref.apply_adjoint(F[1])) <= APPLY_TOL


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_full_size_properties(gpu, cfg):
    inp = inputs.make_config(cfg)
    op = ProductConvolutionOperator.from_inputs(inp)
    F = normal_vectors({"c3": 2, "c4": 4}[cfg], 2, inp.n_points)
    f, h = F[0], F[1]
    Af, Ah = op.apply_batch(F)
    # linearity (test_pc_operator.cpp:87-95)
    assert rel(op.apply(2.5 * f - 0.75 * h), 2.5 * Af - 0.75 * Ah) <= 1e-13
    # adjoint identity <A f, h> = <f, A* h> (test_pc_operator.cpp:75-85)
    lhs, rhs = Af @ h, f @ op.apply_adjoint(h)
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))
    # zero in -> zero out (test_pc_operator.cpp:54-59)
    assert not op.apply(np.zeros(inp.n_points)).any()
    # the oracle on a subset of terms at the full domain size
    ks = [0, inp.rank // 2 + 3, inp.rank - 1]
    sub = inp.subset(ks)
    ref = O.PCOperator.from_inputs(sub)
    opsub = ProductConvolutionOperator.from_inputs(sub)
    assert rel(opsub.apply(f), ref.apply(f)) <= APPLY_TOL
    assert rel(opsub.apply_adjoint(h), ref.apply_adjoint(h)) <= APPLY_TOL


def test_c3_plans_agree(gpu):
    """The two exact plans (global spectral accumulation, local trimmed windows) agree at c3 size."""
    inp = inputs.make_config("c3")
    F = normal_vectors(2, 2, inp.n_points)
    a = ProductConvolutionOperator.from_inputs(inp, mode="global").apply_batch(F)
    b = ProductConvolutionOperator.from_inputs(inp, mode="local").apply_batch(F)
    for i in range(2):
        assert rel(a[i], b[i]) <= 1e-12


def test_single_kernel_exactness_c1_geometry(gpu):
    """Acceptance criterion 1 at config-1 geometry: a translation-invariant blur is reproduced
    exactly (Atilde = A) by the extended impulses (acceptance.cpp:88-112)."""
    n = 128
    blur = inputs.blur_const(n, 2, 3.0)
    nodes = [inputs.uniform_nodes(n, 3)] * 2
    inp = inputs.lattice_operator("c1const", blur, nodes)
    f = normal_vectors(0, 1, n * n)[0]
    truth = inputs.apply_true_blur(blur, f.reshape(n, n)).reshape(-1)
    for mode in MODES:
        op = ProductConvolutionOperator.from_inputs(inp, mode=mode)
        assert rel(op.apply(f), truth) <= 1e-12


def test_cpp_host_example(gpu, tmp_path):
    """The C++ host side (include/pcb/operator.hpp) linked against the in-tree library."""
    import subprocess

    from paper_1805_06018_b200 import lib

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "apply_example")
    libdir = os.path.dirname(lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{root}/include", os.path.join(root, "tests", "cpp", "apply_example.cpp"),
                    f"-L{libdir}", "-lpcop_b200", f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


def test_apply_block_vs_reference_golden(gpu):
    """apply_block (pc_operator.cpp:98-130): batched blocks, both directions, vs the reference."""
    d = np.load(os.path.join(GOLD, "apply_block.npz"))
    inp = inputs.small_lattice(**SMALL["small2d"])
    op = ProductConvolutionOperator.from_inputs(inp)
    n = int(d["n"])
    Ts = [tuple(map(tuple, d[f"b{i}_T"])) for i in range(n)]
    Ss = [tuple(map(tuple, d[f"b{i}_S"])) for i in range(n)]
    fs = [d[f"b{i}_f"] for i in range(n)]
    for adj in (0, 1):
        out = op.apply_blocks(Ts, Ss, fs, adjoint=bool(adj))
        for i in range(n):
            ref = d[f"b{i}_{adj}"]
            assert np.max(np.abs(out[i] - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_apply_block_many_blocks(gpu):
    """More blocks in one call than a grid's y extent (65,535): the batched H-matrix rounds of a larger
    operator pass that many (found by scripts/hmatrix_time.py at n = 96)."""
    inp = inputs.small_lattice(**SMALL["small2d"])
    op = ProductConvolutionOperator.from_inputs(inp)
    n = inp.shape[0]
    rng = np.random.default_rng(11)
    nb = 70_000
    t = rng.integers(0, n - 1, (nb, 2))
    s = np.clip(t + rng.integers(-3, 4, (nb, 2)), 0, n - 2)
    Ts = [(tuple(a), tuple(a + 1)) for a in t]
    Ss = [(tuple(a), tuple(a + 1)) for a in s]
    fs = [rng.uniform(-1, 1, (2, 2)) for _ in range(nb)]
    out = op.apply_blocks(Ts, Ss, fs)
    for i in (0, 65_535, 65_536, nb - 1):
        one = op.apply_block(Ts[i], Ss[i], fs[i])
        assert np.array_equal(out[i], one)


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_apply_block_properties(gpu, cfg):
    """T = S = Omega equals apply (test_pc_operator.cpp:185-194; the FFT path for big blocks), H-matrix
    leaf blocks equal apply-then-restrict, far boxes give exact zeros, domain violations raise."""
    inp = inputs.make_config(cfg)
    op = ProductConvolutionOperator.from_inputs(inp)
    n = inp.shape[0]
    dom = (inp.dom_lo, inp.dom_hi)
    f = normal_vectors(5, 1, inp.n_points)[0]
    for adj in (False, True):
        whole = op.apply_block(dom, dom, f.reshape(inp.shape), adjoint=adj)
        full = (op.apply_adjoint if adj else op.apply)(f)
        assert rel(whole.reshape(-1), full) <= 1e-12
    rng = np.random.default_rng(3)
    Ts, Ss, fs = [], [], []
    for _ in range(32):
        t = rng.integers(0, n - 8, 2)
        s = np.clip(t + rng.integers(-12, 12, 2), 0, n - 8)
        Ts.append((tuple(t), tuple(t + 7)))
        Ss.append((tuple(s), tuple(s + 7)))
        fs.append(rng.uniform(-1, 1, (8, 8)))
    for adj in (False, True):
        out = op.apply_blocks(Ts, Ss, fs, adjoint=adj)
        for i in (0, 7, 31):
            full = np.zeros(inp.shape)
            s0, s1 = Ss[i]
            full[s0[0]:s1[0] + 1, s0[1]:s1[1] + 1] = fs[i]
            g = (op.apply_adjoint if adj else op.apply)(full.reshape(-1)).reshape(inp.shape)
            t0, t1 = Ts[i]
            ref = g[t0[0]:t1[0] + 1, t0[1]:t1[1] + 1]
            assert np.max(np.abs(out[i] - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
    far = op.apply_block(((0, 0), (3, 3)), ((n - 4, n - 4), (n - 1, n - 1)), np.ones((4, 4)))
    assert not far.any()
    with pytest.raises(ValueError, match="boxes must lie inside the domain"):
        op.apply_block(((0, 0), (n, 3)), ((0, 0), (3, 3)), np.ones((4, 4)))


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_bundled_gather_matches_per_entry_gather(gpu, name, monkeypatch):
    """The frequency-domain bundles of the LOCAL apply gather (phase-shifted spectra summed, one
    C2R per bundle) agree with the one-C2R-per-entry gather at full config size."""
    inp = inputs.make_config(name)
    F = normal_vectors(8, 2, inp.n_points)
    monkeypatch.setenv("PCB_BUNDLE", "0")
    a = ProductConvolutionOperator.from_inputs(inp, mode="local").apply_batch(F)
    monkeypatch.setenv("PCB_BUNDLE", "1")
    b = ProductConvolutionOperator.from_inputs(inp, mode="local").apply_batch(F)
    for i in range(2):
        assert rel(b[i], a[i]) <= 1e-14


@pytest.mark.parametrize("name", ["c2", "c3"])
@pytest.mark.parametrize("bundle", ["1", "0"])
def test_split3_rows_match_power_of_two_rows(gpu, name, bundle, monkeypatch):
    """PCB_MIXED_LAST=2: last-axis sizes 3 * 2^a (192, 384) run as three interleaved power-of-two
    sub-lines in the row passes (radix-3 butterfly in the forward gather / the inverse's output
    pass).  Same operator as the power-of-two plan: apply and adjoint, bundled and per-entry gathers,
    and the spectra built through the same forward kernels."""
    inp = inputs.make_config(name)
    F = normal_vectors(12, 2, inp.n_points)
    monkeypatch.setenv("PCB_BUNDLE", bundle)
    monkeypatch.setenv("PCB_MIXED_LAST", "0")
    p2 = ProductConvolutionOperator.from_inputs(inp, mode="local")
    monkeypatch.setenv("PCB_MIXED_LAST", "2")
    s3 = ProductConvolutionOperator.from_inputs(inp, mode="local")
    assert s3.info["spectra_bytes"] < p2.info["spectra_bytes"]  # some classes moved to 192 / 384
    a, b = p2.apply_batch(F), s3.apply_batch(F)
    aa, ba = p2.apply_adjoint_batch(F), s3.apply_adjoint_batch(F)
    for i in range(2):
        assert rel(b[i], a[i]) <= 1e-13
        assert rel(ba[i], aa[i]) <= 1e-13


def test_split3_rows_vs_oracle_1d(gpu, monkeypatch):
    """A 1-D operator whose line is 3 * 2^a under PCB_MIXED_LAST=2 (one sub-line CTA), vs the oracle."""
    inp = inputs.small_lattice(n=300, dim=1, m=2, sigma=6.0)
    ref = O.PCOperator.from_inputs(inp)
    F = normal_vectors(13, 2, inp.n_points)
    monkeypatch.setenv("PCB_MIXED_LAST", "0")
    p2 = ProductConvolutionOperator.from_inputs(inp, mode="local")
    monkeypatch.setenv("PCB_MIXED_LAST", "2")
    op = ProductConvolutionOperator.from_inputs(inp, mode="local")
    assert op.info["spectra_bytes"] < p2.info["spectra_bytes"]  # the 348-point term runs at 384, not 512
    G, GA = op.apply_batch(F), op.apply_adjoint_batch(F)
    for i in range(2):
        assert rel(G[i], ref.apply(F[i])) <= APPLY_TOL
        assert rel(GA[i], ref.apply_adjoint(F[i])) <= APPLY_TOL


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "small2d", "small3d", "small1d"])
def test_row_families_match_per_term_rows(gpu, name, monkeypatch):
    """Separable (tent) weights: terms sharing a last-axis weight factor share their row
    transforms, scaled per term by the lead-axis factor; the adjoint shares the rows of g and
    (2-D) sums each family's rows before one C2R.  Same operator as the per-term passes
    (PCB_FAMILIES=0) and as the oracle."""
    inp = inputs.make_config(name) if name.startswith("c") else inputs.small_lattice(**SMALL[name])
    F = normal_vectors(9, 2, inp.n_points)
    monkeypatch.setenv("PCB_FAMILIES", "0")
    off = ProductConvolutionOperator.from_inputs(inp, mode="local")
    monkeypatch.setenv("PCB_FAMILIES", "1")
    on = ProductConvolutionOperator.from_inputs(inp, mode="local")
    assert off.info["n_row_families"] == 0
    if inp.dim > 1:
        assert 0 < on.info["n_row_families"] < inp.rank
    a, b = off.apply_batch(F), on.apply_batch(F)
    for i in range(2):
        assert rel(b[i], a[i]) <= 1e-14
    # adjoint: shared rows of g and, in 2-D, one C2R per (output line, family)
    aa, ba = off.apply_adjoint_batch(F), on.apply_adjoint_batch(F)
    for i in range(2):
        assert rel(ba[i], aa[i]) <= 1e-14
    if name.startswith("small"):
        ref = O.PCOperator.from_inputs(inp)
        for i in range(2):
            assert rel(b[i], ref.apply(F[i])) <= APPLY_TOL
            assert rel(ba[i], ref.apply_adjoint(F[i])) <= APPLY_TOL


def test_non_separable_weights_use_per_term_rows(gpu):
    """Weights that do not factor (a random perturbation of the tents) keep per-term rows."""
    inp = inputs.small_lattice(n=24, dim=2, m=3, sigma=1.7)
    rng = np.random.default_rng(5)
    for w in inp.weights:
        w.values[...] = w.values * (1.0 + 0.1 * rng.random(w.values.shape))
    op = ProductConvolutionOperator.from_inputs(inp, mode="local")
    assert op.info["n_row_families"] == 0
    F = normal_vectors(4, 2, inp.n_points)
    ref = O.PCOperator.from_inputs(inp)
    G = op.apply_batch(F)
    for i in range(2):
        assert rel(G[i], ref.apply(F[i])) <= APPLY_TOL


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "small2d", "small2d_zeroext"])
def test_column_chains_match_per_term_inverse(gpu, name, monkeypatch):
    """2-D LOCAL column chains (members' spectra summed in registers, one axis-0 inverse and one T
    region per chain) give the same operator as one inverse per term (PCB_CHAINS=0), and the
    oracle on the small cases; the adjoint (wider windows for chain members) agrees too."""
    inp = inputs.make_config(name) if name.startswith("c") else inputs.small_lattice(**SMALL[name])
    F = normal_vectors(10, 2, inp.n_points)
    monkeypatch.setenv("PCB_CHAINS", "0")
    off = ProductConvolutionOperator.from_inputs(inp, mode="local")
    monkeypatch.setenv("PCB_CHAINS", "1")
    monkeypatch.setenv("PCB_CHAIN_BETA", "200")  # long chains: the strongest exercise
    on = ProductConvolutionOperator.from_inputs(inp, mode="local")
    assert off.info["n_column_chains"] == 0
    assert on.info["n_chained_terms"] > 0
    a, b = off.apply_batch(F), on.apply_batch(F)
    aa, ba = off.apply_adjoint_batch(F), on.apply_adjoint_batch(F)
    for i in range(2):
        assert rel(b[i], a[i]) <= 1e-14
        assert rel(ba[i], aa[i]) <= 1e-14
    if not name.startswith("c") or name == "c1":
        ref = O.PCOperator.from_inputs(inp)
        for i in range(2):
            assert rel(b[i], ref.apply(F[i])) <= APPLY_TOL
            assert rel(ba[i], ref.apply_adjoint(F[i])) <= APPLY_TOL


@pytest.mark.parametrize("name", ["c4", "small3d"])
def test_plane_families_match_per_term_mid(gpu, name, monkeypatch):
    """3-D plane families (terms of one row family sharing the axis-1 factor share the axis-1
    forward transforms; the cols pass applies a_k(x0)) give the same operator as per-term mid
    passes (PCB_PLANE_FAMILIES=0) and as the oracle."""
    inp = inputs.make_config(name) if name.startswith("c") else inputs.small_lattice(**SMALL[name])
    F = normal_vectors(12, 2, inp.n_points)
    monkeypatch.setenv("PCB_PLANE_FAMILIES", "0")
    a = ProductConvolutionOperator.from_inputs(inp, mode="local").apply_batch(F)
    monkeypatch.setenv("PCB_PLANE_FAMILIES", "1")
    b = ProductConvolutionOperator.from_inputs(inp, mode="local").apply_batch(F)
    for i in range(2):
        assert rel(b[i], a[i]) <= 1e-14
    if name.startswith("small"):
        ref = O.PCOperator.from_inputs(inp)
        for i in range(2):
            assert rel(b[i], ref.apply(F[i])) <= APPLY_TOL


@pytest.mark.parametrize("name", ["c1", "small3d"])
def test_graph_replay_matches_direct_launches(gpu, name, monkeypatch):
    """Device-pointer applies replay a captured CUDA graph per (adjoint, B, F, G): bitwise equal to
    kernel-by-kernel launches (PCB_GRAPHS=0), on repeated calls, new inputs in the same buffers,
    other buffers, the adjoint, and on a side stream."""
    import torch

    inp = inputs.make_config(name) if name.startswith("c") else inputs.small_lattice(**SMALL[name])
    F = torch.from_numpy(normal_vectors(3, 3, inp.n_points)).cuda()
    s = torch.cuda.current_stream().cuda_stream
    monkeypatch.setenv("PCB_GRAPHS", "0")
    direct = ProductConvolutionOperator.from_inputs(inp, mode="local")
    monkeypatch.setenv("PCB_GRAPHS", "1")
    graph = ProductConvolutionOperator.from_inputs(inp, mode="local")
    Gd, Gg = torch.empty_like(F), torch.empty_like(F)
    for adjoint in (False, True):
        direct.apply_batch_dev(3, F.data_ptr(), Gd.data_ptr(), s, adjoint=adjoint)
        for _ in range(3):
            Gg.zero_()
            graph.apply_batch_dev(3, F.data_ptr(), Gg.data_ptr(), s, adjoint=adjoint)
            torch.cuda.synchronize()
            assert torch.equal(Gg, Gd)
    F2 = F.flip(0).contiguous()
    G2 = torch.empty_like(F)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        graph.apply_batch_dev(3, F2.data_ptr(), G2.data_ptr(), side.cuda_stream)
        F.copy_(F2)  # same buffer, new inputs
        graph.apply_batch_dev(3, F.data_ptr(), Gg.data_ptr(), side.cuda_stream)
    torch.cuda.synchronize()
    direct.apply_batch_dev(3, F2.data_ptr(), Gd.data_ptr(), s)
    torch.cuda.synchronize()
    assert torch.equal(G2, Gd) and torch.equal(Gg, Gd)
