"""GPU checks beyond parity: the FFT engine unit test, the library's NCCL shard reduce on a 1-rank
communicator, cost-balanced k-shards, and the host-buffer pipeline with many sub-batches (pinned
and pageable).  (compute-sanitizer is disabled on this GPU pool -- its wrapper refuses to run --
so out-of-bounds writes are caught by the library's own guard bands, test_guard_bands.)"""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1805_06018_b200 import build, inputs
from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("cfg", list(dict.fromkeys(build.FFT_UNIT_CONFIGS)), ids=lambda c: "_".join(c))
def test_fft_engine_unit(gpu, cfg):
    """fft.cuh for every compiled line length (8..4096, 2^a * {1,3,9}), forward and inverse, both
    register orders, vs a long-double DFT: relative l2 < 1e-14 (tests/cuda/fft_unit.cu)."""
    exe = build.fft_unit_path(cfg)
    if not os.path.exists(exe):
        exe = build.build_tools()[list(dict.fromkeys(build.FFT_UNIT_CONFIGS)).index(cfg)]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "all lengths OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("graphs", ["1", "0"])
def test_guard_bands(gpu, graphs):
    """No kernel writes out of bounds: every device allocation carries 64 KiB canary bands
    (PCB_GUARD=1) and every entry point runs on c1/c3/c4/1-D/3-D/long-line operators
    (tests/guard_target.py), with CUDA graphs on and off."""
    env = dict(os.environ, PCB_GUARD="1", PCB_GRAPHS=graphs)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "guard_target.py")], capture_output=True,
                       text=True, timeout=900, env=env)
    assert r.returncode == 0 and "GUARD TARGET OK" in r.stdout, (r.stdout + r.stderr)[-4000:]


def test_nccl_reduce_one_rank(gpu):
    """The shard reduce inside the library (pcb_options.nccl_id) on a 1-rank communicator: the
    chunked apply + ncclReduce / ncclAllReduce pipeline gives the unsharded result (a sum over one
    rank is exact), device and host paths, apply, adjoint and the estimator update."""
    from paper_1805_06018_b200 import lib

    inp = inputs.make_config("c2")
    F = normal_vectors(1, 6, inp.n_points)
    ref = ProductConvolutionOperator.from_inputs(inp)
    G0, GA0 = ref.apply_batch(F), ref.apply_adjoint_batch(F)
    for red in ("all", "root"):
        op = ProductConvolutionOperator.from_inputs(inp, shard=(0, 1), nccl_id=lib.comm_unique_id(), reduce=red)
        assert op.info["comm_nranks"] == 1 and op.info["comm_version"] > 0
        assert np.array_equal(op.apply_batch(F), G0)
        assert np.array_equal(op.apply_adjoint_batch(F), GA0)
        import torch

        dF = torch.from_numpy(F).cuda()
        dG = torch.empty_like(dF)
        op.apply_batch_dev(6, dF.data_ptr(), dG.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(dG.cpu().numpy(), G0)
        yt, cells, ea, er = op.probe_estimate(F[:2], F[:2] * 0.5, [], want_ytilde=True)
        assert np.array_equal(yt, GA0[:2])
        op.close()


def test_k_shards_partition_and_sum(gpu):
    """Cost-balanced k-shards (no communicator): each shard keeps exactly the planner's block
    (pcb_plan_shards) and the partials sum to the full apply."""
    from paper_1805_06018_b200 import sharding

    inp = inputs.make_config("c3")
    F = normal_vectors(2, 2, inp.n_points)
    full = ProductConvolutionOperator.from_inputs(inp).apply_batch(F)
    acc = np.zeros_like(full)
    for s in range(3):
        op = ProductConvolutionOperator.from_inputs(inp, shard=(s, 3))
        ks = sharding.k_terms(inp, s, 3)
        assert op.info["rank_active"] == len(ks)
        assert (op.info["term_lo"], op.info["term_hi"]) == (ks[0], ks[-1] + 1)
        acc += op.apply_batch(F)
        op.close()
    assert rel(acc, full) <= 1e-14


@pytest.mark.parametrize("cfg", ["c2", "c3"])
@pytest.mark.parametrize("B", [5, 7])
def test_host_pipeline_many_sub_batches(gpu, cfg, B):
    """pcb_apply_batch with 1 MiB sub-batches (many of them, ping-pong staging slots, half-size
    edges), pinned and pageable host buffers, apply and adjoint: bitwise equal to the device path."""
    import torch

    inp = inputs.make_config(cfg)
    op = ProductConvolutionOperator.from_inputs(inp, host_sub_mb=1)
    F = normal_vectors(9, B, inp.n_points)
    dF = torch.from_numpy(F).cuda()
    dG = torch.empty_like(dF)
    for adj in (False, True):
        op.apply_batch_dev(B, dF.data_ptr(), dG.data_ptr(), torch.cuda.current_stream().cuda_stream, adjoint=adj)
        torch.cuda.synchronize()
        want = dG.cpu().numpy()
        got = op.apply_adjoint_batch(F) if adj else op.apply_batch(F)  # pageable numpy
        assert np.array_equal(got, want)
        Fp = torch.from_numpy(F).pin_memory()
        Gp = torch.empty_like(Fp).pin_memory()
        from paper_1805_06018_b200 import lib

        fn = lib.load().pcb_apply_adjoint_batch if adj else lib.load().pcb_apply_batch
        lib.check(fn(op._h, B, Fp.data_ptr(), Gp.data_ptr()))
        assert np.array_equal(Gp.numpy(), want)
        # repeated calls replay the cached graphs (same keys every call)
        again = op.apply_adjoint_batch(F) if adj else op.apply_batch(F)
        assert np.array_equal(again, want)
        # caller-owned buffers page-locked in place (pcb_host_register): the copy-engine path
        G = np.empty_like(F)
        with lib.host_registered(F, G):
            lib.check(fn(op._h, B, F.ctypes.data, G.ctypes.data))
            with pytest.raises(lib.PcbError):  # already registered
                lib.check(lib.load().pcb_host_register(F.ctypes.data, F.nbytes))
        assert np.array_equal(G, want)
        with pytest.raises(lib.PcbError):  # not registered any more
            lib.check(lib.load().pcb_host_unregister(F.ctypes.data))
    op.close()


@pytest.mark.parametrize("cfg,ndev", [("c2", 2), ("c3", 3), ("c4", 2)])
def test_multi_device_handle(gpu, cfg, ndev):
    """pcb_create_multi with every shard on GPU 0 (the box has one): the scatter / all-gather of F,
    the per-shard partials and the library's slice-parallel reduction run exactly as across
    devices; apply and adjoint (device and host buffers), the estimator and entries equal the
    single handle's to rounding (the shard sums reorder the k-sum)."""
    import torch

    inp = inputs.make_config(cfg)
    F = normal_vectors(5, 4, inp.n_points)
    ref = ProductConvolutionOperator.from_inputs(inp)
    G0, GA0 = ref.apply_batch(F), ref.apply_adjoint_batch(F)
    op = ProductConvolutionOperator.from_inputs(inp, devices=[0] * ndev)
    assert op.info["shard_count"] == ndev and op.info["rank_active"] == inp.rank
    assert rel(op.apply_batch(F), G0) <= 1e-14
    assert rel(op.apply_adjoint_batch(F), GA0) <= 1e-14
    dF = torch.from_numpy(F).cuda()
    dG = torch.empty_like(dF)
    for adj, want in ((False, G0), (True, GA0)):
        op.apply_batch_dev(4, dF.data_ptr(), dG.data_ptr(), torch.cuda.current_stream().cuda_stream, adjoint=adj)
        torch.cuda.synchronize()
        assert rel(dG.cpu().numpy(), want) <= 1e-14
    again = op.apply_batch(F)  # deterministic: the reduction sums in shard order
    assert np.array_equal(again, op.apply_batch(F))
    rng = np.random.default_rng(1)
    y = np.stack([rng.integers(0, n, 64) for n in inp.shape], 1)
    x = np.stack([rng.integers(0, n, 64) for n in inp.shape], 1)
    assert np.array_equal(op.entries(y, x), ref.entries(y, x))
    yt, _, ea, er = op.probe_estimate(F[:2], 0.5 * F[:2], [], want_ytilde=True)
    _, _, ea0, er0 = ref.probe_estimate(F[:2], 0.5 * F[:2], [])
    assert abs(ea - ea0) <= 1e-13 * ea0 and abs(er - er0) <= 1e-13 * er0
    op.close()
