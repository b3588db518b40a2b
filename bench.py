#!/usr/bin/env python
"""Benchmark: Atilde-apply vectors/s (fp64) on B200 for a BASELINE.json configuration.

One "step" = one apply of the product-convolution operator to the configuration's batch of
vectors (c3: 64 vectors on 1024^2, r = 256).  Contract (README / task):
  * W >= 3 untimed warm-up steps, then K timed steps, each bracketed by CUDA events on the
    launching stream; L2 is flushed (a 256 MiB write) between timed steps, outside the events;
  * multi-GPU: one process per GPU (torchrun).  ``--shard rhs`` (default): weak scaling, every
    rank applies the config's B vectors of its own (independent units, no collective), value =
    all ranks' vectors / max-over-ranks time.  ``--shard k``: the terms are sharded and the
    partial outputs all-reduced over NCCL inside the timed region (strong scaling);
  * ``e2e``: the same metric through the host C-ABI call ``pcb_apply_batch`` with pinned host
    buffers (H2D + kernels + D2H inside the timed region);
  * ``roofline``: the dominant kernel's algorithmic bytes / its CUDA-event time, measured
    live in this run (pcb_profile_begin/end bracket every launch on its stream);
  * ``cpu_baseline``: the reference's own apply (oracle/_ref, compiled from its sources) on
    the host cores, bounded sample, rank 0 only.
``--impl reference`` runs only that reference timing as the headline line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Atilde-apply vectors/sec (fp64)"
UNIT = "vectors/s"

# workload definitions; c3 is the headline (BASELINE.json north_star target)
WORKLOADS = {
    "c1": dict(B=1, seed=0),
    "c2": dict(B=16, seed=1),
    "c3": dict(B=64, seed=2),
    "c4": dict(B=8, seed=4),
}


def family_of(name: str) -> str:
    for fam in ("rows_fwd", "rows_inv", "mid", "cols"):
        if name.startswith(fam):
            return fam
    return name


def fp64_peak_tflops():
    """Measured DFMA peak (scripts/fp64_peak.cu on this pool's B200, profiles/fp64_peak_r01.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")) as f:
            return float(json.load(f)["fp64_fma_tflops"]), "measured DFMA microbenchmark (profiles/fp64_peak_r01.json)"
    except Exception:
        return 37.0, "vendor nominal (no measurement found)"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_sample(cfg: str, threads: int, budget_terms: int = 0):
    """Reference ProductConvolutionOperator::apply (oracle/_ref, verbatim sources) on the host.

    Runs `threads` concurrent applies (apply is pure and thread-safe, pc_operator.hpp:15-16) of
    the operator restricted to the first `nt` terms, on the reference's own full-box extended
    impulses (impulse.cpp:74).  vectors/s = threads * (nt / r) / wall (extrapolated when nt < r).
    """
    from oracle import ref_lib  # CPU-baseline leg only
    from paper_1805_06018_b200 import inputs
    from paper_1805_06018_b200.operator import normal_vectors

    blur, nodes = inputs.config_spec(cfg)
    r = int(np.prod([len(a) for a in nodes]))
    nt = budget_terms or {"c1": r, "c2": r, "c3": 6, "c4": 2}.get(cfg, 4)
    nt = min(nt, r)
    kind = "reference" if ref_lib.available() else "port"
    inp = inputs.lattice_operator(cfg, blur, nodes, full_box=True, ks=list(range(nt)))
    F = normal_vectors(WORKLOADS[cfg]["seed"], threads, inp.n_points)
    if kind == "reference":
        op = ref_lib.RefOperator(inp)
        t0 = time.perf_counter()
        op.apply_batch(F, threads=threads)
        wall = time.perf_counter() - t0
        backend = "shimmed reference apply (pc_operator.cpp:45-56) with in-tree radix-2 FFT (FFTW absent)"
    else:  # numpy restatement, single thread (no reference build on this box)
        from oracle import pcop_oracle
        op = pcop_oracle.PCOperator.from_inputs(inp)
        threads = 1
        t0 = time.perf_counter()
        op.apply(F[0])
        wall = time.perf_counter() - t0
        backend = "numpy restatement (oracle/pcop_oracle.py), numpy.fft"
    value = threads * (nt / r) / wall
    sample = (f"{cfg}: {threads} concurrent applies x {nt}/{r} terms (full-box phi^E), wall {wall:.2f} s"
              + ("" if nt == r else f", extrapolated x{r / nt:.1f} to all terms") + f"; {backend}")
    return {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample}


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):  # untimed samples (page-in, thread spin-up)
        cpu_reference_sample(args.config, threads)
    vals = []
    for _ in range(max(1, args.steps)):
        cb = cpu_reference_sample(args.config, threads)
        vals.append(cb["value"])
    v = float(np.mean(vals))
    cb["value"] = v
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": WORKLOADS[args.config]["B"] / v * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json config shapes)",
            "config": {"workload": args.config, "global_batch": WORKLOADS[args.config]["B"]},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="auto", choices=["auto", "global", "local"])
    ap.add_argument("--shard", default="rhs", choices=["rhs", "k"])
    ap.add_argument("--batch", type=int, default=0, help="override the config batch")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="(ncu) run warmup + steps, print nothing else")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if not args.profile_only else args.warmup

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_1805_06018_b200 import inputs, lib
    from paper_1805_06018_b200.operator import ProductConvolutionOperator, normal_vectors

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # PCB_BENCH_FORCE_DIST=1: run the process-group path (init, barriers, max-over-ranks
    # all-reduces, the k-shard all-reduce) even at world size 1, to exercise it on one GPU
    use_dist = world > 1 or os.environ.get("PCB_BENCH_FORCE_DIST") == "1"
    if use_dist:
        dist.init_process_group("nccl", device_id=dev)

    cfg = args.config
    wl = WORKLOADS[cfg]
    B = args.batch or wl["B"]
    inp = inputs.make_config(cfg)
    N = inp.n_points
    # --shard rhs (default): weak scaling -- every rank applies the config's B vectors of its own
    # (rank r draws seed + r; rank 0 is the single-GPU workload), no collective.  --shard k: the
    # terms are split across ranks and the partial outputs all-reduced (strong scaling).
    weak = args.shard == "rhs"
    if weak:
        shard = (0, 1)
        Bl = B
        seed = wl["seed"] + rank
    else:
        shard = (rank, world) if world > 1 else (0, 1)
        Bl = B
        seed = wl["seed"]
    B_total = B * world if weak else B
    op = ProductConvolutionOperator.from_inputs(inp, mode=args.mode, max_batch=max(1, min(Bl, 64)), shard=shard,
                                                device=local_rank)
    info = op.info
    F_host = normal_vectors(seed, Bl, N)
    F = torch.from_numpy(F_host).to(dev)
    G = torch.empty_like(F)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    def step():
        op.apply_batch_dev(Bl, F.data_ptr(), G.data_ptr(), sptr)
        if args.shard == "k" and use_dist:
            dist.all_reduce(G)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if args.profile_only:
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        return

    # ---- timed region (device events per step, L2 flushed between steps) ----
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = lib.launch_count()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    launches = lib.launch_count() - launches0
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(np.sum(step_ms))
    if use_dist:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = B_total * args.steps / (total_ms * 1e-3)

    # ---- per-kernel profile (same workload, CUDA events around each launch on its stream) ----
    op.profile_begin()
    for _ in range(2):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    prof = op.profile_end()
    fam_ms = {}
    for name, (ms, _n) in prof.items():
        fam = family_of(name)
        fam_ms[fam] = fam_ms.get(fam, 0.0) + ms / 2
    dom_fam = max(fam_ms, key=fam_ms.get)
    dom_ms = fam_ms[dom_fam]
    hbm, peak_src = peaks()
    fp64_peak, fp64_src = fp64_peak_tflops()
    kb = info["kernel_bytes"][dom_fam] * Bl
    kf = info["kernel_flops"][dom_fam] * Bl
    achieved = kb / (dom_ms * 1e-3) / 1e9
    achieved_tf = kf / (dom_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{cfg}_{info['mode']}.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(dom_fam)
        except Exception:
            traffic = None

    # ---- e2e through the host C-ABI (pinned buffers, H2D + kernels + D2H per step) ----
    Fh = torch.from_numpy(F_host).pin_memory()
    Gh = torch.empty_like(Fh).pin_memory()
    Fn, Gn = Fh.numpy(), Gh.numpy()
    op.apply_batch(Fn)  # warm
    e2e_ms = []
    for _ in range(max(3, min(args.steps, 10))):
        flush.zero_()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rc = lib.load().pcb_apply_batch(op._h, Bl, Fn.ctypes.data, Gn.ctypes.data)
        b.record(stream)
        torch.cuda.synchronize()
        lib.check(rc)
        if args.shard == "k" and use_dist:
            t = torch.from_numpy(Gn).to(dev)
            dist.all_reduce(t)
        e2e_ms.append(a.elapsed_time(b))
    e2e_total = float(np.sum(e2e_ms))
    if use_dist:
        t = torch.tensor([e2e_total], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = B_total * len(e2e_ms) / (e2e_total * 1e-3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(cfg, os.cpu_count() or 1)
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable", "sample": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded mt19937_64 normal vectors; config blur operator built per BASELINE.json)",
            "config": {"workload": cfg, "global_batch": B_total, "per_gpu_batch": Bl, "n": inp.shape, "r": inp.rank,
                       "mode": info["mode"], "fft_size": info["fft_size"], "n_groups": info["n_groups"],
                       "shard": args.shard if world > 1 else "none", "parallelism": f"{args.shard}{world}",
                       "l2": "flushed between timed steps (256 MiB write) and inputs > L2",
                       "spectra_bytes": info["spectra_bytes"]},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(B_total * N * 8),
                    "d2h_bytes_per_step": int(B_total * N * 8)},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": dom_fam, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
                         "traffic": traffic,
                         "algorithmic_bytes": "bytes the kernel must read and write once per step in this "
                                              "pipeline (pcb_info.kernel_bytes x vectors)",
                         "kernel_ms_per_step": dom_ms, "kernel_share_of_step": dom_ms / (total_ms / args.steps),
                         "fp64": {"achieved": achieved_tf, "peak": fp64_peak, "unit": "TFLOP/s",
                                  "frac": achieved_tf / fp64_peak, "peak_source": fp64_src}},
            "pipeline_roofline": {"algorithmic_bytes_per_vector": info["bytes_per_vector"],
                                  "per_gpu": True,
                                  "achieved_gbs": info["bytes_per_vector"] * value / world / 1e9,
                                  "frac_hbm": info["bytes_per_vector"] * value / world / 1e9 / hbm,
                                  "nominal_tflops": info["flops_per_vector"] * value / world / 1e12,
                                  "frac_fp64": info["flops_per_vector"] * value / world / 1e12 / fp64_peak,
                                  "definition": "SURVEY 8(d): every stored half spectrum read once + f + g"},
            "kernels_ms_per_step": {k: round(v[0] / 2, 4) for k, v in prof.items()},
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
