#!/usr/bin/env python
"""Benchmark: Atilde-apply vectors/s (fp64) on B200 for a BASELINE.json configuration.

One "step" = one apply of the product-convolution operator to the configuration's batch of
vectors (c3: 64 vectors on 1024^2, r = 256).  Contract (README / task):
  * W >= 3 untimed warm-up steps, then K timed steps, each bracketed by CUDA events on the
    launching stream; L2 is flushed (a 256 MiB write) between timed steps, outside the events;
  * multi-GPU: one process per GPU (torchrun).  ``--shard k`` (default for c3/c4, BASELINE.json
    "sharded over 8 GPUs by k"): strong scaling, the config's B vectors, terms split by the
    planner's modelled cost, the partials summed by ncclReduce INSIDE libpcop_b200 (its own
    communicator) within every timed apply; a shard-by-RHS weak-scaling measurement rides along
    as ``rhs_weak``.  ``--shard rhs``: weak scaling, every rank applies B vectors of its own;
    value = all ranks' vectors / max-over-ranks time;
  * ``e2e``: the same metric through the host C-ABI call ``pcb_apply_batch`` with pinned host
    buffers (H2D + kernels + reduce + D2H inside the timed region); ``pageable_value`` the same
    with plain numpy buffers;
  * ``roofline``: SURVEY 8(d) algorithmic bytes (spectra once per vector + f + g at the FFT sizes
    used) / the dominant kernel's CUDA-event time (and / the step time), measured live in this
    run (pcb_profile_begin/end bracket every launch on its stream); ``traffic`` = ncu DRAM bytes
    of the same build (profiles/traffic_<cfg>_<mode>.json, matched by source hash);
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


def emit(line: dict) -> None:  # replaced in main() by the writer to the saved stdout
    print(json.dumps(line), flush=True)
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


def host_cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# terms per reference sample: c1/c2 in full; c3/c4 have uniform per-term FFT sizes on the reference's
# full-box phi^E (2048^2 / 256^3), so a block of terms is timed and scaled by r / nt
REF_TERMS = {"c1": 0, "c2": 0, "c3": 4, "c4": 1}
REF_LATENCY_TERMS = {"c1": 0, "c2": 0, "c3": 16, "c4": 4}
REF_BACKEND = "shimmed reference apply (pc_operator.cpp:45-56) with the in-tree radix-2 FFT behind the fftw3.h shim (FFTW absent)"


class RefSampler:
    """The reference ProductConvolutionOperator::apply (oracle/_ref: its own sources compiled
    verbatim, oracle/Makefile) on the host cores.  Never loads the product library: the inputs come
    from paper_1805_06018_b200.inputs (pure numpy) and the vectors from the reference build's own
    mt19937_64 stream (ref_lib.normal_vectors).

    sample(threads, k0, nt): `threads` concurrent applies (apply is pure and thread-safe,
    pc_operator.hpp:15-16) of the operator restricted to the terms k0 .. k0+nt-1 (mod r), each on
    its own vector; vectors/s = threads * (nt / r) / wall.  The reference's per-term cost is uniform
    at c3/c4 (P_k = 2048^2 / 256^3 for every term), so the r / nt scaling is exact up to noise."""

    def __init__(self, cfg: str):
        from oracle import ref_lib  # CPU-baseline leg / reference arm only
        from paper_1805_06018_b200 import inputs

        if not ref_lib.available():
            raise FileNotFoundError("oracle/_ref/libpcopref.so missing (make -C oracle)")
        self.ref_lib = ref_lib
        self.inputs = inputs
        self.cfg = cfg
        self.blur, self.nodes = inputs.config_spec(cfg)
        self.r = int(np.prod([len(a) for a in self.nodes]))
        self.N = self.blur.n ** self.blur.dim
        self.F = ref_lib.normal_vectors(WORKLOADS[cfg]["seed"], max(1, os.cpu_count() or 1), self.N)
        self._ops = {}

    def _op(self, ks):
        key = tuple(ks)
        if key not in self._ops:
            inp = self.inputs.lattice_operator(self.cfg, self.blur, self.nodes, full_box=True, ks=list(ks))
            self._ops = {key: self.ref_lib.RefOperator(inp)}  # keep one operator alive at a time
        return self._ops[key]

    def sample(self, threads: int, k0: int, nt: int):
        nt = min(nt or self.r, self.r)
        ks = [(k0 + i) % self.r for i in range(nt)]
        op = self._op(ks)
        t0 = time.perf_counter()
        op.apply_batch(self.F[:threads], threads=threads)
        wall = time.perf_counter() - t0
        return threads * (nt / self.r) / wall, wall, ks


def cpu_reference_sample(cfg: str, threads: int):
    """cpu_baseline of the GPU arm: T-core throughput on nt terms plus 1-core latency on the
    latency block (16 terms at c3), both scaled to all r terms; ~10-30 s of CPU work."""
    rs = RefSampler(cfg)
    nt = REF_LATENCY_TERMS[cfg] or rs.r
    rs.sample(1, 0, 1)  # page-in
    v_t, wall_t, ks = rs.sample(threads, 0, nt)
    v_1, wall_1, _ = rs.sample(1, 0, nt)
    scale = rs.r / len(ks)
    sample = (f"{cfg}: {threads} concurrent applies on distinct vectors x terms {ks[0]}..{ks[-1]} "
              f"({len(ks)}/{rs.r}, full-box phi^E), wall {wall_t:.2f} s"
              + ("" if len(ks) == rs.r else f", extrapolated x{scale:.1f} to all terms (uniform per-term cost)")
              + f"; 1-core latency from one apply on the same terms ({wall_1:.2f} s); {REF_BACKEND}")
    return {"value": v_t, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample,
            "latency_1core_s_per_vector": wall_1 * scale, "throughput_1core": v_1,
            "host_cpu": host_cpu_model(), "fft_backend": "in-tree radix-2 (oracle/shim/shim_fft.cpp)",
            "terms_sampled": len(ks)}


def workload_config(cfg: str) -> dict:
    """The workload both arms run (identical in the GPU and reference lines)."""
    from paper_1805_06018_b200 import inputs

    blur, nodes = inputs.config_spec(cfg)
    return {"workload": cfg, "global_batch": WORKLOADS[cfg]["B"], "n": [blur.n] * blur.dim,
            "r": int(np.prod([len(a) for a in nodes])), "seed": WORKLOADS[cfg]["seed"],
            "desc": inputs.CONFIGS[cfg]["desc"]}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU apply, all host threads, rank 0 only.  Warm-up
    samples are 1-term applies (page-in, thread spin-up); timed step i applies T vectors over the
    term block starting at i * nt, so the K steps cover K * nt distinct terms (c3: 4 per step,
    >= 16 over the run; c4: 1 per step); value = mean over steps of T * (nt / r) / wall."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    rs = RefSampler(args.config)
    nt = REF_TERMS[args.config] or rs.r
    for i in range(args.warmup):
        rs.sample(threads, i, 1)
    vals, walls, covered = [], [], set()
    for i in range(max(1, args.steps)):
        v, w, ks = rs.sample(threads, i * nt, nt)
        vals.append(v)
        walls.append(w)
        covered.update(ks)
    lat_nt = REF_LATENCY_TERMS[args.config] or rs.r
    _, wall_1, ks1 = rs.sample(1, 0, lat_nt)
    v = float(np.mean(vals))
    cb = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
          "sample": (f"{args.config}: per step {threads} concurrent applies on distinct vectors x {nt}/{rs.r} terms "
                     f"(full-box phi^E; step i covers terms i*{nt}..), mean step wall {np.mean(walls):.2f} s, "
                     f"{len(covered)} distinct terms over the run"
                     + ("" if nt == rs.r else f", extrapolated x{rs.r / nt:.1f} to all terms (uniform per-term cost)")
                     + f"; {REF_BACKEND}"),
          "latency_1core_s_per_vector": wall_1 * rs.r / len(ks1), "latency_terms_sampled": len(ks1),
          "host_cpu": host_cpu_model(), "fft_backend": "in-tree radix-2 (oracle/shim/shim_fft.cpp)",
          "terms_covered": len(covered)}
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": WORKLOADS[args.config]["B"] / v * 1e3, "higher_is_better": True,
            "scaling": "strong" if args.shard == "k" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded mt19937_64 normal vectors; config blur "
                                                         "operator built per BASELINE.json)",
            "config": workload_config(args.config), "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def source_hash() -> str:
    """Hash of the sources the library is built from: a traffic file measured on another build is
    not used (roofline.traffic is null then)."""
    import hashlib

    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_1805_06018_b200", "csrc")
    files = sorted(os.path.join(csrc, f) for f in os.listdir(csrc)) + [
        os.path.join(ROOT, "include", "pcb", "pcb.h"), os.path.join(ROOT, "paper_1805_06018_b200", "build.py")]
    for f in files:
        if os.path.isfile(f):
            h.update(os.path.basename(f).encode())
            h.update(open(f, "rb").read())
    return h.hexdigest()[:16]


def main():
    # exactly one JSON line on stdout: everything else the process writes to fd 1 (NCCL's init
    # banner and NCCL_DEBUG=INFO log lines, library prints) goes to stderr
    json_out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    os.environ.setdefault("NCCL_DEBUG", "INFO")  # NCCL init logs (ranks, NVLS / transport choice) on stderr
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    global emit
    emit = lambda line: (json_out.write(json.dumps(line) + "\n"), json_out.flush())  # noqa: E731
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="auto", choices=["auto", "global", "local"])
    ap.add_argument("--shard", default="auto", choices=["auto", "rhs", "k"],
                    help="auto: k for c3/c4 (BASELINE.json: 'sharded over 8 GPUs by k'), rhs otherwise")
    ap.add_argument("--reduce", default="root", choices=["root", "all"], help="k-shard combine (ncclReduce / AllReduce)")
    ap.add_argument("--batch", type=int, default=0, help="override the config batch")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the shard-by-RHS secondary measurement")
    ap.add_argument("--profile-only", action="store_true", help="(ncu) run warmup + steps, print nothing else")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if not args.profile_only else args.warmup
    if args.shard == "auto":
        args.shard = "k" if args.config in ("c3", "c4") else "rhs"

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
    # the process group is plumbing only (barriers, max-over-ranks timing, the NCCL id broadcast);
    # the shard reduce itself runs inside libpcop_b200 on its own communicator.
    # PCB_BENCH_FORCE_DIST=1 runs that path at world size 1 (a 1-rank communicator) on one GPU.
    use_dist = world > 1 or os.environ.get("PCB_BENCH_FORCE_DIST") == "1"
    if use_dist:
        dist.init_process_group("nccl", device_id=dev)

    cfg = args.config
    wl = WORKLOADS[cfg]
    B = args.batch or wl["B"]
    inp = inputs.make_config(cfg)
    N = inp.n_points
    kshard = args.shard == "k"
    nccl_id = None
    if kshard and use_dist:
        box = [lib.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        nccl_id = box[0]
    # --shard k: strong scaling -- the config's B vectors, the terms split by modelled cost, the
    # partial outputs summed by the library (ncclReduce to rank 0) inside every apply.
    # --shard rhs: weak scaling -- every rank applies B vectors of its own (seed + rank), no collective.
    seed = wl["seed"] if kshard else wl["seed"] + rank
    B_total = B if kshard else B * world
    t_create = time.perf_counter()
    op = ProductConvolutionOperator.from_inputs(inp, mode=args.mode, max_batch=max(1, min(B, 64)),
                                                shard=(rank, world) if kshard else (0, 1), device=local_rank,
                                                nccl_id=nccl_id, reduce=args.reduce)
    t_create = time.perf_counter() - t_create
    info = op.info
    F_host = normal_vectors(seed, B, N)
    F = torch.from_numpy(F_host).to(dev)
    G = torch.empty_like(F)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    def step():
        op.apply_batch_dev(B, F.data_ptr(), G.data_ptr(), sptr)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if args.profile_only:
        for _ in range(args.steps):
            flush.zero_()
            step()
        torch.cuda.synchronize()
        return

    def max_over_ranks(v: float) -> float:
        if not use_dist:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps):
        """K steps, CUDA events per step on the launching stream, L2 flushed between steps
        (outside the events), barrier + synchronize on both sides; max over ranks."""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(steps):
            flush.zero_()
            ev[i][0].record(stream)
            fn()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        return max_over_ranks(float(np.sum([a.elapsed_time(b) for a, b in ev])))

    # ---- timed region ----
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    launches0 = lib.launch_count()
    total_ms = timed(step, args.steps)
    launches = lib.launch_count() - launches0
    clk = clocks.stop()
    value = B_total * args.steps / (total_ms * 1e-3)
    step_ms = total_ms / args.steps

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
    # SURVEY 8(d) algorithmic bytes: every stored half spectrum read once per vector + f read + g
    # written, at the FFT sizes actually used (this shard's terms)
    alg_vec = info["bytes_per_vector"]
    alg_step = alg_vec * B
    achieved = alg_step / (dom_ms * 1e-3) / 1e9
    achieved_step = alg_step / (step_ms * 1e-3) / 1e9
    kb = info["kernel_bytes"][dom_fam] * B
    kf = info["kernel_flops"][dom_fam] * B
    src_hash = source_hash()
    traffic = traffic_total = None
    traffic_note = "no ncu capture of this build"
    tpath = os.path.join(ROOT, "profiles", f"traffic_{cfg}_{info['mode']}.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            if tj.get("source_hash") == src_hash and tj.get("batch") == B:
                traffic = tj["per_step"].get(dom_fam)
                traffic_total = sum(tj["per_step"].values())
                traffic_note = f"ncu dram__bytes_read+write.sum per step, {os.path.basename(tpath)} (same source hash)"
            else:
                traffic_note = f"{os.path.basename(tpath)} was measured on another build ({tj.get('source_hash')})"
        except Exception as e:
            traffic_note = f"unreadable traffic file: {e}"

    # ---- e2e through the host C-ABI: pinned (the copy-engine path) and pageable numpy buffers ----
    def e2e(Fn, Gn, reps):
        lib.check(lib.load().pcb_apply_batch(op._h, B, Fn.ctypes.data, Gn.ctypes.data))  # warm
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            torch.cuda.synchronize()
            if use_dist:
                dist.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            rc = lib.load().pcb_apply_batch(op._h, B, Fn.ctypes.data, Gn.ctypes.data)
            b.record(stream)
            torch.cuda.synchronize()
            lib.check(rc)
            tot += a.elapsed_time(b)
        return B_total * reps / (max_over_ranks(tot) * 1e-3)

    Fh = torch.from_numpy(F_host).pin_memory()
    Gh = torch.empty_like(Fh).pin_memory()
    reps = max(3, min(args.steps, 10))
    e2e_value = e2e(Fh.numpy(), Gh.numpy(), reps)
    Gp = np.empty_like(F_host)
    e2e_pageable = e2e(F_host, Gp, max(2, reps // 2))
    # the same caller-owned numpy buffers page-locked in place (pcb_host_register): what a binding that
    # reuses its std::vector buffers gets; the registration itself is timed separately
    t0 = time.perf_counter()
    reg = lib.host_registered(F_host, Gp)
    reg.__enter__()
    reg_ms = (time.perf_counter() - t0) * 1e3
    try:
        e2e_registered = e2e(F_host, Gp, max(2, reps // 2))
    finally:
        reg.__exit__(None, None, None)

    # ---- secondary: shard-by-RHS weak scaling (every rank its own B vectors, no collective) ----
    rhs = None
    if kshard and world > 1 and not args.no_secondary:
        op_r = ProductConvolutionOperator.from_inputs(inp, mode=args.mode, max_batch=max(1, min(B, 64)),
                                                      device=local_rank)
        Fr = torch.from_numpy(normal_vectors(wl["seed"] + rank, B, N)).to(dev)
        Gr = torch.empty_like(Fr)
        fn = lambda: op_r.apply_batch_dev(B, Fr.data_ptr(), Gr.data_ptr(), sptr)  # noqa: E731
        for _ in range(args.warmup):
            fn()
        ms_r = timed(fn, args.steps)
        rhs = {"value": B * world * args.steps / (ms_r * 1e-3), "unit": UNIT, "scaling": "weak",
               "global_batch": B * world, "ms_per_step": ms_r / args.steps}
        op_r.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(cfg, os.cpu_count() or 1)
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable", "sample": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong" if kshard else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded mt19937_64 normal vectors; config blur operator built per BASELINE.json)",
            "config": workload_config(cfg) if B == wl["B"] else dict(workload_config(cfg), global_batch=B_total),
            "plan": {"parallelism": f"{'k' if kshard else 'rhs'}{world}", "per_gpu_batch": B,
                     "global_batch": B_total, "mode": info["mode"], "fft_size": info["fft_size"],
                     "n_groups": info["n_groups"], "spectra_bytes": info["spectra_bytes"],
                     "terms_this_rank": info["rank_active"], "shard_cost_share": info["shard_cost"] / max(info["total_cost"], 1e-300),
                     "reduce": (f"nccl {args.reduce} inside libpcop_b200 (comm ranks {info['comm_nranks']}, "
                                f"NCCL {info['comm_version']})") if nccl_id else "none",
                     "create_s": round(t_create, 3),
                     "l2": "flushed between timed steps (256 MiB write) and inputs > L2"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(B * N * 8 * world),
                    "d2h_bytes_per_step": int(B * N * 8 * world),
                    "path": "pcb_apply_batch, pinned host buffers (H2D + kernels + reduce + D2H)",
                    "pageable_value": e2e_pageable, "registered_value": e2e_registered, "register_ms": reg_ms},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": dom_fam, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs, burst copy)",
                         "traffic": traffic, "traffic_ratio": (traffic / alg_step) if traffic else None,
                         "traffic_note": traffic_note, "source_hash": src_hash,
                         "algorithmic_bytes_per_step": alg_step,
                         "algorithmic_bytes": "SURVEY 8(d): r*16*P^(d-1)*(P/2+1) summed over this shard's terms at "
                                              "the FFT sizes used + 16*N, per vector, x vectors per step",
                         "kernel_ms_per_step": dom_ms, "kernel_share_of_step": dom_ms / step_ms,
                         "step": {"achieved": achieved_step, "frac": achieved_step / hbm,
                                  "traffic": traffic_total,
                                  "traffic_ratio": (traffic_total / alg_step) if traffic_total else None},
                         "kernel_io": {"achieved": kb / (dom_ms * 1e-3) / 1e9, "frac": kb / (dom_ms * 1e-3) / 1e9 / hbm,
                                       "definition": "the dominant kernel's own inputs+outputs once (incl. the S/T "
                                                     "intermediates; pcb_info.kernel_bytes) / its time"},
                         "fp64": {"achieved": kf / (dom_ms * 1e-3) / 1e12, "peak": fp64_peak, "unit": "TFLOP/s",
                                  "frac": kf / (dom_ms * 1e-3) / 1e12 / fp64_peak, "peak_source": fp64_src,
                                  "step_tflops": info["flops_per_vector"] * B / (step_ms * 1e-3) / 1e12}},
            "kernels_ms_per_step": {k: round(v[0] / 2, 4) for k, v in prof.items()},
            "model_ms_per_vector": {"local": info["model_ms_local"], "global": info["model_ms_global"],
                                    "measured": step_ms / B},
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        if rhs:
            line["rhs_weak"] = rhs
        emit(line)
    op.close()
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
