"""bench.py's driver contract: one JSON line on stdout with the required keys, for the reference
arm (runs on the CPU: the reference's own apply from oracle/_ref, never the product library) and,
on a GPU, for our arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e"]


def run_bench(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout[-2000:]  # exactly one line on stdout
    return json.loads(lines[0])


@pytest.mark.skipif(not __import__("oracle.ref_lib", fromlist=["x"]).available(),
                    reason="reference build (oracle/_ref) not built")
def test_reference_arm_contract():
    d = run_bench(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1"])
    for k in BASE + ["impl", "cpu_baseline"]:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["latency_1core_s_per_vector"] > 0
    assert cb["host_cpu"] and cb["terms_covered"] == 16
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "c1" and d["config"]["r"] == 16


def test_reference_arm_does_not_load_the_product():
    """The reference arm runs the reference alone: libpcop_b200.so is never mapped."""
    from oracle import ref_lib

    if not ref_lib.available():
        pytest.skip("reference build (oracle/_ref) not built")
    code = ("import runpy,sys; sys.argv=['bench.py','--impl','reference','--config','c1','--steps','1',"
            "'--warmup','1']; runpy.run_path('bench.py', run_name='__main__'); "
            "m=open('/proc/self/maps').read(); sys.stderr.write('MAPPED=%d\\n' % ('libpcop_b200' in m))")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "MAPPED=0" in r.stderr


@pytest.mark.gpu
def test_gpu_arm_contract(gpu):
    d = run_bench(["--config", "c1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"])
    for k in BASE + ["roofline", "gpu_launches", "clocks", "plan"]:
        assert k in d, k
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert d["gpu_launches"] > 0 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == d["config"]["global_batch"] * 128 * 128 * 8
