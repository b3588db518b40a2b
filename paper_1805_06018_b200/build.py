"""Build the in-tree C-ABI library ``paper_1805_06018_b200/lib/libpcop_b200.so`` with nvcc for sm_100a.

No torch extension machinery: the product is a plain shared library with the C ABI of
``include/pcb/pcb.h``; Python reaches it through ctypes (``paper_1805_06018_b200.lib``).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
OBJDIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(LIBDIR, "libpcop_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-diag-suppress", "177,128",
          "-Xcompiler", "-fPIC,-fvisibility=hidden", f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]
EXTRA = os.environ.get("PCB_NVCC_EXTRA", "").split()  # experiments
# elements per thread of the power-of-two FFT engines, per kernel family (fft.cuh PCB_E2)
E_ROWS = os.environ.get("PCB_E_ROWS", "8")
E_COLS = os.environ.get("PCB_E_COLS", "16")
E_MID = os.environ.get("PCB_E_MID", "8")
E3_MID = os.environ.get("PCB_E3_MID", "12")  # 3-smooth engines: 12 elements per thread in mid, 24 elsewhere
E3_COLS = os.environ.get("PCB_E3_COLS", "24")  # 3-smooth engines of the cols pass
E3_COLS_SMALL = os.environ.get("PCB_E3_COLS_SMALL", "96")  # cols: 3-smooth lengths <= this use 12 per thread
E_COLS_SMALL = os.environ.get("PCB_E_COLS_SMALL", "64")  # cols: pow2 lengths <= this use 8 elements per thread
RADIX_DESC_ROWS = os.environ.get("PCB_RADIX_DESC_ROWS", "1")  # rows: prefix radices largest first
E3_ROWS_SMALL = os.environ.get("PCB_E3_ROWS_SMALL", "0")  # rows: 3-smooth lengths <= this use 12 per thread
PER_SOURCE = {"kernels_rows.cu": [f"-DPCB_E2={E_ROWS}", f"-DPCB_RADIX_DESC={RADIX_DESC_ROWS}",
                                  f"-DPCB_E3_SMALL_MAX={E3_ROWS_SMALL}"],
              "kernels_cols.cu": [f"-DPCB_E2={E_COLS}", f"-DPCB_E2_SMALL_MAX={E_COLS_SMALL}", f"-DPCB_E3={E3_COLS}",
                                  f"-DPCB_E3_SMALL_MAX={E3_COLS_SMALL}"],
              "kernels_mid.cu": [f"-DPCB_E2={E_MID}", f"-DPCB_E3={E3_MID}"]}
SOURCES = ["kernels_rows.cu", "kernels_cols.cu", "kernels_mid.cu", "kernels_misc.cu", "blur.cu", "hmatrix.cpp", "comm.cpp", "pcop_b200.cpp"]
HEADERS = ["fft.cuh", "kernels.cuh", "kernels_impl.cuh", "comm.h"]


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths if os.path.exists(p))


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJDIR, os.path.splitext(src)[0] + ".o")
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + \
        [os.path.join(ROOT, "include", "pcb", "pcb.h")]
    lang = [] if src.endswith(".cu") else ["-x", "cu"]
    cmd = [NVCC] + ARCH + COMMON + EXTRA + PER_SOURCE.get(src, []) + lang + ["-c", os.path.join(CSRC, src), "-o", obj]
    stamp = obj + ".cmd"  # the object is stale when its sources are newer or its command changed
    if (os.path.exists(obj) and os.path.getmtime(obj) >= _newest(deps) and os.path.exists(stamp)
            and open(stamp).read() == " ".join(cmd)):
        return obj
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    with open(stamp, "w") as f:
        f.write(" ".join(cmd))
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    if not (os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest(objs)):
        cmd = [NVCC] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", LIB] + objs + ["-lcudart_static", "-ldl", "-lrt",
                                                                                         "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


# FFT engine unit test (tests/cuda/fft_unit.cu vs a long-double DFT, every compiled length, both
# directions, both register orders), once per element-count setting the product compiles:
# (PCB_E2, PCB_E3, PCB_E2_SMALL_MAX, PCB_E3_SMALL_MAX, PCB_RADIX_DESC) of cols (16/24, 8 for <= 64,
# 12 for <= 96), rows (8/24, radices largest first) and mid (8/12).  Run by tests/test_gpu_tools.py.
FFT_UNIT_CONFIGS = [(E_COLS, E3_COLS, E_COLS_SMALL, E3_COLS_SMALL, "0"), (E_COLS, E3_COLS, "0", "0", "0"),
                    (E_ROWS, "24", "0", "0", RADIX_DESC_ROWS), (E_ROWS, "24", "0", "0", "0"), (E_MID, E3_MID, "0", "0", "0")]
TOOLDIR = os.path.join(ROOT, "build", "tools")


def fft_unit_path(cfg) -> str:
    return os.path.join(TOOLDIR, "fft_unit_" + "_".join(cfg))


def build_tools(verbose: bool = False) -> list:
    os.makedirs(TOOLDIR, exist_ok=True)
    src = os.path.join(ROOT, "tests", "cuda", "fft_unit.cu")
    deps = [src, os.path.join(CSRC, "fft.cuh")]

    def one(cfg):
        out = fft_unit_path(cfg)
        if os.path.exists(out) and os.path.getmtime(out) >= _newest(deps):
            return out
        e2, e3, s2, s3, desc = cfg
        cmd = [NVCC] + ARCH + ["-O2", "-std=c++17", "--expt-relaxed-constexpr", f"-DPCB_E2={e2}", f"-DPCB_E3={e3}",
                               f"-DPCB_E2_SMALL_MAX={s2}", f"-DPCB_E3_SMALL_MAX={s3}", f"-DPCB_RADIX_DESC={desc}",
                               f"-I{CSRC}", f"-I{os.path.join(ROOT, 'include')}", src, "-o", out]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return out

    cfgs = list(dict.fromkeys(FFT_UNIT_CONFIGS))
    with ThreadPoolExecutor(max_workers=len(cfgs)) as ex:
        return list(ex.map(one, cfgs))


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
    if "--tools" in sys.argv:
        print(build_tools(verbose="-v" in sys.argv))
