"""Generate tests/golden/headline_{c3,c4,c5}.npz: the reference's own outputs at the FULL headline
configurations (BASELINE.json configs 3, 4, 5), as fingerprints (tests/headline_common.py).

Every value comes from the reference library compiled verbatim from /root/reference/proj/core/src
(oracle/_ref/libpcopref.so, oracle/Makefile):
  * c3 (1024^2, r = 256) and c4 (128^3, r = 512): ProductConvolutionOperator::apply /
    ::apply_adjoint (pc_operator.cpp:45-69) with the k-loop split across host threads
    (oracle.ref_lib.apply_split) -- apply on vectors 0, 1 and apply_adjoint on vector 0 of the
    config's seeded batch (c3 seed 2, c4 seed 4);
  * c5 (the c2 operator, 4096 blocks of 8x8 x 8x8 points, origins mt19937_64(3)): ::entry
    (pc_operator.cpp:84-96) for all 16.8 M entries; the fixture keeps the SHA-256 of the whole
    [blk][i][j] array (the GPU gather must be bit-identical) and the values of 16 nonzero blocks.
Run here (needs the oracle build, ~6 min on 8 cores):  python tests/golden/make_headline_golden.py
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from headline_common import c5_origins, c5_pairs, fingerprint, sha256_f64  # noqa: E402
from oracle import ref_lib  # noqa: E402
from paper_1805_06018_b200 import inputs  # noqa: E402
from paper_1805_06018_b200.operator import normal_vectors  # noqa: E402

SEEDS = {"c3": 2, "c4": 4}


def make_cfg(cfg: str, out: dict):
    inp = inputs.make_config(cfg)
    F = normal_vectors(SEEDS[cfg], 2, inp.n_points)
    t = time.time()
    G = ref_lib.apply_split(inp, F, adjoint=False)
    print(f"{cfg} apply x2: {time.time() - t:.1f} s", flush=True)
    t = time.time()
    GA = ref_lib.apply_split(inp, F[:1], adjoint=True)
    print(f"{cfg} adjoint x1: {time.time() - t:.1f} s", flush=True)
    for b in range(2):
        for k, v in fingerprint(G[b], inp.shape).items():
            out[f"apply{b}_{k}"] = v
    for k, v in fingerprint(GA[0], inp.shape).items():
        out[f"adjoint0_{k}"] = v
    out["checksum"] = np.array(inp.checksum())
    out["seed"] = np.array(SEEDS[cfg])


def make_c5(out: dict):
    inp = inputs.make_config("c2")
    ref = ref_lib.RefOperator(inp)
    org = c5_origins()
    y, x = c5_pairs(org)
    t = time.time()
    E = ref_lib.entries_split(ref, y, x).reshape(4096, 64, 64)
    print(f"c5 entries: {time.time() - t:.1f} s", flush=True)
    nz = np.flatnonzero(np.abs(E).reshape(4096, -1).max(axis=1) > 0)
    keep = nz[np.linspace(0, len(nz) - 1, min(16, len(nz))).astype(int)] if len(nz) else nz
    out.update(origins=org, sha256=np.array(sha256_f64(E)), nonzero_blocks=nz, keep=keep, blocks=E[keep],
               abs_max=np.array(np.abs(E).max()), checksum=np.array(inp.checksum()))
    print(f"c5: {len(nz)} nonzero blocks of 4096", flush=True)


def main():
    which = sys.argv[1:] or ["c5", "c3", "c4"]
    for cfg in which:
        out = {}
        make_c5(out) if cfg == "c5" else make_cfg(cfg, out)
        np.savez_compressed(os.path.join(HERE, f"headline_{cfg}.npz"), **out)
        print("wrote", f"headline_{cfg}.npz", flush=True)


if __name__ == "__main__":
    main()
