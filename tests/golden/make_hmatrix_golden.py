"""Generate tests/golden/hmatrix_ref_{randomized,cur}.pchm.gz: the reference's own H-matrix
(assemble_hmatrix + save_hmatrix, hmatrix.cpp:338-471, compiled verbatim into oracle/_ref against
the Eigen shim) of the 12x12 two-tent blur operator (inputs.small_lattice(n=12, m=2, sigma=3.0)),
tol 1e-8, leaf_cap 16.  Run here:  python tests/golden/make_hmatrix_golden.py"""
import gzip
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref_lib  # noqa: E402
from paper_1805_06018_b200 import inputs  # noqa: E402

SPEC = dict(n=12, dim=2, m=2, sigma=3.0)
TOL, LEAF = 1e-8, 16


def main():
    inp = inputs.small_lattice(**SPEC)
    op = ref_lib.RefOperator(inp)
    for method in ("randomized", "cur"):
        H = ref_lib.RefHMatrix.assemble(op, TOL, LEAF, method)
        tmp = os.path.join(HERE, f".tmp_{method}.pchm")
        H.save(tmp)
        with open(tmp, "rb") as f, open(os.path.join(HERE, f"hmatrix_ref_{method}.pchm.gz"), "wb") as g:
            g.write(gzip.compress(f.read(), mtime=0))
        os.remove(tmp)
        print(method, H.info())
    with open(os.path.join(HERE, "hmatrix_ref.checksum"), "w") as f:
        f.write(inp.checksum() + "\n")


if __name__ == "__main__":
    main()
