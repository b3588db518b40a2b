"""Build an A/B variant of the library into build/ab/<tag>.so (env PCB_E_ROWS / PCB_E_COLS / PCB_E_MID /
PCB_NVCC_EXTRA select it).  usage: PCB_E_ROWS=8 python scripts/build_variant.py rows8"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06018_b200 import build as b  # noqa: E402

tag = sys.argv[1]
b.OBJDIR = os.path.join(b.ROOT, "build", "obj_" + tag)
b.LIB = os.path.join(b.ROOT, "build", "ab", tag + ".so")
os.makedirs(os.path.dirname(b.LIB), exist_ok=True)
print(b.build())
