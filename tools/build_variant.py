"""Build an experiment variant of the engine: python tools/build_variant.py NAME [-DMACRO[=V] ...]
-> paper_2106_15869_b200/NAME.so (compare with tools/ab.py NAME.so ..., diagnostics: tools/diag_density.py)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_15869_b200 import _native as n  # noqa: E402

out = os.path.join(os.path.dirname(n.LIB), sys.argv[1] + ".so")
subprocess.check_call([n.nvcc(), *n.NVCC_FLAGS, *sys.argv[2:], "-I", os.path.join(n.ROOT, "include"), "-o", out, n.SRC])
print(out)
