import sys, os, shutil
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["EIK_DIAG_PRINT"] = "1"
from paper_2106_15869_b200 import _native
_native.LIB = _native.LIB.replace("libeik_ifim.so", "libeik_ifim_diag.so")
import runpy
sys.argv = ["probe", sys.argv[1] if len(sys.argv) > 1 else "256"]
runpy.run_path(os.path.join(os.path.dirname(__file__), "probe_perf.py"), run_name="__main__")
