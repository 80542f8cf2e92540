import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_15869_b200 import _native
_native.LIB = _native.LIB.replace("libeik_ifim.so", sys.argv[1])
import runpy
sys.argv = ["probe", "512"]
runpy.run_path(os.path.join(os.path.dirname(__file__), "probe_perf.py"), run_name="__main__")
