#!/bin/bash
# cfg2 probe for several engine variants: tools/cfg2_ab.sh libA.so libB.so ...
for v in "$@"; do
  python - "$v" <<'PY'
import sys
v = sys.argv[1]
sys.path.insert(0, ".")
from paper_2106_15869_b200 import _native
_native.LIB = _native.LIB.replace("libeik_ifim.so", v)
sys.argv = ["cfg2_probe", "4096"]
import runpy
runpy.run_path("tools/cfg2_probe.py", run_name="__main__")
PY
done
