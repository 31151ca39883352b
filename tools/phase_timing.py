"""Per-phase K3 cycles (needs a FGT_PHASE_TIMING=1 build via FGT1D_LIB)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import subprocess
from paper_1909_09825_b200 import _capi
L = _capi.lib()
L.fgt_debug_phase_cycles.restype = ctypes.c_int
L.fgt_debug_phase_cycles.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
import runpy
sys.argv = ["plan_timing.py", sys.argv[1] if len(sys.argv) > 1 else "1e8"]
buf = (ctypes.c_ulonglong * 8)()
L.fgt_debug_phase_cycles(buf)
runpy.run_path(os.path.join(os.path.dirname(__file__), "plan_timing.py"), run_name="__main__")
L.fgt_debug_phase_cycles(buf)
segs = max(buf[4], 1)
names = ["loads+degrees", "carries", "pass2", "output"]
tot = sum(buf[i] for i in range(4))
for i, n in enumerate(names):
    print(f"{n:15s} {buf[i] / segs:10.0f} cycles/segment  {100 * buf[i] / tot:5.1f}%")
