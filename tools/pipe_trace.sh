# Phase trace of fgt_transform_host at N = M = 1e8 (GPU box): gpurun_out/pipe_trace.log
FGT_PIPE_TRACE=1 python - > gpurun_out/pipe_trace.log 2>&1 <<'PY'
import ctypes, os, sys, time
sys.path.insert(0, '.')
import torch
from paper_1909_09825_b200 import _capi
from paper_1909_09825_b200.soe import soe_for_tolerance
PD = ctypes.POINTER(ctypes.c_double)
n = 100_000_000
L = _capi.lib(); dev = torch.device("cuda", 0)
sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
def gen(sid, sort=True):
    raw = torch.empty(n, dtype=torch.float64, device=dev)
    _capi.check(L.fgt_uniform_points_device(raw.data_ptr(), n, 0, sid, 0, sh))
    return raw.sort().values if sort else raw
x, y = gen(3), gen(0); a = gen(1, False) * 2 - 1
hx, hy, ha = x.cpu().pin_memory(), y.cpu().pin_memory(), a.cpu().pin_memory()
hu = torch.empty(n, dtype=torch.float64).pin_memory()
del x, y, a
soe = soe_for_tolerance(1e-10); tr, ti, wr, wi, sc = soe.arrays()
sp = (tr.ctypes.data_as(PD), ti.ctypes.data_as(PD), wr.ctypes.data_as(PD), wi.ctypes.data_as(PD), sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), len(soe), 1)
for i in range(int(os.environ.get("REPS", "3"))):
    print("---", flush=True)
    _capi.check(L.fgt_transform_host(ctypes.cast(hx.data_ptr(), PD), n, ctypes.cast(hy.data_ptr(), PD), n,
                ctypes.cast(ha.data_ptr(), PD), 1e-3, *sp, ctypes.cast(hu.data_ptr(), PD), 0, sh))
PY
