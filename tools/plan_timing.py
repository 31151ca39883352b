"""Break down one step (plan create / apply / destroy) with host timers and
per-kernel device times (ncu launch list is taken separately)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_09825_b200 import _capi
from paper_1909_09825_b200.soe import soe_for_tolerance
PD = ctypes.POINTER(ctypes.c_double)
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
L = _capi.lib(); dev = torch.device("cuda", 0)
sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
def gen(sid, sort=True):
    raw = torch.empty(n, dtype=torch.float64, device=dev)
    _capi.check(L.fgt_uniform_points_device(raw.data_ptr(), n, 0, sid, 0, sh))
    if not sort: return raw
    out = torch.empty_like(raw); perm = torch.empty(n, dtype=torch.int32, device=dev)
    _capi.check(L.fgt_sort_device(raw.data_ptr(), n, out.data_ptr(), perm.data_ptr(), sh)); return out
x, y = gen(3), gen(0); a = gen(1, False) * 2 - 1; u = torch.empty(n, dtype=torch.float64, device=dev)
soe = soe_for_tolerance(1e-10); tr, ti, wr, wi, sc = soe.arrays()
sp = (tr.ctypes.data_as(PD), ti.ctypes.data_as(PD), wr.ctypes.data_as(PD), wi.ctypes.data_as(PD), sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), len(soe), 1)
fl = _capi.FGT_DEVICE_PTRS | _capi.FGT_BORROW
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = ctypes.c_void_p()
    _capi.check(L.fgt_plan_create(ctypes.cast(x.data_ptr(), PD), n, ctypes.cast(y.data_ptr(), PD), n, 1e-3, *sp, fl, 0, sh, ctypes.byref(h)))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    _capi.check(L.fgt_apply_general(h, ctypes.cast(a.data_ptr(), PD), n, ctypes.cast(u.data_ptr(), PD), 1, fl, sh))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    L.fgt_plan_destroy(h)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"plan {1e3*(t1-t0):.3f} ms  apply {1e3*(t2-t1):.3f} ms  destroy {1e3*(t3-t2):.3f} ms")
