"""Wall time of fgt_batch_create / fgt_plan_destroy on the cfg 5 shape (the
create call ends with a stream synchronize, so wall = host + device time)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1909_09825_b200 import _capi  # noqa: E402
from paper_1909_09825_b200.soe import soe_for_tolerance  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
n = 65536
L = _capi.lib()
dev = torch.device("cuda", 0)
PD = ctypes.POINTER(ctypes.c_double)
PI64 = ctypes.POINTER(ctypes.c_int64)
x = torch.sort(torch.rand(B, n, dtype=torch.float64, device=dev), dim=1).values.contiguous()
y = torch.sort(torch.rand(B, n, dtype=torch.float64, device=dev), dim=1).values.contiguous()
off = np.arange(B + 1, dtype=np.int64) * n
deltas = np.ascontiguousarray(10.0 ** np.random.default_rng(0).uniform(-6, -1, B))
soe = soe_for_tolerance(1e-10)
tr, ti, wr, wi, sc = soe.arrays()
sp = (tr.ctypes.data_as(PD), ti.ctypes.data_as(PD), wr.ctypes.data_as(PD), wi.ctypes.data_as(PD),
      sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), len(soe), 1)
sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
fl = _capi.FGT_DEVICE_PTRS | _capi.FGT_BORROW
tc, td = [], []
for it in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = ctypes.c_void_p()
    _capi.check(L.fgt_batch_create(B, ctypes.cast(x.data_ptr(), PD), off.ctypes.data_as(PI64),
                                   ctypes.cast(y.data_ptr(), PD), off.ctypes.data_as(PI64),
                                   deltas.ctypes.data_as(PD), *sp, fl, 0, sh, ctypes.byref(h)))
    t1 = time.perf_counter()
    L.fgt_plan_destroy(h)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    tc.append(1e3 * (t1 - t0))
    td.append(1e3 * (t2 - t1))
print("create ms", [round(v, 3) for v in tc])
print("destroy ms", [round(v, 3) for v in td])
