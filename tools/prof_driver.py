"""Small driver for ncu captures: one presorted cfg3-shaped transform (N=M=n)."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1909_09825_b200 import _capi  # noqa: E402
from paper_1909_09825_b200.soe import soe_for_tolerance  # noqa: E402

PD = ctypes.POINTER(ctypes.c_double)
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=1e7)
ap.add_argument("--delta", type=float, default=1e-3)
ap.add_argument("--tol", type=float, default=1e-10)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
n = int(args.n)
L = _capi.lib()
dev = torch.device("cuda", 0)
sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def gen(stream_id, sort=True):
    raw = torch.empty(n, dtype=torch.float64, device=dev)
    _capi.check(L.fgt_uniform_points_device(raw.data_ptr(), n, 0, stream_id, 0, sh))
    if not sort:
        return raw
    out = torch.empty_like(raw)
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    _capi.check(L.fgt_sort_device(raw.data_ptr(), n, out.data_ptr(), perm.data_ptr(), sh))
    return out


x, y = gen(3), gen(0)
a = gen(1, sort=False) * 2.0 - 1.0
u = torch.empty(n, dtype=torch.float64, device=dev)
soe = soe_for_tolerance(args.tol)
tr, ti, wr, wi, sc = soe.arrays()
sp = (tr.ctypes.data_as(PD), ti.ctypes.data_as(PD), wr.ctypes.data_as(PD), wi.ctypes.data_as(PD),
      sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), len(soe), 1)
flags = _capi.FGT_DEVICE_PTRS | _capi.FGT_BORROW
for _ in range(args.reps):
    h = ctypes.c_void_p()
    _capi.check(L.fgt_plan_create(ctypes.cast(x.data_ptr(), PD), n, ctypes.cast(y.data_ptr(), PD),
                                  n, args.delta, *sp, flags, 0, sh, ctypes.byref(h)))
    _capi.check(L.fgt_apply_general(h, ctypes.cast(a.data_ptr(), PD), n, ctypes.cast(u.data_ptr(), PD),
                                    1, flags, sh))
    L.fgt_plan_destroy(h)
torch.cuda.synchronize()
print("ok", float(u[:4].sum()))
