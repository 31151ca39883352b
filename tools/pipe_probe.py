"""Probe of the host-link pipeline (GPU box): pure upload time of the cfg-3
inputs, upload with a concurrent download (duplex), and fgt_transform_host
with phase stamps (FGT_PIPE_TRACE) for a few chunk sizes."""
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
    return raw.sort().values if sort else raw
x, y = gen(3), gen(0); a = gen(1, False) * 2 - 1
hx, hy, ha = x.cpu().pin_memory(), y.cpu().pin_memory(), a.cpu().pin_memory()
hu = torch.empty(n, dtype=torch.float64).pin_memory()
d = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(4)]
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
def up_all():
    with torch.cuda.stream(s_in):
        for k, h in enumerate((hy, ha, hx)):
            d[k].copy_(h, non_blocking=True)
def run(f, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts)
print("upload 3 arrays          %.2f ms" % run(up_all), flush=True)
def duplex():
    up_all()
    with torch.cuda.stream(s_out):
        hu.copy_(d[3], non_blocking=True)
print("upload + download 1 arr  %.2f ms" % run(duplex), flush=True)
def down():
    with torch.cuda.stream(s_out):
        hu.copy_(d[3], non_blocking=True)
print("download 1 array         %.2f ms" % run(down), flush=True)
del d
soe = soe_for_tolerance(1e-10); tr, ti, wr, wi, sc = soe.arrays()
sp = (tr.ctypes.data_as(PD), ti.ctypes.data_as(PD), wr.ctypes.data_as(PD), wi.ctypes.data_as(PD), sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), len(soe), 1)
os.environ["FGT_PIPE_TRACE"] = "0"
for chunk in (6250000, 12500000, 25000000, 50000000):
    os.environ["FGT_PIPE_CHUNK"] = str(chunk)
    def tr_():
        _capi.check(L.fgt_transform_host(ctypes.cast(hx.data_ptr(), PD), n, ctypes.cast(hy.data_ptr(), PD), n,
                    ctypes.cast(ha.data_ptr(), PD), 1e-3, *sp, ctypes.cast(hu.data_ptr(), PD), 0, sh))
    print(f"transform_host chunk={chunk}: %.2f ms" % run(tr_), flush=True)
