"""Python host API of the transform path, mirroring the reference.

C++ reference (proj/include/fgt1d/transform.hpp)      here
  TransformRequest / TransformResult (:17-26)          TransformRequest / list of floats
  TransformPlan (:32-47)                               TransformPlan (device plan handle)
  plan(request, soe, precompute) (:53-54)              plan()
  precompute_gap_table(plan) (:58)                     precompute_gap_table()
  apply_same / apply_general (:65-75)                  apply_same() / apply_general()
  direct(request, subset) (:80-81)                     direct()
  preset_mode_count / preset_soe (:86-89)              soe.preset_mode_count / soe.preset_soe
  detail::mode_sums (:101-102)                         mode_sums()
Python binding (proj/bindings/pymodule.cpp)
  gauss_transform (:37-60, :151-155)                   gauss_transform()
  direct_transform (:62-72, :156-158)                  direct_transform()
  uniform_points (:159-161)                            uniform_points()

Every compute call goes through the C ABI (libfgt1d_b200.so) on the GPU.
"""
import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from .soe import SoeApprox, SoeForm, cf_soe, fold, validate

_PD = ctypes.POINTER(ctypes.c_double)
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PU8 = ctypes.POINTER(ctypes.c_uint8)


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))


def _ptr(a):
    return a.ctypes.data_as(_PD)


@dataclass
class TransformRequest:
    targets: list = field(default_factory=list)
    sources: list = field(default_factory=list)
    strengths: list = field(default_factory=list)
    delta: float = 1.0


class TransformPlan:
    """Device-resident plan: sorted copies, permutations, folded SOE, tile
    partition.  Reusable across strength vectors (transform.hpp:28-31)."""

    def __init__(self, handle, soe, delta, M, N):
        self._h = handle
        self.soe = soe
        self.delta = delta
        self._M, self._N = M, N
        self.precomputed = False
        self.gap_exponentials = []
        self._sorted = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _capi.lib().fgt_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def _info(self):
        M, N, ntiles = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        ne, same, ts, ss = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _capi.check(_capi.lib().fgt_plan_info(self._h, ctypes.byref(M), ctypes.byref(N),
                                              ctypes.byref(ne), ctypes.byref(same),
                                              ctypes.byref(ts), ctypes.byref(ss),
                                              ctypes.byref(ntiles)))
        return dict(M=M.value, N=N.value, n_modes=ne.value, same_points=bool(same.value),
                    targets_were_sorted=bool(ts.value), sources_were_sorted=bool(ss.value),
                    ntiles=ntiles.value)

    @property
    def same_points(self):
        return self._info()["same_points"]

    def _fetch_sorted(self):
        if self._sorted is None:
            sx = np.empty(self._M)
            sy = np.empty(self._N)
            tp = np.empty(self._M, dtype=np.int64)
            sp = np.empty(self._N, dtype=np.int64)
            _capi.check(_capi.lib().fgt_plan_copy_sorted(self._h, _ptr(sx), tp.ctypes.data_as(_PI64),
                                                         _ptr(sy), sp.ctypes.data_as(_PI64)))
            self._sorted = (sx, tp, sy, sp)
        return self._sorted

    @property
    def sorted_targets(self):
        return self._fetch_sorted()[0]

    @property
    def target_perm(self):
        return self._fetch_sorted()[1]

    @property
    def sorted_sources(self):
        return self._fetch_sorted()[2]

    @property
    def source_perm(self):
        return self._fetch_sorted()[3]


def _soe_args(soe):
    tr, ti, wr, wi, sc = soe.arrays()
    keep = (tr, ti, wr, wi, sc)
    return keep, (_ptr(tr), _ptr(ti), _ptr(wr), _ptr(wi), sc.ctypes.data_as(_PU8), len(soe),
                  int(soe.form))


def plan(request, soe, precompute=False):
    """fgt::plan (transform.cpp:200-219): validation order and error classes
    follow the reference (ValueError for domain / invalid-argument errors)."""
    x = _f64(request.targets)
    y = _f64(request.sources)
    a = _f64(request.strengths)
    delta = float(request.delta)
    if not (np.isfinite(delta) and delta > 0.0):
        raise ValueError("delta must be positive and finite")
    if not np.all(np.isfinite(x)):
        raise ValueError("target coordinates must be finite")
    if not np.all(np.isfinite(y)):
        raise ValueError("source coordinates must be finite")
    if a.size != y.size:
        raise ValueError("one strength per source required")
    validate(soe)
    folded = soe if soe.form == SoeForm.FOLDED else fold(soe)
    keep, sargs = _soe_args(folded)
    h = ctypes.c_void_p()
    _capi.check(_capi.lib().fgt_plan_create(_ptr(x), x.size, _ptr(y), y.size, delta, *sargs, 0, -1,
                                            None, ctypes.byref(h)))
    p = TransformPlan(h.value, folded, delta, x.size, y.size)
    if precompute:
        precompute_gap_table(p)
    return p


def precompute_gap_table(p):
    """transform.cpp:221-237 -- API parity only; the device path forms gap
    factors on the fly and never reads the table."""
    if p.precomputed:
        return
    M, ne = p._M, len(p.soe)
    if M >= 2 and ne > 0:
        out = np.empty(2 * ne * (M - 1))
        _capi.check(_capi.lib().fgt_plan_gap_table(p.handle, _ptr(out)))
        p.gap_exponentials = (out[0::2] + 1j * out[1::2]).tolist()
    p.precomputed = True


def _apply(p, strengths, threads, same):
    a = _f64(strengths)
    out = np.empty(p._M)
    fn = _capi.lib().fgt_apply_same if same else _capi.lib().fgt_apply_general
    _capi.check(fn(p.handle, _ptr(a), a.size, _ptr(out), int(threads), 0, None))
    return out


def apply_general(p, strengths, num_threads=1):
    return _apply(p, strengths, num_threads, False)


def apply_same(p, strengths, num_threads=1):
    return _apply(p, strengths, num_threads, True)


def direct(request, target_subset=None):
    """fgt::direct on the device (double-double accumulation)."""
    x, y, a = _f64(request.targets), _f64(request.sources), _f64(request.strengths)
    if a.size != y.size:
        raise ValueError("one strength per source required")
    sub = None if target_subset is None or len(target_subset) == 0 else np.ascontiguousarray(
        np.asarray(target_subset, dtype=np.int64))
    n = x.size if sub is None else sub.size
    out = np.empty(n)
    _capi.check(_capi.lib().fgt_direct(_ptr(x), x.size, _ptr(y), y.size, _ptr(a), float(request.delta),
                                       None if sub is None else sub.ctypes.data_as(_PI64),
                                       0 if sub is None else sub.size, _ptr(out)))
    return out


def mode_sums(p, strengths):
    """detail::mode_sums: (hp, hm) as complex arrays [n_modes][M], sorted-target order."""
    a = _f64(strengths)
    if a.size != p._N:
        raise ValueError("strengths length must match the planned source count")
    ne, M = len(p.soe), p._M
    hp = np.empty(2 * ne * M)
    hm = np.empty(2 * ne * M)
    _capi.check(_capi.lib().fgt_mode_sums(p.handle, _ptr(a), _ptr(hp), _ptr(hm)))
    return ((hp[0::2] + 1j * hp[1::2]).reshape(ne, M), (hm[0::2] + 1j * hm[1::2]).reshape(ne, M))


class BatchPlan:
    """B independent presorted transforms planned together (BASELINE cfg 5)."""

    def __init__(self, targets, sources, deltas, soe):
        self.t_off = np.concatenate([[0], np.cumsum([len(t) for t in targets])]).astype(np.int64)
        self.s_off = np.concatenate([[0], np.cumsum([len(s) for s in sources])]).astype(np.int64)
        x = _f64(np.concatenate([np.asarray(t, dtype=np.float64) for t in targets]) if targets else [])
        y = _f64(np.concatenate([np.asarray(v, dtype=np.float64) for v in sources]) if sources else [])
        d = _f64(deltas)
        if d.size != len(targets) or len(sources) != len(targets):
            raise ValueError("one delta, target set and source set per transform")
        folded = soe if soe.form == SoeForm.FOLDED else fold(soe)
        self.soe = folded
        self._keep, sargs = _soe_args(folded)
        h = ctypes.c_void_p()
        _capi.check(_capi.lib().fgt_batch_create(len(targets), _ptr(x), self.t_off.ctypes.data_as(_PI64),
                                                 _ptr(y), self.s_off.ctypes.data_as(_PI64), _ptr(d),
                                                 *sargs, 0, -1, None, ctypes.byref(h)))
        self._h = h.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _capi.lib().fgt_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def apply(self, strengths):
        a = _f64(np.concatenate([np.asarray(v, dtype=np.float64) for v in strengths]) if strengths else [])
        if a.size != self.s_off[-1]:
            raise ValueError("strengths must match the batch's sources")
        out = np.empty(int(self.t_off[-1]))
        _capi.check(_capi.lib().fgt_apply_general(self._h, _ptr(a), a.size, _ptr(out), 1, 0, None))
        return [out[self.t_off[b]:self.t_off[b + 1]] for b in range(len(self.t_off) - 1)]


def batch_transform(targets, sources, strengths, deltas, soe):
    """Independent transforms u_b = G_{delta_b}(x_b, y_b) alpha_b in one batched plan
    (each x_b, y_b sorted)."""
    return BatchPlan(targets, sources, deltas, soe).apply(strengths)


def _is_cuda_tensor(v):
    return type(v).__module__.startswith("torch") and getattr(v, "is_cuda", False)


def gauss_transform_device(targets, sources, strengths, delta, soe=None, ne=4):
    """Device-array entry: float64 CUDA tensors in, a CUDA
    tensor of potentials (original target order) out, on the current stream;
    nothing crosses PCIe.  Same validation and error classes as gauss_transform."""
    import torch
    x = targets.reshape(-1).to(torch.float64).contiguous()
    y = sources.reshape(-1).to(torch.float64).contiguous()
    a = strengths.reshape(-1).to(torch.float64).contiguous()
    if a.numel() != y.numel():
        raise ValueError("one strength per source required")
    use = (soe if soe.form == SoeForm.FOLDED else fold(soe)) if soe is not None else fold(
        cf_soe(2 * int(ne)))
    validate(use)
    keep, sargs = _soe_args(use)
    dev = x.device
    st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    fl = _capi.FGT_DEVICE_PTRS
    L = _capi.lib()
    h = ctypes.c_void_p()
    _capi.check(L.fgt_plan_create(ctypes.cast(x.data_ptr(), _PD), x.numel(),
                                  ctypes.cast(y.data_ptr(), _PD), y.numel(), float(delta), *sargs,
                                  fl, dev.index or 0, st, ctypes.byref(h)))
    try:
        u = torch.empty(x.numel(), dtype=torch.float64, device=dev)
        same = ctypes.c_int()
        _capi.check(L.fgt_plan_info(h, None, None, None, ctypes.byref(same), None, None, None))
        fn = L.fgt_apply_same if same.value else L.fgt_apply_general
        _capi.check(fn(h, ctypes.cast(a.data_ptr(), _PD), a.numel(), ctypes.cast(u.data_ptr(), _PD),
                       1, fl, st))
    finally:
        L.fgt_plan_destroy(h)
    del keep
    return u


def gauss_transform(targets, sources, strengths, delta, soe=None, ne=4, threads=1):
    """pymodule.cpp:37-60: plan(precompute) then apply_same / apply_general.
    CUDA tensors are transformed on the device (gauss_transform_device)."""
    if _is_cuda_tensor(targets):
        return gauss_transform_device(targets, sources, strengths, delta, soe, ne)
    use = (soe if soe.form == SoeForm.FOLDED else fold(soe)) if soe is not None else fold(
        cf_soe(2 * int(ne)))
    return transform_host(targets, sources, strengths, delta, use).tolist()


def transform_host(targets, sources, strengths, delta, soe):
    """One-shot transform of host arrays through fgt_transform_host: the
    plan -> apply_general result (apply_same agrees on identical sets), with
    the PCIe uploads / downloads overlapped for large presorted inputs.
    Validation order and error classes as plan() (transform.cpp:200-219)."""
    x = _f64(targets)
    y = _f64(sources)
    a = _f64(strengths)
    delta = float(delta)
    if not (np.isfinite(delta) and delta > 0.0):
        raise ValueError("delta must be positive and finite")
    if not np.all(np.isfinite(x)):
        raise ValueError("target coordinates must be finite")
    if not np.all(np.isfinite(y)):
        raise ValueError("source coordinates must be finite")
    if a.size != y.size:
        raise ValueError("one strength per source required")
    validate(soe)
    keep, sargs = _soe_args(soe)
    u = np.empty(x.size)
    _capi.check(_capi.lib().fgt_transform_host(_ptr(x), x.size, _ptr(y), y.size, _ptr(a), delta,
                                               *sargs, _ptr(u), -1, None))
    del keep
    return u


def direct_transform(targets, sources, strengths, delta):
    return direct(TransformRequest(targets, sources, strengths, delta)).tolist()


# -- counter RNG (rng.hpp:6-39, rng.cpp:7-29), vectorised ---------------------

_GOLD = np.uint64(0x9E3779B97F4A7C15)


def _mix64(z):
    with np.errstate(over="ignore"):
        z = z + _GOLD
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def counter_rand(seed, stream, i):
    with np.errstate(over="ignore"):
        base = _mix64(np.uint64(seed) ^ (np.uint64(stream) * np.uint64(0xA24BAED4963EE407)))
        return _mix64(base + np.asarray(i, dtype=np.uint64) * _GOLD)


def uniform_points_array(count, seed, stream=0, offset=0):
    i = np.arange(offset, offset + count, dtype=np.uint64)
    return (counter_rand(seed, stream, i) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def uniform_points(count, seed, stream=0):
    return uniform_points_array(count, seed, stream).tolist()


def chebyshev_points(count):
    """(1 + cos(pi (2i - 1) / (2 count))) / 2 for i = 1..count (rng.cpp:31-40)."""
    i = np.arange(1, int(count) + 1, dtype=np.float64)
    return ((1.0 + np.cos(3.14159265358979323846 * (2.0 * i - 1.0) / (2.0 * float(count)))) / 2.0)


def gen_points(dist, count, seed, stream):
    """fgt1d_cli.cpp:170-179: 'uniform' (counter RNG) or 'chebyshev' points."""
    if dist == "uniform":
        return uniform_points_array(count, seed, stream)
    if dist == "chebyshev":
        return chebyshev_points(count)
    raise ValueError(f"unknown distribution '{dist}' (expected uniform or chebyshev)")


def measure_error(request, potentials, seed):
    """Sampled relative error (fgt1d_cli.cpp:198-218, acceptance bench_error):
    100 target indices min(M-1, floor(u M)) from the eval-index stream, the
    direct sum at them (device, double-double), max |u - u_direct| / |u_direct|
    skipping |u_direct| < 1e-3 max|u_direct| (near-cancellation guard)."""
    M = len(request.targets)
    u = uniform_points_array(100, seed, K_STREAM_EVAL_INDICES)
    idx = np.minimum(M - 1, (u * M).astype(np.int64))
    ud = direct(request, idx)
    umax = np.max(np.abs(ud)) if ud.size else 0.0
    got = np.asarray(potentials)[idx]
    keep = np.abs(ud) >= 1e-3 * umax
    if not np.any(keep):
        return 0.0
    return float(np.max(np.abs(got[keep] - ud[keep]) / np.abs(ud[keep])))


def preset_for_ne(ne):
    """fgt1d_cli.cpp:181-195: precision presets for n_e = 3..6, otherwise
    fold(cf_soe(2 n_e)) for 1..7."""
    from .soe import preset_soe
    if 3 <= ne <= 6:
        return preset_soe(ne - 3)
    if 1 <= ne <= 7:
        return fold(cf_soe(2 * ne))
    raise ValueError("--ne must be between 1 and 7")


def delta_sweep(N, ne, deltas, seed=0, dist="uniform"):
    """fgt1d_cli.cpp:317-352: same-point transform of N points (strengths from
    the strengths stream) for each delta, error by measure_error.  Returns
    [{"delta": d, "error": e}, ...]."""
    if N < 1:
        raise ValueError("--N must be at least 1")
    for d in deltas:
        if not (d > 0.0 and np.isfinite(d)):
            raise ValueError("all --delta values must be positive")
    soe = preset_for_ne(int(ne))
    y = gen_points(dist, N, seed, K_STREAM_SOURCES)
    a = uniform_points_array(N, seed, K_STREAM_STRENGTHS)
    rows = []
    for d in deltas:
        req = TransformRequest(y, y, a, float(d))
        p = plan(req, soe, True)
        res = apply_same(p, a, 1)
        rows.append({"delta": float(d), "error": measure_error(req, res, seed)})
    return rows


K_STREAM_SOURCES = 0
K_STREAM_STRENGTHS = 1
K_STREAM_EVAL_INDICES = 2
K_STREAM_TARGETS = 3
