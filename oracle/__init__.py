"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the SOE fast Gauss transform.

Two checkers, both CPU-only, used exclusively by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs (never by the product):

  * C restatement  (oracle/fgt_oracle.c -> oracle/_build/liboracle.so): the
    reference algorithm, operation for operation (proj/src/transform.cpp).
  * the reference itself (oracle/_ref/libfgt1d_ref.so, built from
    /root/reference/proj/src/{transform,soe,rng}.cpp by oracle/build_ref.sh),
    when it was built.

Parity pinning: tests/test_oracle.py checks the restatement against the
reference's golden potentials (proj/tests/test_transform.cpp:19-26) and
bit-for-bit against the reference library on seeded inputs.
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfgt1d_ref.so")
TABLE_DIR = os.path.join(os.path.dirname(HERE), "paper_1909_09825_b200", "data")

_PD = ctypes.POINTER(ctypes.c_double)
_PI64 = ctypes.POINTER(ctypes.c_int64)


def _p(a):
    return a.ctypes.data_as(_PD)


def _f(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = ctypes.CDLL(ORACLE_SO)
        L.oracle_transform.restype = ctypes.c_int
        L.oracle_transform.argtypes = [_PD, ctypes.c_int64, _PD, ctypes.c_int64, _PD, ctypes.c_double,
                                       _PD, _PD, _PD, _PD, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       _PD]
        L.oracle_direct.restype = ctypes.c_int
        L.oracle_direct.argtypes = [_PD, ctypes.c_int64, _PD, ctypes.c_int64, _PD, ctypes.c_double,
                                    _PI64, ctypes.c_int64, _PD]
        L.oracle_sort_with_perm.restype = None
        L.oracle_sort_with_perm.argtypes = [_PD, ctypes.c_int64, _PD, _PI64]
        L.oracle_mode_sums.restype = ctypes.c_int
        L.oracle_mode_sums.argtypes = [_PD, ctypes.c_int64, _PD, _PI64, ctypes.c_int64, _PD,
                                       ctypes.c_double, _PD, _PD, ctypes.c_int, _PD, _PD]
        L.oracle_gap_table.restype = None
        L.oracle_gap_table.argtypes = [_PD, ctypes.c_int64, ctypes.c_double, _PD, _PD, ctypes.c_int,
                                       _PD]
        L.oracle_counter_rand.restype = ctypes.c_uint64
        L.oracle_counter_rand.argtypes = [ctypes.c_uint64] * 3
        L.oracle_uniform01.restype = ctypes.c_double
        L.oracle_uniform01.argtypes = [ctypes.c_uint64] * 3
        _oracle = L
    return _oracle


def ref_available():
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise ImportError(f"{REF_SO} missing: run oracle/build_ref.sh (needs /root/reference)")
        L = ctypes.CDLL(REF_SO)
        L.fgt_ref_last_error.restype = ctypes.c_char_p
        L.fgt_ref_set_table_dir.argtypes = [ctypes.c_char_p]
        L.fgt_ref_transform.restype = ctypes.c_int
        L.fgt_ref_transform.argtypes = [_PD, ctypes.c_int64, _PD, ctypes.c_int64, _PD,
                                        ctypes.c_double, ctypes.c_int, _PD, _PD, _PD, _PD,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, _PD, _PD]
        L.fgt_ref_direct.restype = ctypes.c_int
        L.fgt_ref_direct.argtypes = [_PD, ctypes.c_int64, _PD, ctypes.c_int64, _PD,
                                     ctypes.c_double, _PI64, ctypes.c_int64, _PD]
        L.fgt_ref_plan.restype = ctypes.c_int
        L.fgt_ref_plan.argtypes = [_PD, ctypes.c_int64, _PD, ctypes.c_int64, _PD, ctypes.c_double,
                                   ctypes.c_int, _PD, _PI64, _PD, _PI64,
                                   ctypes.POINTER(ctypes.c_int)]
        L.fgt_ref_mode_sums.restype = ctypes.c_int
        L.fgt_ref_mode_sums.argtypes = [_PD, ctypes.c_int64, _PD, ctypes.c_int64, _PD,
                                        ctypes.c_double, ctypes.c_int, _PD, _PD]
        L.fgt_ref_max_error.restype = ctypes.c_int
        L.fgt_ref_max_error.argtypes = [ctypes.c_int, ctypes.c_int, _PD, _PD]
        L.fgt_ref_gap_table.restype = ctypes.c_int
        L.fgt_ref_gap_table.argtypes = [_PD, ctypes.c_int64, ctypes.c_double, ctypes.c_int, _PD]
        L.fgt_ref_uniform_points.restype = ctypes.c_int
        L.fgt_ref_uniform_points.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, _PD]
        L.fgt_ref_counter_rand.restype = ctypes.c_uint64
        L.fgt_ref_counter_rand.argtypes = [ctypes.c_uint64] * 3
        L.fgt_ref_set_table_dir(TABLE_DIR.encode())
        _ref = L
    return _ref


# ---- SOE tables (read from the committed text tables) -----------------------

def load_table(n):
    """Full-form CF table n as (t, w) complex arrays (proj/src/soe.cpp:250-337 format)."""
    with open(os.path.join(TABLE_DIR, f"cf_n{n}.soe")) as f:
        rows = [l.split() for l in f.read().splitlines()[1:] if l.strip()]
    v = np.array([[float(x) for x in r] for r in rows])
    return v[:, 0] + 1j * v[:, 1], v[:, 2] + 1j * v[:, 3]


def folded_table(n):
    """fold(cf_soe(n)) restated (soe.cpp:143-215): (t, mw) with mw = m_k w_k."""
    t, w = load_table(n)
    ent = []
    used = [False] * len(t)
    for k in range(len(t)):
        if used[k]:
            continue
        if abs(t[k].imag) <= 1e-12 * abs(t[k]):
            used[k] = True
            ent.append((complex(t[k].real, 0.0), complex(w[k].real, 0.0), 1.0))
            continue
        want = np.conj(t[k])
        for j in range(len(t)):
            if j != k and not used[j] and abs(t[j] - want) <= 1e-12 * abs(t[k]) and \
                    (t[j].imag > 0) != (t[k].imag > 0) and abs(t[j].imag) > 1e-12 * abs(t[j]):
                up, dn = (k, j) if t[k].imag > 0 else (j, k)
                used[k] = used[j] = True
                ent.append((0.5 * (t[up] + np.conj(t[dn])), 0.5 * (w[up] + np.conj(w[dn])), 2.0))
                break
    ent.sort(key=lambda e: (e[0].real, e[0].imag))
    tt = np.array([e[0] for e in ent])
    mw = np.array([e[2] * e[1] for e in ent])
    return tt, mw


# ---- oracle (C restatement) -------------------------------------------------

def transform(x, y, alpha, delta, ne=6, mode=2, threads=1, soe=None):
    """plan + apply (mode 0 general, 1 same, 2 auto), original order."""
    x, y, alpha = _f(x), _f(y), _f(alpha)
    t, mw = soe if soe is not None else folded_table(2 * ne)
    tr, ti = np.ascontiguousarray(t.real), np.ascontiguousarray(t.imag)
    mr, mi = np.ascontiguousarray(mw.real), np.ascontiguousarray(mw.imag)
    out = np.empty(x.size)
    rc = oracle_lib().oracle_transform(_p(x), x.size, _p(y), y.size, _p(alpha), float(delta),
                                       _p(tr), _p(ti), _p(mr), _p(mi), len(t), mode, threads,
                                       _p(out))
    if rc:
        raise ValueError(f"oracle_transform rc={rc}")
    return out


def direct(x, y, alpha, delta, subset=None):
    x, y, alpha = _f(x), _f(y), _f(alpha)
    sub = None if subset is None else np.ascontiguousarray(np.asarray(subset, dtype=np.int64))
    n = x.size if sub is None else sub.size
    out = np.empty(n)
    rc = oracle_lib().oracle_direct(_p(x), x.size, _p(y), y.size, _p(alpha), float(delta),
                                    None if sub is None else sub.ctypes.data_as(_PI64),
                                    0 if sub is None else sub.size, _p(out))
    if rc:
        raise ValueError("target subset index out of range")
    return out


def sort_with_perm(v):
    v = _f(v)
    s = np.empty(v.size)
    p = np.empty(v.size, dtype=np.int64)
    oracle_lib().oracle_sort_with_perm(_p(v), v.size, _p(s), p.ctypes.data_as(_PI64))
    return s, p


def mode_sums(x, y, alpha, delta, ne):
    """(hp, hm) [ne][M] at sorted targets, like detail::mode_sums."""
    xs, _ = sort_with_perm(x)
    ys, sp = sort_with_perm(y)
    a = _f(alpha)
    t, _mw = folded_table(2 * ne)
    tr, ti = np.ascontiguousarray(t.real), np.ascontiguousarray(t.imag)
    hp = np.empty(2 * ne * xs.size)
    hm = np.empty(2 * ne * xs.size)
    oracle_lib().oracle_mode_sums(_p(xs), xs.size, _p(ys), sp.ctypes.data_as(_PI64), ys.size, _p(a),
                                  float(delta), _p(tr), _p(ti), ne, _p(hp), _p(hm))
    return ((hp[0::2] + 1j * hp[1::2]).reshape(ne, -1), (hm[0::2] + 1j * hm[1::2]).reshape(ne, -1))


# ---- the reference library itself -------------------------------------------

def ref_transform(x, y, alpha, delta, ne=6, mode=2, threads=1, precompute=True):
    """Reference plan -> precompute_gap_table -> apply; returns (u, (t_sort, t_pre, t_rem))."""
    L = ref_lib()
    x, y, alpha = _f(x), _f(y), _f(alpha)
    out = np.empty(x.size)
    times = np.zeros(3)
    rc = L.fgt_ref_transform(_p(x), x.size, _p(y), y.size, _p(alpha), float(delta), ne, None, None,
                             None, None, 0, 0, mode, threads, 1 if precompute else 0, _p(out),
                             _p(times))
    if rc:
        raise ValueError(L.fgt_ref_last_error().decode())
    return out, tuple(times)


def ref_direct(x, y, alpha, delta, subset=None):
    L = ref_lib()
    x, y, alpha = _f(x), _f(y), _f(alpha)
    sub = None if subset is None else np.ascontiguousarray(np.asarray(subset, dtype=np.int64))
    n = x.size if sub is None else sub.size
    out = np.empty(n)
    rc = L.fgt_ref_direct(_p(x), x.size, _p(y), y.size, _p(alpha), float(delta),
                          None if sub is None else sub.ctypes.data_as(_PI64),
                          0 if sub is None else sub.size, _p(out))
    if rc:
        raise ValueError(L.fgt_ref_last_error().decode())
    return out


def ref_plan(x, y, alpha, delta, ne=4):
    L = ref_lib()
    x, y, alpha = _f(x), _f(y), _f(alpha)
    sx, sy = np.empty(x.size), np.empty(y.size)
    tp, sp = np.empty(x.size, dtype=np.int64), np.empty(y.size, dtype=np.int64)
    same = ctypes.c_int()
    rc = L.fgt_ref_plan(_p(x), x.size, _p(y), y.size, _p(alpha), float(delta), ne, _p(sx),
                        tp.ctypes.data_as(_PI64), _p(sy), sp.ctypes.data_as(_PI64),
                        ctypes.byref(same))
    if rc:
        raise ValueError(L.fgt_ref_last_error().decode())
    return sx, tp, sy, sp, bool(same.value)


def ref_mode_sums(x, y, alpha, delta, ne):
    L = ref_lib()
    x, y, alpha = _f(x), _f(y), _f(alpha)
    hp = np.empty(2 * ne * x.size)
    hm = np.empty(2 * ne * x.size)
    rc = L.fgt_ref_mode_sums(_p(x), x.size, _p(y), y.size, _p(alpha), float(delta), ne, _p(hp),
                             _p(hm))
    if rc:
        raise ValueError(L.fgt_ref_last_error().decode())
    return ((hp[0::2] + 1j * hp[1::2]).reshape(ne, -1), (hm[0::2] + 1j * hm[1::2]).reshape(ne, -1))


def ref_max_error(n, fold_it=False):
    L = ref_lib()
    e, a = ctypes.c_double(), ctypes.c_double()
    rc = L.fgt_ref_max_error(n, 1 if fold_it else 0, ctypes.byref(e), ctypes.byref(a))
    if rc:
        raise ValueError(L.fgt_ref_last_error().decode())
    return e.value, a.value


def ref_gap_table(x, delta, ne):
    """The reference's precompute_gap_table for targets x (mode-major, complex)."""
    L = ref_lib()
    x = _f(x)
    out = np.empty(2 * ne * max(x.size - 1, 0))
    rc = L.fgt_ref_gap_table(_p(x), x.size, float(delta), ne, _p(out))
    if rc:
        raise ValueError(L.fgt_ref_last_error().decode())
    return out[0::2] + 1j * out[1::2]


def ref_uniform_points(count, seed, stream):
    """rng::uniform_points of the reference library."""
    L = ref_lib()
    out = np.empty(int(count))
    rc = L.fgt_ref_uniform_points(int(count), int(seed), int(stream), _p(out))
    if rc:
        raise ValueError(L.fgt_ref_last_error().decode())
    return out


def gap_table(xs_sorted, delta, ne):
    """C restatement of precompute_gap_table on sorted targets (complex)."""
    xs = _f(xs_sorted)
    t, _mw = folded_table(2 * ne)
    tr, ti = np.ascontiguousarray(t.real), np.ascontiguousarray(t.imag)
    out = np.empty(2 * ne * max(xs.size - 1, 0))
    oracle_lib().oracle_gap_table(_p(xs), xs.size, float(delta), _p(tr), _p(ti), len(t), _p(out))
    return out[0::2] + 1j * out[1::2]
