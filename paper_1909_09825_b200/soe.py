"""SOE representation for the Python host API.

Mirrors the reference's SoeApprox (proj/include/fgt1d/soe.hpp:24-39) and the
pieces of proj/src/soe.cpp the transform path touches: validate (:107-132),
fold / unfold (:143-235), evaluate (:100-105), and the coefficient-table text
format (:250-337).  Table data comes from the compiled-in CF tables of the C
ABI (fgt_cf_soe), i.e. "SOE node/weight table lookup by tolerance".
"""
import ctypes
from dataclasses import dataclass
import enum
import math

import numpy as np

from . import _capi


class SoeForm(enum.IntEnum):
    FULL = _capi.FGT_SOE_FULL
    FOLDED = _capi.FGT_SOE_FOLDED


class SoeApprox:
    """nodes t_k (Re > 0), weights w_k, form, self_conjugate flags (folded)."""

    def __init__(self, nodes=(), weights=(), form=SoeForm.FULL, self_conjugate=()):
        self.nodes = [complex(t) for t in nodes]
        self.weights = [complex(w) for w in weights]
        self.form = SoeForm(form)
        self.self_conjugate = [int(b) for b in self_conjugate]

    def __len__(self):
        return len(self.nodes)

    def multiplier(self, k):
        if self.form == SoeForm.FULL:
            return 1.0
        return 1.0 if self.self_conjugate[k] else 2.0

    def __repr__(self):
        return f"SoeApprox(n={len(self)}, form={'full' if self.form == SoeForm.FULL else 'folded'})"

    def arrays(self):
        n = len(self)
        t = np.array(self.nodes, dtype=complex).reshape(n)
        w = np.array(self.weights, dtype=complex).reshape(n)
        sc = np.array(self.self_conjugate if self.form == SoeForm.FOLDED else [0] * n,
                      dtype=np.uint8).reshape(n)
        return (np.ascontiguousarray(t.real), np.ascontiguousarray(t.imag),
                np.ascontiguousarray(w.real), np.ascontiguousarray(w.imag), sc)


def validate(soe):
    """soe.cpp:107-132 (ValueError == std::invalid_argument in the binding)."""
    if len(soe.nodes) != len(soe.weights):
        raise ValueError("SOE node/weight count mismatch")
    if soe.form == SoeForm.FOLDED:
        if len(soe.self_conjugate) != len(soe.nodes):
            raise ValueError("folded SOE requires one self-conjugate flag per node")
    elif soe.self_conjugate:
        raise ValueError("full-form SOE must not carry fold flags")
    for k, (t, w) in enumerate(zip(soe.nodes, soe.weights)):
        if not (math.isfinite(t.real) and math.isfinite(t.imag) and math.isfinite(w.real)
                and math.isfinite(w.imag)):
            raise ValueError("SOE coefficients must be finite")
        if not t.real > 0.0:
            raise ValueError("SOE nodes must lie in the open right half-plane")
        if soe.form == SoeForm.FOLDED:
            if t.imag < 0.0:
                raise ValueError("folded SOE stores the Im(t) >= 0 representative of each pair")
            if soe.self_conjugate[k] and t.imag != 0.0:
                raise ValueError("self-conjugate folded node must have a real t")


def _from_capi(n, folded):
    L = _capi.lib()
    cnt = n if not folded else (n + 1) // 2
    buf = [np.zeros(cnt) for _ in range(4)]
    sc = np.zeros(cnt, dtype=np.uint8)
    ptrs = [b.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for b in buf]
    got = L.fgt_cf_soe(n, 1 if folded else 0, *ptrs, sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
    if got < 0:
        _capi.check(-got)
    t = buf[0][:got] + 1j * buf[1][:got]
    w = buf[2][:got] + 1j * buf[3][:got]
    if folded:
        return SoeApprox(t, w, SoeForm.FOLDED, sc[:got].tolist())
    return SoeApprox(t, w, SoeForm.FULL)


def cf_soe(n):
    """Near-best rational SOE of order n (2..14), full form (cf.hpp:34)."""
    return _from_capi(int(n), False)


def fold(soe):
    """soe.cpp:143-215."""
    validate(soe)
    if soe.form == SoeForm.FOLDED:
        return soe
    n = len(soe)
    kind = []
    for k in range(n):
        t, w = soe.nodes[k], soe.weights[k]
        if abs(t.imag) <= 1e-12 * abs(t):
            if abs(w.imag) > 1e-9 * (1.0 + abs(w)):
                raise ValueError(f"fold: real node {k} carries a non-real weight; the sum cannot "
                                 "be real-valued")
            kind.append(0)
        else:
            kind.append(1 if t.imag > 0.0 else -1)
    used = [False] * n
    ent, flags = [], []
    for k in range(n):
        if used[k]:
            continue
        if kind[k] == 0:
            used[k] = True
            ent.append((complex(soe.nodes[k].real, 0.0), complex(soe.weights[k].real, 0.0)))
            flags.append(1)
            continue
        want = soe.nodes[k].conjugate()
        tol = 1e-12 * abs(soe.nodes[k])
        match = None
        for j in range(n):
            if j == k or used[j] or kind[j] == 0 or kind[j] == kind[k]:
                continue
            if abs(soe.nodes[j] - want) <= tol:
                match = j
                break
        if match is None:
            raise ValueError(f"fold: node {k} has no conjugate partner")
        used[k] = used[match] = True
        up, dn = (k, match) if kind[k] > 0 else (match, k)
        ent.append((0.5 * (soe.nodes[up] + soe.nodes[dn].conjugate()),
                    0.5 * (soe.weights[up] + soe.weights[dn].conjugate())))
        flags.append(0)
    order = sorted(range(len(ent)), key=lambda i: (ent[i][0].real, ent[i][0].imag))
    return SoeApprox([ent[i][0] for i in order], [ent[i][1] for i in order], SoeForm.FOLDED,
                     [flags[i] for i in order])


def unfold(soe):
    """soe.cpp:217-235."""
    validate(soe)
    if soe.form == SoeForm.FULL:
        return soe
    ent = []
    for k in range(len(soe)):
        ent.append((soe.nodes[k], soe.weights[k]))
        if not soe.self_conjugate[k]:
            ent.append((soe.nodes[k].conjugate(), soe.weights[k].conjugate()))
    ent.sort(key=lambda e: (e[0].real, e[0].imag))
    return SoeApprox([e[0] for e in ent], [e[1] for e in ent], SoeForm.FULL)


def evaluate(soe, x, delta):
    """S(x; delta) = Re sum_k m_k w_k exp(-t_k |x| / sqrt(delta)) (soe.cpp:100-105)."""
    validate(soe)
    if not math.isfinite(x):
        raise ValueError("evaluate: x must be finite")
    if not (math.isfinite(delta) and delta > 0.0):
        raise ValueError("evaluate: delta must be positive and finite")
    s = abs(x) / math.sqrt(delta)
    acc = 0j
    for k in range(len(soe)):
        t = soe.nodes[k]
        if t.real * s > 745.0:
            continue
        acc += soe.multiplier(k) * soe.weights[k] * complex(np.exp(-t * s))
    return acc.real


# -- SOE error on the standard grid (soe.cpp:38-101, 236-248) ----------------

ERROR_GRID_LOG_POINTS = 100000  # soe.hpp kErrorGridLogPoints


def error_grid_point(i):
    """0 for i <= 0, else 10^(-5 + 7 (i-1)/(kErrorGridLogPoints-1)) (soe.cpp:236-240)."""
    if i <= 0:
        return 0.0
    return 10.0 ** (-5.0 + 7.0 * (i - 1) / (ERROR_GRID_LOG_POINTS - 1))


@dataclass
class ErrorReport:
    n: int                 # exponentials (folded pairs count 2)
    max_abs_error: float   # max |exp(-x^2/4) - S(x)| over the grid
    argmax_x: float        # grid point attaining it (smallest on ties)


def _max_error(soe, real, cplx):
    validate(soe)
    i = np.arange(1, ERROR_GRID_LOG_POINTS + 1, dtype=np.float64)
    x = np.concatenate([[0.0], 10.0 ** (-5.0 + 7.0 * (i - 1) / (ERROR_GRID_LOG_POINTS - 1))])
    s = x.astype(real)
    acc = np.zeros(x.size, dtype=cplx)
    for k in range(len(soe)):  # mode order as eval_sum (soe.cpp:22-35)
        t = cplx(soe.nodes[k])
        w = cplx(soe.weights[k])
        keep = real(t.real) * s <= real(745.0)
        term = real(soe.multiplier(k)) * w * np.exp(-t * s)
        acc += np.where(keep, term, cplx(0))
    g = np.exp(-s * s / real(4))
    e = np.abs(g - acc.real).astype(np.float64)
    j = int(np.argmax(e))  # first maximum: ties keep the smaller x
    n = int(sum(soe.multiplier(k) for k in range(len(soe))))
    return ErrorReport(n, float(e[j]), float(x[j]))


def max_error(soe):
    """fgt::max_error (soe.hpp:76): double accumulation."""
    return _max_error(soe, np.float64, np.complex128)


def max_error_extended(soe):
    """fgt::max_error_extended (soe.hpp:78-81): long-double accumulation."""
    return _max_error(soe, np.longdouble, np.clongdouble)


def preset_mode_count(p):
    """Precision preset (transform.hpp:86-89) -> n_e."""
    r = _capi.lib().fgt_preset_mode_count(int(p))
    if r < 0:
        _capi.check(-r)
    return r


def preset_soe(p):
    """fold(cf_soe(2 n_e)) (transform.cpp:304-306)."""
    return _from_capi(2 * preset_mode_count(p), True)


def mode_count_for_tolerance(tol):
    r = _capi.lib().fgt_mode_count_for_tolerance(float(tol))
    if r < 0:
        _capi.check(-r)
    return r


def soe_for_tolerance(tol):
    """Table lookup by tolerance (north_star): folded CF SOE with the fewest modes
    whose documented transform error is <= tol."""
    return _from_capi(2 * mode_count_for_tolerance(tol), True)


# -- coefficient tables (soe.cpp:250-337) -----------------------------------

def write_coefficient_table(f, soe, source_tag=""):
    validate(soe)
    f.write(f"soe n={len(soe)} form={'folded' if soe.form == SoeForm.FOLDED else 'full'}")
    if source_tag:
        f.write(f" source={source_tag}")
    f.write("\n")
    for t, w in zip(soe.nodes, soe.weights):
        f.write("%.16e %.16e %.16e %.16e\n" % (t.real, t.imag, w.real, w.imag))


def read_coefficient_table(f):
    header = f.readline()
    if not header:
        raise ValueError("coefficient table: empty input")
    toks = header.split()
    if not toks or toks[0] != "soe":
        raise ValueError("coefficient table: header must start with 'soe'")
    n, form = -1, ""
    for kv in toks[1:]:
        if "=" not in kv:
            raise ValueError(f"coefficient table: malformed header field '{kv}'")
        k, v = kv.split("=", 1)
        if k == "n":
            try:
                n = int(v)
            except ValueError:
                raise ValueError("coefficient table: bad n value")
        elif k == "form":
            form = v
    if n < 0:
        raise ValueError("coefficient table: missing n")
    if form not in ("full", "folded"):
        raise ValueError("coefficient table: missing or bad form")
    out = SoeApprox(form=SoeForm.FOLDED if form == "folded" else SoeForm.FULL)
    for line in f:
        if not line.strip():
            continue
        parts = line.split()
        try:
            tr, ti, wr, wi = (float(p) for p in parts[:4])
            if len(parts) < 4:
                raise ValueError
        except ValueError:
            raise ValueError(f"coefficient table: malformed row '{line.rstrip()}'")
        out.nodes.append(complex(tr, ti))
        out.weights.append(complex(wr, wi))
        if out.form == SoeForm.FOLDED:
            if ti < 0.0:
                raise ValueError("coefficient table: folded rows must have Im(t) >= 0")
            out.self_conjugate.append(1 if ti == 0.0 else 0)
    if len(out) != n:
        raise ValueError("coefficient table: row count does not match header n")
    validate(out)
    return out


def save_coefficient_table(path, soe, source_tag="python"):
    with open(path, "w") as f:
        write_coefficient_table(f, soe, source_tag)


def load_coefficient_table(path):
    try:
        f = open(path)
    except OSError:
        raise ValueError(f"cannot open for reading: {path}")
    with f:
        return read_coefficient_table(f)
