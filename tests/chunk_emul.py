"""Numpy emulation of the per-chunk device work (test infrastructure only):
the chunk aggregates and the chunk finish of fgt_apply_chunk_aggregate /
fgt_apply_chunk_finish, written directly from the merged-stream recurrences
(reference transform.cpp:119-149 restated; decay as transform.cpp:60-68)."""
import numpy as np


def decay(s, g):
    a = s.real * g
    return np.where(g == 0, 1.0 + 0j, np.where(a > 745.0, 0j, np.exp(-s * g)))


def merged(x, y, a):
    """Merged stream (sources before targets at equal coordinates)."""
    z = np.concatenate([y, x])
    kind = np.concatenate([np.zeros(y.size, int), np.ones(x.size, int)])
    b = np.concatenate([a, np.zeros(x.size)])
    order = np.lexsort((kind, z))
    return z[order], b[order], kind[order]


def chunk_aggregate(z, b, zprev, s):
    g = np.diff(np.concatenate([[zprev], z]))
    A, F, G, P = 1 + 0j, 0j, 0j, 1 + 0j
    for gi, bi in zip(g, b):
        d = decay(s, gi)
        F = d * F + bi
        P = P * d
        G = G + bi * P
    return P, F, G


def chunk_finish(z, b, kind, zprev, s, mw, cf, cb):
    g = np.diff(np.concatenate([[zprev], z]))
    d = decay(s, g)
    out = np.zeros(z.size)
    H = cf
    for i in range(z.size):
        H = d[i] * H + b[i]
        out[i] += (mw * H).real
    K = cb
    for i in reversed(range(z.size)):
        out[i] += (mw * K).real
        K = d[i] * (K + b[i])
    return out[kind == 1]
