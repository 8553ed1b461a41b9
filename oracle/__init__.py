"""CPU oracle for the colour-coding hot path (TEST INFRASTRUCTURE ONLY).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  The product package
`paper_1804_09764_b200` never imports it and shares no code with it.

Thin ctypes wrapper over `oracle/oracle.c` (plain C + OpenMP); see that file's
header for what each function computes and which PAPER.md passage it follows.
Parity status of each function is listed in DESIGN.md section "Oracle pins".
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRCS = [os.path.join(_HERE, "oracle.c"), os.path.join(_HERE, "dp_body.inc"), os.path.join(_HERE, "dp_root_body.inc")]

NUM_EXACT, NUM_LONGDOUBLE, NUM_DOUBLE = 0, 1, 2


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    newest = max(os.path.getmtime(s) for s in _SRCS)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fopenmp", "-fPIC", "-shared",
                               "-o", _SO + ".tmp", _SRCS[0], "-lm"])
        os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        lib.or_mix.restype = u64
        lib.or_mix.argtypes = [u64]
        lib.or_color.argtypes = [i64, i32, u64, vp]
        lib.or_brute_count.restype = ctypes.c_int
        lib.or_brute_count.argtypes = [i64, vp, vp, i32, vp, vp, i32, vp, vp]
        lib.or_aut.restype = ctypes.c_int
        lib.or_aut.argtypes = [i32, vp, vp]
        lib.or_combine_row.restype = ctypes.c_int
        lib.or_combine_row.argtypes = [i32, i32, i32, vp, vp, vp]
        lib.or_dp_count.restype = ctypes.c_int
        lib.or_dp_count.argtypes = [i64, vp, vp, i32, vp, vp, i32, i32, vp, vp, vp, vp, vp]
        lib.or_dp_count_kc.restype = ctypes.c_int
        lib.or_dp_count_kc.argtypes = [i64, vp, vp, i32, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp]
        lib.or_dp_root_at.restype = ctypes.c_int
        lib.or_dp_root_at.argtypes = [i64, vp, vp, i32, vp, vp, i32, i64, vp, vp, vp]
        lib.or_estimate.restype = ctypes.c_double
        lib.or_estimate.argtypes = [i32, vp, i32, u64]
        lib.or_mom.restype = ctypes.c_double
        lib.or_mom.argtypes = [i32, vp, i32, u64, i32]
        lib.or_niter.restype = ctypes.c_int64
        lib.or_niter.argtypes = [ctypes.c_double, ctypes.c_double, i32, ctypes.c_double]
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data if a is not None and a.size else None


def _parent(parent):
    return np.ascontiguousarray(parent, dtype=np.int32)


def mix(x: int) -> int:
    """SplitMix64 finaliser (reading C-2)."""
    return int(_load().or_mix(x & 0xFFFFFFFFFFFFFFFF))


def color(n: int, k: int, seed: int) -> np.ndarray:
    """col(seed, v) = ((mix(mix(seed) ^ v) >> 32) * k) >> 32, v = original vertex id (reading C-2)."""
    out = np.empty(max(n, 1), dtype=np.uint8)[:n]
    if n:
        _load().or_color(n, k, seed & 0xFFFFFFFFFFFFFFFF, out.ctypes.data)
    return out


def brute_count(g, parent, colors=None) -> int:
    """Exact count of maps of the definition (105-108): colourful maps
    if `colors` is given, else all injective edge-preserving maps."""
    par = _parent(parent)
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    col = None if colors is None else np.ascontiguousarray(colors, dtype=np.uint8)
    rc = _load().or_brute_count(g.n, _ptr(g.row_ptr), _ptr(g.col), len(par), par.ctypes.data,
                                _ptr(col), 1 if col is not None else 0,
                                ctypes.byref(lo), ctypes.byref(hi))
    if rc:
        raise OracleError(f"or_brute_count rc={rc}")
    return (hi.value << 64) | lo.value


def aut(parent) -> int:
    """|Aut(T)| as the number of injective edge-preserving maps T -> T."""
    par = _parent(parent)
    out = ctypes.c_uint64()
    rc = _load().or_aut(len(par), par.ctypes.data, ctypes.byref(out))
    if rc:
        raise OracleError(f"or_aut rc={rc}")
    return out.value


def combine_row(k: int, a: int, p: int, A, N) -> np.ndarray:
    """T(S u Y) = sum A(S) N(Y) over disjoint S, Y (Eq. 1's split sum), colex-indexed rows."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    N = np.ascontiguousarray(N, dtype=np.float64)
    T = np.zeros(math.comb(k, a + p), dtype=np.float64)
    assert A.size == math.comb(k, a) and N.size == math.comb(k, p)
    rc = _load().or_combine_row(k, a, p, A.ctypes.data, N.ctypes.data, T.ctypes.data)
    if rc:
        raise OracleError(f"or_combine_row rc={rc}")
    return T


def subtree_sizes(parent):
    k = len(parent)
    size = [1] * k
    # parent indices may be larger than the child's; walk up from every vertex
    for v in range(k):
        p = parent[v]
        while p >= 0:
            size[p] += 1
            p = parent[p]
    return size


class DPResult:
    def __init__(self, total, exact, table, root):
        self.total = total      # int (exact) or float
        self.exact = exact
        self.table = table      # np.ndarray n x C(k, s_x) or None
        self.root = root        # np.ndarray n or None


def dp_count(g, parent, colors, numtype=NUM_EXACT, keep_x=-1, want_root=False, colours=None) -> DPResult:
    """The fold-children DP of Eq. 1 with d = 1; returns X = sum_v D_root(v,[k]).
    colours (>= k, default k): a colouring with more colours than template
    vertices: tables over the colours-universe, X sums the root
    table over every colour set of size k."""
    par = _parent(parent)
    k = len(par)
    kc = k if colours is None else int(colours)
    col = np.ascontiguousarray(colors, dtype=np.uint8)
    assert col.size == g.n
    table = None
    if keep_x >= 0:
        s = subtree_sizes(list(par))[keep_x]
        table = np.zeros((g.n, math.comb(kc, s)), dtype=np.float64)
    root = np.zeros(g.n, dtype=np.float64) if want_root else None
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    ld = ctypes.c_longdouble()
    rc = _load().or_dp_count_kc(g.n, _ptr(g.row_ptr), _ptr(g.col), k, par.ctypes.data, _ptr(col), kc,
                                numtype, keep_x, _ptr(table), _ptr(root), ctypes.byref(lo),
                                ctypes.byref(hi), ctypes.byref(ld))
    if rc == 2:
        raise OverflowError("oracle DP overflowed the exact u128 type")
    if rc:
        raise OracleError(f"or_dp_count rc={rc}")
    if numtype == NUM_EXACT:
        return DPResult((hi.value << 64) | lo.value, True, table, root)
    return DPResult(float(ld.value), False, table, root)


def dp_root_at(g, parent, colors, v0: int, numtype=NUM_EXACT):
    """D_root(v0, [k]): the DP's per-vertex root count at ONE vertex (each
    template vertex's table evaluated only within its depth of v0)."""
    par = _parent(parent)
    k = len(par)
    col = np.ascontiguousarray(colors, dtype=np.uint8)
    assert col.size == g.n
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    ld = ctypes.c_longdouble()
    rc = _load().or_dp_root_at(g.n, _ptr(g.row_ptr), _ptr(g.col), k, par.ctypes.data, _ptr(col), numtype, int(v0),
                               ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(ld))
    if rc == 2:
        raise OverflowError("oracle DP overflowed the exact u128 type")
    if rc:
        raise OracleError(f"or_dp_root_at rc={rc}")
    return (hi.value << 64) | lo.value if numtype == NUM_EXACT else float(ld.value)


def estimate(X, k: int, aut_t: int) -> float:
    """mean_j X_j * k^k/k! / |Aut(T)| (readings C-1, C-10)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    return float(_load().or_estimate(len(X), X.ctypes.data, k, aut_t))


def median_of_means(X, k: int, aut_t: int, t: int) -> float:
    """Median of t group means of C_j = X_j k^k/k!/|Aut(T)| (Alg. 1 last line; SPEC.md 455-463)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    r = _load().or_mom(len(X), X.ctypes.data, k, aut_t, t)
    if r < 0:
        raise OracleError("median_of_means: need 1 <= t <= len(X)")
    return float(r)


def niter(eps: float, delta: float, k: int, c: float = 1.0) -> int:
    """Niter = ceil(c e^k ln(1/delta) / eps^2), >= 1 (Alg. 1 line 3)."""
    r = int(_load().or_niter(eps, delta, k, c))
    if r < 0:
        raise OracleError("niter: need eps > 0, 0 < delta <= 1, k >= 1, c > 0")
    return r
