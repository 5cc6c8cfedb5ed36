"""CPU oracle for the CSK hot path (arXiv 2004.02480) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2004_02480_b200`` never imports it and shares no code with it.

This module is argument marshalling around ``csk_oracle.c`` (plain C99,
single-threaded, ``-ffp-contract=off``); every arithmetic step lives in the C
file and cites the paper there.  ``materialize_S`` and ``dense_S_product`` are
the plain Definition-1 matrix used to pin the sketch by brute force.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csk_oracle.c")
_LIB = os.path.join(_HERE, "libcsk_oracle.so")

CONVERGED, MAX_ITERS, STAGNATED = 0, 1, 2
TERMINATION_NAMES = {CONVERGED: "converged", MAX_ITERS: "max_iters", STAGNATED: "stagnated"}


def build(force: bool = False) -> str:
    """Compile csk_oracle.c with gcc (plain C99, no BLAS/OpenMP, fp-contract off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fPIC",
                               "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64, u64, dbl = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        lib.oracle_splitmix64_next.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
        lib.oracle_splitmix64_next.restype = u64
        lib.oracle_hash.argtypes = [u64, i64, i64, P, P]
        lib.oracle_hash.restype = None
        lib.oracle_sketch_dense.argtypes = [P, i64, P, i64, i64, i64, P, P, P, P]
        lib.oracle_sketch_dense.restype = None
        lib.oracle_sketch_csr.argtypes = [P, P, P, P, i64, i64, i64, P, P, P, P]
        lib.oracle_sketch_csr.restype = None
        lib.oracle_row_norms.argtypes = [P, i64, i64, P]
        lib.oracle_row_norms.restype = None
        lib.oracle_residual.argtypes = [P, P, i64, i64, P, P]
        lib.oracle_residual.restype = None
        lib.oracle_solve.argtypes = [P, P, P, i64, i64, P, P, dbl, i64,
                                     ctypes.POINTER(i64), ctypes.POINTER(dbl),
                                     ctypes.POINTER(i64), P, P, P, i64, P]
        lib.oracle_solve.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def splitmix64_stream(seed: int, count: int) -> list[int]:
    """The first ``count`` outputs of the sequential SplitMix64 stream."""
    lib = _load()
    st = ctypes.c_uint64(seed & (2**64 - 1))
    return [int(lib.oracle_splitmix64_next(ctypes.byref(st))) for _ in range(count)]


def hash_map(seed: int, m: int, d: int) -> tuple[np.ndarray, np.ndarray]:
    """(h int32[m], s int8[m]) of Definition 1 from ``seed`` (reading R-1)."""
    h = np.empty(m, np.int32)
    s = np.empty(m, np.int8)
    _load().oracle_hash(seed & (2**64 - 1), m, d, _p(h), _p(s))
    return h, s


def sketch_dense(A, b, d: int, h=None, s=None, seed: int = 0):
    """(A~, b~) = (S A, S b), S = Phi D; row-order accumulation."""
    A = _f64(A)
    b = _f64(b)
    m, n = A.shape
    if h is None:
        h, s = hash_map(seed, m, d)
    h = np.ascontiguousarray(h, np.int32)
    s = np.ascontiguousarray(s, np.int8)
    At = np.empty((d, n), np.float64)
    bt = np.empty(d, np.float64)
    _load().oracle_sketch_dense(_p(A), n, _p(b), m, n, d, _p(h), _p(s), _p(At), _p(bt))
    return At, bt


def sketch_csr(row_ptr, col, val, b, n: int, d: int, h=None, s=None, seed: int = 0):
    """CSR variant of ``sketch_dense`` (stored pair order within a row)."""
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val = _f64(val)
    b = _f64(b)
    m = row_ptr.shape[0] - 1
    if h is None:
        h, s = hash_map(seed, m, d)
    h = np.ascontiguousarray(h, np.int32)
    s = np.ascontiguousarray(s, np.int8)
    At = np.empty((d, n), np.float64)
    bt = np.empty(d, np.float64)
    _load().oracle_sketch_csr(_p(row_ptr), _p(col), _p(val), _p(b), m, n, d,
                              _p(h), _p(s), _p(At), _p(bt))
    return At, bt


def row_norms(At) -> np.ndarray:
    """nsq_j = ||A~^(j)||^2, fma left to right (P:62 / P:122)."""
    At = _f64(At)
    d, n = At.shape
    nsq = np.empty(d, np.float64)
    _load().oracle_row_norms(_p(At), d, n, _p(nsq))
    return nsq


def residual(At, bt, x) -> np.ndarray:
    """r = b~ - A~ x, fma left to right."""
    At, bt, x = _f64(At), _f64(bt), _f64(x)
    d, n = At.shape
    r = np.empty(d, np.float64)
    _load().oracle_residual(_p(At), _p(bt), d, n, _p(x), _p(r))
    return r


@dataclass
class SolveResult:
    x: np.ndarray
    iterations: int
    final_res: float
    termination: int
    last_index: int
    idx_trace: np.ndarray | None = None
    res_trace: np.ndarray | None = None
    x_trace: np.ndarray | None = None
    extra: dict = field(default_factory=dict)


def solve(At, bt, nsq, x0=None, x_star=None, tol: float = 1e-6, max_iters: int = 50000,
          trace: int = 0, trace_x: bool = False) -> SolveResult:
    """Algorithm 1 loop with the P:180 stopping rule; see csk_oracle.c O-4.

    ``trace`` > 0 records i_k and the stop quantity for the first ``trace`` iterations
    (and x_k when ``trace_x``).
    """
    At, bt, nsq = _f64(At), _f64(bt), _f64(nsq)
    d, n = At.shape
    x = np.zeros(n, np.float64) if x0 is None else _f64(x0).copy()
    xs = None if x_star is None else _f64(x_star)
    it = ctypes.c_int64(0)
    fr = ctypes.c_double(0.0)
    last = ctypes.c_int64(-1)
    idx_tr = np.full(trace, -1, np.int64) if trace else None
    res_tr = np.full(trace, np.nan) if trace else None
    x_tr = np.full((trace, n), np.nan) if (trace and trace_x) else None
    work = np.empty(d, np.float64)
    rc = _load().oracle_solve(_p(At), _p(bt), _p(nsq), d, n, _p(x), _p(xs), float(tol),
                              int(max_iters), ctypes.byref(it), ctypes.byref(fr),
                              ctypes.byref(last), _p(idx_tr), _p(res_tr), _p(x_tr),
                              int(trace), _p(work))
    if rc < 0:
        raise ValueError("oracle_solve: " + ("all rows of the sketch are zero" if rc == -2
                                             else "invalid argument"))
    k = it.value
    return SolveResult(x=x, iterations=k, final_res=fr.value, termination=rc,
                       last_index=last.value,
                       idx_trace=None if idx_tr is None else idx_tr[:min(k, trace)],
                       res_trace=None if res_tr is None else res_tr[:min(k + 1, trace)],
                       x_trace=None if x_tr is None else x_tr[:min(k + 1, trace)])


def csk(A, b, d: int, seed: int = 0, x0=None, x_star=None, tol: float = 1e-6,
        max_iters: int = 50000, **kw) -> SolveResult:
    """Whole Algorithm 1: sketch once, then the MWRK-on-sketch loop."""
    At, bt = sketch_dense(A, b, d, seed=seed)
    nsq = row_norms(At)
    return solve(At, bt, nsq, x0=x0, x_star=x_star, tol=tol, max_iters=max_iters, **kw)


def mwrk(A, b, x0=None, x_star=None, tol: float = 1e-6, max_iters: int = 50000, **kw):
    """MWRK (Remark 1): the same loop on (A, b) with S = I."""
    A = _f64(A)
    return solve(A, b, row_norms(A), x0=x0, x_star=x_star, tol=tol, max_iters=max_iters, **kw)


# --------------------------------------------------------------------------
# Definition 1 written out as a dense matrix -- tiny inputs only.
# --------------------------------------------------------------------------
def materialize_S(h, s, d: int) -> np.ndarray:
    """S = Phi D as an explicit d x m matrix: S[h(i), i] = s_i, zero elsewhere."""
    m = len(h)
    S = np.zeros((d, m), np.float64)
    for i in range(m):
        S[int(h[i]), i] = float(s[i])
    return S


def dense_S_product(S: np.ndarray, A: np.ndarray) -> np.ndarray:
    """(S A)[j,k] = sum_i S[j,i] A[i,k] by the textbook triple loop, i ascending."""
    d, m = S.shape
    n = A.shape[1]
    out = np.zeros((d, n), np.float64)
    for j in range(d):
        for k in range(n):
            acc = 0.0
            for i in range(m):
                acc = acc + float(S[j, i]) * float(A[i, k])
            out[j, k] = acc
    return out
