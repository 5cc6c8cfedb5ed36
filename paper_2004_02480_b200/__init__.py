"""B200-native Count-Sketch Kaczmarz (CSK) hot path -- thin Python binding of libcsk.

Every function here is argument marshalling around the C ABI in ``include/csk.h``
(same names): it checks dtypes/devices, passes ``data_ptr()``s and the current CUDA
stream, and raises on a non-OK status.  All arithmetic runs in the CUDA kernels of
``csrc/`` (sm_100a).  There is no CPU fallback: importing this package without the
built ``libcsk.so`` raises, and every call needs CUDA tensors.

Method: Zhang & Li, arXiv 2004.02480 -- Algorithm 1: sketch once
(A~ = S A, b~ = S b, S = Phi D of Definition 1), then the maximal-weighted-
residual Kaczmarz loop on (A~, b~) until RES <= tol.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# CSK_LIB=prof selects the debug build with the in-kernel phase profiler (tools/loop_probe.py),
# CSK_LIB=checked the build with device-side bounds checks (CSK_DCHECK)
# CSK_LIB=/path/to/libcsk_*.so loads another build of the same ABI (A/B timing of kernel versions)
_lib_env = os.environ.get("CSK_LIB", "")
LIB_PATH = (_lib_env if _lib_env.endswith(".so") else
            os.path.join(_PKG, {"prof": "libcsk_prof.so", "checked": "libcsk_checked.so"}.get(_lib_env, "libcsk.so")))

CSK_OK, CSK_E_ARG, CSK_E_ZERO_SKETCH, CSK_E_UNSUPPORTED, CSK_E_CUDA, CSK_E_NCCL, CSK_E_NOMEM = range(7)
CONVERGED, MAX_ITERS, STAGNATED = 0, 1, 2
STOP_RES, STOP_RESIDUAL = 0, 1
MAX_N = 2048
SOLVE_ASYNC = 1
SOLVE_NO_TMEM = 4
SOLVE_FORCE_TMEM = 8
SOLVE_NO_STREAM_RING = 16


class CskError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_STATUS = {0: "CSK_OK", 1: "CSK_E_ARG", 2: "CSK_E_ZERO_SKETCH", 3: "CSK_E_UNSUPPORTED",
           4: "CSK_E_CUDA", 5: "CSK_E_NCCL", 6: "CSK_E_NOMEM"}


class Report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("final_res", ctypes.c_double),
                ("termination", ctypes.c_int32), ("stop_mode", ctypes.c_int32),
                ("last_index", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class SolveOpts(ctypes.Structure):
    _fields_ = [("num_ctas", ctypes.c_int32), ("smem_rows", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("cluster_size", ctypes.c_int32),
                ("trace_cap", ctypes.c_int64), ("idx_trace", ctypes.c_void_p),
                ("res_trace", ctypes.c_void_p), ("x_trace", ctypes.c_void_p),
                ("phase_cycles", ctypes.c_void_p), ("reg_rows", ctypes.c_int32),
                ("group_warps", ctypes.c_int32), ("r_trace", ctypes.c_void_p),
                ("r_trace_cap", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, i64, u64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
    sigs = {
        "csk_abi_version": ([], ctypes.c_int),
        "csk_ctx_create": ([i32, ctypes.POINTER(P)], i32),
        "csk_ctx_destroy": ([P], i32),
        "csk_last_error": ([P], ctypes.c_char_p),
        "csk_status_string": ([i32], ctypes.c_char_p),
        "csk_hash": ([P, u64, i64, i64, i64, P, P, P], i32),
        "csk_plan": ([P, u64, i64, i64, i64, P, P, P, P, P], i32),
        "csk_sketch": ([P, P, i64, P, i64, i64, i64, u64, P, P, P, P], i32),
        "csk_sketch_with_map": ([P, P, i64, P, i64, i64, i64, P, P, P, P, P, P], i32),
        "csk_sketch_csr": ([P, P, P, P, P, i64, i64, i64, u64, P, P, P, P], i32),
        "csk_sketch_planned": ([P, P, i64, P, i64, i64, i64, P, P, P, P, P, P], i32),
        "csk_row_norms": ([P, P, i64, i64, P, P], i32),
        "csk_solve": ([P, P, P, P, i64, i64, P, P, dbl, i64, ctypes.POINTER(Report), P], i32),
        "csk_solve_ex": ([P, P, P, P, i64, i64, P, P, dbl, i64, ctypes.POINTER(SolveOpts),
                          ctypes.POINTER(Report), P], i32),
        "csk_solve_wait": ([P, ctypes.POINTER(Report)], i32),
        "csk_ctx_set_timing": ([P, i32], i32),
        "csk_last_kernel_ms": ([P, i32, ctypes.POINTER(ctypes.c_float)], i32),
        "csk_last_solve_tiers": ([P, P], i32),
        "csk_last_solve_geometry": ([P, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                     ctypes.POINTER(ctypes.c_int32)], i32),
        "csk_run": ([P, P, i64, P, i64, i64, i64, u64, P, P, dbl, i64, ctypes.POINTER(Report), P], i32),
        "csk_run_host": ([P, P, i64, P, i64, i64, i64, u64, P, P, dbl, i64,
                          ctypes.POINTER(Report), P], i32),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _extend_sharded(lib)
    return lib


def _extend_sharded(lib):
    P, i64, u64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double
    pi64 = ctypes.POINTER(ctypes.c_int64)
    extra = {
        "csk_shard_range": ([i64, i32, i32, pi64, pi64], i32),
        "csk_comm_unique_id": ([P], i32),
        "csk_comm_create": ([P, P, i32, i32], i32),
        "csk_comm_destroy": ([P], i32),
        "csk_sketch_sharded": ([P, P, i64, P, i64, i64, i64, i64, i64, u64, P, P, P, pi64, pi64, P], i32),
        "csk_solve_sharded": ([P, P, P, P, i64, i64, i64, i64, P, P, dbl, i64, ctypes.POINTER(Report), P], i32),
        "csk_solve_virtual_ranks": ([P, P, P, P, i64, i64, i32, P, P, dbl, i64, P, ctypes.POINTER(Report), P], i32),
        "csk_solve_virtual_ranks_ex": ([P, P, P, P, i64, i64, i32, P, P, dbl, i64, P, ctypes.POINTER(SolveOpts),
                                        ctypes.POINTER(Report), P], i32),
        "csk_sketch_csr_sharded": ([P, P, P, P, P, i64, i64, i64, i64, i64, u64, i32, P, P, P, pi64, pi64, P], i32),
        "csk_sketch_csr_routed_virtual": ([P, P, P, P, P, i64, i64, i64, u64, i32, P, P, P, P], i32),
    }
    for name, (args, res) in extra.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


lib = _load()


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _need(t: torch.Tensor, dtype, name, dims=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if dims is not None and t.dim() != dims:
        raise ValueError(f"{name} must be {dims}-D")


class Context:
    """Owns a ``csk_ctx_t`` (workspaces, plan scratch, optional NCCL communicator)."""

    def __init__(self, device: int | None = None):
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        h = ctypes.c_void_p()
        st = lib.csk_ctx_create(device, ctypes.byref(h))
        if st != CSK_OK:
            raise CskError(st, "csk_ctx_create failed (needs an sm_100 GPU)")
        self.handle = h

    def close(self):
        if self.handle:
            lib.csk_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def check(self, st: int):
        if st != CSK_OK:
            raise CskError(st, lib.csk_last_error(self.handle).decode())


_default: Context | None = None


def default_context() -> Context:
    global _default
    if _default is None or _default.device != torch.cuda.current_device():
        _default = Context()
    return _default


# ------------------------------------------------------------------ S1/S2 plan
def csk_hash(m: int, d: int, seed: int = 0, row_offset: int = 0, ctx: Context | None = None):
    """(h int32[m], sign int8[m]) of Definition 1, counter-form SplitMix64."""
    ctx = ctx or default_context()
    h = torch.empty(m, dtype=torch.int32, device="cuda")
    s = torch.empty(m, dtype=torch.int8, device="cuda")
    ctx.check(lib.csk_hash(ctx.handle, seed & (2**64 - 1), row_offset, m, d, _ptr(h), _ptr(s), _stream()))
    return h, s


def csk_plan(m: int, d: int, seed: int = 0, row_offset: int = 0, h=None, sign=None,
             ctx: Context | None = None):
    """(perm int32[m] with sign in bit 31, offsets int32[d+1]) -- stable bucketing by h."""
    ctx = ctx or default_context()
    perm = torch.empty(m, dtype=torch.int32, device="cuda")
    offsets = torch.empty(d + 1, dtype=torch.int32, device="cuda")
    if h is not None:
        _need(h, torch.int32, "h", 1)
        _need(sign, torch.int8, "sign", 1)
    ctx.check(lib.csk_plan(ctx.handle, seed & (2**64 - 1), row_offset, m, d, _ptr(h), _ptr(sign),
                           _ptr(perm), _ptr(offsets), _stream()))
    return perm, offsets


# ------------------------------------------------------------------ S3/S4 sketch
def csk_sketch(A: torch.Tensor, b: torch.Tensor, d: int, seed: int = 0, with_norms: bool = True,
               ctx: Context | None = None, out=None):
    """(A~, b~, nsq) = (S A, S b, row norms of A~) (Algorithm 1 "Initialize")."""
    ctx = ctx or default_context()
    _need(A, torch.float64, "A", 2)
    _need(b, torch.float64, "b", 1)
    if A.stride(1) != 1:
        raise ValueError("A must be row-major (stride(1) == 1)")
    m, n = A.shape
    if out is None:
        At = torch.empty(d, n, dtype=torch.float64, device=A.device)
        bt = torch.empty(d, dtype=torch.float64, device=A.device)
        nsq = torch.empty(d, dtype=torch.float64, device=A.device) if with_norms else None
    else:
        At, bt, nsq = out
    ctx.check(lib.csk_sketch(ctx.handle, _ptr(A), A.stride(0), _ptr(b.contiguous()), m, n, d,
                             seed & (2**64 - 1), _ptr(At), _ptr(bt), _ptr(nsq), _stream()))
    return At, bt, nsq


def csk_sketch_planned(A: torch.Tensor, b: torch.Tensor, d: int, perm: torch.Tensor, offsets: torch.Tensor,
                       with_norms: bool = True, ctx: Context | None = None, out=None):
    """Sketch with a cached plan (perm, offsets from csk_plan for the same seed, m, d)."""
    ctx = ctx or default_context()
    _need(A, torch.float64, "A", 2)
    _need(b, torch.float64, "b", 1)
    _need(perm, torch.int32, "perm", 1)
    _need(offsets, torch.int32, "offsets", 1)
    if A.stride(1) != 1:
        raise ValueError("A must be row-major (stride(1) == 1)")
    m, n = A.shape
    if out is None:
        At = torch.empty(d, n, dtype=torch.float64, device=A.device)
        bt = torch.empty(d, dtype=torch.float64, device=A.device)
        nsq = torch.empty(d, dtype=torch.float64, device=A.device) if with_norms else None
    else:
        At, bt, nsq = out
    ctx.check(lib.csk_sketch_planned(ctx.handle, _ptr(A), A.stride(0), _ptr(b.contiguous()), m, n, d, _ptr(perm),
                                     _ptr(offsets), _ptr(At), _ptr(bt), _ptr(nsq), _stream()))
    return At, bt, nsq


def csk_sketch_with_map(A, b, d: int, h, sign, with_norms: bool = True, ctx: Context | None = None):
    """Sketch with an explicit map (test hook; d == m allowed, Remark 1 P:69)."""
    ctx = ctx or default_context()
    _need(A, torch.float64, "A", 2)
    _need(h, torch.int32, "h", 1)
    _need(sign, torch.int8, "sign", 1)
    m, n = A.shape
    At = torch.empty(d, n, dtype=torch.float64, device=A.device)
    bt = torch.empty(d, dtype=torch.float64, device=A.device)
    nsq = torch.empty(d, dtype=torch.float64, device=A.device) if with_norms else None
    ctx.check(lib.csk_sketch_with_map(ctx.handle, _ptr(A), A.stride(0), _ptr(b.contiguous()), m, n, d,
                                      _ptr(h), _ptr(sign), _ptr(At), _ptr(bt), _ptr(nsq), _stream()))
    return At, bt, nsq


def csk_sketch_csr(row_ptr, col, val, b, n: int, d: int, seed: int = 0, with_norms: bool = True,
                   ctx: Context | None = None):
    """CSR-input sketch (config C5)."""
    ctx = ctx or default_context()
    _need(row_ptr, torch.int64, "row_ptr", 1)
    _need(col, torch.int32, "col", 1)
    _need(val, torch.float64, "val", 1)
    _need(b, torch.float64, "b", 1)
    m = row_ptr.shape[0] - 1
    At = torch.empty(d, n, dtype=torch.float64, device=val.device)
    bt = torch.empty(d, dtype=torch.float64, device=val.device)
    nsq = torch.empty(d, dtype=torch.float64, device=val.device) if with_norms else None
    ctx.check(lib.csk_sketch_csr(ctx.handle, _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(b), m, n, d,
                                 seed & (2**64 - 1), _ptr(At), _ptr(bt), _ptr(nsq), _stream()))
    return At, bt, nsq


def csk_row_norms(At: torch.Tensor, ctx: Context | None = None):
    """nsq_j = ||A~^(j)||^2."""
    ctx = ctx or default_context()
    _need(At, torch.float64, "A_tilde", 2)
    At = At.contiguous()
    d, n = At.shape
    nsq = torch.empty(d, dtype=torch.float64, device=At.device)
    ctx.check(lib.csk_row_norms(ctx.handle, _ptr(At), d, n, _ptr(nsq), _stream()))
    return nsq


# ------------------------------------------------------------------ S5-S8 loop
@dataclass
class SolveResult:
    x: torch.Tensor
    iterations: int
    final_res: float
    termination: int
    stop_mode: int
    last_index: int
    idx_trace: torch.Tensor | None = None
    res_trace: torch.Tensor | None = None
    x_trace: torch.Tensor | None = None
    r_trace: torch.Tensor | None = None


def _trace_opts(opts, d: int, n: int, device, trace: int, trace_x: bool, trace_r: int):
    """Device trace buffers (NaN / -1 filled) wired into a SolveOpts."""
    idx_t = res_t = x_t = r_t = None
    if trace:
        idx_t = torch.full((trace,), -1, dtype=torch.int64, device=device)
        res_t = torch.full((trace,), float("nan"), dtype=torch.float64, device=device)
        if trace_x:
            x_t = torch.full((trace, n), float("nan"), dtype=torch.float64, device=device)
        opts.trace_cap = trace
        opts.idx_trace = idx_t.data_ptr()
        opts.res_trace = res_t.data_ptr()
        opts.x_trace = None if x_t is None else x_t.data_ptr()
    if trace_r:
        r_t = torch.full((trace_r, d), float("nan"), dtype=torch.float64, device=device)
        opts.r_trace = r_t.data_ptr()
        opts.r_trace_cap = trace_r
    return idx_t, res_t, x_t, r_t


def _result(x, rep, traces, trace: int, trace_r: int) -> "SolveResult":
    idx_t, res_t, x_t, r_t = traces
    k = rep.iterations
    return SolveResult(x=x, iterations=k, final_res=rep.final_res, termination=rep.termination,
                       stop_mode=rep.stop_mode, last_index=rep.last_index,
                       idx_trace=None if idx_t is None else idx_t[:min(k, trace)],
                       res_trace=None if res_t is None else res_t[:min(k + 1, trace)],
                       x_trace=None if x_t is None else x_t[:min(k + 1, trace)],
                       r_trace=None if r_t is None else r_t[:min(k + 1, trace_r)])


def csk_solve(At, bt, nsq, x0=None, x_star=None, tol: float = 1e-6, max_iters: int = 50_000,
              num_ctas: int = 0, smem_rows: int = 0, cluster_size: int = 0, trace: int = 0,
              trace_x: bool = False, phase_cycles: torch.Tensor | None = None,
              reg_rows: int = 0, group_warps: int = 0, tmem: bool | None = None,
              stream_ring: bool = True, trace_r: int = 0, ctx: Context | None = None) -> SolveResult:
    """Algorithm 1 loop with the P:180 stopping rule, one persistent kernel.

    ``trace`` records i_k and the stop quantity (and x_k with ``trace_x``) for the first ``trace``
    iterations; ``trace_r`` records the whole residual vector r_k = b~ - A~ x_k (the values the
    kernel scores) for the first ``trace_r`` iterations (``r_trace``: trace_r x d)."""
    ctx = ctx or default_context()
    _need(At, torch.float64, "A_tilde", 2)
    _need(bt, torch.float64, "b_tilde", 1)
    _need(nsq, torch.float64, "nsq", 1)
    At = At.contiguous()
    d, n = At.shape
    x = torch.zeros(n, dtype=torch.float64, device=At.device) if x0 is None else x0.clone().contiguous()
    xs = None if x_star is None else x_star.contiguous()
    opts = SolveOpts()
    opts.num_ctas = num_ctas
    opts.smem_rows = smem_rows
    opts.cluster_size = cluster_size
    opts.reg_rows = reg_rows
    opts.group_warps = group_warps
    opts.flags = ((SOLVE_NO_TMEM if tmem is False else 0) | (SOLVE_FORCE_TMEM if tmem is True else 0)
                  | (0 if stream_ring else SOLVE_NO_STREAM_RING))
    traces = _trace_opts(opts, d, n, At.device, trace, trace_x, trace_r)
    if phase_cycles is not None:
        opts.phase_cycles = phase_cycles.data_ptr()
    rep = Report()
    ctx.check(lib.csk_solve_ex(ctx.handle, _ptr(At), _ptr(bt.contiguous()), _ptr(nsq.contiguous()),
                               d, n, _ptr(x), _ptr(xs), float(tol), int(max_iters),
                               ctypes.byref(opts), ctypes.byref(rep), _stream()))
    return _result(x, rep, traces, trace, trace_r)


def csk_solve_async(At, bt, nsq, x, x_star=None, tol: float = 1e-6, max_iters: int = 50_000,
                    num_ctas: int = 0, smem_rows: int = 0, cluster_size: int = 0,
                    ctx: Context | None = None):
    """Launch the loop without waiting (CSK_SOLVE_ASYNC); x (in/out) is updated in place.
    Call ``csk_solve_wait(ctx)`` for the report."""
    ctx = ctx or default_context()
    # the same checks as csk_solve; x is updated in place, so it must be a contiguous fp64 CUDA tensor
    _need(At, torch.float64, "A_tilde", 2)
    _need(bt, torch.float64, "b_tilde", 1)
    _need(nsq, torch.float64, "nsq", 1)
    _need(x, torch.float64, "x", 1)
    if x_star is not None:
        _need(x_star, torch.float64, "x_star", 1)
    for t, nm in ((At, "A_tilde"), (bt, "b_tilde"), (nsq, "nsq"), (x, "x"), (x_star, "x_star")):
        if t is not None and not t.is_contiguous():
            raise ValueError(f"{nm} must be contiguous (csk_solve_async passes raw pointers)")
    d, n = At.shape
    if bt.shape[0] != d or nsq.shape[0] != d or x.shape[0] != n or (x_star is not None and x_star.shape[0] != n):
        raise ValueError("csk_solve_async: shape mismatch")
    opts = SolveOpts()
    opts.num_ctas = num_ctas
    opts.smem_rows = smem_rows
    opts.cluster_size = cluster_size
    opts.flags = SOLVE_ASYNC
    ctx.check(lib.csk_solve_ex(ctx.handle, _ptr(At), _ptr(bt), _ptr(nsq), d, n, _ptr(x), _ptr(x_star),
                               float(tol), int(max_iters), ctypes.byref(opts), None, _stream()))


def csk_ctx_set_timing(on: bool = True, ctx: Context | None = None):
    """Record CUDA events around the sketch and loop kernels of later calls on `ctx`."""
    ctx = ctx or default_context()
    ctx.check(lib.csk_ctx_set_timing(ctx.handle, 1 if on else 0))


def csk_last_kernel_ms(which: str, ctx: Context | None = None) -> float:
    """Duration (ms) of the last timed 'sketch' (k_sketch_dense) or 'loop' (k_loop) launch."""
    ctx = ctx or default_context()
    ms = ctypes.c_float()
    ctx.check(lib.csk_last_kernel_ms(ctx.handle, {"sketch": 0, "loop": 1}[which], ctypes.byref(ms)))
    return ms.value


def csk_last_solve_geometry(ctx: Context | None = None) -> dict:
    """{'num_ctas', 'cluster_size', 'smem_rows'} of the last solve on ``ctx``."""
    ctx = ctx or default_context()
    g, c, r = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    ctx.check(lib.csk_last_solve_geometry(ctx.handle, ctypes.byref(g), ctypes.byref(c), ctypes.byref(r)))
    return {"num_ctas": g.value, "cluster_size": c.value, "smem_rows": r.value}


def csk_last_solve_tiers(ctx: Context | None = None) -> dict:
    """Row tiers per row group of the last solve on ``ctx`` (csk_last_solve_tiers, loop.cu)."""
    ctx = ctx or default_context()
    out = (ctypes.c_int32 * 8)()
    ctx.check(lib.csk_last_solve_tiers(ctx.handle, ctypes.cast(out, ctypes.c_void_p)))
    keys = ["num_ctas", "cluster_size", "reg_rows", "tmem_rows", "smem_rows", "group_warps", "ring_stages",
            "ring_rows"]
    return dict(zip(keys, list(out)))


def csk_solve_wait(ctx: Context | None = None) -> Report:
    ctx = ctx or default_context()
    rep = Report()
    ctx.check(lib.csk_solve_wait(ctx.handle, ctypes.byref(rep)))
    return rep


def csk_run(A, b, d: int, seed: int = 0, x0=None, x_star=None, tol: float = 1e-6,
            max_iters: int = 50_000, ctx: Context | None = None):
    """Whole Algorithm 1 on device buffers: plan + sketch + norms + loop."""
    ctx = ctx or default_context()
    _need(A, torch.float64, "A", 2)
    _need(b, torch.float64, "b", 1)
    m, n = A.shape
    x = torch.zeros(n, dtype=torch.float64, device=A.device) if x0 is None else x0.clone().contiguous()
    rep = Report()
    ctx.check(lib.csk_run(ctx.handle, _ptr(A), A.stride(0), _ptr(b.contiguous()), m, n, d,
                          seed & (2**64 - 1), _ptr(x), _ptr(x_star), float(tol), int(max_iters),
                          ctypes.byref(rep), _stream()))
    return x, rep


def csk_run_host(A, b, d: int, seed: int = 0, x0=None, x_star=None, tol: float = 1e-6,
                 max_iters: int = 50_000, ctx: Context | None = None):
    """Whole Algorithm 1 from HOST (CPU, ideally pinned) tensors; copies in and out."""
    ctx = ctx or default_context()
    for t, nm in ((A, "A"), (b, "b")):
        if t.is_cuda or t.dtype != torch.float64:
            raise TypeError(f"{nm} must be a host fp64 tensor")
    m, n = A.shape
    x = torch.zeros(n, dtype=torch.float64) if x0 is None else x0.clone().contiguous()
    rep = Report()
    ctx.check(lib.csk_run_host(ctx.handle, _ptr(A), A.stride(0), _ptr(b.contiguous()), m, n, d,
                               seed & (2**64 - 1), _ptr(x), _ptr(x_star), float(tol), int(max_iters),
                               ctypes.byref(rep), _stream()))
    return x, rep


# ------------------------------------------------------------------ S9/S10 sharded path
NCCL_UID_BYTES = 128


def shard_range(total: int, nranks: int, rank: int) -> tuple[int, int]:
    """Rows [lo, hi) of A~ owned by `rank` (equal ceil blocks; host-only)."""
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    st = lib.csk_shard_range(total, nranks, rank, ctypes.byref(lo), ctypes.byref(hi))
    if st != CSK_OK:
        raise CskError(st, "csk_shard_range: bad arguments")
    return lo.value, hi.value


def comm_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0; the caller broadcasts the 128 bytes)."""
    buf = ctypes.create_string_buffer(NCCL_UID_BYTES)
    st = lib.csk_comm_unique_id(buf)
    if st != CSK_OK:
        raise CskError(st, "ncclGetUniqueId failed")
    return buf.raw


def comm_create(uid: bytes, nranks: int, rank: int, ctx: Context | None = None):
    ctx = ctx or default_context()
    buf = ctypes.create_string_buffer(bytes(uid), NCCL_UID_BYTES)
    ctx.check(lib.csk_comm_create(ctx.handle, buf, nranks, rank))


def comm_destroy(ctx: Context | None = None):
    ctx = ctx or default_context()
    ctx.check(lib.csk_comm_destroy(ctx.handle))


def csk_sketch_sharded(A_local, b_local, row_offset: int, m: int, d: int, nranks: int, rank: int,
                       seed: int = 0, ctx: Context | None = None):
    """S9: this rank's rows of (A, b) -> its bucket rows of (A~, b~, nsq) (NCCL reduce-scatter)."""
    ctx = ctx or default_context()
    _need(A_local, torch.float64, "A_local", 2)
    _need(b_local, torch.float64, "b_local", 1)
    ml, n = A_local.shape
    lo, hi = shard_range(d, nranks, rank)
    rows = max(hi - lo, 0)
    At = torch.empty(max(rows, 1), n, dtype=torch.float64, device=A_local.device)
    bt = torch.empty(max(rows, 1), dtype=torch.float64, device=A_local.device)
    nsq = torch.empty(max(rows, 1), dtype=torch.float64, device=A_local.device)
    dlo, dhi = ctypes.c_int64(), ctypes.c_int64()
    ctx.check(lib.csk_sketch_sharded(ctx.handle, _ptr(A_local), A_local.stride(0), _ptr(b_local.contiguous()),
                                     ml, row_offset, m, n, d, seed & (2**64 - 1), _ptr(At), _ptr(bt), _ptr(nsq),
                                     ctypes.byref(dlo), ctypes.byref(dhi), _stream()))
    return At[:rows], bt[:rows], nsq[:rows], dlo.value, dhi.value


SHARD_REDUCE_SCATTER, SHARD_ROUTE_ROWS = 0, 1


def csk_sketch_csr_sharded(row_ptr, col, val, b_local, row_offset: int, m: int, n: int, d: int, nranks: int,
                           rank: int, seed: int = 0, mode: int = SHARD_ROUTE_ROWS, ctx: Context | None = None):
    """S9 for CSR input: this rank's rows [row_offset, row_offset + len(b_local)) -> its bucket rows of
    (A~, b~, nsq).  mode SHARD_ROUTE_ROWS (rows to their bucket owners; bit-identical to one GPU) or
    SHARD_REDUCE_SCATTER (partial A~ + ncclReduceScatter)."""
    ctx = ctx or default_context()
    _need(row_ptr, torch.int64, "row_ptr", 1)
    _need(col, torch.int32, "col", 1)
    _need(val, torch.float64, "val", 1)
    _need(b_local, torch.float64, "b_local", 1)
    ml = row_ptr.shape[0] - 1
    lo, hi = shard_range(d, nranks, rank)
    rows = max(hi - lo, 0)
    dev = val.device
    At = torch.empty(max(rows, 1), n, dtype=torch.float64, device=dev)
    bt = torch.empty(max(rows, 1), dtype=torch.float64, device=dev)
    nsq = torch.empty(max(rows, 1), dtype=torch.float64, device=dev)
    dlo, dhi = ctypes.c_int64(), ctypes.c_int64()
    ctx.check(lib.csk_sketch_csr_sharded(ctx.handle, _ptr(row_ptr.contiguous()), _ptr(col.contiguous()),
                                         _ptr(val.contiguous()), _ptr(b_local.contiguous()), ml, row_offset, m, n, d,
                                         seed & (2**64 - 1), int(mode), _ptr(At), _ptr(bt), _ptr(nsq),
                                         ctypes.byref(dlo), ctypes.byref(dhi), _stream()))
    return At[:rows], bt[:rows], nsq[:rows], dlo.value, dhi.value


def csk_sketch_csr_routed_virtual(row_ptr, col, val, b, n: int, d: int, nranks: int, seed: int = 0,
                                  ctx: Context | None = None):
    """The row-routing decomposition of S9 with `nranks` virtual ranks on this GPU (test hook)."""
    ctx = ctx or default_context()
    _need(row_ptr, torch.int64, "row_ptr", 1)
    _need(col, torch.int32, "col", 1)
    _need(val, torch.float64, "val", 1)
    _need(b, torch.float64, "b", 1)
    m = row_ptr.shape[0] - 1
    At = torch.empty(d, n, dtype=torch.float64, device=val.device)
    bt = torch.empty(d, dtype=torch.float64, device=val.device)
    nsq = torch.empty(d, dtype=torch.float64, device=val.device)
    ctx.check(lib.csk_sketch_csr_routed_virtual(ctx.handle, _ptr(row_ptr.contiguous()), _ptr(col.contiguous()),
                                                _ptr(val.contiguous()), _ptr(b.contiguous()), m, n, d,
                                                seed & (2**64 - 1), int(nranks), _ptr(At), _ptr(bt), _ptr(nsq),
                                                _stream()))
    return At, bt, nsq


def csk_solve_sharded(At_local, bt_local, nsq_local, d_lo: int, d_hi: int, d: int, n: int,
                      x0=None, x_star=None, tol: float = 1e-6, max_iters: int = 50_000,
                      ctx: Context | None = None):
    """S10: Algorithm 1 loop with A~ rows sharded across ranks (x replicated)."""
    ctx = ctx or default_context()
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.zeros(n, dtype=torch.float64, device=dev) if x0 is None else x0.clone().contiguous()
    rep = Report()
    ctx.check(lib.csk_solve_sharded(ctx.handle, _ptr(At_local.contiguous()), _ptr(bt_local.contiguous()),
                                    _ptr(nsq_local.contiguous()), d_lo, d_hi, d, n, _ptr(x), _ptr(x_star),
                                    float(tol), int(max_iters), ctypes.byref(rep), _stream()))
    return x, rep


def csk_solve_virtual_ranks(At, bt, nsq, nranks: int, x0=None, x_star=None, tol: float = 1e-6,
                            max_iters: int = 50_000, trace: int = 0, trace_x: bool = False, trace_r: int = 0,
                            ctx: Context | None = None):
    """The sharded loop with `nranks` virtual ranks on this GPU (loopback exchange).

    Returns (x, copies, report), or (x, copies, report, SolveResult with the traces) when any
    trace is requested (virtual rank 0's i_k / RES / x_k; r_k of every rank by global row)."""
    ctx = ctx or default_context()
    _need(At, torch.float64, "A_tilde", 2)
    At = At.contiguous()
    d, n = At.shape
    x = torch.zeros(n, dtype=torch.float64, device=At.device) if x0 is None else x0.clone().contiguous()
    copies = torch.empty(nranks, n, dtype=torch.float64, device=At.device)
    rep = Report()
    opts = SolveOpts()
    traces = _trace_opts(opts, d, n, At.device, trace, trace_x, trace_r)
    ctx.check(lib.csk_solve_virtual_ranks_ex(ctx.handle, _ptr(At), _ptr(bt.contiguous()), _ptr(nsq.contiguous()),
                                             d, n, nranks, _ptr(x), _ptr(x_star), float(tol), int(max_iters),
                                             _ptr(copies), ctypes.byref(opts), ctypes.byref(rep), _stream()))
    if trace or trace_r:
        return x, copies, rep, _result(x, rep, traces, trace, trace_r)
    return x, copies, rep
