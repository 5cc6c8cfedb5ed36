"""CPU-side checks of the C-ABI library: it builds, loads, and exports every symbol
declared in include/*.h (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    inc = os.path.join(ROOT, "include")
    for fn in os.listdir(inc):
        if fn.endswith(".h"):
            src = open(os.path.join(inc, fn)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(csk_[a-z0-9_]+)\s*\(", src))
    return names


@pytest.fixture(scope="module")
def lib():
    # by path: importing the package would load the (maybe not yet built) libcsk.so
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_csk_build", os.path.join(ROOT, "paper_2004_02480_b200", "_build.py"))
    _build = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(_build)
    path = _build.build()
    return ctypes.CDLL(path)


def test_header_declares_boundary():
    names = _declared()
    for must in ["csk_sketch", "csk_row_norms", "csk_solve", "csk_hash", "csk_plan",
                 "csk_sketch_csr", "csk_run", "csk_run_host", "csk_ctx_create"]:
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in sorted(_declared()) if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_version_and_status_strings(lib):
    lib.csk_abi_version.restype = ctypes.c_int
    assert lib.csk_abi_version() == 2
    lib.csk_status_string.restype = ctypes.c_char_p
    assert lib.csk_status_string(0) == b"CSK_OK"
    assert lib.csk_status_string(2) == b"CSK_E_ZERO_SKETCH"


def test_ctx_create_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    lib.csk_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    assert lib.csk_ctx_create(0, ctypes.byref(h)) != 0


def test_shard_range_host_logic(lib):
    """Bucket ownership used by the sharded sketch/loop (host-only function)."""
    if not hasattr(lib, "csk_shard_range"):
        pytest.skip("sharded API not built")
    f = lib.csk_shard_range
    i64 = ctypes.c_int64
    f.argtypes = [i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    for total in [1, 7, 10, 10000, 40001]:
        for P in [1, 2, 3, 4, 8]:
            prev = 0
            for p in range(P):
                lo, hi = i64(), i64()
                assert f(total, P, p, ctypes.byref(lo), ctypes.byref(hi)) == 0
                assert lo.value == prev and hi.value >= lo.value
                prev = hi.value
            assert prev == total
