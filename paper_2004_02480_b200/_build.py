"""Build libcsk.so (the C-ABI library of include/csk.h) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libcsk.so")
PROF_LIB = os.path.join(PKG, "libcsk_prof.so")  # debug build with the in-kernel phase profiler
CHECKED_LIB = os.path.join(PKG, "libcsk_checked.so")  # debug build with device-side bounds checks
SOURCES = ["api.cu", "plan.cu", "sketch.cu", "loop.cu", "comm.cu", "route.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dirs():
    try:
        import nvidia.nccl as nn  # torch's bundled NCCL (2.28.x)
        base = list(nn.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib")
    except Exception:  # pragma: no cover
        return None, None


def flags(extra=()):
    inc, lib = _nccl_dirs()
    f = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "--fmad=false", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-I", os.path.join(ROOT, "include")]
    if inc:
        f += ["-I", inc]
    # experiment knob (A/B builds only): extra nvcc flags, e.g. -DCSK_CSR_STAGE_PAIRS=64
    f += os.environ.get("CSK_EXTRA_NVCC", "").split()
    return f + list(extra)


def link_flags():
    inc, lib = _nccl_dirs()
    f = ["-shared"]
    if lib:
        f += ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath", "-Xlinker", lib]
    return f


def sources():
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(ROOT, "include", "csk.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, prof: bool = False, checked: bool = False) -> str:
    lib = PROF_LIB if prof else CHECKED_LIB if checked else LIB
    if not force and not needs_build(lib):
        return lib
    objdir = os.path.join(PKG, "build_prof" if prof else "build_checked" if checked else "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        extra = ((["-Xptxas", "-v"] if verbose else []) + (["-DCSK_PHASE_PROF=1"] if prof else [])
                 + (["-DCSK_CHECKED=1"] if checked else []))
        cmd = [NVCC, "-c", src, "-o", obj] + flags(extra)
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        if verbose:
            sys.stderr.write(out.decode())
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC] + objs + ["-o", tmp, "-gencode", "arch=compute_100a,code=sm_100a"] + link_flags()
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, prof="--prof" in sys.argv,
                checked="--checked" in sys.argv))
