"""Registers and spills per kernel of one csrc/*.cu file: python tools/ptxas_stats.py loop.cu"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2004_02480_b200"))
import _build  # noqa: E402

src = os.path.join(ROOT, "paper_2004_02480_b200", "csrc", sys.argv[1])
out = subprocess.run([_build.NVCC, "-c", src, "-o", "/tmp/ptxas_stats.o"] + _build.flags(["-Xptxas", "-v"]),
                     capture_output=True, text=True)
cur, sp = None, ("0", "0")
for line in (out.stdout + out.stderr).split("\n"):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        sp = (m.group(1), m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        name = subprocess.run(["c++filt"], input=cur, capture_output=True, text=True).stdout.strip()
        name = re.sub(r"csk::\(anonymous namespace\)::", "", name).replace("(csk::LoopParams)", "")
        print(f"{m.group(1):>4} regs  spill st/ld {sp[0]:>4}/{sp[1]:<4} {name}")
        cur, sp = None, ("0", "0")
if out.returncode:
    print(out.stderr[-3000:])
