"""Per-source-line warp-stall samples of one kernel in an .ncu-rep (run here, no GPU).

python tools/ncu_lines.py report.ncu-rep lib.so kernel_substring [top]
Maps each sampled SASS offset to its CUDA source line with nvdisasm -g (needs -lineinfo)."""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
import os


def main(rep, lib, kname, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    I = {k: i for i, k in enumerate(h)}
    data = rows[2:]
    S = "Warp Stall Sampling (All Samples)"
    addrs = [int(r[I["Address"]], 16) for r in data]
    base = min(addrs)
    # cubin of the library -> SASS offsets with line info
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=td, capture_output=True)
        cubins = [os.path.join(td, f) for f in os.listdir(td) if f.endswith(".cubin")]
        off2line = {}
        for cb in cubins:
            dis = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
            fn = None
            line = None
            for l in dis.split("\n"):
                m = re.match(r"\s*\.text\.(\S+):", l)
                if m:
                    fn = m.group(1)
                    continue
                m = re.search(r'## File ".*?([^/"]+)", line (\d+)', l)
                if m:
                    line = f"{m.group(1)}:{m.group(2)}"
                    continue
                m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
                if m and fn and kname in fn:
                    off2line[int(m.group(1), 16)] = line
    agg = collections.Counter()
    stall = collections.defaultdict(collections.Counter)
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    for r, a in zip(data, addrs):
        ln = off2line.get(a - base, "?")
        s = int(r[I[S]] or 0)
        agg[ln] += s
        for c in cols:
            stall[ln][c[6:]] += int(r[I[c]] or 0)
    tot = sum(agg.values()) or 1
    print(f"# {rep}: {tot} samples, kernel {kname}")
    for ln, s in agg.most_common(int(top)):
        print(f"{s:9d} {100 * s / tot:5.1f}%  {ln:16s} {stall[ln].most_common(3)}")


if __name__ == "__main__":
    main(*sys.argv[1:])
