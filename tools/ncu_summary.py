"""Summarise an .ncu-rep (run here, no GPU): key SOL/memory metrics + top stall lines.
python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    print(f"# ncu summary of {rep}")
    print(f"kernel: {vals[hdr.index('Kernel Name')]}")
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"{k:60s} {vals[i]:>18s} {units[i]}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source=sass"))))
    h = src[1]
    I = {k: i for i, k in enumerate(h)}
    rows = src[2:]
    S = "Warp Stall Sampling (All Samples)"
    tot = sum(int(x[I[S]] or 0) for x in rows) or 1
    stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    agg = {c: sum(int(x[I[c]] or 0) for x in rows) for c in stall_cols}
    print(f"\nwarp-stall samples: {tot}")
    for c, v in sorted(agg.items(), key=lambda t: -t[1])[:8]:
        print(f"  {c:32s} {v:9d} {100 * v / tot:5.1f}%")
    print("\ntop instructions (samples, share, SASS, top stall reasons):")
    for x in sorted(rows, key=lambda x: -int(x[I[S]] or 0))[:20]:
        s = int(x[I[S]] or 0)
        rs = sorted([(int(x[I[c]] or 0), c) for c in stall_cols], reverse=True)[:2]
        print(f"  {s:8d} {100 * s / tot:5.1f}%  {x[1].strip()[:60]:60s} {rs}")

    by_line(rep)


def by_line(rep, top=25):
    """Per CUDA source line (-lineinfo): instructions executed and stall samples, top lines."""
    out = ncu(rep, "--page", "source", "--csv", "--print-source=cuda,sass")
    fname, hdr, lines = "", None, []
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = {k: i for i, k in enumerate(row)}
            continue
        if hdr is None or not row[0]:
            continue
        try:
            ie = int(row[hdr["Instructions Executed"]] or 0)
            sm = int(row[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, KeyError, IndexError):
            continue
        lines.append((fname, int(row[0]), row[1].strip(), ie, sm))
    if not lines:
        return
    ti = sum(x[3] for x in lines) or 1
    ts = sum(x[4] for x in lines) or 1
    print(f"\nby source line (instructions executed {ti}, stall samples {ts}):")
    print("  inst%  stall%  file:line  source")
    keep = sorted(lines, key=lambda x: -(x[3] / ti + x[4] / ts))[:top]
    for f, ln, src, ie, sm in keep:
        print(f"  {100 * ie / ti:5.1f}  {100 * sm / ts:5.1f}   {f}:{ln}  {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1])
