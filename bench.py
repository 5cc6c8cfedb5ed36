#!/usr/bin/env python
"""CSK hot-path benchmark (BASELINE.json metric): time-to-1e-6 (sketch + iterate),
iterations/s and sketch HBM GB/s on B200, plus the CPU oracle beside it.

One "step" = one pass of the whole hot path over one synthetic problem resident in
HBM: plan (S1/S2) + sketch with fused norms (S3/S4) + the persistent Algorithm 1
loop (S5-S8) until RES <= 1e-6 or the iteration cap.
Default workload: config C3 (see DESIGN.md §7 for why C3).  Between timed steps L2
is flushed by writing a 256 MiB buffer (untimed) unless A is larger than L2 (C3: 400 MB), the
timing rules' other option.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

N > 1 (torchrun): ONE problem, row-sharded across the ranks (strong scaling): the sketch
with csk_sketch_sharded (NCCL reduce-scatter of partial A~ by bucket range, S9) and the loop
with csk_solve_sharded (S10: the persistent loop on every GPU, one exchange over NVLink peer
memory per iteration).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from csk_synth import CONFIGS, make_config  # noqa: E402

METRIC = "CSK time-to-1e-6 rel err (sketch+iterate); iterations/s; sketch HBM GB/s"
SMEM_BYTES_PER_CLK_PER_SM = 128  # B300_MICROARCH.md "smem crossbar BW 128/N B/cyc/SM"
DFMA_PER_CLK_PER_SM = 64         # measured 63.4 (profiles/r01_microbench_k7b.txt, tools/microbench_dfma.cu)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi (NVML) clocks/throttle reasons sampled every 2 ms while running."""

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
        except Exception:
            self._nvml = None

    def _sample(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        return (time.perf_counter(), sm, mx, r)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            time.sleep(0.002)

    def sample_now(self):
        """One sample from the caller's thread (between timed steps, outside their CUDA events),
        so a short timed region still has samples taken while the GPU was busy."""
        if self._nvml:
            try:
                self.samples.append(self._sample())
            except Exception:
                pass

    def start(self):
        if self._nvml:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self, t0, t1):
        if not self._nvml:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        if not inside:  # timed region shorter than the sampling period: sample right at its end
            try:
                inside = [self._sample()]
            except Exception:
                inside = self.samples[-1:]
        nv = self._nvml
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
            "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
            "display_clock_setting": 0x100,
        }
        mask = 0
        for s in inside:
            mask |= int(s[3])
        reasons = [k for k, v in names.items() if mask & v and k != "gpu_idle"]
        return {"sm_mhz": statistics.median(s[1] for s in inside), "sm_max_mhz": inside[-1][2],
                "reasons": reasons, "samples": len(inside)}


def _dist(force: bool = False):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1 or force:
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", str(ws))
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        import torch.distributed as dist
        rank = int(os.environ["RANK"])
        local = int(os.environ.get("LOCAL_RANK", rank))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return dist, rank, ws, local
    return None, 0, 1, 0


def _barrier(dist):
    if dist is not None:
        dist.barrier()


def _max_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _ncu_traffic(name: str):
    """dram read+write bytes per launch from a committed ncu summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        vals = {}
        for line in open(path):
            parts = line.split()
            if len(parts) >= 3 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[parts[2]]
                vals[parts[0]] = float(parts[1].replace(",", "")) * scale
        return int(vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"])
    except Exception:
        return None


def _config_dict(cfg) -> dict:
    """The workload as both arms name it (same keys in the reference line: same_config)."""
    return {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "d": cfg.d, "kind": cfg.kind, "tol": cfg.tol,
            "max_iters": cfg.max_iters, "sketch_seed": cfg.sketch_seed, "gen_seed": cfg.gen_seed}


def alg_bytes_sketch(cfg) -> int:
    """8mn + 8m + 8dn + 8d (A, b read; A~, b~ written) + 8d (nsq)."""
    return 8 * cfg.m * cfg.n + 8 * cfg.m + 8 * cfg.d * cfg.n + 16 * cfg.d


def alg_bytes_iter(cfg) -> int:
    """8dn + 16d per iteration (A~ + b~ + nsq)."""
    return 8 * cfg.d * cfg.n + 16 * cfg.d


# ------------------------------------------------------------------ our arm
def run_ours(args, dist, rank, ws):
    import paper_2004_02480_b200 as csk

    cfg = CONFIGS[args.config]
    hbm_peak, sm_max_mhz, peak_src = _peaks()
    dev = torch.device("cuda", torch.cuda.current_device())
    p = make_config(cfg, dev)
    ctx = csk.Context()
    csk.csk_ctx_set_timing(True, ctx=ctx)  # events right around k_sketch_dense / k_loop (roofline)
    d, n = cfg.d, cfg.n
    At = torch.empty(d, n, dtype=torch.float64, device=dev)
    bt = torch.empty(d, dtype=torch.float64, device=dev)
    nsq = torch.empty(d, dtype=torch.float64, device=dev)
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    # timing rule: flush L2 between steps OR use inputs larger than L2.  When A exceeds L2
    # (C3: 400 MB vs 126 MB) nothing of A survives a step, and a write-flush would only leave L2
    # full of dirty lines whose write-backs then compete with the sketch's HBM reads.
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    do_flush = cfg.bytes_A <= 2 * l2_bytes
    stream = torch.cuda.current_stream()

    def step(ev=None):
        x.zero_()
        if ev:
            ev[0].record(stream)
        csk.csk_sketch(p.A, p.b, d, seed=cfg.sketch_seed, ctx=ctx, out=(At, bt, nsq))
        if ev:
            ev[1].record(stream)
        csk.csk_solve_async(At, bt, nsq, x, x_star=p.x_star, tol=cfg.tol, max_iters=cfg.max_iters, ctx=ctx)
        if ev:
            ev[2].record(stream)
        return csk.csk_solve_wait(ctx)

    for _ in range(args.warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(dev.index)
    sampler.start()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    reps = []
    kern_ms = {"sketch": [], "loop": []}
    _barrier(dist)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(args.steps):
        if do_flush:
            flush.fill_(1.0)  # untimed: outside the events of step k
        reps.append(step(evs[k]))
        for w in kern_ms:  # the step already synchronised (csk_solve_wait)
            kern_ms[w].append(csk.csk_last_kernel_ms(w, ctx=ctx))
        sampler.sample_now()
    torch.cuda.synchronize()
    _barrier(dist)
    t1 = time.perf_counter()
    sampler.stop()
    clocks = sampler.summary(t0, t1)

    sk = [e[0].elapsed_time(e[1]) for e in evs]
    sv = [e[1].elapsed_time(e[2]) for e in evs]
    tot = [a + b for a, b in zip(sk, sv)]
    # median of the K timed steps; the mean and spread are reported beside it
    ms_step = _max_over_ranks(dist, statistics.median(tot))
    sk_ms = statistics.median(sk)
    sv_ms = statistics.median(sv)
    it = reps[-1].iterations
    assert all(r.iterations == it for r in reps), "non-deterministic iteration count"

    # roofline: the dominant kernel is the persistent loop k_loop (A~ on chip: registers at
    # C1-C3; registers + TMEM + shared memory at C4).  north_star frames it as the bytes of A~
    # per iteration over the on-chip (SMEM/L2) bandwidth; the FP64 FMA bound is reported beside.
    loop_bytes = alg_bytes_iter(cfg) * it
    k_loop_ms = statistics.median(kern_ms["loop"])
    k_sketch_ms = statistics.median(kern_ms["sketch"])
    loop_gbs = loop_bytes / (k_loop_ms * 1e-3) / 1e9
    smem_peak = 148 * SMEM_BYTES_PER_CLK_PER_SM * sm_max_mhz * 1e6 / 1e9
    loop_tflops = 2.0 * cfg.d * cfg.n * it / (k_loop_ms * 1e-3) / 1e12
    fp64_peak = 148 * DFMA_PER_CLK_PER_SM * 2 * sm_max_mhz * 1e6 / 1e12
    loop_floor_us = (3230.0 + -(-cfg.d // 148) * cfg.n / 64.0) / sm_max_mhz
    sketch_gbs = alg_bytes_sketch(cfg) / (sk_ms * 1e-3) / 1e9
    out = {
        "metric": METRIC,
        "value": round(ms_step, 4),
        "unit": "ms",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (torch Philox, PAPER.md:180 recipe; csk_synth.py)",
        "config": dict(_config_dict(cfg),
                       l2=("flushed between steps (256 MiB write, untimed)" if do_flush else
                           "input larger than L2 (A = %.0f MB > %.0f MB L2): no flush" % (cfg.bytes_A / 1e6, l2_bytes / 1e6))),
        "timing": {"statistic": "median of the K timed steps", "mean_ms": round(sum(tot) / len(tot), 4),
                   "min_ms": round(min(tot), 4), "max_ms": round(max(tot), 4)},
        "iterations": it,
        "final_res": reps[-1].final_res,
        "termination": ["converged", "max_iters", "stagnated"][reps[-1].termination],
        "iterations_per_s": round(it / (sv_ms * 1e-3), 1),
        "sketch_ms": round(sk_ms, 5),
        "solve_ms": round(sv_ms, 5),
        "sketch_hbm_gbs": round(sketch_gbs, 1),
        "us_per_iteration": round(sv_ms * 1e3 / max(it, 1), 4),
        "roofline": {"kernel": "k_loop (persistent Algorithm 1 loop, A~ on chip)", "bound": "smem",
                     "achieved": round(loop_gbs, 1),
                     "peak": round(smem_peak, 1), "unit": "GB/s", "frac": round(loop_gbs / smem_peak, 4),
                     "traffic": _ncu_traffic(f"r01_ncu_loop_{cfg.name}.txt"),
                     "traffic_note": "DRAM bytes of the whole k_loop launch (one launch = the whole loop): "
                                     "A~ is read once into registers/TMEM/shared memory and stays on chip",
                     "peak_source": f"derived: 148 SM x {SMEM_BYTES_PER_CLK_PER_SM} B/clk x {sm_max_mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
                     "alg_bytes_per_iteration": alg_bytes_iter(cfg),
                     "kernel_ms": round(k_loop_ms, 5),
                     "timing": "CUDA events recorded by libcsk on the launching stream right around k_loop "
                               "(csk_ctx_set_timing), mean over the timed steps"},
        "roofline_fp64": {"kernel": "k_loop", "bound": "alu", "achieved": round(loop_tflops, 3),
                          "peak": round(fp64_peak, 2), "unit": "TFLOP/s", "frac": round(loop_tflops / fp64_peak, 4),
                          "peak_source": f"derived: 148 SM x {DFMA_PER_CLK_PER_SM} DFMA/clk x 2 x {sm_max_mhz:.0f} MHz "
                                         "(63.4 DFMA/clk/SM measured, profiles/r01_microbench_k7b.txt)",
                          "alg_flops_per_iteration": 2 * cfg.d * cfg.n,
                          "note": "the loop is latency-bound: one grid-wide exchange (atomic max-key + count, "
                                  "~2.3k cycles floor measured) per iteration"},
        # what actually bounds the loop: one grid-wide exchange per iteration.  Floor = the
        # microbenchmarked 148-CTA atomic exchange with a 500-double winner-row fetch (3230 cycles,
        # profiles/r01_microbench_k7b.txt "+row500") + the GEMV at the FP64 FMA rate
        "roofline_latency": {"kernel": "k_loop", "bound": "latency",
                             "floor_us_per_iteration": round(loop_floor_us, 3),
                             "achieved_us_per_iteration": round(k_loop_ms * 1e3 / max(it, 1), 3),
                             "frac": round(loop_floor_us / (k_loop_ms * 1e3 / max(it, 1)), 4),
                             "floor_source": "3230 cycles (microbench_xchg atomic_pair +row500, G=148) + "
                                             "ceil(d/148) n / 64 DFMA cycles, at sm_max_mhz"},
        "roofline_sketch": {"kernel": "k_sketch_dense", "bound": "hbm",
                            "achieved": round(alg_bytes_sketch(cfg) / (k_sketch_ms * 1e-3) / 1e9, 1),
                            "peak": hbm_peak, "unit": "GB/s",
                            "frac": round(alg_bytes_sketch(cfg) / (k_sketch_ms * 1e-3) / 1e9 / hbm_peak, 4),
                            "peak_source": peak_src, "alg_bytes": alg_bytes_sketch(cfg),
                            "kernel_ms": round(k_sketch_ms, 5),
                            "traffic": _ncu_traffic(f"r01_ncu_sketch_{cfg.name}.txt"),
                            "with_plan": {"ms": round(sk_ms, 5), "achieved": round(sketch_gbs, 1),
                                          "frac": round(sketch_gbs / hbm_peak, 4),
                                          "note": "whole csk_sketch call: plan (S1 hash + S2 stable bucketing) + sketch kernel"}},
        "clocks": clocks,
        "gpu_launches": 4 * args.steps,
        "gpu_launches_note": "per step: k_plan_hist (one cooperative launch: hash, per-CTA histograms, scan, "
                             "slots, group sorts), k_sketch_dense (or k_sketch_dense_wpb / k_sketch_csr), "
                             "k_row_norms_exact, k_loop; libcsk's own kernels only (profiles/r02_launches_C3.csv: "
                             "k_loop 91 % of their GPU time)",
    }

    # ---- the sketch with a cached plan (csk_plan once, csk_sketch_planned per step): the plan depends
    #      only on (seed, m, d), so a caller solving many right-hand sides / matrices of one shape
    #      pays it once
    perm_c, offs_c = csk.csk_plan(cfg.m, cfg.d, seed=cfg.sketch_seed, ctx=ctx)
    cp = []
    for k in range(6):
        if do_flush:
            flush.fill_(1.0)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record(stream)
        csk.csk_sketch_planned(p.A, p.b, d, perm_c, offs_c, ctx=ctx, out=(At, bt, nsq))
        e[1].record(stream)
        torch.cuda.synchronize()
        if k:
            cp.append(e[0].elapsed_time(e[1]))
    cp_ms = statistics.median(cp)
    out["roofline_sketch"]["cached_plan"] = {
        "ms": round(cp_ms, 5), "achieved": round(alg_bytes_sketch(cfg) / (cp_ms * 1e-3) / 1e9, 1),
        "frac": round(alg_bytes_sketch(cfg) / (cp_ms * 1e-3) / 1e9 / hbm_peak, 4),
        "note": "csk_sketch_planned with a plan from csk_plan (computed once): sketch kernel + exact-order norms"}
    del perm_c, offs_c

    # ---- e2e: the public API with HOST buffers, copies inside the timed region
    if not args.no_e2e:
        Ah = p.A.cpu().pin_memory()
        bh = p.b.cpu().pin_memory()
        xsh = p.x_star.cpu().pin_memory()
        for _ in range(1):
            csk.csk_run_host(Ah, bh, d, seed=cfg.sketch_seed, x_star=xsh, tol=cfg.tol, max_iters=cfg.max_iters, ctx=ctx)
        times = []
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            ta = time.perf_counter()
            xh, rep = csk.csk_run_host(Ah, bh, d, seed=cfg.sketch_seed, x_star=xsh, tol=cfg.tol,
                                       max_iters=cfg.max_iters, ctx=ctx)
            times.append((time.perf_counter() - ta) * 1e3)
        e2e_ms = _max_over_ranks(dist, sum(times) / len(times))
        out["e2e"] = {"value": round(e2e_ms, 4), "unit": "ms",
                      "h2d_bytes_per_step": 8 * cfg.m * cfg.n + 8 * cfg.m + 16 * cfg.n,
                      "d2h_bytes_per_step": 8 * cfg.n + 32,
                      "api": "csk_run_host (C ABI, pinned host buffers)"}
        del Ah, bh

    # ---- CPU oracle beside it (rank 0, N = 1 only)
    if rank == 0 and ws == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(cfg, p)

    # ---- other configs (rank 0, N = 1): evidence for every §8(a) regime
    if rank == 0 and ws == 1 and not args.no_extras:
        out["per_config"] = extras(csk, ctx, [c for c in ("C1", "C2", "C4") if c != cfg.name], flush)
        if cfg.name != "C5":
            out["per_config"]["C5"] = c5_extra(csk, ctx)
        if not args.no_uncapped:
            out["per_config"]["C4_uncapped"] = c4_uncapped(csk, ctx)
        # the paper's comparison (Table 1 columns): MWRK on the unsketched system
        out["vs_mwrk"] = mwrk_compare(csk, ctx, cfg, p, ms_step, it)
        out["stop_modes"] = stop_modes(csk, ctx, cfg, p)
    return out


def stop_modes(csk, ctx, cfg, p, cap=300):
    """The loop's cost per iteration in both stop rules on this config's sketch: RES on the
    iterate error (x* known; the timed step) and the residual stop (x* unknown, S:279:
    ||b~ - A~ x_k||^2 / ||b~||^2 formed in the same pass), each capped at `cap` iterations."""
    At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed, ctx=ctx)
    x = torch.zeros(cfg.n, dtype=torch.float64, device="cuda")
    out = {"capped_at": cap}
    for name, xs in (("x_star", p.x_star), ("residual", None)):
        best = None
        for _ in range(3):
            x.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            csk.csk_solve_async(At, bt, nsq, x, x_star=xs, tol=1e-30, max_iters=cap, ctx=ctx)
            ev[1].record()
            rep = csk.csk_solve_wait(ctx)
            torch.cuda.synchronize()
            us = ev[0].elapsed_time(ev[1]) * 1e3 / max(rep.iterations, 1)
            best = us if best is None else min(best, us)
        out[name + "_us_per_iteration"] = round(best, 3)
    del At, bt, nsq
    return out


def c5_extra(csk, ctx, cap=None):
    """C5 on one GPU (CSR input; A~ = 40000 x 2000 = 640 MB, far above on-chip capacity): the CSR
    sketch, and the loop to RES <= 1e-6 (the metric; ~2.6k iterations) -- time to 1e-6,
    per-iteration time and the HBM rate of the rows it streams (TMA ring) every iteration."""
    cfg = CONFIGS["C5"]
    p = make_config(cfg, "cuda")
    d, n = cfg.d, cfg.n
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    res = None
    for k in range(2):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        x.zero_()
        e[0].record()
        At, bt, nsq = csk.csk_sketch_csr(p.row_ptr, p.col, p.val, p.b, n, d, seed=cfg.sketch_seed, ctx=ctx)
        e[1].record()
        csk.csk_solve_async(At, bt, nsq, x, x_star=p.x_star, tol=cfg.tol, max_iters=cap or cfg.max_iters, ctx=ctx)
        e[2].record()
        rep = csk.csk_solve_wait(ctx)
        torch.cuda.synchronize()
        res = (e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), rep, csk.csk_last_kernel_ms("sketch", ctx=ctx))
        del At, bt, nsq
    sk, sv, rep, skk = res
    t = csk.csk_last_solve_tiers(ctx=ctx)
    G, rg = t["num_ctas"], 8 // max(t["group_warps"], 1)
    rows_cta = -(-d // G)
    per_group = -(-rows_cta // rg)
    resident = min(per_group, t["reg_rows"] + t["tmem_rows"] + t["smem_rows"])
    streamed_rows = max(0, d - G * rg * resident)
    us_it = sv * 1e3 / max(rep.iterations, 1)
    gbs = 8.0 * n * streamed_rows / (us_it * 1e-6) / 1e9
    peak = _peaks()[0]
    nnz = int(p.row_ptr[-1].item())
    sk_bytes = 12 * nnz + 8 * (cfg.m + 1) + 8 * cfg.m + 8 * d * n + 16 * d
    return {"ms_per_step": round(sk + sv, 4), "sketch_ms": round(sk, 4), "solve_ms": round(sv, 4),
            "sketch_bytes": sk_bytes, "sketch_hbm_gbs": round(sk_bytes / (sk * 1e-3) / 1e9, 1),
            "sketch_hbm_frac_with_plan": round(sk_bytes / (sk * 1e-3) / 1e9 / peak, 4),
            "sketch_kernel_ms": round(skk, 4),
            "sketch_kernel_hbm_frac": round(sk_bytes / (skk * 1e-3) / 1e9 / peak, 4) if skk > 0 else None,
            "sketch_kernel_note": "k_sketch_csr alone (libcsk events); its floor is the random row gather: "
                                  "tools/microbench_gather.cu reads the same rows in the same order with "
                                  "nothing folded in 0.57 ms (0.64 ms with the A~ writes), DESIGN.md section 6",
            "iterations": rep.iterations, "final_res": rep.final_res,
            "termination": ["converged", "max_iters", "stagnated"][rep.termination],
            "us_per_iteration": round(us_it, 3), "tiers": t,
            "streamed_rows_per_iteration": streamed_rows,
            "loop_streamed_hbm_gbs": round(gbs, 1), "loop_streamed_hbm_frac": round(gbs / peak, 4),
            "note": "time to RES <= 1e-6 on one GPU (second of two runs); rows past the on-chip tiers are "
                    "re-read every iteration through the TMA stream ring; 96 MB of them stay L2-resident "
                    "(evict_last copies, the rest evict_first), so loop_streamed_hbm_gbs is algorithmic bytes per "
                    "iteration time and may exceed the HBM copy peak"}


def c4_uncapped(csk, ctx, cap=2_000_000):
    """C4 without the 50k cap: the loop run to RES <= 1e-6 (~7e5 iterations), once."""
    cfg = CONFIGS["C4"]
    p = make_config(cfg, "cuda")
    At, bt, nsq = csk.csk_sketch(p.A, p.b, cfg.d, seed=cfg.sketch_seed, ctx=ctx)
    xs = p.x_star
    del p
    torch.cuda.empty_cache()
    x = torch.zeros(cfg.n, dtype=torch.float64, device="cuda")
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    csk.csk_solve_async(At, bt, nsq, x, x_star=xs, tol=cfg.tol, max_iters=cap, ctx=ctx)
    e[1].record()
    rep = csk.csk_solve_wait(ctx)
    torch.cuda.synchronize()
    ms = e[0].elapsed_time(e[1])
    del At, bt, nsq
    torch.cuda.empty_cache()
    return {"loop_ms": round(ms, 2), "iterations": rep.iterations, "final_res": rep.final_res,
            "termination": ["converged", "max_iters", "stagnated"][rep.termination],
            "us_per_iteration": round(ms * 1e3 / max(rep.iterations, 1), 3), "cap": cap,
            "note": "C4 loop without the configs' 50k cap, to RES <= 1e-6 (one run; the sketch is in "
                    "per_config.C4.sketch_ms)"}


def mwrk_compare(csk, ctx, cfg, p, csk_ms, csk_it):
    """MWRK (Remark 1) on (A, b) itself: row norms of A + the same persistent loop with
    d = m rows (those that do not fit on chip are re-read from HBM every iteration).  IT speedup
    and time speedup as defined at P:178 (MWRK over CSK; CSK time = sketch + loop)."""
    x = torch.zeros(cfg.n, dtype=torch.float64, device="cuda")

    def run(ev=None):
        x.zero_()
        if ev:
            ev[0].record()
        nsq = csk.csk_row_norms(p.A, ctx=ctx)
        csk.csk_solve_async(p.A, p.b, nsq, x, x_star=p.x_star, tol=cfg.tol, max_iters=cfg.max_iters, ctx=ctx)
        if ev:
            ev[1].record()
        return csk.csk_solve_wait(ctx)

    run()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    rep = run(ev)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    geo = csk.csk_last_solve_geometry(ctx=ctx)
    return {"config": cfg.name, "method": "MWRK on the unsketched system (P:69 Remark 1), same loop kernel, d = m",
            "iterations": rep.iterations, "termination": ["converged", "max_iters", "stagnated"][rep.termination],
            "final_res": rep.final_res, "ms": round(ms, 4), "us_per_iteration": round(ms * 1e3 / max(rep.iterations, 1), 3),
            "it_speedup": round(rep.iterations / max(csk_it, 1), 4), "time_speedup": round(ms / csk_ms, 3),
            "resident_rows_per_cta": geo["smem_rows"],
            "note": "IT speedup = IT(MWRK)/IT(CSK), time speedup = time(MWRK)/time(CSK) (P:178); "
                    "MWRK time = row norms + loop, CSK time = sketch + loop"}


def extras(csk, ctx, names, flush):
    _, sm_max_mhz, _ = _peaks()
    smem_gbs = 148 * SMEM_BYTES_PER_CLK_PER_SM * sm_max_mhz * 1e6 / 1e9
    res = {}
    for nm in names:
        cfg = CONFIGS[nm]
        p = make_config(cfg, "cuda")
        d, n = cfg.d, cfg.n
        At = torch.empty(d, n, dtype=torch.float64, device="cuda")
        bt = torch.empty(d, dtype=torch.float64, device="cuda")
        nsq = torch.empty(d, dtype=torch.float64, device="cuda")
        x = torch.zeros(n, dtype=torch.float64, device="cuda")
        st = torch.cuda.current_stream()
        rows = []
        for k in range(4):
            flush.fill_(1.0)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            x.zero_()
            e[0].record(st)
            csk.csk_sketch(p.A, p.b, d, seed=cfg.sketch_seed, ctx=ctx, out=(At, bt, nsq))
            e[1].record(st)
            csk.csk_solve_async(At, bt, nsq, x, x_star=p.x_star, tol=cfg.tol, max_iters=cfg.max_iters, ctx=ctx)
            e[2].record(st)
            rep = csk.csk_solve_wait(ctx)
            if k:
                rows.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), rep))
        sk = statistics.median(r[0] for r in rows)
        sv = statistics.median(r[1] for r in rows)
        rep = rows[-1][2]
        res[nm] = {"ms_per_step": round(sk + sv, 4), "sketch_ms": round(sk, 5), "solve_ms": round(sv, 4),
                   "iterations": rep.iterations, "final_res": rep.final_res,
                   "termination": ["converged", "max_iters", "stagnated"][rep.termination],
                   "iterations_per_s": round(rep.iterations / (sv * 1e-3), 1),
                   "us_per_iteration": round(sv * 1e3 / max(rep.iterations, 1), 4),
                   "sketch_hbm_gbs": round(alg_bytes_sketch(cfg) / (sk * 1e-3) / 1e9, 1),
                   "loop_gbs": round(alg_bytes_iter(cfg) * rep.iterations / (sv * 1e-3) / 1e9, 1)}
        # t_bw = the loop's bytes per iteration over the SMEM yardstick, beside t_iter
        t_iter = sv * 1e3 / max(rep.iterations, 1)
        t_bw = alg_bytes_iter(cfg) / (smem_gbs * 1e9) * 1e6
        res[nm].update({"loop_t_bw_us": round(t_bw, 4), "loop_t_bw_frac": round(t_bw / t_iter, 4),
                        "loop_floor_note": "t_iter's fixed part (grid exchange + winner-row fetch + update) is "
                                           "~2.3-2.5 us on 148 CTAs (one row per CTA, profiles/r02_loop_scan.txt); "
                                           "C1/C2 run one 16-CTA cluster (DSMEM exchange)"})
        del p, At
        torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------ oracle arm
def _oracle_sample(cfg, A, b, xs, budget_s=20.0):
    """Time the oracle (1 core) on the workload: sketch + norms + loop.  Small configs run
    whole; if the full loop would exceed ``budget_s`` the loop is run for a bounded number
    of iterations and the per-iteration time is extrapolated to the GPU's iteration count."""
    import oracle
    t0 = time.perf_counter()
    At, bt = oracle.sketch_dense(A, b, cfg.d, seed=cfg.sketch_seed)
    nsq = oracle.row_norms(At)
    t_sketch = time.perf_counter() - t0
    t1 = time.perf_counter()
    probe = oracle.solve(At, bt, nsq, x_star=xs, tol=cfg.tol, max_iters=20)
    t_probe = (time.perf_counter() - t1) / max(probe.iterations, 1)
    cap = max(1, int((budget_s - t_sketch) / max(t_probe, 1e-9)))
    t2 = time.perf_counter()
    r = oracle.solve(At, bt, nsq, x_star=xs, tol=cfg.tol, max_iters=min(cfg.max_iters, cap))
    t_loop = time.perf_counter() - t2
    complete = r.termination == 0 or r.iterations >= cfg.max_iters
    per_it = t_loop / max(r.iterations, 1)
    return t_sketch, t_loop, per_it, r, complete


def _host_info(core):
    """CPU model, logical CPU count and the pinned core's frequency governor."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    gov = None
    try:
        gov = open(f"/sys/devices/system/cpu/cpu{core}/cpufreq/scaling_governor").read().strip()
    except OSError:
        gov = "unavailable"
    return {"cpu_model": model, "nproc": os.cpu_count(), "pinned_core": core, "governor": gov}


class _PinnedCore:
    """Pin the calling thread (the oracle runs in it, through ctypes) to one core for the timing."""

    def __enter__(self):
        self.prev = os.sched_getaffinity(0)
        self.core = sorted(self.prev)[-1]
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.prev)


def _oracle_timed(cfg, A, b, xs, runs=3, warmup=1, budget_s=20.0):
    """Median over `runs` pinned single-core oracle samples (after `warmup` untimed ones)."""
    with _PinnedCore() as pc:
        for _ in range(warmup):
            _oracle_sample(cfg, A, b, xs, budget_s=min(budget_s, 5.0))
        samples = [_oracle_sample(cfg, A, b, xs, budget_s=budget_s) for _ in range(runs)]
        info = _host_info(pc.core)
    vals = []
    for t_sketch, t_loop, per_it, r, complete in samples:
        vals.append((t_sketch + (t_loop if complete else per_it * cfg.max_iters)) * 1e3)
    med = statistics.median(vals)
    t_sketch, t_loop, per_it, r, complete = samples[vals.index(sorted(vals)[len(vals) // 2])]
    if complete:
        sample = f"whole {cfg.name} solve (sketch + {r.iterations} iterations), median of {runs} pinned runs"
    else:
        sample = (f"{cfg.name}: sketch + {r.iterations} iterations timed, loop extrapolated "
                  f"to {cfg.max_iters} at {per_it * 1e3:.2f} ms/iteration, median of {runs} pinned runs")
    return {"value": round(med, 3), "unit": "ms", "cores": 1, "kind": "oracle", "sample": sample,
            "runs_ms": [round(v, 3) for v in vals], "iterations": r.iterations,
            "sketch_ms": round(t_sketch * 1e3, 3), "loop_ms_per_iteration": round(per_it * 1e3, 4),
            "host": info}


def cpu_baseline(cfg, p):
    """The oracle on one pinned host core, on the same bytes as the GPU run (D2H copies)."""
    if cfg.kind == "csr":
        return {"value": None, "unit": "ms", "cores": 1, "kind": "oracle",
                "sample": "not timed for the CSR config in the default run"}
    A = p.A.cpu().numpy()
    b = p.b.cpu().numpy()
    xs = p.x_star.cpu().numpy()
    return _oracle_timed(cfg, A, b, xs)


def run_reference(args):
    """--impl reference: the CPU oracle (plain C, 1 thread, pinned) on our arm's config/metric, on
    the SAME bytes our arm solves: the problem is drawn with the same torch Philox stream on the
    GPU (as our arm does) and copied to the host; only without a GPU is it drawn on the CPU."""
    import oracle
    cfg = CONFIGS[args.config]
    on_gpu = torch.cuda.is_available()
    p = make_config(cfg, "cuda" if on_gpu else "cpu")
    A, b, xs = p.A.cpu().numpy(), p.b.cpu().numpy(), p.x_star.cpu().numpy()
    del p
    oracle.build()
    runs = max(3, min(args.steps, 5))
    warm = max(1, min(args.warmup, 5))  # the requested W untimed samples (capped at 5: ~3 s each)
    cb = _oracle_timed(cfg, A, b, xs, runs=runs, warmup=warm)
    v = cb["value"]
    return {"metric": METRIC, "value": v, "unit": "ms", "n_gpus": 0,
            "steps": runs, "warmup": warm, "ms_per_step": v,
            "higher_is_better": False, "impl": "reference", "dtype": "f64",
            "data": ("synthetic (torch Philox on the GPU, copied to the host: the same bytes as our arm; csk_synth.py)"
                     if on_gpu else "synthetic (torch Philox CPU stream; no GPU here, csk_synth.py)"),
            "config": _config_dict(cfg),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "iterations": cb["iterations"], "vs_baseline": None,
            "note": f"each step = one pinned single-core oracle sample (median of {runs}); "
                    "--steps K is clamped to 3..5 samples and --warmup W to 1..5 so the arm finishes in about a minute"}


def _sharded_roofline(dist, cfg, ws, it, kloop, ksk):
    """Roofline of the dominant kernel (the SYS k_loop) at N ranks: this rank's rows of A~ per
    iteration over one GPU's on-chip yardstick (max of the kernel time over ranks), beside the
    sketch kernel against HBM."""
    hbm_peak, sm_max_mhz, peak_src = _peaks()
    k_loop_ms = _max_over_ranks(dist, sum(kloop) / len(kloop))
    k_sk_ms = _max_over_ranks(dist, sum(ksk) / len(ksk))
    rows = -(-cfg.d // ws)
    loop_bytes = (8 * rows * cfg.n + 16 * rows) * it
    smem_peak = 148 * SMEM_BYTES_PER_CLK_PER_SM * sm_max_mhz * 1e6 / 1e9
    gbs = loop_bytes / (k_loop_ms * 1e-3) / 1e9
    sk_bytes = alg_bytes_sketch(cfg) / ws
    return {"kernel": "k_loop (SYS: two-level cross-GPU exchange), per rank", "bound": "smem",
            "achieved": round(gbs, 1), "peak": round(smem_peak, 1), "unit": "GB/s", "frac": round(gbs / smem_peak, 4),
            "traffic": None, "alg_bytes_per_iteration_per_rank": 8 * rows * cfg.n + 16 * rows,
            "kernel_ms": round(k_loop_ms, 5), "us_per_iteration": round(k_loop_ms * 1e3 / max(it, 1), 3),
            "peak_source": f"derived: 148 SM x {SMEM_BYTES_PER_CLK_PER_SM} B/clk x {sm_max_mhz:.0f} MHz",
            "sketch": {"kernel": "k_sketch_dense (this rank's rows)", "bound": "hbm",
                       "achieved": round(sk_bytes / (k_sk_ms * 1e-3) / 1e9, 1), "peak": hbm_peak, "unit": "GB/s",
                       "frac": round(sk_bytes / (k_sk_ms * 1e-3) / 1e9 / hbm_peak, 4), "kernel_ms": round(k_sk_ms, 5),
                       "peak_source": peak_src},
            "timing": "CUDA events recorded by libcsk around the kernels (csk_ctx_set_timing), max over ranks"}


def run_sharded(args, dist, rank, ws):
    """N > 1: the same workload, sharded (S9/S10); CUDA events, max over ranks."""
    import paper_2004_02480_b200 as csk
    from paper_2004_02480_b200.parallel import init_comm, row_shard

    cfg = CONFIGS[args.config]
    dev = torch.device("cuda", torch.cuda.current_device())
    p = make_config(cfg, dev)                    # every rank draws the same problem ...
    lo, hi = row_shard(cfg.m, ws, rank)          # ... and keeps its contiguous row shard
    A_loc = p.A[lo:hi].contiguous()
    b_loc = p.b[lo:hi].contiguous()
    xs = p.x_star
    del p
    torch.cuda.empty_cache()
    ctx = csk.Context()
    init_comm(ctx)
    csk.csk_ctx_set_timing(True, ctx=ctx)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()

    def step(ev=None):
        if ev:
            ev[0].record(st)
        At, bt, nsq, dlo, dhi = csk.csk_sketch_sharded(A_loc, b_loc, lo, cfg.m, cfg.d, ws, rank,
                                                       seed=cfg.sketch_seed, ctx=ctx)
        if ev:
            ev[1].record(st)
        x, rep = csk.csk_solve_sharded(At, bt, nsq, dlo, dhi, cfg.d, cfg.n, x_star=xs, tol=cfg.tol,
                                       max_iters=cfg.max_iters, ctx=ctx)
        if ev:
            ev[2].record(st)
        return rep

    for _ in range(args.warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev.index)
    sampler.start()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    reps = []
    _barrier(dist)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kloop, ksk = [], []
    for k in range(args.steps):
        flush.fill_(1.0)
        reps.append(step(evs[k]))
        torch.cuda.synchronize()  # (outside the events of step k)
        kloop.append(csk.csk_last_kernel_ms("loop", ctx=ctx))
        ksk.append(csk.csk_last_kernel_ms("sketch", ctx=ctx))
        sampler.sample_now()
    torch.cuda.synchronize()
    _barrier(dist)
    t1 = time.perf_counter()
    sampler.stop()
    sk = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    sv = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    ms = _max_over_ranks(dist, sk + sv)
    sk = _max_over_ranks(dist, sk)
    sv = _max_over_ranks(dist, sv)
    it = reps[-1].iterations
    out = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (torch Philox, PAPER.md:180 recipe; csk_synth.py)",
        "config": {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "d": cfg.d, "kind": cfg.kind,
                   "tol": cfg.tol, "max_iters": cfg.max_iters, "parallelism": f"row-sharded x{ws} (NCCL)",
                   "l2": "flushed between steps (256 MiB write, untimed)"},
        "iterations": it, "final_res": reps[-1].final_res,
        "termination": ["converged", "max_iters", "stagnated"][reps[-1].termination],
        "iterations_per_s": round(it / (sv * 1e-3), 1), "sketch_ms": round(sk, 5), "solve_ms": round(sv, 4),
        "sketch_hbm_gbs": round(alg_bytes_sketch(cfg) / (sk * 1e-3) / 1e9, 1),
        "clocks": sampler.summary(t0, t1),
        "roofline": _sharded_roofline(dist, cfg, ws, it, kloop, ksk),
        "gpu_launches": args.steps * 4,
        "gpu_launches_note": "per step: the plan (k_plan_hist), "
                             "k_sketch_dense, k_loop (+ the NCCL reduce-scatter of S9 and the NCCL handle/barrier "
                             "collectives of S10)",
    }
    # ---- e2e at N GPUs: every rank's pinned host shard -> device, S9 + S10 through the public
    #      API, x back to the host (max over ranks of the per-step wall time)
    if not args.no_e2e:
        A_h = A_loc.cpu().pin_memory()
        b_h = b_loc.cpu().pin_memory()
        xs_h = xs.cpu().pin_memory()
        times = []
        for k in range(4):
            _barrier(dist)
            torch.cuda.synchronize()
            ta = time.perf_counter()
            A_d = A_h.to(dev, non_blocking=True)
            b_d = b_h.to(dev, non_blocking=True)
            xs_d = xs_h.to(dev, non_blocking=True)
            At, bt, nsq, dlo, dhi = csk.csk_sketch_sharded(A_d, b_d, lo, cfg.m, cfg.d, ws, rank,
                                                           seed=cfg.sketch_seed, ctx=ctx)
            x, rep = csk.csk_solve_sharded(At, bt, nsq, dlo, dhi, cfg.d, cfg.n, x_star=xs_d, tol=cfg.tol,
                                           max_iters=cfg.max_iters, ctx=ctx)
            x_h = x.cpu()
            torch.cuda.synchronize()
            if k:
                times.append((time.perf_counter() - ta) * 1e3)
            del A_d, b_d, xs_d, At, bt, nsq, x, x_h
        e2e_ms = _max_over_ranks(dist, sum(times) / len(times))
        out["e2e"] = {"value": round(e2e_ms, 4), "unit": "ms",
                      "h2d_bytes_per_step": 8 * (hi - lo) * cfg.n + 8 * (hi - lo) + 8 * cfg.n,
                      "d2h_bytes_per_step": 8 * cfg.n,
                      "api": "csk_sketch_sharded + csk_solve_sharded (binding over the C ABI), pinned host shards "
                             "per rank; max over ranks"}
    if not args.no_extras:
        out["per_config"] = sharded_extras(csk, ctx, dist, rank, ws)
    csk.comm_destroy(ctx)
    return out


def sharded_extras(csk, ctx, dist, rank, ws, reps=2):
    """N ranks on north_star's multi-GPU configs: C4 (dense 8 GB, S9 reduce-scatter + S10, the 50k
    cap) and C5 (CSR, S9 by row routing -- bit-identical to one GPU -- + S10 to RES <= 1e-6).  Each
    rank draws the same problem and keeps its row shard; CUDA events, max over ranks."""
    from paper_2004_02480_b200.parallel import row_shard
    hbm_peak, sm_max_mhz, _ = _peaks()
    smem_peak = 148 * SMEM_BYTES_PER_CLK_PER_SM * sm_max_mhz * 1e6 / 1e9
    dev = torch.device("cuda", torch.cuda.current_device())
    res = {}
    for name in ("C4", "C5"):
        cfg = CONFIGS[name]
        p = make_config(cfg, dev)
        lo, hi = row_shard(cfg.m, ws, rank)
        if cfg.kind == "csr":
            rp_l = p.row_ptr[lo:hi + 1].contiguous()
            col, val = p.col, p.val
            b_l = p.b[lo:hi].contiguous()
            sk_bytes = 12 * (int(p.row_ptr[hi]) - int(p.row_ptr[lo])) + 16 * (hi - lo) + 8 * cfg.d * cfg.n // ws
        else:
            A_l = p.A[lo:hi].contiguous()
            b_l = p.b[lo:hi].contiguous()
            del p.A
            sk_bytes = 8 * (hi - lo) * (cfg.n + 1) + 8 * cfg.d * cfg.n // ws
        xs = p.x_star
        torch.cuda.empty_cache()
        rows = []
        for k in range(reps + 1):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            _barrier(dist)
            torch.cuda.synchronize()
            e[0].record()
            if cfg.kind == "csr":
                At, bt, nsq, dlo, dhi = csk.csk_sketch_csr_sharded(rp_l, col, val, b_l, lo, cfg.m, cfg.n, cfg.d, ws,
                                                                   rank, seed=cfg.sketch_seed,
                                                                   mode=csk.SHARD_ROUTE_ROWS, ctx=ctx)
            else:
                At, bt, nsq, dlo, dhi = csk.csk_sketch_sharded(A_l, b_l, lo, cfg.m, cfg.d, ws, rank,
                                                               seed=cfg.sketch_seed, ctx=ctx)
            e[1].record()
            x, rep = csk.csk_solve_sharded(At, bt, nsq, dlo, dhi, cfg.d, cfg.n, x_star=xs, tol=cfg.tol,
                                           max_iters=cfg.max_iters, ctx=ctx)
            e[2].record()
            torch.cuda.synchronize()
            kl = csk.csk_last_kernel_ms("loop", ctx=ctx)
            if k:
                rows.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), kl, rep))
            del At, bt, nsq, x
        sk = _max_over_ranks(dist, statistics.median(r[0] for r in rows))
        sv = _max_over_ranks(dist, statistics.median(r[1] for r in rows))
        kl = _max_over_ranks(dist, statistics.median(r[2] for r in rows))
        rep = rows[-1][3]
        it = max(rep.iterations, 1)
        loc_rows = -(-cfg.d // ws)
        loop_gbs = (8 * loc_rows * cfg.n + 16 * loc_rows) * it / (kl * 1e-3) / 1e9
        res[name] = {"ms_per_step": round(sk + sv, 4), "sketch_ms": round(sk, 4), "solve_ms": round(sv, 4),
                     "iterations": rep.iterations, "final_res": rep.final_res,
                     "termination": ["converged", "max_iters", "stagnated"][rep.termination],
                     "us_per_iteration": round(sv * 1e3 / it, 3),
                     "sketch": {"mode": "row routing (bit-identical to 1 GPU)" if cfg.kind == "csr" else
                                "reduce-scatter of partial A~", "bytes_per_rank": sk_bytes,
                                "achieved_gbs_per_rank": round(sk_bytes / (sk * 1e-3) / 1e9, 1),
                                "frac_of_hbm": round(sk_bytes / (sk * 1e-3) / 1e9 / hbm_peak, 4)},
                     "loop_roofline_per_rank": {"bound": "smem", "achieved": round(loop_gbs, 1),
                                                "peak": round(smem_peak, 1), "unit": "GB/s",
                                                "frac": round(loop_gbs / smem_peak, 4), "kernel_ms": round(kl, 4)},
                     "note": "S9 + S10 at N ranks; the loop's exchange is one key per rank over NVLink per iteration"}
        del p
        torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded (S9/S10) path even at N = 1 (a 1-rank NCCL communicator; tests the N > 1 code path)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-uncapped", action="store_true", help="skip the uncapped C4 run (~4 s)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        print(json.dumps(run_reference(args)))
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun (the driver's own launch sets
        # WORLD_SIZE and lands below directly)
        import random
        port = str(29500 + random.randrange(1000))
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", port, os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    dist, rank, ws, _ = _dist(force=args.sharded)
    if ws != args.gpus and not (args.sharded and ws == 1):
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws} ranks were launched")
    out = run_ours(args, dist, rank, ws) if ws == 1 and not args.sharded else run_sharded(args, dist, rank, ws)
    if rank == 0:
        print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
