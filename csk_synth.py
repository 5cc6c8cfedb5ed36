"""Seeded synthetic workloads for the CSK hot path -- shared by tests, bench and smoke.

This module holds NO arithmetic of the method (no hashing, sketching, norms or
iteration): it only draws the problem (A, x*, b = A x*) the paper's experiments
use ("generate A and x* using randn ... b = A x* ... x0 = 0") in the five
shapes BASELINE.json names (configs C1..C5), so that the CUDA path and the CPU
oracle can be fed identical bytes.  The recipe is restated in DESIGN.md §5.

Generation is torch's Philox stream on the requested device, seeded with
``1000 + config index``; x* is drawn first, then A (then any extra structure).
Everything is fp64.  The CSR generator draws, per row, a uniformly random
10-subset of the n columns (top-k of i.i.d. uniforms, an unbiased
without-replacement sample), sorted ascending, with N(0,1) values.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    d: int
    kind: str                 # "gauss" | "lognormal_rows" | "illcond" | "csr"
    gen_seed: int             # torch generator seed (1000 + index)
    sketch_seed: int = 0      # SplitMix64 seed of the count sketch (configs: seed 0)
    tol: float = 1e-6         # RES threshold
    max_iters: int = 50_000   # iteration cap (BASELINE configs)
    nnz_per_row: int = 0      # CSR only

    @property
    def bytes_A(self) -> int:
        if self.kind == "csr":
            nnz = self.m * self.nnz_per_row
            return 12 * nnz + 8 * (self.m + 1)
        return 8 * self.m * self.n


# BASELINE.json "configs" [0..4]
CONFIGS = {
    "C1": Config("C1", 1_000, 50, 500, "gauss", 1000),
    "C2": Config("C2", 20_000, 200, 2_000, "gauss", 1001),
    "C3": Config("C3", 100_000, 500, 5_000, "lognormal_rows", 1002),
    "C4": Config("C4", 1_000_000, 1_000, 10_000, "illcond", 1003),
    "C5": Config("C5", 4_000_000, 2_000, 40_000, "csr", 1004, nnz_per_row=10),
}


@dataclass
class DenseProblem:
    A: torch.Tensor       # m x n fp64, row-major
    b: torch.Tensor       # m
    x_star: torch.Tensor  # n


@dataclass
class CsrProblem:
    row_ptr: torch.Tensor  # int64[m+1]
    col: torch.Tensor      # int32[nnz], ascending within a row
    val: torch.Tensor      # fp64[nnz]
    b: torch.Tensor        # fp64[m]
    x_star: torch.Tensor   # fp64[n]
    n: int


def _gen(device, seed: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def make_dense(m: int, n: int, kind: str = "gauss", seed: int = 1000,
               device="cpu") -> DenseProblem:
    """A, x* ~ randn, b = A x* (P:180); ``kind`` adds the configs' structure."""
    g = _gen(device, seed)
    x_star = torch.randn(n, generator=g, device=device, dtype=torch.float64)
    A = torch.randn(m, n, generator=g, device=device, dtype=torch.float64)
    if kind == "lognormal_rows":      # C3: row i scaled by exp(N(0,1))
        A *= torch.exp(torch.randn(m, 1, generator=g, device=device, dtype=torch.float64))
    elif kind == "illcond":           # C4: columns scaled by logspace(0, 2, n)
        A *= torch.logspace(0, 2, n, device=device, dtype=torch.float64)
    elif kind != "gauss":
        raise ValueError(kind)
    b = A @ x_star
    return DenseProblem(A=A, b=b, x_star=x_star)


def make_csr(m: int, n: int, nnz_per_row: int = 10, seed: int = 1004, device="cpu",
             chunk: int = 100_000) -> CsrProblem:
    """CSR A with exactly ``nnz_per_row`` distinct uniform columns per row, N(0,1) values."""
    g = _gen(device, seed)
    x_star = torch.randn(n, generator=g, device=device, dtype=torch.float64)
    cols = []
    for lo in range(0, m, chunk):
        rows = min(chunk, m - lo)
        u = torch.rand(rows, n, generator=g, device=device, dtype=torch.float32)
        c = torch.topk(u, nnz_per_row, dim=1).indices
        cols.append(torch.sort(c, dim=1).values.to(torch.int32))
        del u
    col = torch.cat(cols).reshape(-1)
    val = torch.randn(m * nnz_per_row, generator=g, device=device, dtype=torch.float64)
    row_ptr = torch.arange(0, m + 1, device=device, dtype=torch.int64) * nnz_per_row
    b = (val.view(m, nnz_per_row) * x_star[col.view(m, nnz_per_row).long()]).sum(dim=1)
    return CsrProblem(row_ptr=row_ptr, col=col, val=val, b=b, x_star=x_star, n=n)


def make_config(cfg: Config | str, device="cpu"):
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if cfg.kind == "csr":
        return make_csr(cfg.m, cfg.n, cfg.nnz_per_row, cfg.gen_seed, device)
    return make_dense(cfg.m, cfg.n, cfg.kind, cfg.gen_seed, device)
