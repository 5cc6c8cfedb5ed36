"""Regenerates the values in hash_seed0_d500.txt with plain Python big-int arithmetic.

Test infrastructure: imports nothing from oracle/ or the package.  Reading R-1
of Definition 1: the SplitMix64 stream seeded with `seed` (Steele, Lea & Flood,
OOPSLA 2014, the sequential form: state += gamma, then the 64-bit finaliser); row i takes draw 2i
for its bucket h = floor(z * d / 2^64) and draw 2i+1 for its sign (-1 iff bit 63 is set).

    python tests/golden/gen_hash_seed0_d500.py      # prints the data lines of the golden file
"""
from __future__ import annotations

GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def splitmix64(seed: int):
    state = seed & M64
    while True:
        state = (state + GAMMA) & M64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        yield z ^ (z >> 31)


def count_sketch_map(seed: int, m: int, d: int):
    g = splitmix64(seed)
    h, s = [], []
    for _ in range(m):
        zh, zs = next(g), next(g)
        h.append((zh * d) >> 64)
        s.append(-1 if zs >> 63 else 1)
    return h, s


def golden_lines() -> list[str]:
    h, s = count_sketch_map(0, 1000, 500)
    cnt = [0] * 500
    for v in h:
        cnt[v] += 1
    h2, _ = count_sketch_map(0, 20000, 2000)
    c2 = [0] * 2000
    for v in h2:
        c2[v] += 1
    return [
        "h " + " ".join(str(v) for v in h[:12]),
        "s " + " ".join("+" if v > 0 else "-" for v in s[:12]),
        f"c1_empty {cnt.count(0)}",
        f"c1_max_bucket {max(cnt)}",
        f"c1_sign_sum {sum(s)}",
        f"c2_empty {c2.count(0)}",
        f"c2_max_bucket {max(c2)}",
    ]


if __name__ == "__main__":
    print("\n".join(golden_lines()))
