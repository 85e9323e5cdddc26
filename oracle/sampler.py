"""O8 -- SpaCO chunk sampler and scales.  TEST INFRASTRUCTURE ONLY.

Alg. 2 line 4: "Randomly select t distinct indices from {1..k}".  The
random source is splitmix64 (Steele, Lea & Flood 2014) with state = seed, so the
host library (csrc/sampler.cpp) and this oracle -- two independent
implementations -- must agree bit for bit (DESIGN.md §3 reading Z7 / O8).

Modes (reading Z7, Z8, Z9):
  PAPER      t distinct indices (partial Fisher-Yates, index r + floor(u*(k-r)/2^64)),
             relay gamma = min(k/t, cap), seed scale s = 1       (Alg. 2 literally)
  HT         same draw, gamma = (k-1)/(t-1), s = k/t              (exactly unbiased for one layer)
  BERNOULLI  include i iff floor(u*k/2^64) < t, gamma = s = k/t   (the paper's independence model)
The cap (<= 0: none) bounds gamma in every mode.  Indices are 0-based and
returned strictly descending (processing order, reading Z10).
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
PAPER, HT, BERNOULLI = 0, 1, 2


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)


def sample_indices(k: int, t: int, seed: int, mode: int = PAPER):
    """The sampled set I (list of 0-based chunk indices, strictly descending)."""
    if not (1 <= t <= k):
        raise ValueError("need 1 <= t <= k")
    if mode == HT and t < 2:
        raise ValueError("HT mode needs t >= 2")
    rng = SplitMix64(seed)
    if mode in (PAPER, HT):
        a = list(range(k))
        for r in range(t):
            j = r + ((rng.next() * (k - r)) >> 64)
            a[r], a[j] = a[j], a[r]
        chosen = a[:t]
    elif mode == BERNOULLI:
        chosen = [i for i in range(k) if ((rng.next() * k) >> 64) < t]
    else:
        raise ValueError("unknown mode")
    return sorted(chosen, reverse=True)


def scales(k: int, t: int, cap: float = 2.0, mode: int = PAPER):
    """(relay gamma, seed scale s) as float32 values (each ratio computed in
    double and rounded once to float32, then capped)."""
    if mode == PAPER:
        g, s = k / t, 1.0
    elif mode == HT:
        g, s = (k - 1) / (t - 1), k / t
    elif mode == BERNOULLI:
        g, s = k / t, k / t
    else:
        raise ValueError("unknown mode")
    g32, s32 = np.float32(g), np.float32(s)
    if cap is not None and cap > 0:
        g32 = min(g32, np.float32(cap))
    return float(g32), float(s32)


def sample_and_scale(k, t, seed, cap=2.0, mode=PAPER):
    """(I, gamma, s) -- what spaco_sample_and_scale must return."""
    g, s = scales(k, t, cap, mode)
    return sample_indices(k, t, seed, mode), g, s
