"""Algorithmic FLOP accounting: only what the method
must compute -- no masked upper triangle, no skipped chunks.

Visible (query, key) pairs of chunk j (0-based, chunk size c):
    Pairs_j = c^2 j + c(c+1)/2            and  sum_j Pairs_j = S(S+1)/2.
Per q-head, a pair costs 4 d FLOPs in the forward (QK^T and PV, 2 d each) and
10 d in the backward (S recompute, dP, dV, dK, dQ: 5 x 2 d).
    fwd_j = 4 d Hq Pairs_j,  bwd_j = 10 d Hq Pairs_j,  F = sum_j fwd_j = 2 d Hq S(S+1)
    SeCO step  = sum_j (fwd_j [stage 1] + fwd_j [rebuild] + bwd_j) = 4.5 F
    SpaCO step = F + sum_{j in I} (fwd_j + bwd_j) = F + 3.5 sum_{j in I} fwd_j
"""
from __future__ import annotations


def pairs(c: int, j: int) -> int:
    return c * c * j + c * (c + 1) // 2


def fwd_flops(hq: int, d: int, c: int, j: int) -> float:
    return 4.0 * d * hq * pairs(c, j)


def bwd_flops(hq: int, d: int, c: int, j: int) -> float:
    return 10.0 * d * hq * pairs(c, j)


def total_fwd(hq: int, d: int, seq: int) -> float:
    return 2.0 * d * hq * seq * (seq + 1)


def seco_step_flops(hq: int, d: int, seq: int, c: int) -> float:
    k = seq // c
    return sum(2 * fwd_flops(hq, d, c, j) + bwd_flops(hq, d, c, j) for j in range(k))


def spaco_step_flops(hq: int, d: int, seq: int, c: int, selected) -> float:
    k = seq // c
    return sum(fwd_flops(hq, d, c, j) for j in range(k)) + \
        sum(fwd_flops(hq, d, c, j) + bwd_flops(hq, d, c, j) for j in selected)
