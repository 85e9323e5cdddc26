"""O7 -- exact expectation of the SpaCO gradient for one attention layer, in closed
form and by exhaustive enumeration of sampled subsets.  TEST INFRASTRUCTURE ONLY.

§5 (Eq. 8-10) derives the compensation from independent survival
probabilities.  For ONE layer a gradient chain touches at most two chunks: the
loss chunk j and (through the relay) the cache chunk i < j.  Split the exact
SeCO gradient of chunk i's own K (likewise V) into
    loc_i   = dK^(i->i)                   (the chunk's own block)
    cross_i = sum_{j>i} dK^(j->i)          (deposited by later chunks, relayed)
Then with inclusion indicators 1[i in I]:
    dQ_j(I) = 1[j in I] s dQ_j
    dK_i(I) = 1[i in I] s loc_i + sum_{j>i} 1[i in I] 1[j in I] s gamma dK^(j->i)
and taking expectations (reading Z7):
    t-of-k uniform:   E = (t/k) s loc + t(t-1)/(k(k-1)) s gamma cross
    Bernoulli(rho):   E = rho s loc + rho^2 s gamma cross
"""
from __future__ import annotations

import itertools
import math

import numpy as np

from .attention import chunk_bwd
from .chunkwise import chunk_bounds, sparse_stage2


def decompose(q, k, v, do, sizes, scale=None, dtype=np.float64):
    """Exact per-chunk parts of the SeCO gradient: dict(dq, loc_k, loc_v, cross_k, cross_v)."""
    bounds = chunk_bounds(sizes)
    q, k, v, do = (np.asarray(a, dtype) for a in (q, k, v, do))
    dq = np.zeros_like(q)
    loc_k, loc_v = np.zeros_like(k), np.zeros_like(v)
    cross_k, cross_v = np.zeros_like(k), np.zeros_like(v)
    for (a, b) in bounds:
        dq_j, dk_src, dv_src = chunk_bwd(q[:, a:b], k, v, do[:, a:b], a, scale, dtype)
        dq[:, a:b] = dq_j
        loc_k[:, a:b] = dk_src[:, a:b]
        loc_v[:, a:b] = dv_src[:, a:b]
        cross_k[:, :a] += dk_src[:, :a]
        cross_v[:, :a] += dv_src[:, :a]
    return dict(dq=dq, loc_k=loc_k, loc_v=loc_v, cross_k=cross_k, cross_v=cross_v)


def closed_form_t_of_k(parts, k, t, gamma, s):
    """E[gradient] under uniform t-of-k sampling (Alg. 2 line 4 literal)."""
    p1 = t / k
    p2 = t * (t - 1) / (k * (k - 1)) if k > 1 else 0.0
    return dict(dq=p1 * s * parts["dq"],
                dk=p1 * s * parts["loc_k"] + p2 * s * gamma * parts["cross_k"],
                dv=p1 * s * parts["loc_v"] + p2 * s * gamma * parts["cross_v"])


def closed_form_bernoulli(parts, rho, gamma, s):
    """E[gradient] under independent inclusion with probability rho (P:303-307 model)."""
    return dict(dq=rho * s * parts["dq"],
                dk=rho * s * parts["loc_k"] + rho * rho * s * gamma * parts["cross_k"],
                dv=rho * s * parts["loc_v"] + rho * rho * s * gamma * parts["cross_v"])


def enumerate_t_of_k(q, k_, v, do, sizes, t, gamma, s, scale=None, dtype=np.float64):
    """Mean of the SpaCO stage-2 gradient over ALL C(k,t) subsets (each equally likely)."""
    kc = len(sizes)
    acc = None
    n = 0
    for subset in itertools.combinations(range(kc), t):
        g = sparse_stage2(q, k_, v, do, sizes, subset, gamma, s, scale, dtype)
        acc = {x: g[x].copy() for x in ("dq", "dk", "dv")} if acc is None else \
            {x: acc[x] + g[x] for x in acc}
        n += 1
    return {x: acc[x] / n for x in acc}


def enumerate_bernoulli(q, k_, v, do, sizes, rho, gamma, s, scale=None, dtype=np.float64):
    """Probability-weighted sum of the SpaCO gradient over all 2^k subsets."""
    kc = len(sizes)
    acc = None
    for mask in itertools.product((0, 1), repeat=kc):
        subset = [i for i in range(kc) if mask[i]]
        w = rho ** len(subset) * (1 - rho) ** (kc - len(subset))
        g = sparse_stage2(q, k_, v, do, sizes, subset, gamma, s, scale, dtype)
        term = {x: w * g[x] for x in ("dq", "dk", "dv")}
        acc = term if acc is None else {x: acc[x] + term[x] for x in acc}
    return acc


def n_subsets(k, t):
    return math.comb(k, t)
