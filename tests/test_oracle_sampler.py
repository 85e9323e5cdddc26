"""Pins for O8 (oracle/sampler.py): published splitmix64 vectors, independent KATs,
the hypergeometric marginal t/k, worked compensation constants from the paper."""
import os
from collections import Counter

import numpy as np
import pytest

from oracle import sampler as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def test_splitmix64_published_vector():
    want = [int(r[0], 16) for r in _rows("splitmix64_seed0.txt")]
    g = S.SplitMix64(0)
    assert [g.next() for _ in range(3)] == want


@pytest.mark.parametrize("row", _rows("sampler_kats.txt"))
def test_sampler_kats(row):
    mode = {"T_OF_K": S.PAPER, "BERNOULLI": S.BERNOULLI}[row[0]]
    k, t, seed = int(row[1]), int(row[2]), int(row[3])
    want = [int(v) for v in row[4].split(",")]
    assert S.sample_indices(k, t, seed, mode) == want


@pytest.mark.parametrize("row", _rows("compensation_constants.txt"))
def test_compensation_constants(row):
    k, t, cap, gamma = int(row[0]), int(row[1]), float(row[2]), float(row[3])
    g, s = S.scales(k, t, cap, S.PAPER)
    assert g == gamma and s == 1.0


def test_uniform_marginal_frequency():
    """Each index is selected with probability t/k = 0.5 (k=8, t=4; S:232 bound 0.5 +- 0.01)."""
    n = 100_000
    c = Counter()
    for seed in range(n):
        c.update(S.sample_indices(8, 4, seed))
    freqs = np.array([c[i] / n for i in range(8)])
    assert np.all(np.abs(freqs - 0.5) < 0.01), freqs


def test_all_subsets_reachable_and_uniform():
    """k=6, t=2: all C(6,2)=15 subsets appear with frequency 1/15 +- 0.01."""
    n = 60_000
    c = Counter(tuple(S.sample_indices(6, 2, seed)) for seed in range(n))
    assert len(c) == 15
    assert all(abs(v / n - 1 / 15) < 0.01 for v in c.values())


def test_bernoulli_marginal():
    n = 50_000
    c = Counter()
    for seed in range(n):
        c.update(S.sample_indices(16, 4, seed, S.BERNOULLI))
    freqs = np.array([c[i] / n for i in range(16)])
    assert np.all(np.abs(freqs - 0.25) < 0.01)


@pytest.mark.parametrize("k,t,mode", [(16, 4, S.PAPER), (32, 32, S.PAPER), (9, 3, S.HT), (16, 4, S.BERNOULLI)])
def test_shape_and_order(k, t, mode):
    for seed in range(50):
        idx = S.sample_indices(k, t, seed, mode)
        assert idx == sorted(set(idx), reverse=True)
        assert all(0 <= i < k for i in idx)
        if mode != S.BERNOULLI:
            assert len(idx) == t


def test_t_equals_k_selects_all():
    assert S.sample_indices(7, 7, 123) == list(range(6, -1, -1))


def test_mode_scales():
    assert S.scales(16, 4, 0, S.HT) == (5.0, 4.0)
    assert S.scales(16, 4, 0, S.BERNOULLI) == (4.0, 4.0)
    assert S.scales(16, 4, 2.0, S.BERNOULLI) == (2.0, 4.0)
    assert S.scales(3, 1, 0, S.PAPER)[0] == np.float32(3.0)


@pytest.mark.parametrize("k,t,mode", [(4, 0, S.PAPER), (4, 5, S.PAPER), (4, 1, S.HT)])
def test_errors(k, t, mode):
    with pytest.raises(ValueError):
        S.sample_indices(k, t, 0, mode)
