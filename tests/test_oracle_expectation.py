"""Pins for O7 (oracle/expectation.py) -- north-star check (b): exhaustive
enumeration of sampled subsets vs the exact closed forms, and unbiasedness of
the compensated estimator in the models where the paper's claim holds exactly."""
import numpy as np
import pytest

from oracle import chunkwise as C
from oracle import expectation as E
from oracle import sampler as S
from synth import make_inputs

TINY = dict(hq=2, hkv=1, seq=64, d=16)
SIZES = [16, 16, 16, 16]


@pytest.fixture(scope="module")
def tiny():
    x = make_inputs(**TINY, seed=21, bf16=False)
    exact = C.seco_step(x.q, x.k, x.v, x.do, SIZES)
    parts = E.decompose(x.q, x.k, x.v, x.do, SIZES)
    return x, exact, parts


def _err(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def test_decomposition_sums_to_seco(tiny):
    x, exact, parts = tiny
    assert _err(parts["loc_k"] + parts["cross_k"], exact["dk"]) < 1e-13
    assert _err(parts["loc_v"] + parts["cross_v"], exact["dv"]) < 1e-13
    assert _err(parts["dq"], exact["dq"]) < 1e-13
    assert np.abs(parts["cross_k"][:, 48:]).max() == 0     # last chunk receives no deposits


@pytest.mark.parametrize("t", [1, 2, 3, 4])
def test_paper_mode_enumeration_matches_closed_form(tiny, t):
    x, exact, parts = tiny
    g, s = S.scales(4, t, 0, S.PAPER)
    mean = E.enumerate_t_of_k(x.q, x.k, x.v, x.do, SIZES, t, g, s)
    cf = E.closed_form_t_of_k(parts, 4, t, g, s)
    for key in ("dq", "dk", "dv"):
        assert _err(mean[key], cf[key]) < 1e-13


def test_paper_mode_is_biased_at_t2(tiny):
    """Literal Alg. 2 (s = 1, gamma = k/t) at k=4, t=2: local factor 1/2, cross factor 1/3."""
    x, exact, parts = tiny
    g, s = S.scales(4, 2, 0, S.PAPER)
    mean = E.enumerate_t_of_k(x.q, x.k, x.v, x.do, SIZES, 2, g, s)
    assert _err(mean["dq"], 0.5 * exact["dq"]) < 1e-13
    want_k = 0.5 * parts["loc_k"] + (1 / 3) * parts["cross_k"]
    assert _err(mean["dk"], want_k) < 1e-13


@pytest.mark.parametrize("t", [2, 3])
def test_ht_mode_unbiased(tiny, t):
    x, exact, parts = tiny
    g, s = S.scales(4, t, 0, S.HT)
    mean = E.enumerate_t_of_k(x.q, x.k, x.v, x.do, SIZES, t, g, s)
    cf = E.closed_form_t_of_k(parts, 4, t, g, s)
    for key in ("dq", "dk", "dv"):
        assert _err(mean[key], cf[key]) < 1e-13
        # unbiased up to the float32 rounding of gamma, s (the ABI returns float)
        assert _err(mean[key], exact[key]) < 3e-7


@pytest.mark.parametrize("t", [1, 2, 3])
def test_bernoulli_mode_unbiased(tiny, t):
    """The paper's survival model: independent inclusion w.p. t/k with
    scaler k/t on every relay reproduces the exact gradient in expectation (Eq. 10)."""
    x, exact, parts = tiny
    g, s = S.scales(4, t, 0, S.BERNOULLI)
    w = E.enumerate_bernoulli(x.q, x.k, x.v, x.do, SIZES, t / 4, g, s)
    cf = E.closed_form_bernoulli(parts, t / 4, g, s)
    for key in ("dq", "dk", "dv"):
        assert _err(w[key], cf[key]) < 1e-13
        # unbiased up to the float32 rounding of gamma = s = k/t
        assert _err(w[key], exact[key]) < 3e-7


def test_enumeration_counts():
    assert E.n_subsets(4, 2) == 6 and E.n_subsets(16, 4) == 1820
