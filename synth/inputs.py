"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no attention, no softmax, no
sampling, no relay).  It only draws numbers and rounds them to bf16 so that the
oracle (``oracle/``) and the CUDA path (``paper_2505_16710_b200``) see the very
same bytes.  Neither side imports the other; both import this.

Recipe (SURVEY.md §8(d) "Concrete synthetic inputs"):
  * Q, K, V, dO ~ N(0, 1) i.i.d. drawn with numpy PCG64(seed), rounded to bf16
    with round-to-nearest-even.  Shapes: Q, dO, O as [Hq][S][d]; K, V as
    [Hkv][S][d] (head-major, one sequence).
  * "peaky" variant (parity only): Q scaled by 4 and key 0 of every kv-head
    scaled by 3 (an attention sink) -- exercises online-softmax rescaling and a
    wide LSE range.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def bf16_round_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns (uint16), round-to-nearest-even (no NaNs expected)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounding_bias = ((u >> 16) & 1) + 0x7FFF
    return ((u + rounding_bias) >> 16).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> float32 values (exact)."""
    return (b.astype(np.uint32) << 16).view(np.float32)


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Values of x rounded to the nearest bf16, returned as float32."""
    return bf16_bits_to_f32(bf16_round_bits(x))


@dataclass
class AttnInputs:
    """One sequence of attention inputs.  *_bits are bf16 bit patterns (uint16);
    the float arrays are the exact float32 values of those bf16 numbers."""
    q: np.ndarray
    k: np.ndarray
    v: np.ndarray
    do: np.ndarray
    q_bits: np.ndarray
    k_bits: np.ndarray
    v_bits: np.ndarray
    do_bits: np.ndarray

    @property
    def shape(self):
        hq, s, d = self.q.shape
        return hq, self.k.shape[0], s, d


def make_inputs(hq: int, hkv: int, seq: int, d: int, seed: int = 0,
                peaky: bool = False, bf16: bool = True) -> AttnInputs:
    """Draw Q, K, V, dO for one sequence.  With bf16=False the values are plain
    float32 normals (the fp32-debug path and the tiny config use these)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    q = rng.standard_normal((hq, seq, d), dtype=np.float32)
    k = rng.standard_normal((hkv, seq, d), dtype=np.float32)
    v = rng.standard_normal((hkv, seq, d), dtype=np.float32)
    do = rng.standard_normal((hq, seq, d), dtype=np.float32)
    if peaky:
        q *= 4.0
        k[:, 0, :] *= 3.0
    if bf16:
        qb, kb, vb, dob = (bf16_round_bits(a) for a in (q, k, v, do))
        return AttnInputs(bf16_bits_to_f32(qb), bf16_bits_to_f32(kb), bf16_bits_to_f32(vb),
                          bf16_bits_to_f32(dob), qb, kb, vb, dob)
    z = np.zeros(0, np.uint16)
    return AttnInputs(q, k, v, do, z, z, z, z)


@dataclass
class StackInputs:
    """Inputs of the L-layer stack (oracle/multilayer.py, paper_2505_16710_b200/model.py):
    x0 [S][Hd] token states entering layer 0, G [S][Hd] the loss cotangent at the top,
    layers[l] = {W_p, A_p, B_p for p in q, k, v, o} ([in][out]).  All float64 arrays whose
    values are exactly representable in the requested dtype (bf16 or float32)."""
    x0: np.ndarray
    G: np.ndarray
    layers: list


def make_stack_inputs(L: int, hd: int, hq: int, hkv: int, d: int, r: int, seq: int, seed: int = 0,
                      bf16: bool = False, w_scale: float = 1.0, lora_scale: float = 0.5) -> StackInputs:
    """Seeded parameters and inputs.  Base weights ~ N(0, w_scale^2 / fan_in); LoRA A, B ~
    N(0, lora_scale^2 / fan_in), B non-zero so that every gradient is non-trivial; x0, G ~
    N(0, 1).  Values are rounded to bf16 (RNE) or to float32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    rnd = round_to_bf16 if bf16 else (lambda a: np.asarray(a, np.float32))

    def draw(shape, scale):
        return rnd((rng.standard_normal(shape) * scale).astype(np.float32)).astype(np.float64)

    dims = {"q": (hd, hq * d), "k": (hd, hkv * d), "v": (hd, hkv * d), "o": (hq * d, hd)}
    layers = []
    for _ in range(L):
        p = {}
        for n, (i, o) in dims.items():
            p["W" + n] = draw((i, o), w_scale / np.sqrt(i))
            p["A" + n] = draw((i, r), lora_scale / np.sqrt(i))
            p["B" + n] = draw((r, o), lora_scale / np.sqrt(r))
        layers.append(p)
    x0 = draw((seq, hd), 1.0)
    G = draw((seq, hd), 1.0)
    return StackInputs(x0, G, layers)
