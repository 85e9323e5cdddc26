"""Seeded input generators shared by oracle tests, GPU parity tests and bench (no method arithmetic)."""
from .inputs import AttnInputs, make_inputs, bf16_round_bits, bf16_bits_to_f32, round_to_bf16  # noqa: F401
