"""Seeded input generators shared by oracle tests, GPU parity tests and bench (no method arithmetic)."""
from .inputs import (AttnInputs, StackInputs, bf16_bits_to_f32, bf16_round_bits, make_inputs,  # noqa: F401
                     make_stack_inputs, round_to_bf16)
