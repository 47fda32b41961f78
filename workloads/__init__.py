"""Seeded synthetic inputs shared by the oracle tests, the CUDA-path tests and bench.py.

This package holds NO arithmetic of the method (no joint diagonalization, no shrink, Sigma
or expand).  It only draws random numbers, rounds them to bf16 once (so both sides consume
the identical bits, SURVEY 8(c) c7 "quantize once, share the bits") and shapes them like
the paper's workloads (Mistral-7B projections, rank-16 LoRAs, 1000+ adapters, clusters).
Recipe and seeds: DESIGN.md section "Input recipe".
"""
from .bf16 import bf16_round, bf16_to_f64, bf16_to_f32  # noqa: F401
from .gen import (  # noqa: F401
    MISTRAL_MODULES,
    rng,
    gen_loras,
    direct_bank,
    cluster_map,
    decode_tokens,
    prefill_tokens,
    activations,
)
