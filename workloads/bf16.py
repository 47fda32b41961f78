"""bf16 rounding of fp64 input draws (round-to-nearest-even, single rounding).

Inputs are rounded to bf16 exactly once here; the resulting uint16 bit patterns are handed to
both the oracle (which up-converts them exactly: bf16 is a subset of fp64) and the CUDA path
(which reinterprets them as torch.bfloat16).  Rounding fp64 -> fp32 -> bf16 could double-round
in rare ties, so the rounding is done directly from fp64.
"""
import numpy as np

_BF16_SIG_BITS = 8          # 1 implicit + 7 stored mantissa bits
_BF16_MIN_EXP = -126        # smallest normal exponent (same as fp32)
_BF16_SUBNORMAL_ULP = 2.0 ** -133
_BF16_MAX = float.fromhex("0x1.fep127")


def bf16_round(a) -> np.ndarray:
    """fp64 array -> uint16 bf16 bit patterns, round-half-to-even, overflow -> +-inf."""
    a = np.asarray(a, dtype=np.float64)
    out = np.empty(a.shape, dtype=np.float64)
    finite = np.isfinite(a)
    m, e = np.frexp(np.where(finite, a, 0.0))          # a = m * 2**e, 0.5 <= |m| < 1
    # value of one ulp at this exponent for a normal bf16: 2**(e - 8)
    q_normal = np.ldexp(np.round(np.ldexp(m, _BF16_SIG_BITS)), e - _BF16_SIG_BITS)
    # subnormal range (|a| < 2**-126): fixed ulp 2**-133
    q_sub = np.round(np.where(finite, a, 0.0) / _BF16_SUBNORMAL_ULP) * _BF16_SUBNORMAL_ULP
    is_sub = (e - 1) < _BF16_MIN_EXP
    out[...] = np.where(is_sub, q_sub, q_normal)
    over = np.abs(out) > _BF16_MAX
    out[over] = np.copysign(np.inf, a[over])
    out[~finite] = a[~finite]
    bits32 = out.astype(np.float32).view(np.uint32)    # exact: out is representable in fp32
    return (bits32 >> 16).astype(np.uint16)


def bf16_to_f32(bits) -> np.ndarray:
    bits = np.asarray(bits, dtype=np.uint16)
    return (bits.astype(np.uint32) << 16).view(np.float32)


def bf16_to_f64(bits) -> np.ndarray:
    """Exact up-conversion of bf16 bit patterns."""
    return bf16_to_f32(bits).astype(np.float64)
