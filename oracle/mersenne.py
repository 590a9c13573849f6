"""Mersenne-prime field Z_p, p = M_gamma = 2^gamma - 1.  TEST INFRASTRUCTURE ONLY.

PAPER.md:129  "the prime p ... is recommended to be a Mersenne prime. The form of a
               Mersenne prime is M_gamma = 2^gamma - 1."
PAPER.md:130-132  "x mod M_gamma = floor(x / 2^gamma) + x mod 2^gamma, so modulus
               operation can be simplified."
SPEC.md:33    known-exponent table; SPEC.md:38,87 canonical residue in [0, 2^gamma - 2];
SPEC.md:42-51,88  fold repeatedly, then one conditional subtract.
"""
from __future__ import annotations

# SPEC.md:33 (known Mersenne prime exponents, at minimum this list).
MERSENNE_EXPONENTS: tuple[int, ...] = (
    3, 5, 7, 13, 17, 19, 31, 61, 89, 107, 127, 521, 607, 1279, 2203, 2281, 3217,
    4253, 4423, 9689, 9941, 11213, 19937, 21701, 23209, 44497, 86243, 110503,
    132049, 216091, 756839, 859433, 1257787, 1398269, 2976221, 3021377, 6972593,
    13466917, 20996011, 24036583, 25964951, 30402457, 32582657, 37156667,
    42643801, 43112609, 57885161, 74207281,
)


def mersenne(gamma: int) -> int:
    """p = M_gamma = 2^gamma - 1."""
    if gamma not in MERSENNE_EXPONENTS:
        raise ValueError(f"gamma={gamma} is not a known Mersenne exponent (SPEC.md:33)")
    return (1 << gamma) - 1


def gamma_for_block(r: int) -> int:
    """Reading A2: the smallest known exponent gamma >= r, so that an r-bit
    block x_i < 2^r <= p lies in Z_p as Eq. 1 requires."""
    for g in MERSENNE_EXPONENTS:
        if g >= r:
            return g
    raise ValueError(f"no Mersenne exponent >= r={r}")


def reduce_mersenne(x: int, gamma: int) -> int:
    """x mod (2^gamma - 1) by the fold identity of PAPER.md:130-132, canonical.

    Step by step: while x has more than gamma bits replace it by
    floor(x / 2^gamma) + (x mod 2^gamma); then the value p itself maps to 0
    (canonical residue; reading A6).  Linear time in the size of x,
    unlike CPython's ``%`` which is quadratic."""
    if x < 0:
        raise ValueError("x must be non-negative")
    p = (1 << gamma) - 1
    while x >> gamma:
        x = (x >> gamma) + (x & p)
    return 0 if x == p else x


def reduce_general(x: int, gamma: int) -> int:
    """Independent general-purpose modulo (Python ``%``), used only to pin the fold."""
    return x % ((1 << gamma) - 1)


def field_mul(a: int, b: int, gamma: int) -> int:
    """(a*b) mod p, canonical (Eq. 2's a_i*x_i)."""
    return reduce_mersenne(a * b, gamma)


def field_add(a: int, b: int, gamma: int) -> int:
    """(a+b) mod p, canonical (Eq. 2's sum)."""
    return reduce_mersenne(a + b, gamma)
