"""CPU ORACLE (test infrastructure only; see oracle/__init__.py): parameter derivation of
the paper's shape, written from SPEC.md:185-225 and the paper.

Every function is the plain definition: a scan over candidates checked with exact
rational arithmetic, no closed-form shortcuts."""
from __future__ import annotations

from fractions import Fraction

from .mersenne import MERSENNE_EXPONENTS


def derive_security_coefficient(epsilon: float) -> int:
    """Smallest s >= 1 with 2^(-s/2-1) <= epsilon: the composition bound
    eps <= 2^(-s/2-1) of PAPER.md:185-188 solved for s.
    The comparison 2^(-s/2-1) <= eps is done exactly: 2^(-(s+2)/2) <= e  <=>  1 <= e^2 2^(s+2)."""
    if not 0 < epsilon < 1:
        raise ValueError("epsilon must be in (0, 1)")
    e = Fraction(epsilon)
    s = 1
    while e * e * (1 << (s + 2)) < 1:
        s += 1
    return s


def select_block_count(ratio: float) -> int:
    """k = floor(1/r): the largest k with k r <= 1 ("k <= 1/r")."""
    if not 0 < ratio < 1:
        raise ValueError("ratio must be in (0, 1)")
    r = Fraction(ratio).limit_denominator(10**12)
    k = 1
    while (k + 1) * r <= 1:
        k += 1
    return k


def select_gamma(target_n: int, k: int) -> tuple[int, bool]:
    """Largest Mersenne exponent gamma with k gamma <= target_n ("n is equal to gamma x k",
    PAPER.md:282); (smallest exponent, True) when none fits."""
    if target_n < 1 or k < 1:
        raise ValueError("target_n and k must be >= 1")
    fits = [g for g in MERSENNE_EXPONENTS if k * g <= target_n]
    return (max(fits), False) if fits else (min(MERSENNE_EXPONENTS), True)


def derive_paper_params(target_n: int, ratio: float, t: int, epsilon: float) -> dict:
    """k, gamma, n = k gamma, s, m = n - t - s; m > 0 and m + s <= gamma."""
    k = select_block_count(ratio)
    gamma, _ = select_gamma(target_n, k)
    n = k * gamma
    s = derive_security_coefficient(epsilon)
    m = n - t - s
    if m <= 0 or m + s > gamma:
        raise ValueError("invariants m > 0, m + s <= gamma violated")
    return {"gamma": gamma, "k": k, "n": n, "s": s, "m": m}
