"""Pins of oracle/mersenne.py (Mersenne field)."""
import random

import pytest

from oracle.mersenne import (MERSENNE_EXPONENTS, field_add, field_mul, gamma_for_block,
                             mersenne, reduce_general, reduce_mersenne)


@pytest.mark.parametrize("x,want", [(20, 6), (7, 0), (0, 0), (50, 1)])
def test_reduce_spec_examples(x, want):
    # SPEC.md:48-51 (gamma = 3, p = 7)
    assert reduce_mersenne(x, 3) == want


def test_field_mul_add_spec_examples():
    assert field_mul(3, 5, 3) == 1
    assert field_mul(0, 6, 3) == 0
    assert field_mul(1, 5, 3) == 5
    assert field_add(4, 5, 3) == 2
    assert field_add(0, 6, 3) == 6
    assert field_add(3, 4, 3) == 0          # SPEC.md:69 (p == 0, canonical)


@pytest.mark.parametrize("gamma", [3, 13, 31, 61, 127])
def test_fold_matches_general_modulo(gamma):
    # 10^4 random x < 2^(2 gamma) vs an independent general modulo.
    rng = random.Random(gamma)
    for _ in range(10_000):
        x = rng.getrandbits(2 * gamma)
        assert reduce_mersenne(x, gamma) == reduce_general(x, gamma)


@pytest.mark.parametrize("gamma", [521, 4423, 86243])
def test_fold_matches_general_modulo_large(gamma):
    rng = random.Random(gamma)
    p = (1 << gamma) - 1
    cases = [rng.getrandbits(2 * gamma + 7) for _ in range(20)]
    cases += [p, 2 * p, p * p, p - 1, p + 1, (1 << (2 * gamma)) - 1, 0]
    for x in cases:
        assert reduce_mersenne(x, gamma) == x % p


def test_field_laws():
    # SPEC.md:82-83
    rng = random.Random(1)
    for g in (13, 61, 127):
        p = (1 << g) - 1
        for _ in range(200):
            a, b, c = (rng.randrange(p) for _ in range(3))
            assert field_mul(a, b, g) == field_mul(b, a, g)
            assert field_add(a, b, g) == field_add(b, a, g)
            assert field_mul(field_mul(a, b, g), c, g) == field_mul(a, field_mul(b, c, g), g)
            assert field_add(field_add(a, b, g), c, g) == field_add(a, field_add(b, c, g), g)
            assert field_mul(a, 1, g) == a and field_add(a, 0, g) == a and field_mul(a, 0, g) == 0


def test_exponent_table_is_mersenne_primes():
    # spot-check primality of the small entries of SPEC.md:33 by trial division
    for g in [e for e in MERSENNE_EXPONENTS if e <= 31]:
        p = (1 << g) - 1
        assert all(p % d for d in range(2, int(p ** 0.5) + 1))
    with pytest.raises(ValueError):
        mersenne(11)   # 2^11 - 1 = 23 * 89 is not in the table


def test_gamma_for_block_reading_A2():
    assert gamma_for_block(1 << 16) == 86243
    assert gamma_for_block(1 << 20) == 1257787
    assert gamma_for_block(1 << 22) == 6972593
    assert gamma_for_block(1 << 23) == 13466917
    assert gamma_for_block(1 << 24) == 20996011
    assert gamma_for_block(16) == 17
