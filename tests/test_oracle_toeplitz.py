"""Toeplitz-hashing PA oracle (NEXT-4 comparator) pinned to SPEC.md's examples, an explicit
matrix product, GF(2) linearity and the Toeplitz shift structure (-m "not gpu")."""
import itertools
import random

import numpy as np
import pytest

from oracle import toeplitz as T


def bits_to_bytes(bits):
    n = len(bits)
    v = int("".join(map(str, bits)), 2) if n else 0
    nb = (n + 7) // 8
    return (v << (8 * nb - n)).to_bytes(nb, "big")


def diag(bits):            # d_t = bits[t]
    return sum(b << t for t, b in enumerate(bits))


def test_spec_examples():
    # n=2, m=2, diagonal=111, x=10 -> 11
    assert T.toeplitz_pa(bits_to_bytes([1, 0]), 2, 2, diag([1, 1, 1])) == bits_to_bytes([1, 1])
    # all-zero diagonal -> all-zero output
    assert T.toeplitz_pa(bits_to_bytes([1, 1, 0, 1]), 4, 3, 0) == bits_to_bytes([0, 0, 0])
    # n = m = 1, diagonal 1, x = 1 -> 1
    assert T.toeplitz_pa(bits_to_bytes([1]), 1, 1, 1) == bits_to_bytes([1])


def test_index_convention_single_diagonal_bit():
    """Reading A14, T[j, i] = d[m-1-j+i]: with only d_t = 1 the output bit j is x_{t-m+1+j}."""
    n, m = 7, 4
    x = [1, 0, 1, 1, 0, 0, 1]
    for t in range(n + m - 1):
        got = T.toeplitz_pa(bits_to_bytes(x), n, m, 1 << t)
        want = [x[t - m + 1 + j] if 0 <= t - m + 1 + j < n else 0 for j in range(m)]
        assert got == bits_to_bytes(want), t


def test_matches_explicit_matrix_exhaustive_small():
    for n, m in [(1, 1), (2, 2), (3, 2), (4, 3), (5, 4)]:
        for xb in itertools.product([0, 1], repeat=n):
            for d in range(1 << (n + m - 1)):
                key = bits_to_bytes(list(xb))
                assert T.toeplitz_pa(key, n, m, d) == T.toeplitz_pa_matrix(key, n, m, d)


def test_matches_explicit_matrix_random():
    rng = random.Random(5)
    for _ in range(100):                      # SPEC.md:302 sizes: n = 64, m = 16
        n, m = 64, 16
        key = bytes(rng.getrandbits(8) for _ in range(8))
        d = rng.getrandbits(n + m - 1)
        assert T.toeplitz_pa(key, n, m, d) == T.toeplitz_pa_matrix(key, n, m, d)


def test_gf2_linearity_and_shift():
    rng = random.Random(9)
    n, m = 300, 77
    d = rng.getrandbits(n + m - 1)
    xa = bytes(rng.getrandbits(8) for _ in range(38))
    xb = bytes(rng.getrandbits(8) for _ in range(38))
    xab = bytes(a ^ b for a, b in zip(xa, xb))
    ha, hb, hab = (int.from_bytes(T.toeplitz_pa(k, n, m, d), "big") for k in (xa, xb, xab))
    assert hab == ha ^ hb
    # Toeplitz structure: row j+1 of T is row j shifted by one column (d index - 1):
    # dropping the first output bit of (d) equals the first m-1 bits of (d >> 1)'s output
    full = T.toeplitz_pa(xa, n, m, d)
    sh = T.toeplitz_pa(xa, n, m - 1, d)                    # rows 0..m-2 use d[m-1-j+i], m-1 -> m-2
    a = format(int.from_bytes(full, "big") >> (8 * len(full) - m), f"0{m}b")
    b = format(int.from_bytes(sh, "big") >> (8 * len(sh) - (m - 1)), f"0{m - 1}b")
    # sh's row j = d[m-2-j+i] = full's row j+1
    assert b == a[1:]


def test_seeded_diagonal_is_philox_stream():
    d = T.expand_diagonal(7, 130)
    w = np.random.Philox(key=np.array([7, (1 << 63) + 2], dtype=np.uint64)).random_raw(3)
    assert d == (int(w[0]) | (int(w[1]) << 64) | (int(w[2]) << 128)) & ((1 << 130) - 1)
