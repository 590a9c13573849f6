"""CPU ORACLE (test infrastructure only; see oracle/__init__.py): Toeplitz-hashing PA, the
comparator of Table 1 / Fig. 3.

Definition ("standard matrix-vector product over GF(2)"):
    output_j = XOR_i T[j, i] x_i,   j < m, i < n,
with T the m x n Toeplitz matrix of the diagonal sequence d (n + m - 1 bits).  Reading A14
(DESIGN.md): "row 0 starting at diagonal index m-1 descending" is T[j, i] = d[m - 1 - j + i]
(row 0 is d[m-1 .. m+n-2]; going down a column the index descends).  x_i = key bit i read
MSB-first from bytes (reading A4); output bit j emitted MSB-first (reading A5).  The seeded
diagonal (reading A15): Philox4x64-10 stream (seed, 2^63 + 2), bit t = bit (t mod 64) of
word floor(t / 64)."""
from __future__ import annotations

import numpy as np

from .seeds import _philox

STREAM_T = (1 << 63) + 2


def expand_diagonal(seed: int, nbits: int) -> int:
    """d as an integer: bit t = d_t (reading A15)."""
    nw = (nbits + 63) // 64
    words = _philox(seed, STREAM_T).random_raw(nw).astype("<u8")
    return int.from_bytes(words.tobytes(), "little") & ((1 << nbits) - 1)


def _key_int_lsb_first(key, n: int) -> int:
    """X = sum_i x_i 2^i with x_i = key bit i, MSB-first within bytes (reading A4)."""
    kb = bytes(np.asarray(key, dtype=np.uint8)) if not isinstance(key, bytes) else key
    nbytes = (n + 7) // 8
    msb = int.from_bytes(kb[:nbytes], "big") >> (8 * nbytes - n)      # bit n-1-i = x_i
    return int(format(msb, f"0{n}b")[::-1], 2) if n else 0


def _emit_msb_first(bits: list[int]) -> bytes:
    m = len(bits)
    z = 0
    for b in bits:
        z = (z << 1) | b
    nb = (m + 7) // 8
    return (z << (8 * nb - m)).to_bytes(nb, "big")


def toeplitz_pa(key, n: int, m: int, d: int) -> bytes:
    """output_j = parity(popcount(W_j & X)), W_j = row j of T as an n-bit mask:
    bit i of W_j = d[m - 1 - j + i] = bit i of (d >> (m - 1 - j))."""
    if n < 1 or m < 1:
        raise ValueError("n, m must be >= 1")
    X = _key_int_lsb_first(key, n)
    mask = (1 << n) - 1
    return _emit_msb_first([(((d >> (m - 1 - j)) & mask & X).bit_count()) & 1 for j in range(m)])


def toeplitz_pa_matrix(key, n: int, m: int, d: int) -> bytes:
    """The same map through an explicit 0/1 matrix and numpy's matrix-vector product (a
    library primitive), for small n, m: an independent route to the definition."""
    T = np.zeros((m, n), dtype=np.int64)
    for j in range(m):
        for i in range(n):
            T[j, i] = (d >> (m - 1 - j + i)) & 1
    X = _key_int_lsb_first(key, n)
    x = np.array([(X >> i) & 1 for i in range(n)], dtype=np.int64)
    return _emit_msb_first([int(v) & 1 for v in (T @ x)])


def toeplitz_pa_seeded(key, n: int, m: int, seed: int) -> bytes:
    return toeplitz_pa(key, n, m, expand_diagonal(seed, n + m - 1))


def toeplitz_bits(key, n: int, m: int, d: int, js) -> list[int]:
    """Output bits j in js only (the same definition, one row at a time): for sampled
    parity at sizes where the whole output is out of the oracle's reach."""
    X = _key_int_lsb_first(key, n)
    mask = (1 << n) - 1
    return [(((d >> (m - 1 - j)) & mask & X).bit_count()) & 1 for j in js]
