"""Philox4x64-10 written out in plain Python from its published definition, as an
independent pin of the oracle's key expansion (reading A7).  Test code only:
neither oracle/ nor the library imports it.

Definition (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3",
SC'11, Philox-4x64): a 256-bit counter (c0, c1, c2, c3) and a 128-bit key (k0, k1);
one round is

    (hi0, lo0) = M0 * c0          (hi1, lo1) = M1 * c2      (full 128-bit products)
    (c0, c1, c2, c3) <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)

and the key is bumped by the Weyl constants (W0, W1) between rounds; ten rounds.  The
stream of 64-bit words for key (k0, k1) is the four outputs of counter 1, then of
counter 2, ... (numpy.random.Philox advances the counter before its first block).
"""
from __future__ import annotations

MASK = (1 << 64) - 1
M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B


def philox4x64_10(ctr: tuple[int, int, int, int], key: tuple[int, int]) -> tuple[int, int, int, int]:
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for rnd in range(10):
        if rnd:
            k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
        p0, p1 = M0 * c0, M1 * c2
        c0, c1, c2, c3 = ((p1 >> 64) ^ c1 ^ k0) & MASK, p1 & MASK, ((p0 >> 64) ^ c3 ^ k1) & MASK, p0 & MASK
    return c0, c1, c2, c3


def stream_words(k0: int, k1: int, count: int) -> list[int]:
    """The first ``count`` 64-bit words of the stream with key (k0, k1)."""
    out: list[int] = []
    ctr = 0
    while len(out) < count:
        ctr += 1
        out.extend(philox4x64_10((ctr & MASK, (ctr >> 64) & MASK, 0, 0), (k0 & MASK, k1 & MASK)))
    return out[:count]


def draw(words: list[int], bits: int) -> int:
    """ceil(bits/64) words little-endian (word 0 least significant), masked to ``bits``."""
    v = 0
    for i, w in enumerate(words[: (bits + 63) // 64]):
        v |= w << (64 * i)
    return v & ((1 << bits) - 1)
