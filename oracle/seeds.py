"""Hash-key expansion a_i, b, c from a 64-bit seed.  TEST INFRASTRUCTURE ONLY.

PAPER.md:142  "Random numbers: a in Z_p^k, b, c in Z_{2^gamma}, gcd(b,2) = 1."
PAPER.md:125,127  "randomly choose function of MMH with input random number a",
                  "... of MH with input random numbers b and c".
SPEC.md:143,168   a_i uniform on [0, 2^gamma - 2] by rejecting the all-ones pattern.
SPEC.md:152       b uniform over odd integers in [1, 2^alpha); c uniform over [0, 2^alpha).

Reading A7: the generator is Philox4x64-10 exactly as numpy implements it
(``numpy.random.Philox``, a library routine).  Stream s uses key (seed, s):
s = i for a_i (global block index, so a shard expands only its own blocks),
s = 2^63 for b, s = 2^63 + 1 for c.  One draw of w bits consumes ceil(w/64) words,
assembled little-endian (word 0 least significant) and masked to w bits.
a_i: redraw (next ceil(gamma/64) words of the same stream) while the draw equals
2^gamma - 1.  b: bit 0 forced to 1 (uniform over odd values).  c: as drawn.
"""
from __future__ import annotations

import numpy as np

STREAM_B = 1 << 63
STREAM_C = (1 << 63) + 1


def _philox(seed: int, stream: int) -> np.random.Philox:
    # explicit uint64 array: a Python list key is converted through float64 by numpy,
    # which silently rounds 2^63 + 1 to 2^63
    return np.random.Philox(key=np.array([seed & (2**64 - 1), stream], dtype=np.uint64))


def _draw(bg: np.random.Philox, bits: int) -> int:
    nw = (bits + 63) // 64
    words = bg.random_raw(nw).astype("<u8")
    return int.from_bytes(words.tobytes(), "little") & ((1 << bits) - 1)


def expand_a(seed: int, i: int, gamma: int) -> int:
    """a_i in [0, 2^gamma - 2] (uniform on Z_p), stream (seed, i)."""
    bg = _philox(seed, i)
    allones = (1 << gamma) - 1
    while True:
        v = _draw(bg, gamma)
        if v != allones:
            return v


def expand_b(seed: int, alpha: int) -> int:
    """b odd in [1, 2^alpha), stream (seed, 2^63)."""
    bg = _philox(seed, STREAM_B)
    return _draw(bg, alpha) | 1


def expand_c(seed: int, alpha: int) -> int:
    """c in [0, 2^alpha), stream (seed, 2^63 + 1)."""
    bg = _philox(seed, STREAM_C)
    return _draw(bg, alpha)


def expand_hash_keys(seed: int, k: int, gamma: int, alpha: int,
                     blocks: range | None = None) -> tuple[list[int], int, int]:
    """(a_i for i in blocks (default all k), b, c)."""
    blocks = range(k) if blocks is None else blocks
    return [expand_a(seed, i, gamma) for i in blocks], expand_b(seed, alpha), expand_c(seed, alpha)
