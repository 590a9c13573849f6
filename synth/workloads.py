"""Workload table and seeded key generator (no method arithmetic here).

Configs are BASELINE.json ``configs`` C1..C5 (C5 is a sweep over r).
Seeds follow SURVEY.md §8(d): key Philox key = (0x6B6579 + cfg#, 0),
hash seed = 0x5EED0000 + cfg#.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    n: int          # input key bits
    r: int          # MMH block length in bits
    m: int          # output key bits
    cfg_no: int     # config number (1-based) -> seeds

    @property
    def key_seed(self) -> int:
        return 0x6B6579 + self.cfg_no

    @property
    def hash_seed(self) -> int:
        return 0x5EED0000 + self.cfg_no

    @property
    def nbytes(self) -> int:
        return (self.n + 7) // 8

    @property
    def k(self) -> int:
        return -(-self.n // self.r)


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


# BASELINE.json configs; C5's m = ceil(n/10) following C1's 104,858 = ceil(1,048,576/10).
CONFIGS: dict[str, Workload] = {
    "C1": Workload("C1", 1_048_576, 1 << 16, 104_858, 1),
    "C2": Workload("C2", 10_485_760, 1 << 20, 1_048_576, 2),
    "C3": Workload("C3", 100_000_000, 1 << 22, 10_000_000, 3),
    "C4": Workload("C4", 260_000_000, 1 << 23, 26_000_000, 4),
    "C5a": Workload("C5a", 1 << 31, 1 << 20, _ceil_div(1 << 31, 10), 5),
    "C5b": Workload("C5b", 1 << 31, 1 << 22, _ceil_div(1 << 31, 10), 5),
    "C5c": Workload("C5c", 1 << 31, 1 << 24, _ceil_div(1 << 31, 10), 5),
}


# the paper's own shape (Algorithm 1 with gamma-bit blocks, reload
# rule, m < gamma): the CV-QKD case of Table 3 (k = 10) with the gamma SPEC
# derives for the 2.6e8-bit block: n = gamma k = 259,649,510, compression
# ratio 0.0972 -> m = round(0.0972 n) = 25,237,932 < gamma.
@dataclass(frozen=True)
class PaperWorkload:
    name: str
    n: int          # key bits (= gamma k, no spare windows)
    gamma: int      # Mersenne exponent, blocks are gamma bits
    k: int          # blocks
    m: int          # output bits (< gamma)
    cfg_no: int

    @property
    def key_seed(self) -> int:
        return 0x6B6579 + self.cfg_no

    @property
    def hash_seed(self) -> int:
        return 0x5EED0000 + self.cfg_no

    @property
    def r(self) -> int:          # block bits (= gamma in the paper's shape)
        return self.gamma

    @property
    def nbytes(self) -> int:
        return (self.n + 7) // 8


PAPER_CONFIGS: dict[str, PaperWorkload] = {
    "P1": PaperWorkload("P1", 259_649_510, 25_964_951, 10, 25_237_932, 11),
}


def get_workload(name: str) -> Workload:
    return CONFIGS[name]


def key_bytes(n_bits: int, key_seed: int) -> np.ndarray:
    """ceil(n/8) uniformly random bytes (uint8 array), Philox4x64-10 stream
    key=(key_seed, 0), 64-bit words serialised little-endian.  Pad bits of the
    last byte are left random on purpose: the hash must ignore them."""
    nbytes = (n_bits + 7) // 8
    nwords = (nbytes + 7) // 8
    bg = np.random.Philox(key=np.array([key_seed & (2**64 - 1), 0], dtype=np.uint64))
    words = bg.random_raw(nwords).astype("<u8")
    return np.frombuffer(words.tobytes(), dtype=np.uint8)[:nbytes].copy()


def special_key(kind: str, n_bits: int, pos: int = 0) -> np.ndarray:
    """Structured keys for edge cases: 'zero', 'ones', 'alt' (1010...),
    'bit' (only key bit ``pos`` set, MSB-first numbering)."""
    nbytes = (n_bits + 7) // 8
    if kind == "zero":
        return np.zeros(nbytes, np.uint8)
    if kind == "ones":
        return np.full(nbytes, 0xFF, np.uint8)
    if kind == "alt":
        return np.full(nbytes, 0xAA, np.uint8)
    if kind == "bit":
        a = np.zeros(nbytes, np.uint8)
        a[pos >> 3] = 0x80 >> (pos & 7)
        return a
    raise ValueError(kind)
