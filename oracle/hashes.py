"""MMH, MH and Algorithm 1, written out from the paper.  TEST INFRASTRUCTURE ONLY.

Every function follows a passage of PAPER.md (LaTeX of arXiv 2105.13678) or
SPEC.md; the readings of ambiguous passages are A1-A13 in DESIGN.md.  Big-integer
products use CPython's ``int.__mul__`` (a library primitive); reductions mod a
Mersenne prime use the fold identity (``oracle.mersenne``), pinned against ``%``.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

from .mersenne import gamma_for_block, mersenne, reduce_mersenne
from .seeds import expand_hash_keys


# --------------------------------------------------------------------------- MMH / MH
def mmh_eval(a: Sequence[int], x: Sequence[int], gamma: int) -> int:
    """g_a(x) = a . x mod p = sum_{i=1..k} a_i x_i mod p   (Eq. 2).

    Reading A9: exactly k products, then (sum) mod p; the order of summation and the
    reduction schedule cannot change an exact result."""
    if len(a) != len(x):
        raise ValueError("length mismatch (SPEC.md:126)")
    acc = 0
    for ai, xi in zip(a, x):
        acc += ai * xi
    return reduce_mersenne(acc, gamma)


def mh_eval(b: int, c: int, y: int, alpha: int, beta: int) -> int:
    """h_{b,c}(y) = ((b*y + c) mod 2^alpha) / 2^(alpha-beta)   (Eq. 4).

    Reading A8: the division is floor division, i.e. the top beta bits of the
    alpha-bit affine value.  b must be odd (Eq. 3)."""
    if beta > alpha:
        raise ValueError("beta > alpha (SPEC.md:135)")
    if b % 2 == 0:
        raise ValueError("b must be odd (PAPER.md:97)")
    mask = (1 << alpha) - 1
    return ((b * y + c) & mask) >> (alpha - beta)


# ----------------------------------------------------- Algorithm 1 in the paper's shape
def bits_to_field_blocks(bits: Sequence[int], gamma: int, k: int):
    """Split + map to Z_p with the reload rule.

    Successive gamma-bit windows, MSB-first, are read as integers; a window
    equal to 2^gamma - 1 is 'cast away and reloaded', i.e. dropped and
    the next gamma bits consumed (reading A10).  Returns (blocks, consumed, rejected)."""
    allones = (1 << gamma) - 1
    blocks, pos, rejected = [], 0, 0
    while len(blocks) < k:
        if pos + gamma > len(bits):
            raise ValueError(f"insufficient input: filled {len(blocks)} of {k} blocks")
        v = 0
        for t in range(gamma):
            v = (v << 1) | (bits[pos + t] & 1)
        pos += gamma
        if v == allones:
            rejected += 1
            continue
        blocks.append(v)
    return blocks, pos, rejected


def pa_run_paper(bits: Sequence[int], gamma: int, k: int, m: int,
                 a: Sequence[int], b: int, c: int):
    """Algorithm 1 with gamma-bit blocks and alpha = gamma
    (SPEC.md:226-234, 252).  Returns (output bits MSB-first, consumed, rejected)."""
    if m >= gamma + 1:
        raise ValueError("Algorithm 1 requires gamma > beta (PAPER.md:143)")
    x, consumed, rejected = bits_to_field_blocks(bits, gamma, k)   # lines 1-5
    y = mmh_eval(a, x, gamma)                                       # lines 6-9
    z = mh_eval(b, c, y, gamma, m)                                  # line 10
    out = [(z >> (m - 1 - j)) & 1 for j in range(m)]               # A5: MSB-first
    return out, consumed, rejected


# --------------------------------------- the r-bit-block shape computed by the library
def plan_params(n: int, r: int, m: int, gamma: int | None = None) -> dict:
    """O1 of SURVEY.md §8(c): k = ceil(n/r); gamma per reading A2 unless given;
    p = 2^gamma - 1; alpha = max(gamma, m) (reading A1)."""
    if n < 1 or r < 1 or m < 1:
        raise ValueError("n, r, m must be >= 1")
    g = gamma_for_block(r) if gamma is None else gamma
    mersenne(g)  # validates the exponent
    if g < r:
        raise ValueError("gamma must be >= r so that every r-bit block lies in Z_p (A2)")
    return {"k": -(-n // r), "gamma": g, "alpha": max(g, m)}


def key_blocks(key: np.ndarray | bytes, n: int, r: int) -> list[int]:
    """O2-O3: key bits kappa_0..kappa_{n-1}, MSB-first from bytes (
    reading A4), bits >= n ignored, zero-extended to k*r bits (reading A3);
    x_i = sum_t kappa_{ir+t} 2^(r-1-t), block 0 = the first r bits."""
    kb = bytes(np.asarray(key, dtype=np.uint8)) if not isinstance(key, bytes) else key
    nbytes = (n + 7) // 8
    if len(kb) < nbytes:
        raise ValueError("key shorter than ceil(n/8) bytes")
    kb = bytearray(kb[:nbytes])
    if n % 8:
        kb[-1] &= (0xFF << (8 - n % 8)) & 0xFF          # ignore pad bits of the last byte
    k = -(-n // r)
    if r % 8 == 0:
        total = k * r // 8
        kb.extend(b"\x00" * (total - len(kb)))
        step = r // 8
        return [int.from_bytes(kb[i * step:(i + 1) * step], "big") for i in range(k)]
    full = int.from_bytes(bytes(kb), "big") >> (8 * nbytes - n)   # n-bit integer
    full <<= k * r - n
    mask = (1 << r) - 1
    return [(full >> ((k - 1 - i) * r)) & mask for i in range(k)]


def mmh_partial(key, n: int, r: int, gamma: int, a: Sequence[int],
                blocks: range | None = None) -> int:
    """MMH over a subset of block indices ("split and separately handle";
    SPEC.md:161 split-merge): sum_{i in blocks} a_i x_i mod p.  ``a`` is indexed by
    global block index i."""
    x = key_blocks(key, n, r)
    blocks = range(len(x)) if blocks is None else blocks
    return mmh_eval([a[i] for i in blocks], [x[i] for i in blocks], gamma)


def merge_residues(ys: Sequence[int], gamma: int) -> int:
    """S6: y = sum_g y_g mod p (Eq. 2 is linear over a partition of the blocks)."""
    return reduce_mersenne(sum(ys), gamma)


def pack_output(z: int, m: int) -> bytes:
    """O7 / reading A5: z emitted MSB-first into ceil(m/8) bytes, trailing pad bits 0."""
    nb = (m + 7) // 8
    return (z << (8 * nb - m)).to_bytes(nb, "big")


def mh_output(y: int, b: int, c: int, alpha: int, m: int) -> bytes:
    """S7: z = h_{b,c}(y) with beta = m (Eq. 4), packed MSB-first."""
    return pack_output(mh_eval(b, c, y, alpha, m), m)


def pa_hash(key, n: int, r: int, m: int, gamma: int,
            a: Sequence[int], b: int, c: int) -> bytes:
    """Algorithm 1 on r-bit blocks: y = g_a(x); z = h_{b,c}(y)."""
    alpha = max(gamma, m)
    y = mmh_partial(key, n, r, gamma, a)
    return mh_output(y, b, c, alpha, m)


def pa_hash_seeded(key, n: int, r: int, m: int, seed: int, gamma: int | None = None) -> bytes:
    """pa_hash with hash keys expanded from ``seed`` (reading A7)."""
    pp = plan_params(n, r, m, gamma)
    a, b, c = expand_hash_keys(seed, pp["k"], pp["gamma"], pp["alpha"])
    return pa_hash(key, n, r, m, pp["gamma"], a, b, c)


# ------------------------------------------ Algorithm 1 in the paper's shape, byte keys
def paper_blocks(key, n: int, gamma: int, k: int):
    """bits_to_field_blocks on an n-bit
    MSB-first byte key, with Python-int slicing instead of a bit list: windows are the
    successive gamma-bit windows at bit offsets t*gamma; a window equal to 2^gamma - 1 is
    cast away and the next one consumed (reading A10).  Returns (blocks, windows used).
    Raises ValueError (SPEC.md:74 InsufficientInput) if fewer than k windows qualify."""
    kb = bytes(np.asarray(key, dtype=np.uint8)) if not isinstance(key, bytes) else key
    nbytes = (n + 7) // 8
    if len(kb) < nbytes:
        raise ValueError("key shorter than ceil(n/8) bytes")
    full = int.from_bytes(kb[:nbytes], "big") >> (8 * nbytes - n)      # the n-bit integer
    allones = (1 << gamma) - 1
    blocks, t = [], 0
    while len(blocks) < k:
        if (t + 1) * gamma > n:
            raise ValueError(f"insufficient input: filled {len(blocks)} of {k} blocks")
        v = (full >> (n - (t + 1) * gamma)) & allones
        t += 1
        if v == allones:
            continue
        blocks.append(v)
    return blocks, t


def pa_hash_paper(key, n: int, gamma: int, k: int, m: int, a: Sequence[int], b: int, c: int) -> bytes:
    """Algorithm 1 exactly as the paper shapes it: k gamma-bit blocks
    with the reload rule, alpha = gamma, beta = m < gamma; output MSB-first."""
    if m >= gamma:
        raise ValueError("Algorithm 1 requires gamma > beta (PAPER.md:143)")
    x, _ = paper_blocks(key, n, gamma, k)
    y = mmh_eval(a, x, gamma)
    return mh_output(y, b, c, gamma, m)


def pa_hash_paper_seeded(key, n: int, gamma: int, k: int, m: int, seed: int) -> bytes:
    """pa_hash_paper with hash keys from ``seed`` (reading A7; alpha = gamma)."""
    a, b, c = expand_hash_keys(seed, k, gamma, gamma)
    return pa_hash_paper(key, n, gamma, k, m, a, b, c)


# ------------------------------------------------- comparator: MH-only PA (NEXT-4)
def mh_only_pa(key, n: int, m: int, b: int, c: int) -> bytes:
    """Modular-arithmetic-hashing-only PA (Table 1): the n
    input bits read MSB-first as an integer x; output = top m bits of (b x + c) mod 2^n,
    i.e. Eq. 4 with alpha = n, beta = m.  Emitted MSB-first (reading A5)."""
    if m > n:
        raise ValueError("m > n (SPEC.md:309)")
    kb = bytes(np.asarray(key, dtype=np.uint8)) if not isinstance(key, bytes) else key
    nbytes = (n + 7) // 8
    x = int.from_bytes(kb[:nbytes], "big") >> (8 * nbytes - n)
    return mh_output(x, b, c, n, m)


def mh_only_pa_seeded(key, n: int, m: int, seed: int) -> bytes:
    """mh_only_pa with b, c from ``seed`` (reading A7 streams, alpha = n)."""
    from .seeds import expand_b, expand_c
    return mh_only_pa(key, n, m, expand_b(seed, n), expand_c(seed, n))
