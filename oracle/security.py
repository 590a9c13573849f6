"""Brute-force universality checks of the two hash families.  TEST INFRASTRUCTURE ONLY.

Appendix A: a (D;N,M) family is delta-universal if any two distinct
inputs collide under at most delta*D functions.  PAPER.md:89 claims delta = 1/|Z_p| for
MMH; Lemma 2 says the composition is (delta1+delta2)-universal.
These enumerations pin ``oracle.hashes.mmh_eval`` / ``mh_eval`` to those statements
(SPEC.md:162,401-409,515-517).
"""
from __future__ import annotations

import itertools
from fractions import Fraction

from .hashes import mh_eval, mmh_eval


def mmh_delta(gamma: int = 3, k: int = 2) -> Fraction:
    """max over x != x' in Z_p^k of #{a in Z_p^k : g_a(x) = g_a(x')} / p^k."""
    p = (1 << gamma) - 1
    dom = list(itertools.product(range(p), repeat=k))
    table = {x: [mmh_eval(a, x, gamma) for a in dom] for x in dom}
    worst = 0
    for i, x in enumerate(dom):
        tx = table[x]
        for x2 in dom[i + 1:]:
            t2 = table[x2]
            worst = max(worst, sum(1 for u, v in zip(tx, t2) if u == v))
    return Fraction(worst, len(dom))


def mh_delta(alpha: int = 4, beta: int = 2) -> Fraction:
    """max over y != y' in Z_{2^alpha} of #{(b odd, c)} colliding / |family|."""
    fam = [(b, c) for b in range(1, 1 << alpha, 2) for c in range(1 << alpha)]
    N = 1 << alpha
    table = [[mh_eval(b, c, y, alpha, beta) for (b, c) in fam] for y in range(N)]
    worst = 0
    for y in range(N):
        for y2 in range(y + 1, N):
            worst = max(worst, sum(1 for u, v in zip(table[y], table[y2]) if u == v))
    return Fraction(worst, len(fam))


def composed_delta(gamma: int = 3, k: int = 2, beta: int = 2) -> Fraction:
    """MMH then MH with alpha = gamma (Algorithm 1): max collision fraction over
    x != x' in Z_p^k, family = all (a, b, c)."""
    p = (1 << gamma) - 1
    alpha = gamma
    dom = list(itertools.product(range(p), repeat=k))
    mh_fam = [(b, c) for b in range(1, 1 << alpha, 2) for c in range(1 << alpha)]
    # y-table per (x, a), then MH collisions counted per (a) over the MH family.
    ytab = {x: [mmh_eval(a, x, gamma) for a in dom] for x in dom}
    # for a pair of MMH outputs (y1, y2), the number of colliding MH functions:
    mhcoll = {}
    for y1 in range(1 << alpha):
        for y2 in range(1 << alpha):
            mhcoll[(y1, y2)] = sum(1 for (b, c) in mh_fam
                                   if mh_eval(b, c, y1, alpha, beta) == mh_eval(b, c, y2, alpha, beta))
    worst = 0
    for i, x in enumerate(dom):
        for x2 in dom[i + 1:]:
            tot = sum(mhcoll[(u, v)] for u, v in zip(ytab[x], ytab[x2]))
            worst = max(worst, tot)
    return Fraction(worst, len(dom) * len(mh_fam))
