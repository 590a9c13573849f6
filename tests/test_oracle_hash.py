"""Pins of oracle/hashes.py, oracle/seeds.py, oracle/security.py, oracle/schoolbook.c.

Each check ties the oracle to something other than itself: a value printed in the
paper/SPEC, a closed form, a brute-force enumeration, an independent formulation
(bit strings instead of integer shifts) or an independent library routine.
"""
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import hashes, schoolbook, security, seeds
from oracle.hashes import (bits_to_field_blocks, key_blocks, mh_eval, mmh_eval,
                           pa_run_paper)
from synth import key_bytes, special_key

import philox_ref  # noqa: E402  (tests/ is on sys.path under pytest)


# ------------------------------------------------------------------ SPEC examples
def test_mmh_spec_examples():
    assert mmh_eval([3, 5], [2, 6], 3) == 1
    assert mmh_eval([0, 0], [4, 5], 3) == 0
    assert mmh_eval([1], [4], 3) == 4


def test_mh_spec_examples():
    assert mh_eval(3, 1, 5, 3, 2) == 0
    assert mh_eval(1, 0, 5, 3, 3) == 5
    assert mh_eval(5, 3, 7, 4, 2) == 1
    with pytest.raises(ValueError):
        mh_eval(3, 1, 5, 3, 4)                       # beta > alpha


def test_mh_is_top_bits_exhaustive():
    # MH output is the beta most significant bits of the alpha-bit affine
    # value, all inputs at alpha <= 8 (checked through a bit-string formulation).
    for alpha in range(1, 7):
        for beta in range(1, alpha + 1):
            for b in range(1, 1 << alpha, 2):
                for c in range(0, 1 << alpha, 3):
                    for y in range(1 << alpha):
                        s = format((b * y + c) % (2 ** alpha), f"0{alpha}b")
                        assert mh_eval(b, c, y, alpha, beta) == int(s[:beta], 2)


def test_bits_to_field_blocks_spec_examples():
    # SPEC.md:76-78
    assert bits_to_field_blocks([1, 1, 1, 0, 1, 0, 1, 1, 0], 3, 2) == ([2, 6], 9, 1)
    assert bits_to_field_blocks([0] * 6, 3, 2) == ([0, 0], 6, 0)
    with pytest.raises(ValueError):
        bits_to_field_blocks([1] * 9, 3, 1)


def test_pa_run_spec_example():
    # gamma=3, k=2, m=2, a=(3,5), b=3, c=1, bits 010 110 -> output 10
    out, consumed, rejected = pa_run_paper([0, 1, 0, 1, 1, 0], 3, 2, 2, [3, 5], 3, 1)
    assert out == [1, 0] and consumed == 6 and rejected == 0
    # all-zero input with c = 0 -> all zeros
    out, _, _ = pa_run_paper([0] * 62, 31, 2, 16, [12345, 678], 77, 0)
    assert out == [0] * 16


def test_pa_run_matches_straight_line():
    # SPEC.md:246 / acceptance 5: 100 random instances at gamma=31, k=4, m=16 equal an
    # independent straight-line evaluation with general % and no folding / splitting.
    rng = random.Random(5)
    g, k, m = 31, 4, 16
    p = (1 << g) - 1
    for _ in range(100):
        bits = [rng.getrandbits(1) for _ in range(g * k + 3 * g)]
        a = [rng.randrange(p) for _ in range(k)]
        b, c = rng.getrandbits(g) | 1, rng.getrandbits(g)
        out, consumed, _ = pa_run_paper(bits, g, k, m, a, b, c)
        xs, pos = [], 0
        while len(xs) < k:
            v = int("".join(map(str, bits[pos:pos + g])), 2)
            pos += g
            if v != p:
                xs.append(v)
        y = sum(ai * xi for ai, xi in zip(a, xs)) % p
        z = ((b * y + c) % 2 ** g) // 2 ** (g - m)
        assert out == [int(ch) for ch in format(z, f"0{m}b")]
        assert consumed == pos


@pytest.mark.parametrize("n,r,m", [(1000, 64, 50), (4096, 256, 300), (3001, 512, 520), (2048, 1024, 1)])
def test_rbit_pa_hash_m_below_gamma_straight_line(n, r, m):
    # The library's r-bit shape with m < gamma, where the paper fixes alpha = gamma
    # (reading A1 reduces to it): an independent straight-line
    # Algorithm 1 with general % and bit strings -- key bits MSB-first, zero-extended to
    # k r bits (A3, A4), x_i the r-bit windows, y = sum a_i x_i % p,
    # z = ((b y + c) % 2^gamma) // 2^(gamma - m), output bits MSB-first (A5).
    pp = hashes.plan_params(n, r, m)
    g, k = pp["gamma"], pp["k"]
    assert m < g and pp["alpha"] == g
    rng = random.Random(n + r + m)
    key = bytes(rng.getrandbits(8) for _ in range((n + 7) // 8))
    p = 2 ** g - 1
    a = [rng.randrange(p) for _ in range(k)]
    b, c = rng.getrandbits(g) | 1, rng.getrandbits(g)
    bits = "".join(format(byte, "08b") for byte in key)[:n].ljust(k * r, "0")
    xs = [int(bits[i * r:(i + 1) * r], 2) for i in range(k)]
    y = sum(ai * xi for ai, xi in zip(a, xs)) % p
    z = ((b * y + c) % 2 ** g) // 2 ** (g - m)
    zb = format(z, f"0{m}b").ljust(-(-m // 8) * 8, "0")
    want = bytes(int(zb[8 * t:8 * t + 8], 2) for t in range(len(zb) // 8))
    assert hashes.pa_hash(key, n, r, m, g, a, b, c) == want
    # and the seeded entry point uses alpha = gamma for b and c
    a2, b2, c2 = seeds.expand_hash_keys(11, k, g, g)
    assert hashes.pa_hash_seeded(key, n, r, m, 11) == hashes.pa_hash(key, n, r, m, g, a2, b2, c2)


# ---------------------------------------------------------- brute-force universality
def test_mmh_universality_bruteforce():
    # MMH collision probability delta = 1/|Z_p|; SPEC.md:515 gamma=3, k=2.
    assert security.mmh_delta(3, 2) == Fraction(1, 7)


def test_mh_universality_bruteforce():
    # measured delta <= 2^(1-beta); measured value 1/4 = 2^-beta.
    d = security.mh_delta(4, 2)
    assert d <= Fraction(1, 2)
    assert d == Fraction(1, 4)


def test_composition_lemma2_bruteforce():
    # Lemma 2: composed family is (delta1 + delta2)-universal.
    d = security.composed_delta(3, 2, 2)
    assert d <= security.mmh_delta(3, 2) + security.mh_delta(3, 2)
    assert d == Fraction(560, 1568)


# ------------------------------------------------------------------ invariants
def test_mmh_linearity_and_split_merge():
    # SPEC.md:160-161
    rng = random.Random(9)
    g, k = 127, 9
    p = (1 << g) - 1
    for _ in range(50):
        a = [rng.randrange(p) for _ in range(k)]
        x = [rng.randrange(p) for _ in range(k)]
        x2 = [rng.randrange(p) for _ in range(k)]
        s = [(u + v) % p for u, v in zip(x, x2)]
        assert mmh_eval(a, s, g) == (mmh_eval(a, x, g) + mmh_eval(a, x2, g)) % p
        cut = sorted(rng.sample(range(1, k), 3))
        parts = [range(0, cut[0]), range(cut[0], cut[1]), range(cut[1], cut[2]), range(cut[2], k)]
        ys = [mmh_eval([a[i] for i in P], [x[i] for i in P], g) for P in parts]
        assert hashes.merge_residues(ys, g) == mmh_eval(a, x, g)


def _blocks_by_bitstring(key, n, r):
    s = "".join(format(int(v), "08b") for v in key)[:n]
    k = -(-n // r)
    s = s + "0" * (k * r - n)
    return [int(s[i * r:(i + 1) * r], 2) for i in range(k)]


@pytest.mark.parametrize("n,r", [(64, 16), (1000, 64), (1003, 48), (777, 40), (4097, 128),
                                 (333, 17), (100, 7)])
def test_key_blocks_bit_order(n, r):
    # readings A3/A4 via an independent bit-string formulation
    key = key_bytes(n, n * 31 + r)
    assert key_blocks(key, n, r) == _blocks_by_bitstring(key, n, r)


def test_pack_output_bit_order():
    rng = random.Random(3)
    for m in (1, 7, 8, 9, 31, 64, 100):
        z = rng.getrandbits(m)
        s = format(z, f"0{m}b")
        s += "0" * (-len(s) % 8)
        want = bytes(int(s[i:i + 8], 2) for i in range(0, len(s), 8))
        assert hashes.pack_output(z, m) == want


def test_rotation_closed_form():
    # a_i = 2^j  =>  a_i x_i mod M_gamma is the gamma-bit left rotation of x_i by j
    # (2^gamma = 1 mod p).  Checked with string rotation.
    rng = random.Random(4)
    for g in (17, 89, 521, 4423):
        p = (1 << g) - 1
        for _ in range(20):
            x = rng.randrange(p)
            j = rng.randrange(g)
            s = format(x, f"0{g}b")
            rot = int(s[j:] + s[:j], 2)
            rot = 0 if rot == p else rot
            assert mmh_eval([1 << j], [x], g) == rot


def test_identity_and_canonical_zero_end_to_end():
    n, r, m = 256, 64, 89
    g = 89
    key = key_bytes(n, 77)
    x = key_blocks(key, n, r)
    # identity: a = (1,0,..), b = 1, c = 0, alpha = m = gamma -> z = x_0
    out = hashes.pa_hash(key, n, r, m, g, [1, 0, 0, 0], 1, 0)
    assert int.from_bytes(out, "big") >> (8 * len(out) - m) == x[0]
    # canonical zero (A6): Y = p -> y = 0 -> z = top m bits of c
    p = (1 << g) - 1
    key1 = np.zeros(2 * r // 8, np.uint8)
    key1[r // 8 - 1] = 1
    key1[2 * r // 8 - 1] = 1                       # x_0 = x_1 = 1
    c = random.Random(1).getrandbits(g)
    out = hashes.pa_hash(key1, 2 * r, r, m, g, [p - 1, 1], 12345 | 1, c)
    assert out == hashes.pack_output(c >> (g - m), m)


# ------------------------------------------------------------------ seeds (A7)
def test_seed_expansion_contract():
    a, b, c = seeds.expand_hash_keys(1234, 5, 89, 200)
    assert all(0 <= v < (1 << 89) - 1 for v in a)
    assert b % 2 == 1 and 0 < b < (1 << 200) and 0 <= c < (1 << 200)
    # raw Philox words, little-endian, masked: numpy stream key (seed, i)
    w = np.random.Philox(key=np.array([1234, 3], dtype=np.uint64)).random_raw(2)
    assert a[3] == (int(w[0]) | (int(w[1]) << 64)) & ((1 << 89) - 1)


def test_philox_stream_equals_written_out_definition():
    # numpy.random.Philox (the oracle's generator, reading A7) against Philox4x64-10 written
    # out from its definition (tests/philox_ref.py), on the stream keys the oracle uses:
    # a_i (seed, i), b (seed, 2^63), c (seed, 2^63 + 1), and a key with every bit set
    for key in [(0, 0), (1234, 3), (0x5EED0004, seeds.STREAM_B), (0x5EED0004, seeds.STREAM_C),
                (2**64 - 1, 2**64 - 1)]:
        want = philox_ref.stream_words(*key, 11)
        assert [int(v) for v in seeds._philox(*key).random_raw(11)] == want


@pytest.mark.parametrize("seed,alpha", [(0x5EED0001, 104_858), (0x5EED0004, 26_000_000 // 1000),
                                        (7, 1), (7, 64), (7, 65), (2**64 - 1, 200)])
def test_expand_b_c_pinned_to_reference_streams(seed, alpha):
    # PAPER.md:142 "b, c in Z_{2^gamma}, gcd(b,2) = 1"; reading A7: b = draw of stream
    # (seed, 2^63) with bit 0 forced, c = draw of stream (seed, 2^63 + 1) as drawn.  The
    # words come from the written-out Philox, not from numpy, so a key-conversion slip
    # (2^63 + 1 rounded to 2^63 gives c the stream of b) fails here.
    nw = (alpha + 63) // 64
    b_ref = philox_ref.draw(philox_ref.stream_words(seed, 1 << 63, nw), alpha) | 1
    c_ref = philox_ref.draw(philox_ref.stream_words(seed, (1 << 63) + 1, nw), alpha)
    assert seeds.expand_b(seed, alpha) == b_ref
    assert seeds.expand_c(seed, alpha) == c_ref
    if alpha >= 64:
        # the two streams differ (c is not b's stream with bit 0 as drawn)
        assert c_ref != philox_ref.draw(philox_ref.stream_words(seed, 1 << 63, nw), alpha)


def test_expand_a_pinned_to_reference_stream():
    # a_i: ceil(gamma/64) words of stream (seed, i), all-ones rejected
    for seed, i, g in [(99, 0, 89), (99, 30, 521), (2**63, 5, 4423), (5, 1, 3)]:
        ws = philox_ref.stream_words(seed, i, 64 * ((g + 63) // 64))
        nw = (g + 63) // 64
        allones = (1 << g) - 1
        t = 0
        while True:
            v = philox_ref.draw(ws[t * nw:(t + 1) * nw], g)
            t += 1
            if v != allones:
                break
        assert seeds.expand_a(seed, i, g) == v


def test_seed_rejection_of_all_ones():
    # an all-ones draw is rejected and the next draw taken
    hits = 0
    for i in range(400):
        bg = np.random.Philox(key=np.array([99, i], dtype=np.uint64))
        first = int(bg.random_raw(1)[0]) & 7
        second = int(bg.random_raw(1)[0]) & 7
        a = seeds.expand_a(99, i, 3)
        if first == 7:
            hits += 1
            assert a == second if second != 7 else a != 7
        else:
            assert a == first
    assert hits > 0


def test_seed_uniformity_chi_square():
    # over 10^4 draws at gamma=3 each residue within 5 sigma of uniform
    counts = [0] * 7
    for i in range(10_000):
        counts[seeds.expand_a(2024, i, 3)] += 1
    mu = 10_000 / 7
    sd = (10_000 * (1 / 7) * (6 / 7)) ** 0.5
    assert all(abs(cnt - mu) < 5 * sd for cnt in counts)


# ------------------------------------------------------------------ schoolbook C oracle
@pytest.mark.parametrize("n,r,m", [(4096, 256, 700), (100_003, 1024, 5000), (65_536, 2048, 6000),
                                   (300_000, 4096, 30_000)])
def test_schoolbook_equals_python_int(n, r, m):
    # schoolbook (plain C) == CPython int multiplication (independent library routine)
    key = key_bytes(n, n + r)
    pp = hashes.plan_params(n, r, m)
    a, b, c = seeds.expand_hash_keys(n ^ r, pp["k"], pp["gamma"], pp["alpha"])
    assert schoolbook.pa_hash(key, n, r, m, pp["gamma"], a, b, c, nthreads=2) == \
        hashes.pa_hash(key, n, r, m, pp["gamma"], a, b, c)


def test_schoolbook_partial_and_merge():
    n, r, g = 50_000, 512, 521
    key = key_bytes(n, 3)
    k = -(-n // r)
    a, _, _ = seeds.expand_hash_keys(5, k, g, g)
    cuts = [0, 13, 50, k]
    ys = [schoolbook.mmh_partial(key, n, r, g, a[cuts[j]:cuts[j + 1]], cuts[j], cuts[j + 1])
          for j in range(3)]
    assert schoolbook.merge(ys, g) == hashes.mmh_partial(key, n, r, g, a)
    assert ys[1] == hashes.mmh_partial(key, n, r, g, a, range(13, 50))


@pytest.mark.parametrize("kind", ["zero", "ones", "alt", "bit"])
def test_special_keys_oracles_agree(kind):
    n, r, m = 8192, 512, 900
    key = special_key(kind, n, pos=n - 1)
    pp = hashes.plan_params(n, r, m)
    a, b, c = seeds.expand_hash_keys(11, pp["k"], pp["gamma"], pp["alpha"])
    py = hashes.pa_hash(key, n, r, m, pp["gamma"], a, b, c)
    assert schoolbook.pa_hash(key, n, r, m, pp["gamma"], a, b, c, nthreads=2) == py
    if kind == "zero":
        assert py == hashes.pack_output(c >> (pp["alpha"] - m), m)


def test_paper_blocks_match_bit_list_version():
    # the byte-key fast path of Algorithm 1's split + reload equals bits_to_field_blocks
    import random
    rng = random.Random(7)
    for gamma in (5, 7, 13, 17):
        k = 4
        for trial in range(30):
            nb = rng.randrange(k * gamma // 8 + 2, k * gamma // 8 + 12)
            kb = bytearray(rng.getrandbits(8) for _ in range(nb))
            # plant all-ones windows to exercise the reload rule
            n = 8 * nb - rng.randrange(0, 8)
            bits = [(kb[i >> 3] >> (7 - (i & 7))) & 1 for i in range(n)]
            for t in range(n // gamma):
                if rng.random() < 0.3:
                    for q in range(t * gamma, (t + 1) * gamma):
                        bits[q] = 1
            kb = bytearray((n + 7) // 8)
            for i, bit in enumerate(bits):
                kb[i >> 3] |= bit << (7 - (i & 7))
            try:
                want, used, _ = hashes.bits_to_field_blocks(bits, gamma, k)
            except ValueError:
                with pytest.raises(ValueError):
                    hashes.paper_blocks(bytes(kb), n, gamma, k)
                continue
            got, t_used = hashes.paper_blocks(bytes(kb), n, gamma, k)
            assert got == want and t_used * gamma == used


def test_pa_hash_paper_spec_example():
    # gamma=3, k=2, m=2, a=(3,5), b=3, c=1, bits 010 110 -> 10
    key = bytes([0b01011000])
    assert hashes.pa_hash_paper(key, 6, 3, 2, 2, [3, 5], 3, 1) == bytes([0b10000000])


def test_mh_only_pa_spec_example():
    # n=4, m=2, b=5, c=3, x=0111 (7) -> (38 mod 16) = 6 -> 01
    assert hashes.mh_only_pa(bytes([0b01110000]), 4, 2, 5, 3) == bytes([0b01000000])
    # b=1, c=0, m=n -> identity
    assert hashes.mh_only_pa(bytes([0xA5, 0x3C]), 16, 16, 1, 0) == bytes([0xA5, 0x3C])


def test_mh_only_equals_mh_eval_exhaustive():
    # mh_only_pa(n, m) == mh_eval with alpha = n, beta = m, exhaustive at n <= 8
    n, m = 6, 3
    for x in range(1 << n):
        for b in range(1, 1 << n, 2):
            for c in (0, 5, 63):
                key = bytes([x << 2])
                got = hashes.mh_only_pa(key, n, m, b, c)
                assert got == bytes([hashes.mh_eval(b, c, x, n, m) << 5])
