"""Seeded random shapes (-m gpu): MMH-MH in r-bit mode, paper mode and the Toeplitz
comparator, each bit-exact against the oracle.  Shapes are drawn to cross the planner's
regimes (limb widths, prime counts, transform lengths, column splits, ragged key and output
tails, m above and below gamma, many blocks on short transforms)."""
import os
import random

import numpy as np
import pytest
import torch

from oracle import hashes, mersenne, toeplitz
from synth import key_bytes

pytestmark = pytest.mark.gpu

RNG = random.Random(int(os.environ.get("PA_FUZZ_SEED", "20261020")))
SCALE = int(os.environ.get("PA_FUZZ_SCALE", "1"))           # more shapes for a one-off stress run
SHAPES = []
for _ in range(24 * SCALE):
    r = 16 * RNG.choice([1, 2, 3, 7, 16, 61, 64, 100, 256, 1000, 4096])
    n = RNG.randint(1, 40) * r + RNG.randint(-r + 1, r - 1) if RNG.random() < 0.8 else RNG.randint(1, 3 * r)
    n = max(1, n)
    m = RNG.randint(1, max(1, 2 * n))
    SHAPES.append((n, r, m, RNG.getrandbits(32)))


def _dev(b):
    return torch.from_numpy(np.frombuffer(bytes(b), dtype=np.uint8).copy()).cuda()


@pytest.mark.parametrize("n,r,m,seed", SHAPES)
def test_fuzz_mmh_mh(n, r, m, seed):
    from paper_2105_13678_b200 import PAContext
    key = key_bytes(n, seed ^ 0x55)
    ctx = PAContext(n, r, m, seed=seed)
    got = bytes(ctx.hash(_dev(key)).cpu().numpy())
    ctx.close()
    assert got == hashes.pa_hash_seeded(key, n, r, m, seed)


PAPER = []
for _ in range(6 * SCALE):
    g = RNG.choice([89, 107, 127, 521, 607, 1279, 2203])
    k = RNG.randint(1, 12)
    n = k * g + RNG.randint(0, 2 * g)
    m = RNG.randint(1, g - 1)
    PAPER.append((n, g, k, m, RNG.getrandbits(32)))


@pytest.mark.parametrize("n,g,k,m,seed", PAPER)
def test_fuzz_paper_mode(n, g, k, m, seed):
    from paper_2105_13678_b200 import PAContext
    key = key_bytes(n, seed ^ 0xAA)
    ctx = PAContext(n, 0, m, g, seed=seed, paper_k=k)
    got = bytes(ctx.hash(_dev(key)).cpu().numpy())
    ctx.close()
    assert got == hashes.pa_hash_paper_seeded(key, n, g, k, m, seed)


TZ = []
for _ in range(6 * SCALE):
    n = RNG.randint(1, 60_000)
    m = RNG.randint(1, 20_000)
    lr = RNG.choice([0, 9, 10])
    TZ.append((n, m, lr, RNG.getrandbits(32)))


@pytest.mark.parametrize("n,m,lr,seed", TZ)
def test_fuzz_toeplitz(n, m, lr, seed):
    from paper_2105_13678_b200 import PAContext
    key = key_bytes(n, seed ^ 0x33)
    ctx = PAContext(n, 0, m, 0, seed=seed, toeplitz=True, limb_bits=lr)
    got = bytes(ctx.hash(_dev(key)).cpu().numpy())
    ctx.close()
    assert got == toeplitz.toeplitz_pa_seeded(key, n, m, seed)
