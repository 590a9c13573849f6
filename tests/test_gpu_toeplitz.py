"""Toeplitz-hashing PA comparator (NEXT-4) on the GPU against the oracle (oracle/toeplitz.py),
bit-exact: small shapes whole, block-split shapes (forced r) whole, the C4 shape sampled."""
import random

import numpy as np
import pytest
import torch

from oracle import toeplitz as OT
from synth import CONFIGS, key_bytes

pytestmark = pytest.mark.gpu


def _hash(n, m, seed, key, limb_bits=0, tz_group_blocks=0):
    from paper_2105_13678_b200 import PAContext
    ctx = PAContext(n, 0, m, 0, seed=seed, toeplitz=True, limb_bits=limb_bits, tz_group_blocks=tz_group_blocks)
    out = torch.empty(ctx.nbytes_out, dtype=torch.uint8, device="cuda")
    ctx.hash(torch.from_numpy(np.frombuffer(key, dtype=np.uint8).copy()).cuda(), out)
    torch.cuda.synchronize()
    info = ctx.query()
    ctx.close()
    return bytes(out.cpu().numpy()), info


@pytest.mark.parametrize("n,m", [(1, 1), (2, 2), (7, 3), (8, 8), (100, 37), (37, 100), (513, 512), (1000, 999),
                                 (4096, 409), (70_001, 7_001)])
def test_toeplitz_small_whole(n, m):
    key = key_bytes(n, 0x500 + n)
    got, _ = _hash(n, m, 99, key)
    assert got == OT.toeplitz_pa_seeded(key, n, m, 99)


@pytest.mark.parametrize("n,m,lr", [(5000, 1500, 9), (4096, 4096, 9), (20_000, 3_333, 10), (100_000, 16 * 512, 9),
                                    (9_999, 17, 9), (600, 5000, 9)])
def test_toeplitz_block_split_whole(n, m, lr):
    """r forced below max(n, m): several input blocks (sum over b in the transform domain)
    and several output blocks (one inverse each), ragged tails on both sides."""
    key = key_bytes(n, 0x600 + n)
    got, info = _hash(n, m, 7, key, limb_bits=lr)
    assert info["r"] == 1 << lr and info["k"] == -(-n // (1 << lr)) and info["alpha"] == -(-m // (1 << lr))
    assert got == OT.toeplitz_pa_seeded(key, n, m, 7)


@pytest.mark.parametrize("n,m,lr,grp", [(40_000, 20_000, 9, 1), (40_000, 20_000, 9, 3), (5_000, 9_500, 9, 2),
                                        (70_001, 10_000, 10, 5), (600, 5000, 9, 1)])
def test_toeplitz_input_groups_and_many_output_blocks(n, m, lr, grp):
    """Input blocks accumulated in groups of `grp` (each group's counts exact, parities XORed:
    the path n >= prime takes with groups of floor((prime - 1) / r) blocks) and more than 16
    output blocks (MAC launches of at most 16 accumulators), against the oracle."""
    key = key_bytes(n, 0x900 + n)
    got, info = _hash(n, m, 5, key, limb_bits=lr, tz_group_blocks=grp)
    assert info["tz_group_blocks"] == grp and info["alpha"] == -(-m // (1 << lr))
    assert got == OT.toeplitz_pa_seeded(key, n, m, 5)


def test_toeplitz_special_keys():
    n, m = 3000, 1000
    for key in (bytes(375), b"\xff" * 375, b"\xaa" * 375):
        got, _ = _hash(n, m, 3, key)
        assert got == OT.toeplitz_pa_seeded(key, n, m, 3)
    assert _hash(n, m, 3, bytes(375))[0] == bytes(125)          # zero key -> zero output (linear map)


def test_toeplitz_c4_shape_sampled():
    """The bench shape (C4: n = 2.6e8, m = 2.6e7; r = 2^22, 62 x 7 blocks, L = 2^23): 24 output
    bits, spread over all seven output blocks and both block edges, checked one by one."""
    w = CONFIGS["C4"]
    key = key_bytes(w.n, w.key_seed).tobytes()
    got, info = _hash(w.n, w.m, w.hash_seed, key)
    assert info["k"] == 62 and info["alpha"] == 7 and info["mmh"]["log2_len"] == 23
    r = 1 << 22
    rng = random.Random(1)
    js = sorted({0, 1, r - 1, r, 2 * r + 5, 6 * r, w.m - 1, w.m - 2} | {rng.randrange(w.m) for _ in range(16)})
    d = OT.expand_diagonal(w.hash_seed, w.n + w.m - 1)
    want = OT.toeplitz_bits(key, w.n, w.m, d, js)
    for j, b in zip(js, want):
        assert (got[j >> 3] >> (7 - (j & 7))) & 1 == b, j
    assert all(v == 0 for v in [got[-1] & ((1 << (8 * len(got) - w.m)) - 1)])   # pad bits zero


def test_toeplitz_host_path_and_graph_replay():
    from paper_2105_13678_b200 import PAContext
    n, m = 50_000, 9_000
    key = key_bytes(n, 0x777)
    want = OT.toeplitz_pa_seeded(key, n, m, 11)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = PAContext(n, 0, m, 0, seed=11, toeplitz=True, limb_bits=12)
        hk = torch.from_numpy(np.frombuffer(key, dtype=np.uint8).copy()).pin_memory()
        ho = torch.empty(ctx.nbytes_out, dtype=torch.uint8).pin_memory()
        for _ in range(3):                      # graph capture, then replays
            ctx.hash_host(hk, ho)
            assert bytes(ho.numpy()) == want
        kd = hk.cuda()
        od = torch.empty(ctx.nbytes_out, dtype=torch.uint8, device="cuda")
        for _ in range(3):
            ctx.hash(kd, od)
        torch.cuda.synchronize()
        assert bytes(od.cpu().numpy()) == want
        ctx.close()
