"""Multi-rank host logic on CPU (-m "not gpu"): world_size-2 gloo process group.

The CUDA kernels cannot run here, so each rank's per-shard residue and the root's merge
are the ORACLE's (tests may use oracle/); what is under test is the library's host-side
multi-GPU logic in paper_2105_13678_b200/pa.py -- shard ranges, key slicing, the residue
all-gather (gather_residues / shard_gather_merge) and root-only output -- against the
unsharded oracle hash (split-merge)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hashes, seeds
from synth import key_bytes


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _words_tensor(v: int, gamma: int) -> torch.Tensor:
    nw = (gamma + 31) // 32
    return torch.from_numpy(np.frombuffer(v.to_bytes(4 * nw, "little"), dtype="<i4").copy())


def _int(words: torch.Tensor) -> int:
    return int.from_bytes(words.numpy().astype("<i4").tobytes(), "little")


def _worker(rank, world, port, n, r, m, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_13678_b200.pa import key_slice_bytes, shard_gather_merge, shard_ranges
        pp = hashes.plan_params(n, r, m)
        k, gamma, alpha = pp["k"], pp["gamma"], pp["alpha"]
        b0, b1 = shard_ranges(k, world)[rank]
        key = key_bytes(n, 0x77)
        lo, hi = key_slice_bytes(n, r, (b0, b1))
        key_slice = key[lo:hi]
        # a_i of this shard only (stream s = global block index, reading A7)
        a_shard = {i: seeds.expand_a(seed, i, gamma) for i in range(b0, b1)}

        def partial(ks):
            # residue of the shard from ITS key slice only (blocks renumbered from b0)
            nbits = min(n - b0 * r, (b1 - b0) * r)
            xs = hashes.key_blocks(np.asarray(ks), nbits, r)
            y = hashes.mmh_eval([a_shard[b0 + j] for j in range(len(xs))], xs, gamma)
            return _words_tensor(y, gamma)

        def merge(parts):
            assert parts.shape == (world, (gamma + 31) // 32)
            y = hashes.merge_residues([_int(p) for p in parts], gamma)
            b, c = seeds.expand_b(seed, alpha), seeds.expand_c(seed, alpha)
            return hashes.mh_output(y, b, c, alpha, m)

        out = shard_gather_merge(partial, merge, key_slice)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,r,m", [(100_003, 1024, 5_000), (65_536, 4096, 20_000)])
def test_gloo_two_ranks_equals_single(n, r, m):
    world, seed = 2, 1234
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(i, world, port, n, r, m, seed, q)) for i in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[1] is None                       # output exists on the root only
    want = hashes.pa_hash_seeded(key_bytes(n, 0x77), n, r, m, seed)
    assert res[0] == want


def _stream_worker(rank, world, port, n, r, m, seed, nkeys, q):
    """NEXT-3 rotating-root stream: key j's residues are gathered to rank j mod G."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_13678_b200.pa import key_slice_bytes, shard_ranges, stream_gather_merge
        pp = hashes.plan_params(n, r, m)
        k, gamma, alpha = pp["k"], pp["gamma"], pp["alpha"]
        b0, b1 = shard_ranges(k, world)[rank]
        lo, hi = key_slice_bytes(n, r, (b0, b1))
        slices = [key_bytes(n, 0x100 + j)[lo:hi] for j in range(nkeys)]
        a_shard = {i: seeds.expand_a(seed, i, gamma) for i in range(b0, b1)}

        def partial(ks):
            nbits = min(n - b0 * r, (b1 - b0) * r)
            xs = hashes.key_blocks(np.asarray(ks), nbits, r)
            return _words_tensor(hashes.mmh_eval([a_shard[b0 + j] for j in range(len(xs))], xs, gamma), gamma)

        def merge(parts):
            y = hashes.merge_residues([_int(p) for p in parts], gamma)
            return hashes.mh_output(y, seeds.expand_b(seed, alpha), seeds.expand_c(seed, alpha), alpha, m)

        q.put((rank, stream_gather_merge(partial, merge, slices)))
    finally:
        dist.destroy_process_group()


def test_gloo_rotating_root_stream():
    world, seed, nkeys = 2, 4321, 3
    n, r, m = 50_000, 2048, 3_000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stream_worker, args=(i, world, port, n, r, m, seed, nkeys, q)) for i in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(res[0]) == [0, 2] and sorted(res[1]) == [1]      # roots rotate: j mod G
    for rank, outs in res.items():
        for j, out in outs.items():
            assert out == hashes.pa_hash_seeded(key_bytes(n, 0x100 + j), n, r, m, seed), (rank, j)


# ----------------------------------------------------------- transform-domain exchange
def _crt_primes(bits_needed: int) -> list[int]:
    """Primes below 2^30 whose product exceeds 2^bits_needed (deterministic Miller-Rabin)."""
    def is_prime(v):
        if v < 2:
            return False
        for sp in (2, 3, 5, 7, 11, 13):
            if v % sp == 0:
                return v == sp
        d, s = v - 1, 0
        while d % 2 == 0:
            d, s = d // 2, s + 1
        for a in (2, 3, 5, 7, 11):
            x = pow(a, d, v)
            if x in (1, v - 1):
                continue
            for _ in range(s - 1):
                x = x * x % v
                if x == v - 1:
                    break
            else:
                return False
        return True
    ps, prod, v = [], 1, (1 << 30) - 1
    while prod.bit_length() <= bits_needed:
        if is_prime(v):
            ps.append(v)
            prod *= v
        v -= 2
    return ps


def _acc_worker(rank, world, port, n, r, m, seed, nkeys, q):
    """The multi-GPU exchange of include/pa.h (pa_mmh_acc / pa_tail_merge): every rank
    sends a LINEAR image of its blocks' exact sum Y_g = sum_{i in shard} a_i x_i (here its
    residues mod CRT primes, as the transform-domain accumulator is mod the NTT primes),
    the root sums the images mod each prime, recombines, folds mod p and runs MH.  Rank
    compute is the oracle's (no GPU); under test are shard_gather_merge /
    stream_gather_merge with a modular sum across ranks, and the root placement."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_13678_b200.pa import (key_slice_bytes, shard_gather_merge, shard_ranges,
                                               stream_gather_merge)
        pp = hashes.plan_params(n, r, m)
        k, gamma, alpha = pp["k"], pp["gamma"], pp["alpha"]
        primes = _crt_primes(k.bit_length() + r + gamma + 1)
        b0, b1 = shard_ranges(k, world)[rank]
        lo, hi = key_slice_bytes(n, r, (b0, b1))
        a_shard = {i: seeds.expand_a(seed, i, gamma) for i in range(b0, b1)}

        def acc(ks):
            nbits = min(n - b0 * r, (b1 - b0) * r)
            xs = hashes.key_blocks(np.asarray(ks), nbits, r)
            Y = sum(a_shard[b0 + j] * x for j, x in enumerate(xs))          # exact, no mod p
            return torch.tensor([Y % qq for qq in primes], dtype=torch.int64)

        def tail(parts):
            assert parts.shape == (world, len(primes))
            res = [int(v) % qq for v, qq in zip(parts.sum(0).tolist(), primes)]
            M, Y = 1, 0
            for rr, qq in zip(res, primes):                                 # CRT (Garner)
                t = ((rr - Y) * pow(M, -1, qq)) % qq
                Y += M * t
                M *= qq
            y = Y % ((1 << gamma) - 1)
            return hashes.mh_output(y, seeds.expand_b(seed, alpha), seeds.expand_c(seed, alpha), alpha, m)

        one = shard_gather_merge(acc, tail, key_bytes(n, 0x200)[lo:hi])
        many = stream_gather_merge(acc, tail, [key_bytes(n, 0x300 + j)[lo:hi] for j in range(nkeys)])
        q.put((rank, (one, many)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_transform_domain_exchange(world):
    n, r, m, seed, nkeys = 100_003, 1024, 5_000, 99, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_acc_worker, args=(i, world, port, n, r, m, seed, nkeys, q)) for i in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] == hashes.pa_hash_seeded(key_bytes(n, 0x200), n, r, m, seed)
    assert all(res[g][0] is None for g in range(1, world))
    for g in range(world):
        assert sorted(res[g][1]) == [j for j in range(nkeys) if j % world == g]
        for j, out in res[g][1].items():
            assert out == hashes.pa_hash_seeded(key_bytes(n, 0x300 + j), n, r, m, seed), (g, j)
