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
