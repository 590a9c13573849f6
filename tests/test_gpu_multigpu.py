"""GPU parity of the multi-GPU split (SURVEY.md §8(b,e)) through the C ABI, on one GPU.

- pa_mmh_acc / pa_tail_merge: G shard contexts (the ranks' block ranges) each produce the
  transform-domain accumulator of their blocks; the sum, inverse-transformed and finished
  on one context, must equal the CPU oracle's hash of the whole key (MMH is linear over a
  partition of the blocks).
- Multi-GPU contexts (pa_params.world/rank/nccl_id) with a one-rank NCCL communicator run
  the library's own ncclReduce path (pa_hash, and pa_hash_batch with the rotating root)
  against the oracle.  NCCL across several ranks needs a multi-GPU node.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import hashes  # noqa: E402
from synth import CONFIGS, key_bytes  # noqa: E402


def _P():
    from paper_2105_13678_b200 import pa
    return pa


@pytest.mark.parametrize("n,r,m,G", [(100_003, 1024, 5_000, 1), (100_003, 1024, 5_000, 2),
                                     (262_157, 2048, 30_001, 3), (300_000, 4096, 4_000, 5),
                                     (1 << 20, 1 << 16, 104_858, 4)])
def test_transform_merge_equals_oracle(n, r, m, G):
    P = _P()
    seed = 77
    key = key_bytes(n, 0x51 + G)
    k = -(-n // r)
    ctxs, parts = [], []
    for (b0, b1) in P.shard_ranges(k, G):
        ctx = P.PAContext(n, r, m, seed=seed, block_range=(b0, b1))
        lo, hi = P.key_slice_bytes(n, r, (b0, b1))
        parts.append(ctx.mmh_acc(torch.from_numpy(key[lo:hi].copy()).cuda()))
        ctxs.append(ctx)
    acc = torch.stack(parts)
    want = hashes.pa_hash_seeded(key, n, r, m, seed)
    for ctx in (ctxs[0], ctxs[-1]):
        out = ctx.tail_merge(acc)
        torch.cuda.synchronize()
        assert bytes(out.cpu().numpy()) == want
    # the whole-key context's accumulator is the parts' sum mod each NTT prime
    whole = P.PAContext(n, r, m, seed=seed)
    wa = whole.mmh_acc(torch.from_numpy(key).cuda()).to(torch.int64).cpu()
    info = whole.query()
    L = 1 << info["mmh"]["log2_len"]
    q = torch.tensor(info["mmh"]["primes"], dtype=torch.int64).repeat_interleave(L)
    s = acc.to(torch.int64).cpu().sum(0) % q
    assert torch.equal(s, wa)
    assert bool((wa < q).all())
    out = whole.tail_merge(wa.to(torch.int32).cuda().unsqueeze(0))
    torch.cuda.synchronize()
    assert bytes(out.cpu().numpy()) == want
    for ctx in ctxs + [whole]:
        ctx.close()


def _one_rank_ctx(P, n, r, m, seed, **kw):
    try:
        nid = P.nccl_unique_id()
    except Exception as e:  # pragma: no cover
        pytest.fail(f"NCCL not loadable on the GPU box: {e}")
    return P.PAContext(n, r, m, seed=seed, world=1, rank=0, nccl_id=nid, **kw)


@pytest.mark.parametrize("on_stream", [False, True])
@pytest.mark.parametrize("p2p", [False, True])
def test_nccl_one_rank_hash_and_rotating_batch(on_stream, p2p):
    # p2p: the peer-memory exchange (row MAC mode 3 into the root's 64-bit receive buffer,
    # counters waited on / signalled by p2p_wait / p2p_signal) with the rank as its own root
    P = _P()
    n, r, m, seed = 262_157, 2048, 30_001, 4
    s = torch.cuda.Stream() if on_stream else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        ctx = _one_rank_ctx(P, n, r, m, seed, p2p=p2p)
        assert ctx.world == 1 and ctx.rank == 0 and ctx.query()["p2p"] == int(p2p)
        for ks in (1, 2):
            key = key_bytes(n, 0x900 + ks)
            out = ctx.hash(torch.from_numpy(key).cuda())
            s.synchronize()
            assert bytes(out.cpu().numpy()) == hashes.pa_hash_seeded(key, n, r, m, seed)
        keys = [key_bytes(n, 0xA00 + j) for j in range(5)]
        outs = ctx.hash_batch([torch.from_numpy(kk).cuda() for kk in keys])
        s.synchronize()
        for kk, o in zip(keys, outs):
            assert bytes(o.cpu().numpy()) == hashes.pa_hash_seeded(kk, n, r, m, seed)
        info = ctx.query()
        from paper_2105_13678_b200 import _binding as B
        if on_stream and not B.pa_debug_build():          # the debug build captures no graphs
            # new key / output pointers re-capture and update the graphs in place
            assert info["graph_captures"] >= 2 and info["graph_instantiations"] <= info["graph_captures"]
        ctx.close()


@pytest.mark.parametrize("p2p", [False, True])
@pytest.mark.parametrize("pinned", [False, True])
def test_nccl_one_rank_hash_host(p2p, pinned):
    # pa_hash_host on a multi-GPU context: the rank's key slice in from host memory, the merged
    # hash, the output back on rank 0 (one rank: the same H2D, reduce / p2p exchange, tail, D2H)
    P = _P()
    n, r, m, seed = 262_157, 2048, 30_001, 6
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = _one_rank_ctx(P, n, r, m, seed, p2p=p2p)
        for ks in (1, 2, 3):
            key = key_bytes(n, 0xB00 + ks)
            hk = torch.from_numpy(key)
            ho = torch.zeros(ctx.nbytes_out, dtype=torch.uint8)
            if pinned:
                hk, ho = hk.pin_memory(), ho.pin_memory()
            got = ctx.hash_host(hk, ho)
            assert got is ho
            assert bytes(ho.numpy()) == hashes.pa_hash_seeded(key, n, r, m, seed)
        ctx.close()


@pytest.mark.parametrize("p2p", [False, True])
def test_nccl_one_rank_hash_host_batch(p2p):
    # pa_hash_host_batch on a multi-GPU context: slices in from host memory on the copy stream
    # (two staging buffers), rotating root, outputs back to host; five keys, twice
    P = _P()
    n, r, m, seed = 262_157, 2048, 30_001, 9
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = _one_rank_ctx(P, n, r, m, seed, p2p=p2p)
        keys = [key_bytes(n, 0xE00 + j) for j in range(5)]
        want = [hashes.pa_hash_seeded(kk, n, r, m, seed) for kk in keys]
        hk = [torch.from_numpy(kk).pin_memory() for kk in keys]
        for _ in range(2):
            ho = [torch.zeros(ctx.nbytes_out, dtype=torch.uint8).pin_memory() for _ in keys]
            ctx.hash_host_batch(hk, ho)
            assert [bytes(o.numpy()) for o in ho] == want
        outs = ctx.hash_host_batch(keys[:3])             # pageable numpy keys, library-made outputs
        assert [bytes(o) for o in outs] == want[:3]
        ctx.close()


def test_nccl_one_rank_u64_exchange(monkeypatch):
    # the exchange of world > 4 jobs (64-bit sums: acc_export<u64>, ncclUint64 reduce,
    # acc_import_u64), forced on a one-rank communicator with PA_FORCE_X64
    monkeypatch.setenv("PA_FORCE_X64", "1")
    P = _P()
    n, r, m, seed = 262_157, 2048, 30_001, 8
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = _one_rank_ctx(P, n, r, m, seed)
        for ks in (1, 2):
            key = key_bytes(n, 0xC00 + ks)
            out = ctx.hash(torch.from_numpy(key).cuda())
            s.synchronize()
            assert bytes(out.cpu().numpy()) == hashes.pa_hash_seeded(key, n, r, m, seed)
        keys = [key_bytes(n, 0xD00 + j) for j in range(3)]
        outs = ctx.hash_batch([torch.from_numpy(kk).cuda() for kk in keys])
        s.synchronize()
        for kk, o in zip(keys, outs):
            assert bytes(o.cpu().numpy()) == hashes.pa_hash_seeded(kk, n, r, m, seed)
        hk = torch.from_numpy(keys[0]).pin_memory()
        ho = torch.zeros(ctx.nbytes_out, dtype=torch.uint8).pin_memory()
        ctx.hash_host(hk, ho)
        assert bytes(ho.numpy()) == hashes.pa_hash_seeded(keys[0], n, r, m, seed)
        ctx.close()


@pytest.mark.parametrize("p2p", [False, True])
def test_nccl_one_rank_c2_golden(p2p):
    import hashlib
    import json
    import os
    P = _P()
    w = CONFIGS["C2"]
    ctx = _one_rank_ctx(P, w.n, w.r, w.m, w.hash_seed, p2p=p2p)
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "digests.json")))
    key = torch.from_numpy(key_bytes(w.n, w.key_seed)).cuda()
    for _ in range(3):            # the receive buffers alternate; each is zeroed and freed after use
        out = ctx.hash(key)
        torch.cuda.synchronize()
        assert hashlib.sha256(bytes(out.cpu().numpy())).hexdigest() == gold["C2"]["out_sha256"]
    ctx.close()


def test_graph_update_on_new_pointers():
    # verdict r1 #8: a hash on new key/output buffers re-captures and updates the executable
    # graph in place (cudaGraphExecUpdate) instead of re-instantiating; results stay exact
    P = _P()
    n, r, m, seed = 300_001, 4096, 20_000, 8
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = P.PAContext(n, r, m, seed=seed)
        for ks in range(4):
            key = key_bytes(n, 0xB00 + ks)
            kd = torch.from_numpy(key).cuda()                 # a new buffer every time
            out = ctx.hash(kd)
            s.synchronize()
            assert bytes(out.cpu().numpy()) == hashes.pa_hash_seeded(key, n, r, m, seed)
        info = ctx.query()
        from paper_2105_13678_b200 import _binding as B
        if B.pa_debug_build():
            pytest.skip("the bounds-asserting build captures no graphs")
        assert info["graph_captures"] >= 2
        assert info["graph_instantiations"] == 1 and info["graph_updates"] == info["graph_captures"] - 1
        ctx.close()


def test_torch_allocator_and_default_allocator_agree():
    # pa_params.dev_alloc: the context's device memory from PyTorch's caching allocator
    # (default in the binding) or cudaMallocAsync (torch_allocator=False); same results
    P = _P()
    n, r, m, seed = 100_003, 1024, 5_000, 12
    key = key_bytes(n, 0xC00)
    outs = []
    for ta in (True, False):
        before = torch.cuda.memory_allocated()
        ctx = P.PAContext(n, r, m, seed=seed, torch_allocator=ta)
        held = torch.cuda.memory_allocated() - before
        assert (held >= ctx.query()["device_bytes"]) if ta else (held == 0)
        outs.append(bytes(ctx.hash(torch.from_numpy(key).cuda()).cpu().numpy()))
        ctx.close()
        if ta:
            assert torch.cuda.memory_allocated() == before
    assert outs[0] == outs[1] == hashes.pa_hash_seeded(key, n, r, m, seed)


def test_debug_build_catches_out_of_range():
    # under the bounds-asserting build (PA_DEV_LIB=.../_pa_debug.so, scripts/gpu_debug.sh)
    # the checker must catch one out-of-range global address and one shared index
    from paper_2105_13678_b200 import _binding as B
    if B.pa_debug_build() != 1:
        pytest.skip("release build loaded (run the suite with PA_DEV_LIB=_pa_debug.so)")
    torch.cuda.init()
    assert B.pa_debug_selftest() == B.PA_OK
