"""CPU-side checks of the C ABI (-m "not gpu"): the library loads, exports every symbol
include/pa.h declares, validates parameters, plans transforms whose CRT modulus covers
the coefficient bound, and expands hash keys exactly as the oracle does (reading A7)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from paper_2105_13678_b200 import _binding as B
from paper_2105_13678_b200 import pa as P
from oracle import seeds as oseeds
from synth import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "pa.h")).read()
    declared = set(re.findall(r"\b(pa_[a-z0-9_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    lib = ctypes.CDLL(B.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/pa.h but not exported"
    assert declared == set(B.EXPORTED)


@pytest.mark.parametrize("kw,code", [
    (dict(n=0, r=16, m=8), B.PA_E_PARAM),
    (dict(n=100, r=15, m=8), B.PA_E_PARAM),
    (dict(n=100, r=24, m=8), B.PA_E_PARAM),            # r % 16 != 0
    (dict(n=100, r=16, m=0), B.PA_E_PARAM),
    (dict(n=100, r=64, m=8, gamma=61), B.PA_E_PARAM),   # gamma <= r
    (dict(n=100, r=64, m=8, gamma=67), B.PA_E_PARAM),   # not a Mersenne exponent
    (dict(n=1000, r=64, m=100, gamma=89, strict=True), B.PA_E_PARAM),  # m >= gamma
    (dict(n=1000, r=64, m=8, block_range=(3, 3)), B.PA_E_PARAM),
    (dict(n=1000, r=64, m=8, block_range=(0, 17)), B.PA_E_PARAM),
    (dict(n=1000, r=64, m=8, limb_bits=12), B.PA_E_PARAM),
])
def test_plan_rejects(kw, code):
    with pytest.raises(B.PAError) as ei:
        P.plan(**kw)
    assert ei.value.code == code


@pytest.mark.parametrize("name", list(CONFIGS))
def test_plan_configs(name):
    w = CONFIGS[name]
    info = P.plan(w.n, w.r, w.m)
    from oracle.hashes import plan_params
    pp = plan_params(w.n, w.r, w.m)
    assert info["gamma"] == pp["gamma"] and info["alpha"] == pp["alpha"] and info["k"] == pp["k"]
    for st in ("mmh", "mh"):
        s = info[st]
        assert s["bound_log2"] < s["modulus_log2"]
        # independent recomputation of the coefficient bound and the CRT modulus
        Bl = s["limb_bits"]
        if st == "mmh":
            wa, wb, terms = -(-w.r // Bl), -(-pp["gamma"] // Bl), pp["k"]
        else:
            wa, wb, terms = -(-pp["gamma"] // Bl), -(-pp["alpha"] // Bl), 1
        bound = terms * min(wa, wb) * (2 ** Bl - 1) ** 2
        modulus = math.prod(s["primes"])
        assert bound < modulus
        assert (1 << s["log2_len"]) >= wa + wb - 1        # no cyclic wrap-around
        assert s["n_col"] * s["n_row"] == 1 << s["log2_len"]
        for p in s["primes"]:
            assert p < 2 ** 30 and (p - 1) % (1 << s["log2_len"]) == 0
            assert pow(3, p - 1, p) == 1 and all(p % d for d in range(2, 1000))


def test_plan_forced_limb_bits():
    for Bl in (16, 24, 32, 40, 48, 56, 64, 96, 168, 200):
        info = P.plan(1 << 20, 1 << 16, 100_000, limb_bits=Bl)
        assert info["mmh"]["limb_bits"] == Bl and info["mh"]["limb_bits"] == Bl
    with pytest.raises(B.PAError):
        P.plan(1 << 20, 1 << 16, 100_000, limb_bits=264)    # at most 8 words per limb
    with pytest.raises(B.PAError) as e:
        P.plan(1 << 20, 1 << 16, 100_000, limb_bits=256)    # would need > 16 primes
    assert e.value.code == B.PA_E_BOUND


def test_philox_matches_numpy():
    # T1: product-side Philox4x64-10 == numpy.random.Philox (library routine)
    for key in [(0, 0), (5, 7), (2**64 - 1, 2**63), (0x5EED0004, 13)]:
        out = np.zeros(37, dtype=np.uint64)
        B.check(B.pa_philox4x64_10(key[0], key[1], 37, out.ctypes.data))
        want = np.random.Philox(key=np.array(key, dtype=np.uint64)).random_raw(37)
        assert np.array_equal(out, want)


@pytest.mark.parametrize("seed,gamma,alpha", [(1234, 89, 200), (0x5EED0001, 86243, 104858), (7, 17, 40)])
def test_expand_keys_match_oracle(seed, gamma, alpha):
    for i in (0, 1, 5, 1000):
        w = np.zeros((gamma + 31) // 32, dtype="<u4")
        B.check(B.pa_expand_a(seed, i, gamma, w.ctypes.data))
        assert int.from_bytes(w.tobytes(), "little") == oseeds.expand_a(seed, i, gamma)
    bw = np.zeros((alpha + 31) // 32, dtype="<u4")
    cw = np.zeros_like(bw)
    B.check(B.pa_expand_bc(seed, alpha, bw.ctypes.data, cw.ctypes.data))
    assert int.from_bytes(bw.tobytes(), "little") == oseeds.expand_b(seed, alpha)
    assert int.from_bytes(cw.tobytes(), "little") == oseeds.expand_c(seed, alpha)


def test_expand_a_rejection_matches_oracle():
    # gamma = 17: an all-ones first draw is rare; search streams where it happens
    found = 0
    for i in range(300_000):
        w = np.random.Philox(key=np.array([3, i], dtype=np.uint64)).random_raw(1)
        if int(w[0]) & ((1 << 17) - 1) == (1 << 17) - 1:
            out = np.zeros(1, dtype="<u4")
            B.check(B.pa_expand_a(3, i, 17, out.ctypes.data))
            assert int(out[0]) == oseeds.expand_a(3, i, 17) != (1 << 17) - 1
            found += 1
            if found == 2:
                break
    assert found >= 1


def test_shard_ranges():
    assert P.shard_ranges(31, 8) == [(0, 3), (3, 7), (7, 11), (11, 15), (15, 19), (19, 23), (23, 27), (27, 31)]
    for k in (1, 7, 31, 2048):
        for G in (1, 2, 3, 8):
            rs = P.shard_ranges(k, G)
            assert rs[0][0] == 0 and rs[-1][1] == k
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    assert P.key_slice_bytes(1000, 64, (3, 16)) == (24, 125)


def test_ctx_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(B.PAError):
        P.PAContext(1 << 12, 256, 100)
    assert not B.pa_ctx_create(1 << 12, 256, 100, 0, 1)


def test_plan_paper_mode():
    # NEXT-1: Algorithm 1 in the paper's shape (gamma-bit blocks, alpha = gamma)
    info = P.plan(259_649_510, 0, 25_237_932, 25_964_951, paper_k=10)
    assert info["gamma"] == info["alpha"] == 25_964_951 and info["k"] == 10
    for s in (info["mmh"], info["mh"]):
        assert s["bound_log2"] < s["modulus_log2"]
    bad = [dict(n=1000, r=0, m=10, gamma=0, paper_k=3),            # gamma required
           dict(n=1000, r=0, m=107, gamma=107, paper_k=3),         # m < gamma
           dict(n=300, r=0, m=10, gamma=107, paper_k=3),           # n >= k gamma
           dict(n=1000, r=0, m=10, gamma=100, paper_k=3)]          # not a Mersenne exponent
    for kw in bad:
        with pytest.raises(B.PAError):
            P.plan(kw["n"], kw["r"], kw["m"], kw["gamma"], paper_k=kw["paper_k"])
    with pytest.raises(B.PAError):
        P.plan(1000, 0, 10, 107, block_range=(0, 1), paper_k=3)    # no shards


def test_plan_mh_only():
    info = P.plan(260_000_000, 0, 26_000_000, 0, mh_only=True)
    assert info["alpha"] == 260_000_000 and info["mh"]["bound_log2"] < info["mh"]["modulus_log2"]
    for kw in (dict(gamma=89), dict(r=64), dict(paper_k=3), dict(block_range=(0, 1))):
        args = dict(n=1000, r=0, m=10, gamma=0)
        args.update({k: v for k, v in kw.items() if k in ("gamma", "r")})
        with pytest.raises(B.PAError):
            P.plan(args["n"], args["r"], args["m"], args["gamma"], mh_only=True,
                   paper_k=kw.get("paper_k", 0), block_range=kw.get("block_range"))
    with pytest.raises(B.PAError):
        P.plan(100, 0, 101, 0, mh_only=True)                      # m > n


def test_toeplitz_plan():
    """NEXT-4 Toeplitz comparator plan: one prime above n, L = 2r, r x r block counts."""
    info = P.plan(260_000_000, 0, 26_000_000, toeplitz=True)
    assert info["r"] == 1 << 22 and info["k"] == 62 and info["alpha"] == 7
    t = info["mmh"]
    assert t["nprimes"] == 1 and t["log2_len"] == 23 and t["primes"][0] > 260_000_000
    assert t["n_col"] * t["n_row"] == 1 << 23
    small = P.plan(100, 0, 37, toeplitz=True)
    assert small["r"] == 512 and small["k"] == 1 and small["alpha"] == 1
    forced = P.plan(5000, 0, 1500, toeplitz=True, limb_bits=9)
    assert forced["k"] == 10 and forced["alpha"] == 3
    assert info["tz_group_blocks"] == 62                       # n below the prime: one accumulation
    # n above every NTT prime of the length (C5: 2^31 key bits): the input blocks are summed in
    # groups whose counts stay below the prime, floor((p - 1) / r) blocks each; m > 16 r is
    # accumulated 16 output blocks at a time
    big = P.plan(1 << 31, 0, 214_748_365, toeplitz=True)
    q = big["mmh"]["primes"][0]
    assert big["r"] == 1 << 22 and big["k"] == 512 and big["alpha"] == 52 and q < 1 << 31
    assert big["tz_group_blocks"] == (q - 1) // (1 << 22) and big["tz_group_blocks"] * (1 << 22) < q
    assert P.plan(1 << 31, 0, 10, toeplitz=True, tz_group_blocks=3)["tz_group_blocks"] == 3
    with pytest.raises(B.PAError):
        P.plan(100, 0, 1 << 31, toeplitz=True)                # m < 2^31
    with pytest.raises(B.PAError):
        P.plan(100, 16, 10, toeplitz=True)            # r is chosen by the planner
    with pytest.raises(B.PAError):
        P.plan(100, 0, 10, toeplitz=True, limb_bits=8)


@pytest.mark.parametrize("total,n,jobs,rem", [
    (2 * 1000 + 5, 1000, 2, 5),        # SPEC.md pa_stream: 2 full jobs + 5 leftover bits
    (0, 1000, 0, 0),                   # empty input: no jobs, no remainder
    (12, 12, 1, 0), (11, 12, 0, 11), (260_000_000 * 3 + 7, 260_000_000, 3, 7)])
def test_stream_partition(total, n, jobs, rem):
    assert P.stream_partition(total, n) == (jobs, rem)


def test_insecure_length_flag():
    # reading A1: m >= gamma is accepted (alpha = m) but flagged; strict rejects it
    assert P.plan(260_000_000, 1 << 23, 26_000_000)["insecure_length"] == 1     # C4: m > gamma
    assert P.plan(10_485_760, 1 << 20, 1_048_576)["insecure_length"] == 0       # C2: m < gamma
    assert P.plan(4096, 4096, 4423)["insecure_length"] == 1                     # m == gamma


def _host_checker():
    import torch
    ctx = P.PAContext.__new__(P.PAContext)      # the argument checks only (no GPU)
    ctx._torch = torch
    return ctx, torch


def test_host_buffer_checks_reject_bad_buffers():
    # pa_hash_host reads ceil(n/8) and writes ceil(m/8) bytes through raw
    # pointers, so short, strided, non-uint8, read-only or device buffers must be rejected
    ctx, torch = _host_checker()
    ok = np.zeros(100, np.uint8)
    assert ctx._host_u8(ok, 100, "key") == ok.ctypes.data
    assert ctx._host_u8(torch.zeros(100, dtype=torch.uint8), 64, "key") > 0
    bad = [np.zeros(99, np.uint8),                       # short
           np.zeros(200, np.uint8)[::2],                 # strided
           np.zeros(100, np.uint16),                     # wrong dtype
           torch.zeros(200, dtype=torch.uint8)[::2],     # non-contiguous tensor
           torch.zeros(100, dtype=torch.int32),          # wrong tensor dtype
           [0] * 100]                                    # not a buffer
    for b in bad:
        with pytest.raises(ValueError):
            ctx._host_u8(b, 100, "buf")
    ro = np.zeros(100, np.uint8)
    ro.flags.writeable = False
    assert ctx._host_u8(ro, 100, "key") > 0              # a key may be read-only
    with pytest.raises(ValueError):
        ctx._host_u8(ro, 100, "out", writable=True)      # an output may not


def test_plan_multi_gpu_world():
    # rank g of G owns blocks [k g / G, k (g+1) / G); every rank plans the
    # whole key's transform so the transform-domain accumulators are compatible
    n, r, m = 260_000_000, 1 << 23, 26_000_000
    whole = P.plan(n, r, m)
    for G in (1, 2, 3, 8):
        for g in range(G):
            info = P.plan(n, r, m, world=G, rank=g)
            assert (info["block_begin"], info["block_end"]) == P.shard_ranges(31, G)[g]
            assert info["world"] == G and info["rank"] == g
            assert info["mmh"] == whole["mmh"] and info["mh"] == whole["mh"]
            assert info["acc_words"] == whole["mmh"]["nprimes"] << whole["mmh"]["log2_len"]
    # a plain shard context plans the whole key's transform too
    assert P.plan(n, r, m, block_range=(3, 9))["mmh"] == whole["mmh"]
    bad = [dict(world=2, rank=2), dict(world=-1), dict(world=0, rank=1), dict(world=32, rank=0),
           dict(world=2, rank=0, block_range=(0, 3)), dict(world=2, rank=0, paper_k=3)]
    for kw in bad:
        with pytest.raises(B.PAError) as ei:
            if "paper_k" in kw:
                P.plan(1000, 0, 10, 107, **kw)
            else:
                P.plan(n, r, m, **kw)
        assert ei.value.code == B.PA_E_PARAM
    P.plan(n, r, m, world=2, rank=1, block_range=(15, 31))        # the exact range is accepted


def test_nccl_unique_id_host_only():
    # the library loads NCCL at run time (dlopen); the id is 128 bytes and fresh per call
    try:
        a, b = P.nccl_unique_id(), P.nccl_unique_id()
    except B.PAError as e:
        assert e.code == B.PA_E_NCCL
        pytest.skip(f"NCCL not loadable here: {e}")
    assert len(a) == 128 and len(b) == 128 and a != b


def test_debug_build_flag():
    # release _pa.so reports 0 and refuses the self-test; the bounds-asserting build
    # (_pa_debug.so, -DPA_DEBUG) is exercised on the GPU by tests/test_gpu_multigpu.py
    if os.environ.get("PA_DEV_LIB"):
        pytest.skip("a development library is loaded")
    assert B.pa_debug_build() == 0
    assert B.pa_debug_selftest() == B.PA_E_STATE


def test_struct_mirrors_match_library():
    # the ctypes mirrors of pa_params / pa_info have the library's layout size
    pb, ib = ctypes.c_uint64(), ctypes.c_uint64()
    assert B.pa_abi_sizes(ctypes.byref(pb), ctypes.byref(ib)) == 0
    assert pb.value == ctypes.sizeof(B.pa_params)
    assert ib.value == ctypes.sizeof(B.pa_info)


def test_plan_p2p_needs_multi_gpu_context():
    # pa_params.p2p (peer-memory accumulator exchange) is a multi-GPU option only
    n, r, m = 1 << 20, 1 << 16, 104_858
    P.plan(n, r, m, world=2, rank=0, p2p=True)
    for kw in (dict(p2p=True), dict(world=0, rank=0, p2p=True)):
        with pytest.raises(B.PAError) as ei:
            P.plan(n, r, m, **kw)
        assert ei.value.code == B.PA_E_PARAM
