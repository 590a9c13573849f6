"""Model check of the P2P accumulator-exchange protocol (pa_params.p2p; DESIGN.md §8,
csrc/pa_api.cu mg_hash_p2p, csrc/exchange.cuh p2p_wait / p2p_signal), on CPU.

The cross-GPU form needs a multi-GPU node, so its ordering logic is checked here as a model
that follows the library's sequence step by step: G ranks, each with the two hashing streams
of pa_hash_batch (key j on stream j & 1), run the same call sequence; streams interleave at
random.  Per key j with root q = j mod G and receive buffer s = (keys rooted at q so far) & 1:

  every rank r (pre):  wait FREE[q][s] >= EXPF[q][s] + 1, EXPF += 1;  add its partial into
                       q's recv[s] (atomics);  READY[s][r] += 1 on rank q
  root q (post):       wait READY[s][r'] >= EXPR[s][r'] + 1 for all r', EXPR += 1;  import
                       recv[s] and zero it;  FREE[q][s] += 1 on every rank

FREE starts at 1 (every buffer free for its first use), everything else at 0.  Checked: no
deadlock under any sampled schedule, and every import sees exactly that key's G partials --
nothing left over from an earlier key, nothing early from a later one.  The same model with
the FREE wait removed must fail (the check can see a reuse race)."""
import random

import pytest


def run(G: int, K: int, seed: int, skip_free_wait: bool = False):
    rng = random.Random(seed)
    FREE = [[[1, 1] for _ in range(G)] for _ in range(G)]       # FREE[rank][q][s]
    EXPF = [[[0, 0] for _ in range(G)] for _ in range(G)]
    READY = [[[0] * G for _ in range(2)] for _ in range(G)]     # READY[rank][s][r']
    EXPR = [[[0] * G for _ in range(2)] for _ in range(G)]
    recv = [[[] for _ in range(2)] for _ in range(G)]           # recv[rank][s]: partials (key, rank)
    imported = []
    uses = [0] * G
    queues = {(r, st): [] for r in range(G) for st in range(2)}  # (rank, stream) -> ops
    for j in range(K):
        q = j % G
        s = uses[q] & 1
        uses[q] += 1                                               # host-side, identical on every rank
        for r in range(G):
            ops = queues[(r, j & 1)]
            if not skip_free_wait:
                ops.append(("wait_free", q, s))
            ops.append(("add", q, s, j))
            ops.append(("signal_ready", q, s))
            if r == q:
                ops.append(("wait_ready", s))
                ops.append(("import", s, j))
                ops.append(("signal_free", s))

    def runnable(r, op):
        if op[0] == "wait_free":
            _, q, s = op
            return FREE[r][q][s] >= EXPF[r][q][s] + 1
        if op[0] == "wait_ready":
            _, s = op
            return all(READY[r][s][x] >= EXPR[r][s][x] + 1 for x in range(G))
        return True

    def execute(r, op):
        if op[0] == "wait_free":
            _, q, s = op
            EXPF[r][q][s] += 1
        elif op[0] == "add":
            _, q, s, j = op
            recv[q][s].append((j, r))
        elif op[0] == "signal_ready":
            _, q, s = op
            READY[q][s][r] += 1
        elif op[0] == "wait_ready":
            _, s = op
            for x in range(G):
                EXPR[r][s][x] += 1
        elif op[0] == "import":
            _, s, j = op
            imported.append((j, sorted(recv[r][s])))
            recv[r][s] = []
        elif op[0] == "signal_free":
            _, s = op
            for x in range(G):
                FREE[x][r][s] += 1

    while any(queues.values()):
        ready = [k for k, ops in queues.items() if ops and runnable(k[0], ops[0])]
        if not ready:
            return "deadlock", imported
        k = rng.choice(ready)
        execute(k[0], queues[k].pop(0))
    return "done", imported


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_p2p_protocol_no_deadlock_and_exact_sums(G):
    K = 6 * G + 3
    for seed in range(200):
        status, imported = run(G, K, seed)
        assert status == "done", (G, seed)
        assert len(imported) == K
        for j, parts in imported:
            assert parts == [(j, r) for r in range(G)], (G, seed, j, parts)


def test_p2p_model_detects_a_missing_free_wait():
    # without the FREE wait a rank may add a later key's partial into a buffer the root has
    # not imported yet: some schedule must show it (the check is not vacuous)
    bad = 0
    for seed in range(300):
        status, imported = run(2, 12, seed, skip_free_wait=True)
        if status != "done" or any(parts != [(j, r) for r in range(2)] for j, parts in imported):
            bad += 1
    assert bad > 0
