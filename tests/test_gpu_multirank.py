"""The N>1 bench path (block shards -> pa_mmh_acc per rank -> exchange of
the transform-domain accumulators -> pa_tail_merge on the key's root) run end to end as
two and three processes.

The GPU box has one GPU, so the ranks sit on cuda:0 and exchange over gloo (host-staged);
bench.py --verify checks the single-key output (root 0) and the rotating-root stream
outputs (key j on rank j mod G) against the CPU oracle: the golden digest of the config's
key and oracle hashes of the rolled keys.  The library's own NCCL reduce runs as a
one-rank communicator in tests/test_gpu_multigpu.py; NCCL across ranks needs a multi-GPU
node."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("config,nproc", [("C1", 2), ("C2", 2), ("C1", 3)])
def test_multirank_bench_matches_oracle(config, nproc):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + 10 * nproc + int(config[1])),
           "bench.py", "--gpus", str(nproc), "--steps", "5", "--warmup", "3", "--dist-backend", "gloo",
           "--same-device", "--verify", "--config", config, "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == nproc
    assert line["verified_vs_oracle"] is True
    assert line["value"] > 0 and line["gpu_launches"] > 0
    # NEXT-3 rotating-root stream mode ran and was verified against the oracle too
    assert line["stream"]["keys_per_step"] == 2 * nproc and line["stream"]["value"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("p2p", [False, True])
def test_bench_multi_gpu_path_one_rank(p2p):
    """The product N>1 bench path -- library NCCL context, reduce (or peer-memory exchange),
    rotating-root pa_hash_batch, pa_hash_host on the multi-GPU context for e2e -- with a
    one-rank communicator; single-key, stream and e2e outputs checked against the CPU oracle."""
    cmd = [sys.executable, "bench.py", "--one-rank-mg", "--verify", "--config", "C2", "--steps", "5",
           "--warmup", "3"] + (["--p2p"] if p2p else [])
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29650 + int(p2p)), RANK="0", WORLD_SIZE="1")
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, lines                     # exactly one JSON line on stdout
    line = json.loads(lines[0])
    assert line["verified_vs_oracle"] is True
    assert line["e2e"]["verified_vs_oracle"] is True and line["e2e"]["value"] > 0
    assert line["stream"]["value"] > 0 and line["gpu_launches"] > 0
    assert "one_rank_mg=True" in line["validation_only"]
