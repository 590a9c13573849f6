"""The N>1 bench path (block shards -> pa_mmh_partial per rank ->
all-gather of residues -> pa_mh_merge on rank 0) run end to end as two processes.

The GPU box has one GPU, so both ranks sit on cuda:0 and exchange over gloo (host-staged);
the check is that the sharded hash equals the whole-key hash of a single context
(bench.py --verify).  NCCL itself is exercised only on multi-GPU nodes."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["C1", "C2"])
def test_two_rank_bench_matches_whole_key(config):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + int(config[1])),
           "bench.py", "--gpus", "2", "--steps", "5", "--warmup", "3", "--dist-backend", "gloo",
           "--same-device", "--verify", "--config", config, "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["verified_vs_whole_key"] is True
    assert line["value"] > 0 and line["gpu_launches"] > 0
    # NEXT-3 rotating-root stream mode ran and was verified against whole-key hashes too
    assert line["stream"]["keys_per_step"] == 2 and line["stream"]["value"] > 0
