"""Device time of one C4 hash on a plain context, a one-rank NCCL context and a one-rank P2P
context (the multi-GPU code paths with world = 1), 256 MiB L2 flush before each (dev check)."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_13678_b200 import PAContext, pa as P  # noqa: E402
from synth import CONFIGS, key_bytes  # noqa: E402

w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
key = torch.from_numpy(key_bytes(w.n, w.key_seed)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
for name, kw in (("plain", {}), ("nccl1", dict(world=1, rank=0, nccl_id=P.nccl_unique_id())),
                 ("p2p1", dict(world=1, rank=0, nccl_id=P.nccl_unique_id(), p2p=True))):
    ctx = PAContext(w.n, w.r, w.m, seed=w.hash_seed, throughput_only=True, **kw)
    out = torch.empty(ctx.nbytes_out, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ctx.hash(key, out)
    ts = []
    for _ in range(20):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        ctx.hash(key, out)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    res[name] = round(statistics.median(ts), 4)
    res[name + "_out"] = bytes(out[:8].cpu().numpy()).hex()
    ctx.close()
print(json.dumps(res))
