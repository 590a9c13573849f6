"""Does an L2-resident X help the row MAC?  Per-vector times of the MMH forward passes at
increasing block counts (X = nblk * 12 * 2^17 * 4 B: 8 blocks = 50 MB fit L2, 31 do not)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2105_13678_b200 import PAContext  # noqa: E402

torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
res = {}
for nblk in (4, 8, 12, 16, 24, 31):
    n = nblk * (1 << 23)
    ctx = PAContext(n, 1 << 23, 2_600_000, seed=1, limb_bits=168, throughput_only=True)
    key = torch.randint(0, 256, ((n + 7) // 8,), dtype=torch.uint8, device="cuda")
    out = torch.empty(ctx.nbytes_out, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ctx.hash(key, out)
    ctx.set_profiling(True)
    ctx.stage_times(reset=True)
    K = 10
    for _ in range(K):
        flush.fill_(1)
        ctx.hash(key, out)
    torch.cuda.synchronize()
    stt = ctx.stage_times()
    P = ctx.info["mmh"]["nprimes"]
    res[nblk] = {k: round(v[0] / K * 1e3 / (nblk * P), 3) for k, v in stt.items() if k.startswith("mmh_")}
    res[nblk]["plan"] = [ctx.info["mmh"][k] for k in ("limb_bits", "nprimes", "log2_len")]
    ctx.close()
print(json.dumps(res, indent=1))
