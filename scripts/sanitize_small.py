"""Small hashes for compute-sanitizer runs (r-bit mode, paper mode, batch, shards)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_13678_b200 import PAContext
from paper_2105_13678_b200.pa import key_slice_bytes, shard_ranges
from oracle import hashes
from synth import key_bytes

n, r, m, seed = 100_003, 1024, 5_000, 3
key = key_bytes(n, 9)
ctx = PAContext(n, r, m, seed=seed)
out = ctx.hash(torch.from_numpy(key).cuda())
torch.cuda.synchronize()
assert bytes(out.cpu().numpy()) == hashes.pa_hash_seeded(key, n, r, m, seed)
outs = ctx.hash_batch([torch.from_numpy(key).cuda()] * 3)
torch.cuda.synchronize()
assert all(bytes(o.cpu().numpy()) == hashes.pa_hash_seeded(key, n, r, m, seed) for o in outs)
assert bytes(ctx.hash_host(key)) == hashes.pa_hash_seeded(key, n, r, m, seed)
ctx.close()
g, k = 607, 4
pn = 5 * g
pkey = key_bytes(pn, 4)
pctx = PAContext(pn, 0, 100, g, seed=1, paper_k=k)
pout = pctx.hash(torch.from_numpy(pkey).cuda())
pctx.status()
assert bytes(pout.cpu().numpy()) == hashes.pa_hash_paper_seeded(pkey, pn, g, k, 100, 1)
pctx.close()
kk = -(-n // r)
parts = []
for (b0, b1) in shard_ranges(kk, 2):
    c = PAContext(n, r, m, seed=seed, block_range=(b0, b1))
    lo, hi = key_slice_bytes(n, r, (b0, b1))
    parts.append(c.mmh_partial(torch.from_numpy(key[lo:hi].copy()).cuda()))
    if b0 == 0:
        c0 = c
o = c0.mh_merge(torch.stack(parts))
torch.cuda.synchronize()
assert bytes(o.cpu().numpy()) == hashes.pa_hash_seeded(key, n, r, m, seed)
print("sanitize_small ok")
