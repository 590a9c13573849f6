"""Toeplitz comparator (NEXT-4) at the C5 shape, n = 2^31 > every NTT prime of the length:
input blocks summed in groups whose counts stay below the prime (parities XORed), 52 output
blocks in MAC launches of at most 16.  Times the hash and checks sampled output bits against
the oracle (oracle/toeplitz.py toeplitz_bits, one row at a time).  Development check."""
import json, random, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from oracle import toeplitz as OT
from paper_2105_13678_b200 import PAContext
from synth import CONFIGS, key_bytes

w = CONFIGS["C5a"] if "C5a" in CONFIGS else CONFIGS["C5"]
n, m, seed = w.n, w.m, w.hash_seed
key = key_bytes(n, w.key_seed)
t0 = time.time()
ctx = PAContext(n, 0, m, 0, seed=seed, toeplitz=True)
torch.cuda.synchronize()
create_s = time.time() - t0
info = ctx.query()
kd = torch.from_numpy(key).cuda()
out = torch.empty(ctx.nbytes_out, dtype=torch.uint8, device="cuda")
ctx.hash(kd, out); torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(3):
    ev[0].record(); ctx.hash(kd, out); ev[1].record(); torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
got = bytes(out.cpu().numpy())
r = info["r"]; g = info["tz_group_blocks"]
rng = random.Random(5)
js = sorted({0, r - 1, r, 17 * r + 3, m - 1} | {rng.randrange(m) for _ in range(3)})
d = OT.expand_diagonal(seed, n + m - 1)
want = OT.toeplitz_bits(key.tobytes(), n, m, d, js)
ok = all(((got[j >> 3] >> (7 - (j & 7))) & 1) == b for j, b in zip(js, want))
print(json.dumps({"n": n, "m": m, "r": r, "input_blocks": info["k"], "output_blocks": info["alpha"],
                  "prime": info["mmh"]["primes"][0], "group_blocks": g, "groups": -(-info["k"] // g),
                  "device_GB": info["device_bytes"] / 1e9, "create_s": round(create_s, 1),
                  "hash_ms": [round(t, 2) for t in ts], "Mbps": n / (min(ts) * 1e-3) / 1e6,
                  "sampled_bits": len(js), "sampled_ok": ok}))
