"""Per-stage times of the Toeplitz comparator at the C4 shape (dev check)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_13678_b200 import PAContext
from synth import CONFIGS, key_bytes
w = CONFIGS["C4"]
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = PAContext(w.n, 0, w.m, 0, seed=w.hash_seed, toeplitz=True)
kd = torch.from_numpy(key_bytes(w.n, w.key_seed)).cuda()
out = torch.empty(ctx.nbytes_out, dtype=torch.uint8, device="cuda")
for _ in range(2): ctx.hash(kd, out)
ctx.set_profiling(True); ctx.stage_times(reset=True)
for _ in range(5): ctx.hash(kd, out)
st = ctx.stage_times(); ctx.set_profiling(False)
print({k: round(v[0] / 5 * 1e3, 1) for k, v in sorted(st.items())})
print(ctx.query()["mmh"])
