"""Which bench step makes the following pa_hash_host e2e slower? (dev check)"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_13678_b200 import PAContext
from synth import CONFIGS, key_bytes
w = CONFIGS["C4"]
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
key_full = key_bytes(w.n, w.key_seed)
ctx = PAContext(w.n, w.r, w.m, seed=w.hash_seed)
hk = torch.from_numpy(key_full).pin_memory()
ho = torch.empty(ctx.nbytes_out, dtype=torch.uint8).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
kd = torch.from_numpy(key_full).cuda()
out = torch.empty(ctx.nbytes_out, dtype=torch.uint8, device="cuda")
def e2e(tag):
    for _ in range(2): ctx.hash_host(hk, ho)
    t = []
    for _ in range(15):
        flush.fill_(1); torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s); ctx.hash_host(hk, ho); b.record(s); b.synchronize()
        t.append(a.elapsed_time(b))
    print(tag, "e2e median", round(statistics.median(t), 4), "min", round(min(t), 4))
e2e("fresh")
for _ in range(20): ctx.hash(kd, out)
torch.cuda.synchronize()
e2e("after device hashes")
ctx.set_profiling(True); ctx.stage_times(reset=True)
for _ in range(10): ctx.hash(kd, out)
ctx.stage_times(); ctx.set_profiling(False)
e2e("after profiling pass")
e2e("again")
