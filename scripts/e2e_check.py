"""e2e (pa_hash_host) timing, 15 reps after a 256 MiB L2 flush each (dev check)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_13678_b200 import PAContext
from synth import CONFIGS, key_bytes
w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "C4"]
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = PAContext(w.n, w.r, w.m, seed=w.hash_seed)
hk = torch.from_numpy(key_bytes(w.n, w.key_seed)).pin_memory()
ho = torch.empty(ctx.nbytes_out, dtype=torch.uint8).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
if "--batch-first" in sys.argv:
    kd = torch.from_numpy(key_bytes(w.n, w.key_seed)).cuda()
    keys = [kd.clone() for _ in range(8)]
    outs = [torch.empty(ctx.nbytes_out, dtype=torch.uint8, device="cuda") for _ in range(8)]
    for _ in range(3): ctx.hash_batch(keys, outs)
    torch.cuda.synchronize()
for _ in range(3): ctx.hash_host(hk, ho)
t = []
for _ in range(15):
    flush.fill_(1); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s); ctx.hash_host(hk, ho); b.record(s); b.synchronize()
    t.append(a.elapsed_time(b))
print("e2e ms median", round(statistics.median(t), 4), "min", round(min(t), 4), "max", round(max(t), 4))
kd = torch.empty_like(hk, device="cuda")
tc = []
for _ in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s); kd.copy_(hk, non_blocking=True); b.record(s); b.synchronize(); tc.append(a.elapsed_time(b))
print("h2d ms", round(min(tc), 4))
