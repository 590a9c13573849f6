"""One warm-up + one timed pa_hash of a config (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_13678_b200 import PAContext
from synth import CONFIGS, key_bytes
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
w = CONFIGS[name]
ctx = PAContext(w.n, w.r, w.m, seed=w.hash_seed)
key = torch.from_numpy(key_bytes(w.n, w.key_seed)).cuda()
for _ in range(2):
    out = ctx.hash(key)
torch.cuda.synchronize()
print("ok", bytes(out[:8].cpu().numpy()).hex())
