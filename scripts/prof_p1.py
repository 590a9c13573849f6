"""One warm-up + one paper-mode (P1) pa_hash, for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_13678_b200 import PAContext
from synth import PAPER_CONFIGS, key_bytes
w = PAPER_CONFIGS["P1"]
ctx = PAContext(w.n, 0, w.m, w.gamma, seed=w.hash_seed, paper_k=w.k)
key = torch.from_numpy(key_bytes(w.n, w.key_seed)).cuda()
for _ in range(2):
    out = ctx.hash(key)
torch.cuda.synchronize()
ctx.status()
print("ok", bytes(out[:8].cpu().numpy()).hex())
