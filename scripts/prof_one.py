"""Context creation + two warm-up hashes, then ONE pa_hash of a config inside
cudaProfilerStart/Stop (for `ncu --profile-from-start off`: exactly the hash's kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2105_13678_b200 import PAContext  # noqa: E402
from synth import CONFIGS, key_bytes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
w = CONFIGS[name]
ctx = PAContext(w.n, w.r, w.m, seed=w.hash_seed, throughput_only=True)
key = torch.from_numpy(key_bytes(w.n, w.key_seed)).cuda()
for _ in range(2):
    out = ctx.hash(key)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
out = ctx.hash(key)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", bytes(out[:8].cpu().numpy()).hex())
