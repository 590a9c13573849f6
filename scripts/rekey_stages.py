"""Per-stage times of pa_ctx_rekey (device key expansion + transforms) at the C4 shape (dev check)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_13678_b200 import PAContext
from synth import CONFIGS
w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = PAContext(w.n, w.r, w.m, 0, seed=w.hash_seed)
for j in range(2): ctx.rekey(w.hash_seed + 1 + j)
torch.cuda.synchronize()
ctx.set_profiling(True); ctx.stage_times(reset=True)
for j in range(5): ctx.rekey(w.hash_seed + 10 + j)
torch.cuda.synchronize()
st = ctx.stage_times(); ctx.set_profiling(False)
print({k: round(v[0] / 5 * 1e3, 1) for k, v in sorted(st.items())})
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for j in range(5): ctx.rekey(w.hash_seed + 20 + j)
e1.record(s); torch.cuda.synchronize()
print("rekey us", e0.elapsed_time(e1) / 5 * 1e3)
