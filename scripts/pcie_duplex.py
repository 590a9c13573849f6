"""Do H2D key copies and D2H output copies overlap on this box? (dev check for the e2e stream line)"""
import torch
nb, mb, K = 32_500_000, 3_250_000, 8
hk = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(2)]
ho = [torch.empty(mb, dtype=torch.uint8).pin_memory() for _ in range(2)]
dk = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(2)]
do = [torch.empty(mb, dtype=torch.uint8, device="cuda") for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(d2h, h2d=True):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s1); s2.wait_event(e0)
    for j in range(K):
        if h2d:
            with torch.cuda.stream(s1): dk[j & 1].copy_(hk[j & 1], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): ho[j & 1].copy_(do[j & 1], non_blocking=True)
    ev = torch.cuda.Event(); ev.record(s2); s1.wait_event(ev); e1.record(s1); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K
for _ in range(2): run(True)
for _ in range(3):
    print(f"h2d only {run(False):.4f} ms/key   d2h only {run(True, False):.4f}   both {run(True):.4f}")
