"""H2D of one C4 key (32.5 MB pinned): one copy, G sequential chunks, and the same split over two
copy streams (dev check for pa_hash_host's grouped copy)."""
import json
import torch
nb = 32_500_000
hk = torch.empty(nb, dtype=torch.uint8).pin_memory()
dk = torch.empty(nb, dtype=torch.uint8, device="cuda")
ss = [torch.cuda.Stream(), torch.cuda.Stream()]
def run(G, nstream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(ss[0]); ss[1].wait_event(e0)
    for g in range(G):
        lo, hi = nb * g // G, nb * (g + 1) // G
        with torch.cuda.stream(ss[g % nstream]):
            dk[lo:hi].copy_(hk[lo:hi], non_blocking=True)
    ev = torch.cuda.Event(); ev.record(ss[1]); ss[0].wait_event(ev); e1.record(ss[0])
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)
res = {"async_engines": torch.cuda.get_device_properties(0).async_engine_count if hasattr(torch.cuda.get_device_properties(0), "async_engine_count") else None}
for G, ns in [(1, 1), (4, 1), (8, 1), (16, 1), (2, 2), (8, 2), (16, 2)]:
    for _ in range(2): run(G, ns)
    res[f"G{G}_s{ns}"] = round(min(run(G, ns) for _ in range(7)), 4)
print(json.dumps(res))
