"""Timeline of one pa_hash_host (pinned buffers) from the PA_TPROF build: the first CTA start of
every kernel (globaltimer, us from the call's start event), which shows when each copy group's
transforms could begin and what follows the last byte (dev tool)."""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_13678_b200 import PAContext, _binding as B  # noqa: E402
from synth import CONFIGS, key_bytes  # noqa: E402

w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
lib = B._lib
lib.pa_tprof_dump.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = PAContext(w.n, w.r, w.m, seed=w.hash_seed, throughput_only=True)
hk = torch.from_numpy(key_bytes(w.n, w.key_seed)).pin_memory()
ho = torch.empty(ctx.nbytes_out, dtype=torch.uint8).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ctx.hash_host(hk, ho)
dt = np.dtype([("kid", "<u4"), ("blk", "<u4"), ("phase", "<u4"), ("sm", "<u4"), ("t", "<u8"), ("clk", "<u8")])
out = []
for rep in range(3):
    flush.fill_(1)
    torch.cuda.synchronize()
    lib.pa_tprof_reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.hash_host(hk, ho)
    wall = (time.perf_counter() - t0) * 1e3
    buf = np.zeros(1 << 20, dtype=dt)
    n = lib.pa_tprof_dump(buf.ctypes.data, buf.size)
    r = buf[:n]
    r = r[r["phase"] == 0]
    tmin = int(r["t"].min())
    # kernel instances: consecutive records of one kid separated by a gap > 3 us are different launches
    order = np.argsort(r["t"])
    rows, cur = [], None
    for i in order:
        kid, t = int(r["kid"][i]), int(r["t"][i])
        if cur and cur["kid"] == kid and t - cur["last"] < 3000:
            cur["last"] = t; cur["ctas"] += 1
            continue
        cur = {"kid": kid, "first": t, "last": t, "ctas": 1}
        rows.append(cur)
    out.append({"wall_ms": round(wall, 3), "launches": [
        {"kid": hex(x["kid"]), "ctas": x["ctas"], "start_us": round((x["first"] - tmin) / 1e3, 1),
         "last_start_us": round((x["last"] - tmin) / 1e3, 1)} for x in rows]})
print(json.dumps(out[-1], indent=0))
