"""Timeline of one graph-replayed C4 pa_hash from the PA_TPROF build (scripts/build_variant.sh
tprof -DPA_TPROF; PA_DEV_LIB=paper_2105_13678_b200/_pa_tprof.so): per kernel the first and last
CTA start (globaltimer), the gap to the next kernel, and crt_carry's per-phase CTA times."""
import ctypes
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2105_13678_b200 import PAContext, _binding as B  # noqa: E402
from synth import CONFIGS, key_bytes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
w = CONFIGS[cfg]
lib = B._lib
lib.pa_tprof_reset.restype = ctypes.c_int
lib.pa_tprof_dump.restype = ctypes.c_int
lib.pa_tprof_dump.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = PAContext(w.n, w.r, w.m, seed=w.hash_seed, throughput_only=True)
key = torch.from_numpy(key_bytes(w.n, w.key_seed)).cuda()
out = torch.empty(ctx.nbytes_out, dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ctx.hash(key, out)
res = {}
for rep in range(3):
    flush.fill_(1)
    torch.cuda.synchronize()
    lib.pa_tprof_reset()
    ctx.hash(key, out)
    torch.cuda.synchronize()
    dt = np.dtype([("kid", "<u4"), ("blk", "<u4"), ("phase", "<u4"), ("sm", "<u4"), ("t", "<u8"), ("clk", "<u8")])
    buf = np.zeros(1 << 20, dtype=dt)
    n = lib.pa_tprof_dump(buf.ctypes.data, buf.size)
    r = buf[:n]
    t0 = int(r["t"].min())
    kernels = []
    order = []
    for kid in np.unique(r["kid"]):
        e = r[(r["kid"] == kid) & (r["phase"] == 0)]
        order.append((int(e["t"].min()), int(kid)))
    order.sort()
    rows = []
    for i, (ts, kid) in enumerate(order):
        e = r[(r["kid"] == kid) & (r["phase"] == 0)]
        nxt = order[i + 1][0] if i + 1 < len(order) else None
        row = {"kid": hex(kid), "ctas": int(len(e)), "first_start_us": (ts - t0) / 1e3,
               "last_start_us": (int(e["t"].max()) - t0) / 1e3,
               "until_next_kernel_us": ((nxt - ts) / 1e3) if nxt else None}
        if (kid & 0xF000) == 0x5000:
            # carry tiles: every phase mark carries the tile (0x100000 | tile); times relative to
            # phase 7 (ticket known) of the same tile, on the global timer (ns)
            ph = {}
            base = r[(r["kid"] == kid) & (r["phase"] == 7)]
            bt = {int(b): int(t) for b, t in zip(base["blk"], base["t"])}
            ph["ticket_us_after_first_start_median"] = float(np.median([(bt[k] - ts) / 1e3 for k in bt])) if bt else None
            for p in (8, 9, 18, 2, 3, 4, 5):
                a = r[(r["kid"] == kid) & (r["phase"] == p)]
                d = [(int(t) - bt[int(b)]) / 1e3 for b, t in zip(a["blk"], a["t"]) if int(b) in bt]
                if d:
                    ph[f"phase{p}_us_median"] = round(float(np.median(d)), 2)
                    ph[f"phase{p}_us_max"] = round(float(max(d)), 2)
            row.update(ph)
        rows.append(row)
    res[rep] = rows
print(json.dumps(res[2], indent=1))
