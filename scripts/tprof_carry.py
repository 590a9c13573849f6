"""Per-tile phase times of crt_carry from the PA_TPROF build (see scripts/tprof.py)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2105_13678_b200 import PAContext, _binding as B  # noqa: E402
from synth import CONFIGS, key_bytes  # noqa: E402

w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
lib = B._lib
lib.pa_tprof_dump.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = PAContext(w.n, w.r, w.m, seed=w.hash_seed, throughput_only=True)
key = torch.from_numpy(key_bytes(w.n, w.key_seed)).cuda()
out = torch.empty(ctx.nbytes_out, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ctx.hash(key, out)
torch.cuda.synchronize()
lib.pa_tprof_reset()
ctx.hash(key, out)
torch.cuda.synchronize()
dt = np.dtype([("kid", "<u4"), ("blk", "<u4"), ("phase", "<u4"), ("sm", "<u4"), ("t", "<u8"), ("clk", "<u8")])
buf = np.zeros(1 << 20, dtype=dt)
n = lib.pa_tprof_dump(buf.ctypes.data, buf.size)
r = buf[:n]
for kid in (0x508C, 0x500B):
    k = r[r["kid"] == kid]
    t0 = int(k[k["phase"] == 0]["t"].min())
    tiles = {}
    for rec in k[k["phase"] > 0]:
        tiles.setdefault(int(rec["blk"]) & 0xFFFFF, {})[int(rec["phase"])] = (int(rec["t"]) - t0) / 1e3
    print(hex(kid), "tiles", len(tiles))
    ks = sorted(tiles)
    arr = {p: np.array([tiles[t].get(p, np.nan) for t in ks]) for p in (2, 3, 4, 5)}
    for p in (2, 3, 4, 5):
        a = arr[p]
        print(f"  phase{p} end (us after kernel start): min {np.nanmin(a):.2f} med {np.nanmedian(a):.2f} p90 {np.nanpercentile(a, 90):.2f} max {np.nanmax(a):.2f}")
    wait = arr[4] - arr[3]
    print("  look-back wait us: med %.2f p90 %.2f max %.2f" % (np.nanmedian(wait), np.nanpercentile(wait, 90), np.nanmax(wait)))
    worst = np.argsort(-wait)[:8]
    print("  worst tiles:", [(ks[i], round(float(wait[i]), 2), round(float(arr[3][i]), 2)) for i in worst])
    six = [(t, v[6]) for t, v in tiles.items() if 6 in v]
    print("  finish (phase 6):", six, "end max", np.nanmax(arr[5]))
    fl = {}
    for rec in k[k["phase"] >= 10]:
        fl[int(rec["blk"]) & 0xFFFFF] = int(rec["phase"]) - 10
    nind = sum(1 for v in fl.values() if v & 1)
    print("  independent tiles:", nind, "of", len(fl), " allp tiles:", sum(1 for v in fl.values() if v & 2))
    dep = [t for t, v in sorted(fl.items()) if not (v & 1)]
    print("  dependent tiles:", dep[:60])
    for t in ks[300:380:4]:
        print("   tile", t, "flags", fl.get(t), "p3 %.2f p4 %.2f" % (tiles[t].get(3, -1), tiles[t].get(4, -1)))
    # tiles in ticket order: phase 3 times of the first 20 tiles
    print("  phase3 first tiles:", [round(float(x), 2) for x in arr[3][:12]])
