"""Write tests/golden/digests.json: SHA-256 of the expected output key of every
BASELINE.json config, computed ONLY by the CPU oracle (oracle/) on the seeded synthetic
inputs of synth/ (key Philox (0x6B6579 + cfg#, 0), hash seed 0x5EED0000 + cfg#).

Multiprocessing splits the MMH sum over blocks (split-merge); the
per-block products use CPython ints (library multiplication), the reductions the fold
identity -- both pinned by tests/test_oracle_*.py.

    python scripts/gen_golden.py C1 C2 C3 C4      # minutes
    python scripts/gen_golden.py C5a C5b C5c      # tens of minutes
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from multiprocessing import Pool

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import hashes, seeds  # noqa: E402
from synth import CONFIGS, PAPER_CONFIGS, key_bytes  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "digests.json")


def _partial(args):
    name, lo, hi = args
    w = CONFIGS[name]
    pp = hashes.plan_params(w.n, w.r, w.m)
    key = key_bytes(w.n, w.key_seed)
    x = hashes.key_blocks(key, w.n, w.r)
    acc = 0
    for i in range(lo, hi):
        acc += seeds.expand_a(w.hash_seed, i, pp["gamma"]) * x[i]
    return hashes.reduce_mersenne(acc, pp["gamma"])


def _paper_partial(args):
    name, lo, hi = args
    w = PAPER_CONFIGS[name]
    key = key_bytes(w.n, w.key_seed)
    x, _ = hashes.paper_blocks(key, w.n, w.gamma, w.k)
    acc = 0
    for i in range(lo, hi):
        acc += seeds.expand_a(w.hash_seed, i, w.gamma) * x[i]
    return hashes.reduce_mersenne(acc, w.gamma)


def golden_paper(name: str, procs: int) -> dict:
    """Paper mode (NEXT-1): Algorithm 1 with gamma-bit blocks, reload, alpha = gamma."""
    w = PAPER_CONFIGS[name]
    t0 = time.time()
    G = min(procs, w.k)
    cuts = [(name, w.k * g // G, w.k * (g + 1) // G) for g in range(G)]
    with Pool(procs) as pool:
        ys = pool.map(_paper_partial, cuts)
    y = hashes.merge_residues(ys, w.gamma)
    b, c = seeds.expand_b(w.hash_seed, w.gamma), seeds.expand_c(w.hash_seed, w.gamma)
    out = hashes.mh_output(y, b, c, w.gamma, w.m)
    return {"config": name, "mode": "paper (gamma-bit blocks, reload rule, alpha = gamma)", "n": w.n,
            "gamma": w.gamma, "alpha": w.gamma, "k": w.k, "m": w.m, "key_seed": w.key_seed,
            "hash_seed": w.hash_seed,
            "y_sha256": hashlib.sha256(y.to_bytes((w.gamma + 7) // 8, "little")).hexdigest(),
            "out_sha256": hashlib.sha256(out).hexdigest(), "out_head": out[:16].hex(),
            "oracle": "oracle.hashes.paper_blocks + CPython int products, fold reduction",
            "seconds": round(time.time() - t0, 1)}


def golden(name: str, procs: int) -> dict:
    if name in PAPER_CONFIGS:
        return golden_paper(name, procs)
    w = CONFIGS[name]
    pp = hashes.plan_params(w.n, w.r, w.m)
    k = pp["k"]
    t0 = time.time()
    G = min(procs * 4, k)
    cuts = [(name, k * g // G, k * (g + 1) // G) for g in range(G)]
    with Pool(procs) as pool:
        ys = pool.map(_partial, cuts)
    y = hashes.merge_residues(ys, pp["gamma"])
    b, c = seeds.expand_b(w.hash_seed, pp["alpha"]), seeds.expand_c(w.hash_seed, pp["alpha"])
    out = hashes.mh_output(y, b, c, pp["alpha"], w.m)
    return {"config": name, "n": w.n, "r": w.r, "m": w.m, "gamma": pp["gamma"], "alpha": pp["alpha"],
            "k": k, "key_seed": w.key_seed, "hash_seed": w.hash_seed,
            "y_sha256": hashlib.sha256(y.to_bytes((pp["gamma"] + 7) // 8, "little")).hexdigest(),
            "out_sha256": hashlib.sha256(out).hexdigest(), "out_head": out[:16].hex(),
            "oracle": "oracle.hashes (CPython int products, fold reduction)",
            "seconds": round(time.time() - t0, 1)}


def main():
    names = sys.argv[1:] or ["C1", "C2", "C3", "C4"]
    procs = int(os.environ.get("PROCS", os.cpu_count() or 1))
    db = json.load(open(OUT)) if os.path.exists(OUT) else {}
    db["_about"] = ("SHA-256 of expected outputs written by scripts/gen_golden.py from oracle/ only; "
                    "y_sha256 hashes the MMH residue as little-endian ceil(gamma/8) bytes")
    for name in names:
        rec = golden(name, procs)
        db[name] = rec
        print(json.dumps(rec), flush=True)
        json.dump(db, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
