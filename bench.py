"""Benchmark of the MMH-MH privacy-amplification hot path on B200 (one JSON line).

Metric (BASELINE.json): PA throughput in Mbps of INPUT key at n = 2.6e8 bits (config C4),
= n / t_step / 1e6, one step = one full pa_hash (S1..S7: pack, forward NTTs of all 31
blocks, transform-domain multiply-accumulate, inverse, CRT + carries, Mersenne fold, MH).

    python bench.py                               # N=1, C4
    python bench.py --impl reference              # the CPU oracle on a bounded sample
    torchrun --nproc-per-node N bench.py --gpus N # blocks sharded over N ranks, NCCL gather

Timing rules followed: W >= 3 untimed warm-up steps; every timed step is bracketed by
CUDA events on the context stream and preceded (outside the events) by an L2 flush
(a 256 MiB write, > 126 MB L2); device time, max over ranks; nvidia-smi clocks sampled
during the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PA throughput, Mbps of input key at n=2.6e8 bits, 1/2/4/8 B200; % HBM roofline"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
INT_OPS_PER_BFLY = 6     # Shoup butterfly: 3 multiplies + 3 add/sub/correct
INT_OPS_PER_MAC = 6      # Montgomery product (4) + lazy add/correct (2)


def load_peaks() -> dict:
    try:
        return json.load(open(PEAKS))
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


def hbm_view(w, info: dict, ms_per_step: float, peaks: dict, paper: bool) -> dict:
    """the step's bytes over the HBM peak, for two byte counts.
    design = key + precomputed transforms (A^ for the k blocks, B^) + output, the bytes the
    transform-domain design must stream once; min = key + the raw hash keys (k a_i of gamma bits,
    b and c of alpha bits) + output, the bytes any implementation must touch.  The path is
    ALU-bound (`roofline`), so these fractions are context, not its bound."""
    key = (w.n + 7) // 8
    out = (w.m + 7) // 8
    k = info["k"]
    mm, mh = info["mmh"], info["mh"]
    hat = 4 * k * mm["nprimes"] * (1 << mm["log2_len"]) + 4 * mh["nprimes"] * (1 << mh["log2_len"])
    raw = k * ((info["gamma"] + 7) // 8) + 2 * ((info["alpha"] + 7) // 8)
    design, mn = key + hat + out, key + raw + out
    gbs = lambda b: b / (ms_per_step * 1e-3) / 1e9
    peak = peaks.get("hbm_gbs", 6650.0)
    return {"design_bytes": design, "min_bytes": mn, "design_gbs": gbs(design), "min_gbs": gbs(mn),
            "peak_gbs": peak, "design_frac": gbs(design) / peak, "min_frac": gbs(mn) / peak,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if not peaks.get("_fallback") else "fallback"}


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event reasons sampled DURING the timed region: an NVML
    polling thread (1 ms period), falling back to `nvidia-smi -lms 100`."""
    SMI_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                  "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, torch_dev: int):
        self.dev = torch_dev
        self.sm: list[float] = []
        self.reasons: set[str] = set()
        self.smax = None
        self.mode = None
        self._stop = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.dev)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.dev)

    def _poll_nvml(self, nv, h):
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, bit in self.REASONS:
                    if rs & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.001)

    def start(self):
        try:
            nv, h = self._nvml_handle()
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.mode = "nvml (1 ms polling thread)"
            self.t = threading.Thread(target=self._poll_nvml, args=(nv, h), daemon=True)
            self.t.start()
            return
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.SMI_FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.mode = "nvidia-smi -lms 100"
            self.t = threading.Thread(target=self._read_smi, daemon=True)
            self.t.start()
        except Exception:
            self.mode = None

    def _read_smi(self):
        names = [n for n, _ in self.REASONS[:4]]
        for ln in self.proc.stdout:
            f = [x.strip() for x in ln.strip().split(",")]
            if len(f) < 9:
                continue
            try:
                self.sm.append(float(f[1]))
                self.smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    self.reasons.add(nm)

    def stop(self) -> dict:
        if self.mode is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        self._stop.set()
        if self.mode.startswith("nvidia-smi"):
            time.sleep(0.25)
            self.proc.terminate()
        self.t.join(timeout=3)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "sampler": self.mode}


# --------------------------------------------------------------------------- roofline
def stage_ops(info: dict, stage: str) -> float:
    """Algorithmic int32 lane-operations of one launch of a stage:
    radix-2 butterflies of the pass times 6, plus 6 per transform-domain MAC."""
    mmh, mh = info["mmh"], info["mh"]
    nblk = info["block_end"] - info["block_begin"]

    def bfly(pl, nvec, npass_len):
        L = 1 << pl["log2_len"]
        import math
        return nvec * pl["nprimes"] * (L / 2) * math.log2(npass_len)

    if stage == "mmh_fwd_col":
        return INT_OPS_PER_BFLY * bfly(mmh, nblk, mmh["n_col"])
    if stage == "mmh_fwd_row_mac":
        L = 1 << mmh["log2_len"]
        return INT_OPS_PER_BFLY * bfly(mmh, nblk, mmh["n_row"]) + INT_OPS_PER_MAC * nblk * mmh["nprimes"] * L
    if stage == "mmh_inverse":
        return INT_OPS_PER_BFLY * bfly(mmh, 1, 1 << mmh["log2_len"])
    if stage == "mh_fwd_col":
        return INT_OPS_PER_BFLY * bfly(mh, 1, mh["n_col"])
    if stage == "mh_fwd_row_mac":
        return INT_OPS_PER_BFLY * bfly(mh, 1, mh["n_row"]) + INT_OPS_PER_MAC * mh["nprimes"] * (1 << mh["log2_len"])
    if stage == "mh_inverse":
        return INT_OPS_PER_BFLY * bfly(mh, 1, 1 << mh["log2_len"])
    if stage == "mh_row_mac_inv":      # forward row DFT + MAC + inverse row DFT (row_macinv)
        return (2 * INT_OPS_PER_BFLY * bfly(mh, 1, mh["n_row"]) +
                INT_OPS_PER_MAC * mh["nprimes"] * (1 << mh["log2_len"]))
    if stage == "mh_inverse_col":
        return INT_OPS_PER_BFLY * bfly(mh, 1, mh["n_col"])
    return 0.0


def int_peak(peaks: dict, nsm: int = 148) -> tuple[float, str, dict]:
    """The integer roofline denominator in Gop/s (int32 lane-ops).  Measured: the Shoup
    butterfly mix of microbench/int_peak.cu (6 SASS instructions, 3 FMA-pipe + 3 ALU-pipe),
    in lane-ops per SM per clock on a B200, x SMs x sm_max_mhz (profiles/int_peak.json).
    Fallback: the issue model, 1 warp-instruction per clock per SMSP."""
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    try:
        ip = json.load(open(os.path.join(ROOT, "profiles", "int_peak.json")))
        per_clk = float(ip["ops"]["shoup_butterfly"]["lane_ops_per_sm_clk"])
        pipes = {k: round(v["lane_ops_per_sm_clk"], 2) for k, v in ip["ops"].items()}
        return (per_clk * ip.get("sms", nsm) * sm_mhz * 1e6 / 1e9,
                f"measured: Shoup butterfly mix {per_clk:.1f} lane-ops/SM/clk (microbench/int_peak.cu on "
                f"{ip.get('gpu', 'B200')}, profiles/int_peak.json) x {ip.get('sms', nsm)} SMs x {sm_mhz:.0f} MHz",
                pipes)
    except Exception:
        return (nsm * 4 * 32 * sm_mhz * 1e6 / 1e9,
                f"issue model (no profiles/int_peak.json): {nsm} SMs x 4 SMSP x 32 lanes x 1 instr/clk x "
                f"{sm_mhz:.0f} MHz", {})


def roofline(info: dict, stages: dict, peaks: dict, steps: int) -> dict:
    """Dominant kernel stage -> achieved int32 Gop/s vs the measured integer peak.
    `stages` maps stage -> (ms per step, launches per step), from CUDA events recorded
    on the context stream around each launch (pa_ctx_set_profiling)."""
    name, (ms, cnt) = max(stages.items(), key=lambda kv: kv[1][0])
    per_launch_ms = ms / max(cnt, 1)
    ops = stage_ops(info, name)
    peak, note, pipes = int_peak(peaks)
    issue_peak = 148 * 4 * 32 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e9
    achieved = ops / (per_launch_ms * 1e-3) / 1e9 if ops else None
    traffic = None
    ncu_pct = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = prof.get(name, {}).get("dram_bytes_per_launch")
        # issue-slot and per-pipe utilisation of that kernel from the committed --set full capture
        ncu_pct = prof.get(name, {}).get("ncu_pct_of_peak")
    except Exception:
        pass
    share = ms / sum(v[0] for v in stages.values())
    return {"bound": "alu", "kernel": name, "achieved": achieved, "peak": peak, "unit": "Gop/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "ms_per_launch": per_launch_ms, "share_of_step": share, "peak_source": note,
            "issue_model_peak": issue_peak,
            "issue_model_frac": (achieved / issue_peak) if achieved else None,
            "measured_lane_ops_per_sm_clk": pipes,
            "ncu_pct_of_peak": ncu_pct}


# --------------------------------------------------------------------------- CPU oracle
def _cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_part(args):
    """Worker: the oracle's MMH over blocks [lo, hi) of a workload, y_g = sum a_i x_i mod p
    (oracle.hashes.mmh_partial: CPython-int products + fold; PAPER.md:91 split-merge).
    Hash-key expansion (oracle.seeds) is inside the timed part; key generation is not."""
    name, lo, hi = args
    from oracle import hashes, seeds
    from synth import CONFIGS, key_bytes
    w = CONFIGS[name]
    key = key_bytes(w.n, w.key_seed)
    g = hashes.plan_params(w.n, w.r, w.m)["gamma"]
    t0 = time.perf_counter()
    a = {i: seeds.expand_a(w.hash_seed, i, g) for i in range(lo, hi)}
    y = hashes.mmh_partial(key, w.n, w.r, g, a, range(lo, hi))
    return y, time.perf_counter() - t0


def _pool(n):
    from multiprocessing import get_context
    pool = get_context("spawn").Pool(n)
    pool.map(abs, range(n))                                  # workers up before any timing
    return pool


def cpu_oracle_full(w) -> dict:
    """The whole hash of the workload by the CPU oracle as it stands (oracle/hashes.py), on
    all host cores: the k block products split into min(cores, k) contiguous block ranges,
    one oracle mmh_partial per worker process, then merge_residues and the MH (mh_output:
    one CPython-int product) in this process.  Throughput = n / wall time of that whole
    computation; the output is checked against the oracle-written golden digest."""
    import hashlib
    from oracle import hashes, seeds
    cores = os.cpu_count() or 1
    G = max(1, min(cores, w.k))
    with _pool(G) as pool:
        t0 = time.perf_counter()
        parts = pool.map(_oracle_part, [(w.name, w.k * g // G, w.k * (g + 1) // G) for g in range(G)])
        t1 = time.perf_counter()
        pp = hashes.plan_params(w.n, w.r, w.m)
        y = hashes.merge_residues([yg for yg, _ in parts], pp["gamma"])
        b, c = seeds.expand_b(w.hash_seed, pp["alpha"]), seeds.expand_c(w.hash_seed, pp["alpha"])
        out = hashes.mh_output(y, b, c, pp["alpha"], w.m)
        t2 = time.perf_counter()
    digest_ok = None
    try:
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", "digests.json")))
        if w.name in gold:
            digest_ok = hashlib.sha256(out).hexdigest() == gold[w.name]["out_sha256"]
    except Exception:
        pass
    return {"value": w.n / (t2 - t0) / 1e6, "unit": "Mbps", "cores": G, "kind": "oracle",
            "cpu": _cpu_model(), "host_cores": cores,
            "sample": f"the whole {w.name} hash (all {w.k} blocks + MH) by oracle/hashes.py (CPython-int "
                      f"products, fold): blocks split over {G} worker processes, merge + MH in one process",
            "seconds": t2 - t0, "mmh_seconds": t1 - t0, "mh_seconds": t2 - t1,
            "output_matches_golden_digest": digest_ok}


def cpu_oracle_sample(w, pool, nblocks: int) -> dict:
    """A bounded sample of the oracle's work (the --impl reference steps): the MMH terms of
    blocks 0..nblocks-1, one block per worker process, in parallel; Mbps = nblocks r / wall."""
    t0 = time.perf_counter()
    parts = pool.map(_oracle_part, [(w.name, i, i + 1) for i in range(nblocks)])
    wall = time.perf_counter() - t0
    return {"value": nblocks * w.r / wall / 1e6, "seconds": wall, "busy_max": max(s for _, s in parts)}


def run_reference(args, w) -> None:
    """The reference arm of this tier: the CPU oracle as it stands, timed on the host cores.
    Rank 0 only (the other ranks exit without work).  Each step is a bounded sample -- the
    MMH terms of min(cores, k) blocks computed in parallel -- so that W warm-up steps and K
    timed steps finish within a few minutes; the whole-hash figure is the bench line's
    cpu_baseline."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if w.name not in __import__("synth").CONFIGS:
        raise SystemExit("--impl reference runs the r-bit configs")
    cores = os.cpu_count() or 1
    nb = max(1, min(cores, w.k))
    with _pool(nb) as pool:
        for _ in range(args.warmup):
            cpu_oracle_sample(w, pool, nb)
        res = [cpu_oracle_sample(w, pool, nb) for _ in range(args.steps)]
    secs = [r["seconds"] for r in res]
    ms = statistics.median(secs) * 1e3
    v = nb * w.r / (ms * 1e-3) / 1e6
    sample = (f"MMH terms a_i x_i mod p (oracle/hashes.py mmh_partial: CPython-int product + fold, hash-key "
              f"expansion included) of blocks 0..{nb - 1} of {w.name} ({nb * w.r} key bits), one block per "
              f"process on {nb} host cores; Mbps = sampled key bits / wall time")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "Mbps", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int (Python bignum)",
            "data": "synthetic", "config": {"workload": w.name, "n": w.n, "r": w.r, "m": w.m,
                                             "sample": f"{nb} of {w.k} block products per step, in parallel"},
            "cpu_baseline": {"value": v, "unit": "Mbps", "cores": nb, "kind": "oracle", "sample": sample,
                             "cpu": _cpu_model()},
            "e2e": {"value": v, "unit": "Mbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def oracle_check(w, key: "np.ndarray", got: bytes) -> bool:
    """True when `got` is the CPU oracle's hash of `key` under workload w's seed: the golden
    SHA-256 (scripts/gen_golden.py, oracle/ only) for the config's own key, else the oracle
    computed here (oracle/hashes.py; seconds at C1-C2 sizes)."""
    import hashlib
    from synth import key_bytes
    std = key_bytes(w.n, w.key_seed)
    if len(key) == len(std) and bytes(key) == bytes(std):
        try:
            gold = json.load(open(os.path.join(ROOT, "tests", "golden", "digests.json")))
            if w.name in gold:
                return hashlib.sha256(got).hexdigest() == gold[w.name]["out_sha256"]
        except Exception:
            pass
    from oracle import hashes
    return got == hashes.pa_hash_seeded(key, w.n, w.r, w.m, w.hash_seed)


# --------------------------------------------------------------------------- GPU run
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--limb-bits", type=int, default=0, help="force the limb width B (0 = planner)")
    ap.add_argument("--batch", type=int, default=8, help="keys per pa_hash_batch in the stream-mode line")
    ap.add_argument("--no-comparators", dest="comparators", action="store_false",
                    help="skip the MH-only PA comparator measurement")
    ap.add_argument("--only-device", action="store_true",
                    help="timed device steps only (no per-stage pass, no e2e): for ncu launch lists")
    ap.add_argument("--p2p", action="store_true",
                    help="N>1: exchange the accumulators over peer memory (pa_params.p2p) instead of ncclReduce")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N>1 (gloo only to validate the multi-rank path)")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank on cuda:0 (validation of the N>1 host path on a 1-GPU box; not a bench)")
    ap.add_argument("--one-rank-mg", action="store_true",
                    help="run the N>1 code path (library NCCL context, reduce / p2p exchange, multi-GPU e2e, "
                         "rotating-root stream) with a one-rank communicator on one GPU: validates that path, not a bench")
    ap.add_argument("--verify", action="store_true",
                    help="N>1: rank 0 checks the sharded hash against a whole-key single-GPU context")
    args = ap.parse_args()
    if args.impl != "reference":
        args.warmup = max(args.warmup, 3)
    # stdout carries exactly one JSON line: anything native libraries write to fd 1 (NCCL prints
    # its version banner there when NCCL_DEBUG is set) goes to stderr instead
    sys.stdout.flush()
    _real_stdout = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(_real_stdout, "w")

    from synth import CONFIGS, PAPER_CONFIGS, key_bytes
    paper = args.config in PAPER_CONFIGS
    w = PAPER_CONFIGS[args.config] if paper else CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, w)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2105_13678_b200 import PAContext
    from paper_2105_13678_b200.pa import (key_slice_bytes, nccl_context, shard_ranges, transform_merge_hash,
                                           transform_merge_stream)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world
    multi = world > 1 or args.one_rank_mg
    if args.one_rank_mg and world == 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    if args.same_device:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # N>1 product path: the library's own NCCL communicator (pa_params.world/rank/nccl_id)
    # reduces the transform-domain accumulators; torch.distributed only broadcasts the id and
    # brackets the timing.  Validation path (--dist-backend gloo / --same-device, one GPU):
    # the same split through pa_mmh_acc / pa_tail_merge with a gloo exchange.
    lib_nccl = multi and args.dist_backend == "nccl" and not args.same_device
    if multi:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    # a dedicated (non-default) stream: the library then replays each hash as a CUDA graph
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    k = w.k
    if paper and multi:
        raise SystemExit("paper-mode configs (reload rule over the whole key) run on one GPU")
    b0, b1 = shard_ranges(k, world)[rank]
    key_full = key_bytes(w.n, w.key_seed)
    lo, hi = (0, w.nbytes) if paper else key_slice_bytes(w.n, w.r, (b0, b1))
    key_dev = torch.from_numpy(key_full[lo:hi].copy()).to(dev)
    # S0 (untimed in the step): context creation -- plan, host tables, hash-key
    # expansion and the precomputed transforms -- timed once by wall clock
    torch.cuda.synchronize()
    t_create = time.perf_counter()
    if paper:
        ctx = PAContext(w.n, 0, w.m, w.gamma, seed=w.hash_seed, limb_bits=args.limb_bits, paper_k=w.k)
    elif lib_nccl:
        ctx = nccl_context(w.n, w.r, w.m, seed=w.hash_seed, limb_bits=args.limb_bits, throughput_only=True,
                           p2p=args.p2p)
    else:
        ctx = PAContext(w.n, w.r, w.m, seed=w.hash_seed, block_range=(b0, b1) if multi else None,
                        limb_bits=args.limb_bits, throughput_only=True)
    torch.cuda.synchronize()
    ctx_create_ms = (time.perf_counter() - t_create) * 1e3
    info = ctx.query()
    out = torch.empty(ctx.nbytes_out, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        if not multi or lib_nccl:
            return ctx.hash(key_dev, out)
        return transform_merge_hash(ctx, key_dev)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    verified = None
    if multi and args.verify:
        # rank 0 checks the sharded hash against the CPU oracle (golden digest of the config's
        # key, written by scripts/gen_golden.py from oracle/ only)
        res = step()
        torch.cuda.synchronize()
        if rank == 0:
            verified = oracle_check(w, key_full, bytes(res.cpu().numpy()))
            if not verified:
                raise SystemExit("sharded hash differs from the CPU oracle")
    launches0 = ctx.query()["launches_total"]
    if multi:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    evs = []
    for _ in range(args.steps):
        if not args.no_flush:
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    clocks = sampler.stop()
    launches_timed = (ctx.query()["launches_total"] - launches0) % (1 << 32)
    times = [a.elapsed_time(b) for a, b in evs]
    tot = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    if multi:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = tot.item() / args.steps

    if args.only_device:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": w.n / (ms_per_step * 1e-3) / 1e6, "unit": "Mbps",
                              "ms_per_step": ms_per_step, "only_device": True}), flush=True)
        if multi:
            dist.destroy_process_group()
        return
    # ---- N>1 stream mode (NEXT-3): G independent keys per step, the root rotating (key j
    # reduced to and finished on rank j mod G), so the tail + MH no longer serialise on rank 0
    mr_stream = None
    if multi:
        def roll_key(j):
            kb = np.roll(key_full, 977 * j)
            if w.n % 8:
                kb[-1] &= (0xFF << (8 - w.n % 8)) & 0xFF
            return kb
        nkeys = 2 * world
        keys_j = [torch.from_numpy(roll_key(j)[lo:hi].copy()).to(dev) for j in range(nkeys)]

        def stream_step():
            if lib_nccl:
                outs = ctx.hash_batch(keys_j)
                return {j: o for j, o in enumerate(outs) if o is not None}
            return transform_merge_stream(ctx, keys_j)
        for _ in range(2):
            outs_j = stream_step()
        torch.cuda.synchronize()
        if args.verify:
            ok = torch.ones(1, dtype=torch.int32, device=dev)
            for j, o in outs_j.items():
                ok &= int(oracle_check(w, roll_key(j), bytes(o.cpu().numpy())))
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if not ok.item():
                raise SystemExit("rotating-root stream hash differs from the CPU oracle")
            verified = True if verified is None else verified
        dist.barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        bb = torch.cuda.Event(enable_timing=True)
        nst = max(3, args.steps // 5)
        a.record(stream)
        for _ in range(nst):
            stream_step()
        bb.record(stream)
        torch.cuda.synchronize()
        ts = torch.tensor([a.elapsed_time(bb) / nst], dtype=torch.float64, device=dev)
        dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        ms_s = ts.item()
        mr_stream = {"keys_per_step": nkeys, "value": nkeys * w.n / (ms_s * 1e-3) / 1e6, "unit": "Mbps",
                     "ms_per_step": ms_s, "ms_per_key": ms_s / nkeys,
                     "api": ("pa_hash_batch on a multi-GPU context (library NCCL reduce of the transform-domain "
                             "accumulators to rank j mod G, tail + MH there)") if lib_nccl else
                            "transform_merge_stream (pa_mmh_acc, gloo gather to rank j mod G, pa_tail_merge)",
                     "l2": "not flushed between keys (back-to-back stream)"}

    # ---- per-launch times: the same K steps again with CUDA events recorded on the
    # context stream around every launch (pa_ctx_set_profiling); e2e via the host API
    ctx.set_profiling(True)
    ctx.stage_times(reset=True)
    for _ in range(args.steps):
        if not args.no_flush:
            flush.fill_(1)
        step()
    stages = ctx.stage_times()
    ctx.set_profiling(False)
    nsteps_prof = args.steps
    stages = {kname: (v[0], v[1]) for kname, v in stages.items()}

    e2e = None
    if not multi:
        host_key = torch.from_numpy(key_full).pin_memory()
        host_out = torch.empty(ctx.nbytes_out, dtype=torch.uint8).pin_memory()
        for _ in range(2):
            ctx.hash_host(host_key, host_out)
        t, t_copy = [], []
        kd_probe = torch.empty_like(host_key, device=dev)
        for _ in range(max(3, args.steps // 2)):
            if not args.no_flush:
                flush.fill_(1)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            bb = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.hash_host(host_key, host_out)
            bb.record(stream)
            bb.synchronize()
            t.append(a.elapsed_time(bb))
            # the host link is shared with the box's other GPUs: a plain copy of the same key
            # right after each e2e sample shows the PCIe bandwidth that sample saw
            a.record(stream)
            kd_probe.copy_(host_key, non_blocking=True)
            bb.record(stream)
            bb.synchronize()
            t_copy.append(a.elapsed_time(bb))
        e2e_ms = statistics.median(t)
        # end-to-end stream mode: a batch of pinned host keys, H2D overlapping compute
        e2e_stream = None
        if args.batch > 1:
            hkeys = [host_key] + [torch.from_numpy(key_full).pin_memory() for _ in range(args.batch - 1)]
            houts = [torch.empty(ctx.nbytes_out, dtype=torch.uint8).pin_memory() for _ in range(args.batch)]
            ctx.hash_host_batch(hkeys, houts)
            tsb = []
            for _ in range(3):
                a = torch.cuda.Event(enable_timing=True)
                bb = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ctx.hash_host_batch(hkeys, houts)
                bb.record(stream)
                bb.synchronize()
                tsb.append(a.elapsed_time(bb))
            msb = statistics.median(tsb)
            e2e_stream = {"keys_per_batch": args.batch, "value": args.batch * w.n / (msb * 1e-3) / 1e6,
                          "unit": "Mbps", "ms_per_key": msb / args.batch,
                          "h2d_bytes_per_key": (w.n + 7) // 8, "d2h_bytes_per_key": (w.m + 7) // 8,
                          "api": "pa_hash_host_batch (pinned host keys; H2D of key j overlaps the hash of key j-1)"}
        # the PCIe floor: plain pinned copies of the same bytes (context for the e2e number)
        kd = torch.empty_like(host_key, device=dev)
        od = torch.empty(ctx.nbytes_out, dtype=torch.uint8, device=dev)
        th2d, td2h = [], []
        for _ in range(5):
            a = torch.cuda.Event(enable_timing=True); bb = torch.cuda.Event(enable_timing=True)
            a.record(stream); kd.copy_(host_key, non_blocking=True); bb.record(stream); bb.synchronize()
            th2d.append(a.elapsed_time(bb))
            a.record(stream); host_out.copy_(od, non_blocking=True); bb.record(stream); bb.synchronize()
            td2h.append(a.elapsed_time(bb))
        e2e = {"value": w.n / (e2e_ms * 1e-3) / 1e6, "unit": "Mbps", "ms_per_step": e2e_ms,
               "stream": e2e_stream,
               "h2d_bytes_per_step": (w.n + 7) // 8, "d2h_bytes_per_step": (w.m + 7) // 8,
               "api": "pa_hash_host (pinned host buffers, H2D + hash + D2H + sync)",
               "h2d_copy_ms": min(th2d), "d2h_copy_ms": min(td2h),
               "samples_ms": [round(x, 4) for x in t],
               "h2d_copy_ms_interleaved": statistics.median(t_copy),
               "h2d_gbs": (w.n + 7) // 8 / (min(th2d) * 1e-3) / 1e9}

    if multi and lib_nccl:
        # e2e at N GPUs: every rank copies its own key slice from pinned host memory over its own
        # host link (pa_hash_host on the multi-GPU context), rank 0 reads the output back
        host_key = torch.from_numpy(key_full[lo:hi].copy()).pin_memory()
        host_out = torch.empty(ctx.nbytes_out, dtype=torch.uint8).pin_memory() if rank == 0 else None
        for _ in range(2):
            ctx.hash_host(host_key, host_out)
        e2e_ok = True
        if args.verify and rank == 0:
            e2e_ok = oracle_check(w, key_full, bytes(host_out.numpy()))
        t = []
        for _ in range(max(3, args.steps // 2)):
            if not args.no_flush:
                flush.fill_(1)
            torch.cuda.synchronize()
            dist.barrier()
            a = torch.cuda.Event(enable_timing=True)
            bb = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.hash_host(host_key, host_out)
            bb.record(stream)
            bb.synchronize()
            ts = torch.tensor([a.elapsed_time(bb)], dtype=torch.float64, device=dev)
            dist.all_reduce(ts, op=dist.ReduceOp.MAX)
            t.append(ts.item())
        e2e_ms = statistics.median(t)
        e2e = {"value": w.n / (e2e_ms * 1e-3) / 1e6, "unit": "Mbps", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": (w.n + 7) // 8, "d2h_bytes_per_step": (w.m + 7) // 8,
               "h2d_bytes_this_rank": hi - lo,
               "api": "pa_hash_host on the multi-GPU context (each rank: pinned key slice H2D + transforms + "
                      "accumulator merge; rank 0: tail + MH + D2H + sync); max over ranks per step",
               "samples_ms": [round(x, 4) for x in t]}
        if args.verify:
            e2e["verified_vs_oracle"] = e2e_ok
            if not e2e_ok:
                raise SystemExit("multi-GPU pa_hash_host differs from the CPU oracle")
        # e2e stream at N GPUs: 2N pinned host keys (each rank holds its slices), rotating root
        hkeys = [torch.from_numpy(roll_key(j)[lo:hi].copy()).pin_memory() for j in range(nkeys)]
        houts = [torch.empty(ctx.nbytes_out, dtype=torch.uint8).pin_memory() if j % world == rank else None
                 for j in range(nkeys)]
        ctx.hash_host_batch(hkeys, houts)
        if args.verify:
            ok = torch.ones(1, dtype=torch.int32, device=dev)
            for j, o in enumerate(houts):
                if o is not None:
                    ok &= int(oracle_check(w, roll_key(j), bytes(o.numpy())))
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if not ok.item():
                raise SystemExit("multi-GPU pa_hash_host_batch differs from the CPU oracle")
        tsb = []
        for _ in range(3):
            torch.cuda.synchronize()
            dist.barrier()
            a = torch.cuda.Event(enable_timing=True)
            bb = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.hash_host_batch(hkeys, houts)
            bb.record(stream)
            bb.synchronize()
            ts = torch.tensor([a.elapsed_time(bb)], dtype=torch.float64, device=dev)
            dist.all_reduce(ts, op=dist.ReduceOp.MAX)
            tsb.append(ts.item())
        msb = statistics.median(tsb)
        e2e["stream"] = {"keys_per_batch": nkeys, "value": nkeys * w.n / (msb * 1e-3) / 1e6, "unit": "Mbps",
                         "ms_per_key": msb / nkeys, "h2d_bytes_per_key": (w.n + 7) // 8,
                         "d2h_bytes_per_key": (w.m + 7) // 8,
                         "api": "pa_hash_host_batch on the multi-GPU context (pinned slices, H2D of key j overlapping "
                                "the hash of key j-1, rotating root)"}

    # ---- stream mode (pa_hash_batch, NEXT-3): a batch of independent keys, MH / tail of one
    # key overlapping the MMH of the next; reported beside the single-key `value`
    stream_mode = None
    if not multi and args.batch > 1:
        keys_b = [key_dev] + [torch.empty_like(key_dev).copy_(key_dev.roll(j)) for j in range(1, args.batch)]
        outs_b = [torch.empty(ctx.nbytes_out, dtype=torch.uint8, device=dev) for _ in range(args.batch)]
        for _ in range(2):
            ctx.hash_batch(keys_b, outs_b)
        torch.cuda.synchronize()
        tb = []
        for _ in range(max(3, args.steps // 5)):
            if not args.no_flush:
                flush.fill_(1)
            a = torch.cuda.Event(enable_timing=True)
            bb = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.hash_batch(keys_b, outs_b)
            bb.record(stream)
            bb.synchronize()
            tb.append(a.elapsed_time(bb))
        ms_b = statistics.median(tb)
        stream_mode = {"keys_per_batch": args.batch, "value": args.batch * w.n / (ms_b * 1e-3) / 1e6, "unit": "Mbps",
                       "ms_per_batch": ms_b, "ms_per_key": ms_b / args.batch,
                       "api": "pa_hash_batch (device buffers; two buffer sets / streams, graph replay)"}

    # ---- fresh hash keys per job (NEXT-2): pa_ctx_rekey (device Philox expansion + transforms
    # of the a_i and b) before every hash -- the "cold" throughput of a new function per job
    # ---- graph re-binding (verdict r1 #8): pa_hash on alternating output buffers, so every
    # call sees a new pointer set and re-captures + updates its executable graph in place
    # (cudaGraphExecUpdate), against the same calls on one buffer (plain replay)
    graph_rebind = None
    if not multi and not paper:
        outs2 = [torch.empty(ctx.nbytes_out, dtype=torch.uint8, device=dev) for _ in range(2)]
        i0 = ctx.query()
        torch.cuda.synchronize()
        res_t = {}
        for mode in ("same", "alternating"):
            tl = []
            for j in range(max(6, args.steps // 2)):
                o = outs2[0] if mode == "same" else outs2[j & 1]
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                ctx.hash(key_dev, o)
                torch.cuda.synchronize()
                tl.append((time.perf_counter() - t0) * 1e3)
            res_t[mode] = statistics.median(tl[2:])
        i1 = ctx.query()
        graph_rebind = {"host_wall_ms_same_pointers": res_t["same"],
                        "host_wall_ms_new_pointers": res_t["alternating"],
                        "captures": i1["graph_captures"] - i0["graph_captures"],
                        "updates": i1["graph_updates"] - i0["graph_updates"],
                        "instantiations": i1["graph_instantiations"] - i0["graph_instantiations"],
                        "what": "wall time of pa_hash + synchronize; new pointers re-capture and cudaGraphExecUpdate"}

    fresh = None
    if not multi:
        for j in range(2):
            ctx.rekey(w.hash_seed + 1 + j)
            ctx.hash(key_dev, out)
        torch.cuda.synchronize()
        tf, tr = [], []
        for j in range(max(3, args.steps // 5)):
            if not args.no_flush:
                flush.fill_(1)
            a = torch.cuda.Event(enable_timing=True)
            mid = torch.cuda.Event(enable_timing=True)
            bb = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.rekey(w.hash_seed + 100 + j)
            mid.record(stream)
            ctx.hash(key_dev, out)
            bb.record(stream)
            bb.synchronize()
            tf.append(a.elapsed_time(bb))
            tr.append(a.elapsed_time(mid))
        ctx.rekey(w.hash_seed)                                   # restore the benchmarked function
        torch.cuda.synchronize()
        msf = statistics.median(tf)
        fresh = {"value": w.n / (msf * 1e-3) / 1e6, "unit": "Mbps", "ms_per_step": msf,
                 "rekey_ms": statistics.median(tr),
                 "api": "pa_ctx_rekey (device Philox4x64-10 expansion of a_i, b, c + their transforms) then pa_hash"}

    # ---- comparator (NEXT-4; Table 1 / Fig. 3): MH-only PA on the same key and (n, m),
    # top m bits of (b x + c) mod 2^n over the whole key, same kernels and timing rules
    comparators = None
    if not multi and not paper and args.comparators:
        cctx = PAContext(w.n, 0, w.m, 0, seed=w.hash_seed, mh_only=True)
        cout = torch.empty(cctx.nbytes_out, dtype=torch.uint8, device=dev)
        for _ in range(args.warmup):
            cctx.hash(key_dev, cout)
        torch.cuda.synchronize()
        tc = []
        for _ in range(max(3, args.steps // 5)):
            if not args.no_flush:
                flush.fill_(1)
            a = torch.cuda.Event(enable_timing=True)
            bb = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            cctx.hash(key_dev, cout)
            bb.record(stream)
            bb.synchronize()
            tc.append(a.elapsed_time(bb))
        msc = statistics.median(tc)
        ci = cctx.query()
        comparators = {"mh_only_pa": {
            "value": w.n / (msc * 1e-3) / 1e6, "unit": "Mbps", "ms_per_step": msc,
            "plan": {kk: ci["mh"][kk] for kk in ("limb_bits", "nprimes", "log2_len")},
            "what": "modular-arithmetic-hashing-only PA (PAPER.md:66, SPEC.md:305-313): top m bits of "
                    "(b x + c) mod 2^n, one n x n-bit product, same NTT/CRT kernels"}}
        cctx.close()
        # Toeplitz-hashing PA (Table 1's other comparator) on the same key and m
        tctx = PAContext(w.n, 0, w.m, 0, seed=w.hash_seed, toeplitz=True)
        tout = torch.empty(tctx.nbytes_out, dtype=torch.uint8, device=dev)
        for _ in range(args.warmup):
            tctx.hash(key_dev, tout)
        torch.cuda.synchronize()
        tt = []
        for _ in range(max(3, args.steps // 10)):
            if not args.no_flush:
                flush.fill_(1)
            a = torch.cuda.Event(enable_timing=True)
            bb = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            tctx.hash(key_dev, tout)
            bb.record(stream)
            bb.synchronize()
            tt.append(a.elapsed_time(bb))
        mst = statistics.median(tt)
        ti = tctx.query()
        comparators["toeplitz_pa"] = {
            "value": w.n / (mst * 1e-3) / 1e6, "unit": "Mbps", "ms_per_step": mst,
            "plan": {"r": ti["r"], "input_blocks": ti["k"], "output_blocks": ti["alpha"],
                     "log2_len": ti["mmh"]["log2_len"], "prime": ti["mmh"]["primes"][0]},
            "what": "Toeplitz-hashing PA over GF(2) (Table 1, PAPER.md:57-71; SPEC.md:287-304): exact "
                    "single-prime NTT convolution of bit coefficients, r x r block split, parity of counts"}
        tctx.close()

    if rank != 0:
        if multi:
            dist.destroy_process_group()
        return
    peaks = load_peaks()
    roof = roofline(info, {kk: (v[0] / nsteps_prof, v[1] // nsteps_prof) for kk, v in stages.items()}, peaks, 1)
    line = {
        "metric": METRIC, "value": w.n / (ms_per_step * 1e-3) / 1e6, "unit": "Mbps", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (i.i.d. Bernoulli(0.5) key bits from Philox4x64-10; hash keys from seed)",
        "config": {"workload": w.name, "mode": "paper (gamma-bit blocks, reload)" if paper else "r-bit blocks",
                   "n": w.n, "r": w.r, "m": w.m, "k": k, "gamma": info["gamma"],
                   "alpha": info["alpha"],
                   "mmh_plan": {kk: info["mmh"][kk] for kk in ("limb_bits", "nprimes", "log2_len", "n_col", "n_row")},
                   "mh_plan": {kk: info["mh"][kk] for kk in ("limb_bits", "nprimes", "log2_len", "n_col", "n_row")},
                   "parallelism": (f"blocks sharded over {world} ranks; transform-domain accumulators " +
                                   ("added by each rank's row MAC into rank 0's receive buffer over peer memory "
                                    "(p2p)" if args.p2p else "summed by one ncclReduce (library NCCL) to rank 0") +
                                   ", which runs the inverse, CRT, carries, fold and MH") if lib_nccl else (f"{world} ranks, gloo exchange (validation)" if multi
                                                                else "one GPU"),
                   "l2": "flushed (256 MiB write) before every timed step" if not args.no_flush else "not flushed"},
        "gpu_launches": launches_timed,
        "clocks": clocks,
        "roofline": roof,
        "hbm": hbm_view(w, info, ms_per_step, peaks, paper),
        "stages_ms_per_step": {kk: v[0] / nsteps_prof for kk, v in sorted(stages.items())},
        "e2e": e2e,
        "stream": stream_mode if not multi else mr_stream,
        "comparators": comparators,
        "fresh_keys": fresh,
        "graph_rebind": graph_rebind,
        "ctx_create_ms": ctx_create_ms,
    }
    if verified is not None:
        line["verified_vs_oracle"] = verified
    if multi and (args.same_device or args.dist_backend != "nccl" or args.one_rank_mg):
        line["validation_only"] = (f"{world} ranks, backend {args.dist_backend}, same_device={args.same_device}, "
                                   f"one_rank_mg={args.one_rank_mg}")
    if not multi and not args.no_cpu_baseline and not paper:
        line["cpu_baseline"] = cpu_oracle_full(w)
    print(json.dumps(line), flush=True)
    if multi:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
