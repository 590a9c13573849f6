"""Summarise a GPU session's ncu output (gpurun_out/) into tracked files under profiles/.

    python scripts/make_profiles.py r01 [launches.csv] [rep:stage ...]

Writes profiles/<tag>_launches.md (per-launch device times of one timed step and
each kernel's share of that step, from the `--metrics gpu__time_duration.sum` pass),
profiles/<tag>_<stage>.txt (the `--set full` summary of one kernel) and merges
dram bytes per launch into profiles/ncu_traffic.json (read by bench.py)."""
from __future__ import annotations

import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from ncu_summary import summarize  # noqa: E402

PROF = os.path.join(ROOT, "profiles")


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name.replace("void ", "")).replace("pa::", "")
    return name


def launches(path: str, tag: str) -> None:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    iN, iV, iG, iB = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size"), hdr.index("Block Size")
    data = [(short(r[iN]), float(r[iV]) / 1e3, r[iG], r[iB]) for r in rows[1:]]
    # one step = the launches between the last two L2-flush fills (at::...FillFunctor)
    fills = [i for i, d in enumerate(data) if "FillFunctor" in d[0] or "elementwise" in d[0]]
    if len(fills) >= 2:
        step = data[fills[-2] + 1:fills[-1]]
    else:
        step = data[-40:]
    tot = sum(d[1] for d in step)
    out = [f"# {tag}: per-launch device time of one pa_hash step (ncu --metrics gpu__time_duration.sum "
           f"--clock-control none; cold-cache, serialised: compare shares)", "",
           f"step total {tot:.1f} us over {len(step)} launches", "",
           "| # | kernel | grid | block | us | share |", "|---|---|---|---|---|---|"]
    for i, (n, us, g, b) in enumerate(step):
        out.append(f"| {i} | `{n}` | {g} | {b} | {us:.1f} | {100 * us / tot:.1f}% |")
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(out) + "\n")
    print("\n".join(out))


def full(rep: str, stage: str, tag: str) -> None:
    """stage: one name, or comma-separated names of the report's launches in order."""
    recs = summarize(rep)
    names = stage.split(",")
    lines = []
    traffic_path = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for i, rec in enumerate(recs):
        stage = names[min(i, len(names) - 1)]
        lines.append(f"----- {os.path.basename(rep)} (stage {stage})")
        for k, v in rec.items():
            lines.append(f"  {k:80s} {v[:60]}")

        def mb(key):
            v = rec.get(key, "0").split()
            val = float(v[0])
            unit = v[1] if len(v) > 1 else "byte"
            return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        dur = rec.get("gpu__time_duration.sum", "0").split()
        us = float(dur[0]) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(dur[1] if len(dur) > 1 else "usecond", 1.0)
        dram = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
        lines.append(f"  {'achieved DRAM GB/s (read+write / duration, SURVEY.md §8(d) item 4)':80s} "
                     f"{dram / (us * 1e-6) / 1e9 if us else 0:.1f}")
        traffic[stage] = {"kernel": rec.get("Kernel Name"), "dram_bytes_per_launch":
                          mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
                          "dram_read": mb("dram__bytes_read.sum"), "dram_write": mb("dram__bytes_write.sum"),
                          "ncu_pct_of_peak": {kk: float(rec[mk].split()[0]) for kk, mk in (
                              ("issue_active", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                              ("pipe_alu", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                              ("pipe_fma", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                              ("pipe_lsu", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
                              ("warps_active", "sm__warps_active.avg.pct_of_peak_sustained_active")) if mk in rec},
                          "source": f"profiles/{tag}_{names[0] if len(names) == 1 else 'kernels'}.txt"}
    open(os.path.join(PROF, f"{tag}_{names[0] if len(names) == 1 else 'kernels'}.txt"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    os.makedirs(PROF, exist_ok=True)
    tag = sys.argv[1]
    for a in sys.argv[2:]:
        if a.endswith(".csv"):
            launches(a, tag)
        else:
            rep, stage = a.split(":")
            full(rep, stage, tag)
