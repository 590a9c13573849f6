"""Per-CUDA-source-line instruction and stall-sample shares of one kernel from an ncu report
(ncu -i REP --page source --csv --print-source cuda,sass):
python scripts/ncu_lines.py REP REGEX [N] [SKIP]."""
import csv
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"          # matching launches to skip
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{rx}", "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
agg = {}
fname = "?"
hdr = None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue                      # cuda line rows carry '-' in the SASS address column
    try:
        n = float(r[7] or 0)
        s = float(r[4] or 0)
    except ValueError:
        continue
    k = f"{fname}:{r[0]}"
    a = agg.setdefault(k, [0.0, 0.0, r[1][:100]])
    a[0] += n
    a[1] += s
tn = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"warp-instructions {tn:.0f}, stall samples {ts:.0f}")
for k, (n, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * n / tn:5.1f}% inst {100 * s / ts:5.1f}% samp  {k:18s} {src}")
