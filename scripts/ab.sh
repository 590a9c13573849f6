#!/bin/bash
# A/B timing of in-tree library variants: scripts/ab.sh CONFIG base m6 c3 ...  ("base" = _pa.so)
mkdir -p gpurun_out
cfg=$1; shift
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib=paper_2105_13678_b200/_pa_$v.so; fi
  PA_DEV_LIB=$lib timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-comparators --batch 1 --steps 30 \
     > gpurun_out/ab_${v}_$rep.json 2> gpurun_out/ab_${v}_$rep.err
  python - "$v" "gpurun_out/ab_${v}_$rep.json" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
except Exception as e:
    print(sys.argv[1], "FAILED", e); sys.exit()
st = d["stages_ms_per_step"]
print(f"{sys.argv[1]:8s} {d['ms_per_step']*1e3:7.1f} us  " + " ".join(f"{k.replace('mmh_','M').replace('mh_','H')}={v*1e3:.1f}" for k, v in sorted(st.items())))
PY
done; done
