#!/bin/bash
# e2e A/B of in-tree library variants, interleaved: scripts/e2e_ab.sh CONFIG base v1 ...
mkdir -p gpurun_out
cfg=$1; shift
for rep in 1 2 3; do
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib=paper_2105_13678_b200/_pa_$v.so; fi
  echo -n "$v  "; PA_DEV_LIB=$lib timeout 300 python scripts/e2e_check.py $cfg 2>/dev/null | tr '\n' ' '; echo
done; done
