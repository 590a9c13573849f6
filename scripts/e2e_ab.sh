#!/bin/bash
# e2e (pa_hash_host) A/B across in-tree library variants: scripts/e2e_ab.sh base v1 ...
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib=paper_2105_13678_b200/_pa_$v.so; fi
  echo "== $v"; PA_DEV_LIB=$lib timeout 300 python scripts/e2e_check.py C4 2>&1 | tail -2
done; done
