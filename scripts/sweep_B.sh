#!/bin/bash
# forced-limb-width sweep of the C4 step (device time), one line per B
for B in ${@:-96 120 136 144 152 160 168 176 184 192 200}; do
  timeout 120 python bench.py --no-cpu-baseline --steps 20 --limb-bits $B 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms_per_step']
print($B, d['config']['mmh_plan'], d['config']['mh_plan']['limb_bits'], round(d['ms_per_step']*1e3,1), {k:round(v*1e3,1) for k,v in s.items()})"
done
