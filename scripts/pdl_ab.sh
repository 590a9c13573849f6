#!/bin/bash
for cfg in C1 C2 C3 P1; do for rep in 1 2; do
for v in 1 0; do
  r=$(PA_NO_PDL=$v python bench.py --config $cfg --only-device --steps 50 --no-cpu-baseline | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['ms_per_step']*1e3,1))")
  echo "$cfg no_pdl=$v $r us"
done; done; done
