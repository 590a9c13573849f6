#!/bin/bash
# Full ncu capture of the latency-bound tail kernels of one C4 hash (eager launches).
export PA_NO_GRAPH=1
mkdir -p gpurun_out
python scripts/prof_one.py C4 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:row_pass<\(int\)(9|10), \(int\)5, \(int\)(1|2), \(int\)2>|col_pass<.*\(int\)2>|crt_carry<\(int\)11|crt_coeffs<\(int\)11|col_pass<\(int\)8, \(int\)5, \(int\)10, \(int\)0>|row_mac<\(int\)10' \
  -c 12 -o gpurun_out/tail -f python scripts/prof_one.py C4 > gpurun_out/ncu_tail.log 2>&1
tail -2 gpurun_out/ncu_tail.log
