#!/bin/bash
# One GPU session: tests, bench, ncu launch list, full ncu captures of the top kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python bench.py --steps 3 --warmup 3 --only-device > gpurun_out/bench_small.json 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --only-device > gpurun_out/ncu_launch.log 2>&1
python scripts/prof_one.py C4 > gpurun_out/prof_one.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"row_mac|col_pass|pack_key|crt_carry|crt_coeffs" -s 2 -c 7 \
   -o gpurun_out/full -f python scripts/prof_one.py C4 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
