#!/bin/bash
# Round-2 evidence run: GPU test suite, default bench line, launch list and one --set full
# capture of every kernel of one C4 pa_hash (summarised by scripts/make_profiles.py).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python scripts/prof_one.py C4 > gpurun_out/prof_one.log 2>&1 && \
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -o gpurun_out/r02_hash python scripts/prof_one.py C4 > gpurun_out/ncu_full.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --only-device > gpurun_out/bench_small.json 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --only-device > gpurun_out/ncu_launch.log 2>&1
tail -1 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.err; tail -2 gpurun_out/ncu_full.log
