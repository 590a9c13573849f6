#!/bin/bash
# bench line + launch list (plain run first, then ncu on the same command)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python bench.py --steps 3 --warmup 3 --only-device > gpurun_out/bench_small.json 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --only-device > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/bench.err
