#!/bin/bash
# Round-2 session A: integer-pipe microbenchmark, GPU tests, bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 120 ./microbench/int_peak > gpurun_out/int_peak.json 2> gpurun_out/int_peak.err; echo "int_peak rc=$?" >> gpurun_out/int_peak.err
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -1 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.err; cat gpurun_out/int_peak.json
