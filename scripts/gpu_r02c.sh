#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
PA_DEV_LIB=paper_2105_13678_b200/_pa_tprof.so timeout 300 python scripts/tprof.py C4 > gpurun_out/tprof_c4.json 2>&1
tail -1 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.err
