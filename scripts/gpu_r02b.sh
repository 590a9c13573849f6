#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_mg.log 2>&1; echo "pytest_mg rc=$?" >> gpurun_out/pytest_mg.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_mg.log; tail -3 gpurun_out/pytest_gpu.log
