#!/bin/bash
# The whole -m gpu suite on the bounds-asserting build (PA_DEBUG; compute-sanitizer is closed
# on the pool): every global access checked against the live ranges, every shared index
# against the CTA's shared memory; a violation prints the site and traps.
mkdir -p gpurun_out
export PA_DEV_LIB=$PWD/paper_2105_13678_b200/_pa_debug.so
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_debug.log 2>&1
echo "pytest_debug rc=$?" >> gpurun_out/pytest_gpu_debug.log
grep -c "PA_DEBUG bounds violation" gpurun_out/pytest_gpu_debug.log
tail -3 gpurun_out/pytest_gpu_debug.log
