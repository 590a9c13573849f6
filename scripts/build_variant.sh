#!/bin/bash
# A/B build: scripts/build_variant.sh NAME "-DMACRO=V ..." -> paper_2105_13678_b200/_pa_NAME.so
# (select at run time with PA_DEV_LIB=paper_2105_13678_b200/_pa_NAME.so; development only)
set -e
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  $2 -o paper_2105_13678_b200/_pa_$1.so paper_2105_13678_b200/csrc/pa_api.cu
echo "built _pa_$1.so"
