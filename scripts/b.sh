#!/bin/bash
# build the library; print errors and exit 1 on failure
out=$(python /root/repo/paper_2105_13678_b200/build.py 2>&1)
if echo "$out" | grep -q "error"; then echo "$out" | grep -A3 error | head -30; exit 1; fi
echo "build ok"
