#!/bin/bash
# bash scripts/gpu_sanitize.sh TOOL  (one compute-sanitizer tool per gpurun call)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02_sanitize; mkdir -p $O
timeout 300 python scripts/sanitize_tiny.py > $O/plain_$1.log 2>&1 && \
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $1 --print-limit 50 --error-exitcode 9 python scripts/sanitize_tiny.py > $O/$1.log 2>&1
echo "rc=$?" >> $O/$1.log
tail -n 8 $O/$1.log
