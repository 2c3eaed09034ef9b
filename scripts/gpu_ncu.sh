#!/bin/bash
# ncu --set full of the chosen kernels on a short eager bench: bash scripts/gpu_ncu.sh OUT config "regex" [env...]
cd "$GRAFT_REPO_ROOT"
O=$1; CFG=$2; RX=$3; shift 3
mkdir -p $(dirname $O)
CMD="python bench.py --config $CFG --steps 30 --warmup 5 --no-graph --no-cpu-baseline --profile-steps 4"
env "$@" $CMD > ${O}_plain.log 2>&1 && \
env "$@" ncu --set full --clock-control none --import-source on -k "regex:$RX" -s 6 -c 3 -o $O $CMD > ${O}_ncu.log 2>&1
echo "ncu rc=$?"
