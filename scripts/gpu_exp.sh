#!/bin/bash
# knob experiment: bash scripts/gpu_exp.sh OUTDIR "configs" "ENV=a ENV2=b" "ENV=c" ...
cd "$GRAFT_REPO_ROOT"
O=$1; CFGS=$2; shift 2
mkdir -p $O
for cfg in $CFGS; do
  for envs in "$@"; do
    tag=$(echo "$envs" | tr ' =' '_-')
    env $envs timeout 300 python bench.py --config $cfg --steps 1000 --warmup 20 --no-cpu-baseline > $O/b_${cfg}_${tag}.json 2> $O/b_${cfg}_${tag}.err
    python - "$O/b_${cfg}_${tag}.json" "$cfg" "$envs" >> $O/summary.txt 2>&1 <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    k = d["kernels"]
    print(f"{sys.argv[2]:12s} {sys.argv[3]:40s} step {d['ms_per_step']*1e3:7.2f} us  graph med {d['step_time']['graph']['median_us']:7.2f}  "
          f"roof {d['roofline']['frac']:.3f} step_frac {d['step_roofline']['frac']:.3f}")
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
  done
done
cat $O/summary.txt
