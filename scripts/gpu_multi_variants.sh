#!/bin/bash
# compile-time variants at N GPUs: bash scripts/gpu_multi_variants.sh OUTDIR N "configs" "FLAGS A" "FLAGS B" ...
cd "$GRAFT_REPO_ROOT"
O=$1; NG=$2; CFGS=$3; shift 3
mkdir -p $O
for fl in "$@"; do
  tag=$(echo "v$fl" | tr ' =-' '__.')
  EMB_NVCC_EXTRA="$fl" python -c "from paper_2110_09132_b200.build import build; build(force=True)" > $O/build_$tag.log 2>&1 || { echo "build failed $fl"; continue; }
  for cfg in $CFGS; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
      bench.py --gpus $NG --config $cfg --steps 1000 --warmup 20 --no-cpu-baseline > $O/b${NG}_${cfg}_$tag.json 2> $O/b${NG}_${cfg}_$tag.err
    python - "$O/b${NG}_${cfg}_$tag.json" "$cfg" "$fl" >> $O/summary.txt 2>&1 <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]).read().strip().splitlines() if l.startswith("{")][-1])
    print(f"N={d['n_gpus']} {sys.argv[2]:12s} [{sys.argv[3]:30s}] step {d['ms_per_step']*1e3:7.2f} us  {d['value']/1e6:8.1f} Mtok/s  graph med {d['step_time']['graph']['median_us']:7.2f}")
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
  done
done
python -c "from paper_2110_09132_b200.build import build; build(force=True)" > /dev/null 2>&1
cat $O/summary.txt
