#!/bin/bash
# compile-time variant sweep: bash scripts/gpu_variants.sh OUTDIR "configs" "NVCC FLAGS A" "NVCC FLAGS B" ...
# each variant: build (+ -DEMB_TRACE traced pass), bench, trace summary; default build restored at the end
cd "$GRAFT_REPO_ROOT"
O=$1; CFGS=$2; shift 2
mkdir -p $O
for fl in "$@"; do
  tag=$(echo "v$fl" | tr ' =-' '__.')
  EMB_NVCC_EXTRA="$fl" python -c "from paper_2110_09132_b200.build import build; build(force=True)" > $O/build_$tag.log 2>&1 || { echo "build failed $fl"; continue; }
  for cfg in $CFGS; do
    timeout 300 python bench.py --config $cfg --steps 1000 --warmup 20 --no-cpu-baseline > $O/b_${cfg}_$tag.json 2> $O/b_${cfg}_$tag.err
    python - "$O/b_${cfg}_$tag.json" "$cfg" "$fl" >> $O/summary.txt 2>&1 <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:12s} [{sys.argv[3]:40s}] step {d['ms_per_step']*1e3:7.2f} us  graph med {d['step_time']['graph']['median_us']:7.2f}  step_frac {d['step_roofline']['frac']:.3f}")
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
  done
  EMB_NVCC_EXTRA="$fl -DEMB_TRACE" python -c "from paper_2110_09132_b200.build import build; build(force=True)" >> $O/build_$tag.log 2>&1
  for cfg in $CFGS; do
    EMB_TRACE_OUT=$O/tr_${cfg}_$tag timeout 300 python bench.py --config $cfg --steps 400 --warmup 20 --no-cpu-baseline > /dev/null 2>&1
    echo "== $cfg [$fl]" >> $O/traces.txt
    python scripts/trace.py $O/tr_${cfg}_$tag.*.npy >> $O/traces.txt 2>&1
  done
done
python -c "from paper_2110_09132_b200.build import build; build(force=True)" > /dev/null 2>&1
cat $O/summary.txt; cat $O/traces.txt
