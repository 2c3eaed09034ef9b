#!/bin/bash
# multi-GPU kernel trace: bash scripts/gpu_trace_multi.sh OUTDIR N "configs" [ENV=...]
cd "$GRAFT_REPO_ROOT"
O=$1; NG=$2; CFGS=$3; shift 3
mkdir -p $O
EMB_NVCC_EXTRA=-DEMB_TRACE python -c "from paper_2110_09132_b200.build import build; build(force=True)" > $O/build.log 2>&1
for cfg in $CFGS; do
  env "$@" EMB_TRACE_OUT=$O/tr${NG}_$cfg timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
      bench.py --gpus $NG --config $cfg --steps 400 --warmup 20 > $O/b${NG}_$cfg.json 2> $O/b${NG}_$cfg.err
  python scripts/trace.py $O/tr${NG}_$cfg.*.npy > $O/trace${NG}_$cfg.txt 2>&1
  cat $O/trace${NG}_$cfg.txt
done
python -c "from paper_2110_09132_b200.build import build; build(force=True)" >> $O/build.log 2>&1
