#!/bin/bash
# a13 dense priority queue: NCCL AllReduce algorithm (default / NVLS / ring) at N = 2 and 4
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02dq4; mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
run() { n=$1; tag=$2; shift 2; env "$@" timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
   --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $n --config bert_large --dense-queue 24 --steps 20 --warmup 5 \
   > $O/dq${n}_$tag.json 2> $O/dq${n}_$tag.err; echo "$n $tag rc=$?" >> $O/rc.txt; }
for n in 2 $NG; do
  run $n default X=1
  run $n nvls "NCCL_ALGO=allreduce:nvls"
  run $n ring "NCCL_ALGO=allreduce:ring"
done
cat $O/rc.txt
for f in $O/dq*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
    print(sys.argv[1], d["n_gpus"], d["value"], d["unit"], "algbw", d["algbw_gbs"], d["issue_order"]["ok"], round(d["interference"]["overlap_frac"],3))
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
done
