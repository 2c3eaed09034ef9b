#!/bin/bash
# a13 dense priority queue at N = 2 (after the batch-sequence fix), NCCL algorithm variants incl. NVLS
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02dq; mkdir -p $O
run() { tag=$1; shift; env "$@" timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
   --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 2 --config bert_large --dense-queue 24 --steps 20 --warmup 5 \
   > $O/dq_$tag.json 2> $O/dq_$tag.err; echo "$tag rc=$?" >> $O/rc.txt; }
run default NCCL_DEBUG=INFO
run nvls NCCL_DEBUG=INFO NCCL_NVLS_ENABLE=1 NCCL_ALGO=NVLS
run ring NCCL_ALGO=Ring
run gnmt_default X=1
cat $O/rc.txt
grep -h "NVLS\|nvls" $O/dq_default.err | head -5
grep -h "NVLS\|nvls" $O/dq_nvls.err | head -5
for f in $O/dq_*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads([l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")][-1])
    print(sys.argv[1], d["value"], d["unit"], d["issue_order"]["ok"], d["interference"])
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
done
