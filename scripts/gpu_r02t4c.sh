#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02t4c; mkdir -p $O
EMB_NVCC_EXTRA=-DEMB_TRACE python -c "from paper_2110_09132_b200.build import build; build(force=True)" > $O/build.log 2>&1
for mode in coal split; do
  EMB_TRACE_OUT=$O/tr_$mode timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
      bench.py --gpus 4 --config lstm_lm --mode $mode --steps 400 --warmup 20 --no-cpu-baseline > $O/b_$mode.json 2> $O/b_$mode.err
  python scripts/trace.py $O/tr_$mode.0.npy > $O/trace_$mode.txt 2>&1
  echo "== $mode"; cat $O/trace_$mode.txt
done
python -c "from paper_2110_09132_b200.build import build; build(force=True)" >> $O/build.log 2>&1
