#!/bin/bash
# sort with one cluster barrier per pass after the first (EMB_SORT_1BAR): parity + A/B with traces
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bar; mkdir -p $O
EMB_NVCC_EXTRA="-DEMB_SORT_1BAR=1" python -c "from paper_2110_09132_b200.build import build; build(force=True)" > $O/build1.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_colocated.py -q -m gpu --timeout 300 -x > $O/parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
tail -n 2 $O/parity.log
bash scripts/gpu_variants.sh $O "lstm_lm bert_large gnmt" "-DEMB_SORT_1BAR=0" "-DEMB_SORT_1BAR=1" "-DEMB_SORT_1BAR=0" "-DEMB_SORT_1BAR=1" | grep step
grep "== \|sort " $O/traces.txt
cat $O/rc.txt
