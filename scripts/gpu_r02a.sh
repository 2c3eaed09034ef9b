#!/bin/bash
# round-2 first GPU pass: new parity tests (co-located N>1, free-running, pipelined, graph), smoke
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02a
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_colocated.py -x -q -m gpu --timeout 300 > $O/colocated.log 2>&1; echo "colocated rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -k "free or pipelined or graph or null" > $O/parity_new.log 2>&1; echo "parity_new rc=$?" >> $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
cat $O/rc.txt
tail -5 $O/colocated.log $O/parity_new.log
