#!/bin/bash
# round-end style validation on one GPU: every -m gpu test, smoke, default bench, reference arm
cd "$GRAFT_REPO_ROOT"
O=${1:-gpurun_out/r02_end}; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?" >> $O/rc.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -n 3 $O/pytest_gpu.log; tail -n 1 $O/smoke.log
