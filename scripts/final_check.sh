#!/bin/bash
# final check of the committed build: GPU suite + smoke + default bench line + the other configs
D=gpurun_out/final
mkdir -p $D
rm -f gpurun_out/parity_records.jsonl
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo "rc=$?" >> $D/pytest_gpu.log
cp gpurun_out/parity_records.jsonl $D/parity_records.jsonl 2>/dev/null
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "rc=$?" >> $D/smoke.log
timeout 900 python bench.py > $D/bench.log 2>&1; echo "rc=$?" >> $D/bench.log
timeout 900 python bench.py --steps 20 --warmup 5 > $D/bench_cfg3.log 2>&1
for c in 0 1 2 4; do timeout 900 python bench.py --config $c > $D/bench_cfg$c.log 2>&1; done
echo done > $D/DONE
