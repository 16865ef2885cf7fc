#!/bin/bash
mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/o_bench.log; timeout 300 env "$@" python bench.py --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],1))" >> gpurun_out/o_bench.log 2>&1; }
for lib in libnfhmm.so libnfhmm_fb16.so libnfhmm_fb20.so; do for o in 12 16 20 24; do run NFHMM_LIB=$PWD/paper_1206_6468_b200/lib/$lib NFHMM_OVERLAP=$o; done; done
