#!/bin/bash
# config 0 / 2 with the overlap now on for every sequential recursion
mkdir -p gpurun_out/ab
b() { timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-bound-off --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"; }
for rep in 1 2; do
echo "cfg0 default: $(b --config 0)" >> gpurun_out/ab/bench.log
echo "cfg0 overlap0: $(NFHMM_OVERLAP=0 b --config 0)" >> gpurun_out/ab/bench.log
done
echo "cfg2 default: $(b --config 2)" >> gpurun_out/ab/bench.log
