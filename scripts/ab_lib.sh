#!/bin/bash
# How much of the forward-backward the overlap hides at config 3 (NFHMM_SKIP_FB: timing only)
mkdir -p gpurun_out/ab
b() { timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()})"; }
for rep in 1 2; do
echo "default cfg3: $(b)" >> gpurun_out/ab/bench.log
echo "skipfb cfg3 (GEMMs on 132 SMs): $(NFHMM_SKIP_FB=1 b)" >> gpurun_out/ab/bench.log
echo "skipfb overlap0 cfg3 (GEMMs on 148 SMs): $(NFHMM_SKIP_FB=1 NFHMM_OVERLAP=0 b)" >> gpurun_out/ab/bench.log
echo "overlap0 cfg3 (FB serial): $(NFHMM_OVERLAP=0 b)" >> gpurun_out/ab/bench.log
done
