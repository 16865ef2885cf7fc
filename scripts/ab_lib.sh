#!/bin/bash
# A/B: multi-chain forward-backward register cap (FBM_MINB) and the SMs it gets beside the contractions
mkdir -p gpurun_out/ab
L=paper_1206_6468_b200/lib
b() { timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()})"; }
for rep in 1 2; do
echo "base cfg3: $(NFHMM_LIB=$L/libnfhmm_base.so b)" >> gpurun_out/ab/bench.log
echo "mb16 cfg3: $(NFHMM_LIB=$L/libnfhmm_mb16.so b)" >> gpurun_out/ab/bench.log
echo "mb16 ov12 cfg3: $(NFHMM_OVERLAP=12 NFHMM_LIB=$L/libnfhmm_mb16.so b)" >> gpurun_out/ab/bench.log
echo "mb16 ov14 cfg3: $(NFHMM_OVERLAP=14 NFHMM_LIB=$L/libnfhmm_mb16.so b)" >> gpurun_out/ab/bench.log
echo "mb12 cfg3: $(NFHMM_LIB=$L/libnfhmm_mb12.so b)" >> gpurun_out/ab/bench.log
done
echo "base cfg4: $(NFHMM_LIB=$L/libnfhmm_base.so b --config 4 --steps 1)" >> gpurun_out/ab/bench.log
echo "mb16 cfg4: $(NFHMM_LIB=$L/libnfhmm_mb16.so b --config 4 --steps 1)" >> gpurun_out/ab/bench.log
