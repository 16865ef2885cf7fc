#!/bin/bash
# A/B of the overlap partition (SMs left to the forward-backward beside the contractions) on the final
# 3xFP16 build: config 3 and config 4, two repetitions, default first and last
mkdir -p gpurun_out/ab
L=gpurun_out/ab/overlap.log
b() { timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do
echo "cfg3 default(16): $(b)" >> $L
for k in 8 12 20 24 32; do echo "cfg3 overlap$k: $(NFHMM_OVERLAP=$k b)" >> $L; done
echo "cfg3 overlap16 fbfirst: $(NFHMM_FB_FIRST=1 b)" >> $L
echo "cfg3 default(16): $(b)" >> $L
done
for k in 16 8 24 32; do echo "cfg4 overlap$k: $(NFHMM_OVERLAP=$k b --config 4 --steps 2 --warmup 1)" >> $L; done
echo done >> $L
