#!/bin/bash
# A/B of the overlap partition (SMs left to the forward-backward beside the contractions) on the final
# 3xFP16 build, second pass: config 3 between the cliff (12) and the default (16); config 4 with more steps
mkdir -p gpurun_out/ab
L=gpurun_out/ab/overlap2.log
b() { timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do
for k in 16 13 14 15 18; do echo "cfg3 overlap$k: $(NFHMM_OVERLAP=$k b)" >> $L; done
done
for rep in 1 2; do
for k in 16 8 12 4; do echo "cfg4 overlap$k: $(NFHMM_OVERLAP=$k b --config 4 --steps 4 --warmup 2)" >> $L; done
done
echo done >> $L
