#!/bin/bash
# A/B: forward-backward launched first (its one-warp CTAs spread over every SM, the persistent GEMM CTAs
# placed beside them) with a small partition, config 3, final 3xFP16 build
mkdir -p gpurun_out/ab
L=gpurun_out/ab/overlap3.log
b() { timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
echo "cfg3 default(16): $(b)" >> $L
for k in 2 4 8 12; do echo "cfg3 overlap$k fbfirst: $(NFHMM_FB_FIRST=1 NFHMM_OVERLAP=$k b)" >> $L; done
echo "cfg3 default(16): $(b)" >> $L
for k in 2 8; do echo "cfg3 overlap$k fbfirst: $(NFHMM_FB_FIRST=1 NFHMM_OVERLAP=$k b)" >> $L; done
echo done >> $L
