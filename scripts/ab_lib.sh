#!/bin/bash
# A/B: where the overlap cliff below 16 SMs comes from -- CTA pair off, deferral off, config 3
mkdir -p gpurun_out/ab
L=gpurun_out/ab/overlap4.log
b() { timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for k in 16 15; do
echo "cfg3 overlap$k pair0: $(NFHMM_TC_PAIR=0 NFHMM_OVERLAP=$k b)" >> $L
echo "cfg3 overlap$k defer0: $(NFHMM_DEFER=0 NFHMM_OVERLAP=$k b)" >> $L
echo "cfg3 overlap$k tf32: $(NFHMM_RECON=tf32 NFHMM_BACKPROJ=tf32 NFHMM_OVERLAP=$k b)" >> $L
done
echo "cfg3 overlap17: $(NFHMM_OVERLAP=17 b)" >> $L
echo done >> $L
