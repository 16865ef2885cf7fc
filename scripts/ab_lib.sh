#!/bin/bash
# A/B: NFHMM_PRIO=1 (experiment) -- the overlapped sweep's contractions on a high-priority internal stream, so
# pending recursion CTAs cannot take freed SMs ahead of the next contraction; config 3, digests must match
mkdir -p gpurun_out/ab
L=gpurun_out/ab/prio.log
b() { timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['gathered']['L_digest'], d['gathered']['d_hat_digest'])"; }
echo "cfg3 default(16): $(b)" >> $L
for k in 16 12 8 4; do echo "cfg3 prio overlap$k: $(NFHMM_PRIO=1 NFHMM_OVERLAP=$k b)" >> $L; done
echo "cfg3 default(16): $(b)" >> $L
echo "cfg3 prio overlap8: $(NFHMM_PRIO=1 NFHMM_OVERLAP=8 b)" >> $L
echo done >> $L
