#!/bin/bash
mkdir -p gpurun_out/ab2
b() { timeout 300 python bench.py "$@" --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()})"; }
for o in 0 8 12 16 24; do echo "cfg3 overlap $o: $(NFHMM_OVERLAP=$o b)" >> gpurun_out/ab2/bench.log; done
echo "cfg3 defer0 ov24: $(NFHMM_DEFER=0 NFHMM_OVERLAP=24 b)" >> gpurun_out/ab2/bench.log
for o in 0 16 32; do echo "cfg1 overlap $o: $(NFHMM_OVERLAP=$o b --config 1)" >> gpurun_out/ab2/bench.log; done
for o in 0 32 48; do echo "cfg2 overlap $o: $(NFHMM_OVERLAP=$o b --config 2)" >> gpurun_out/ab2/bench.log; done
for o in 0 16 32; do echo "cfg4 overlap $o: $(NFHMM_OVERLAP=$o b --config 4)" >> gpurun_out/ab2/bench.log; done
