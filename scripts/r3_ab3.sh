#!/bin/bash
mkdir -p gpurun_out/ab3
b() { timeout 300 python bench.py "$@" --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"; }
for c in 1 2; do for o in 0 16 32 48 64; do for f in 1 0; do echo "cfg$c overlap $o first $f: $(NFHMM_FB_FIRST=$f NFHMM_OVERLAP=$o b --config $c)" >> gpurun_out/ab3/bench.log; done; done; done
for o in 16 20 24; do echo "cfg3 overlap $o: $(NFHMM_OVERLAP=$o b)" >> gpurun_out/ab3/bench.log; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/ab3/pytest.log 2>&1; echo rc=$? >> gpurun_out/ab3/pytest.log
