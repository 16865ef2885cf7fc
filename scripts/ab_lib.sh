#!/bin/bash
# A/B: current build vs the HEAD build (libnfhmm_base.so), pair on / off
mkdir -p gpurun_out/ab
B=paper_1206_6468_b200/lib/libnfhmm_base.so
b() { timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()}, {k:round(v['frac'],3) for k,v in d['rooflines'].items()})"; }
echo "cur cfg3: $(b)" >> gpurun_out/ab/bench.log
echo "base cfg3: $(NFHMM_LIB=$B b)" >> gpurun_out/ab/bench.log
echo "cur-nopair cfg3: $(NFHMM_TC_PAIR=0 b)" >> gpurun_out/ab/bench.log
echo "cur cfg3: $(b)" >> gpurun_out/ab/bench.log
echo "base cfg3: $(NFHMM_LIB=$B b)" >> gpurun_out/ab/bench.log
echo "cur cfg4: $(b --config 4 --steps 1)" >> gpurun_out/ab/bench.log
echo "base cfg4: $(NFHMM_LIB=$B b --config 4 --steps 1)" >> gpurun_out/ab/bench.log
echo "cur cfg4: $(b --config 4 --steps 1)" >> gpurun_out/ab/bench.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pair or overlap or split or cfg4 or cfg3" > gpurun_out/ab/pytest.log 2>&1; echo rc=$? >> gpurun_out/ab/pytest.log
