#!/bin/bash
# A/B: the committed build (base) vs the two-converter-group build (g2); a short hang check first
mkdir -p gpurun_out/ab
L=paper_1206_6468_b200/lib
NFHMM_LIB=$L/libnfhmm_g2.so timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg3_batched_reduced or edge" > gpurun_out/ab/pytest_quick.log 2>&1; rc=$?; echo rc=$rc >> gpurun_out/ab/pytest_quick.log
[ $rc -ne 0 ] && exit 0
b() { timeout 150 python bench.py --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()}, {k:round(v['frac'],3) for k,v in d['rooflines'].items()})"; }
echo "g2 cfg3: $(NFHMM_LIB=$L/libnfhmm_g2.so b)" >> gpurun_out/ab/bench.log
echo "base cfg3: $(NFHMM_LIB=$L/libnfhmm_base.so b)" >> gpurun_out/ab/bench.log
echo "g2 cfg3: $(NFHMM_LIB=$L/libnfhmm_g2.so b)" >> gpurun_out/ab/bench.log
echo "base cfg3: $(NFHMM_LIB=$L/libnfhmm_base.so b)" >> gpurun_out/ab/bench.log
echo "g2 cfg4: $(NFHMM_LIB=$L/libnfhmm_g2.so b --config 4 --steps 1)" >> gpurun_out/ab/bench.log
echo "base cfg4: $(NFHMM_LIB=$L/libnfhmm_base.so b --config 4 --steps 1)" >> gpurun_out/ab/bench.log
echo "g2 cfg1: $(NFHMM_LIB=$L/libnfhmm_g2.so b --config 1)" >> gpurun_out/ab/bench.log
NFHMM_LIB=$L/libnfhmm_g2.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pair or overlap or split or cfg4 or cfg3 or recon or edge" > gpurun_out/ab/pytest.log 2>&1; echo rc=$? >> gpurun_out/ab/pytest.log
