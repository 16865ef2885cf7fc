#!/bin/bash
# cfg-3 A/B of the overlapped sweep after the 3xFP16 back-projection
mkdir -p gpurun_out/ab
b() { timeout 300 python bench.py "$@" --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()})"; }
echo "default: $(b)" >> gpurun_out/ab/bench.log
echo "nopf: $(NFHMM_TC_DEBUG=256 b)" >> gpurun_out/ab/bench.log
echo "bp tf32: $(NFHMM_BACKPROJ=tf32 b)" >> gpurun_out/ab/bench.log
echo "bp tf32 nopf: $(NFHMM_BACKPROJ=tf32 NFHMM_TC_DEBUG=256 b)" >> gpurun_out/ab/bench.log
echo "overlap 0: $(NFHMM_OVERLAP=0 b)" >> gpurun_out/ab/bench.log
echo "defer 0 ov24: $(NFHMM_DEFER=0 NFHMM_OVERLAP=24 b)" >> gpurun_out/ab/bench.log
echo "all tf32: $(NFHMM_RECON=tf32 b)" >> gpurun_out/ab/bench.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ab/pytest.log 2>&1; echo rc=$? >> gpurun_out/ab/pytest.log
