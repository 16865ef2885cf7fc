#!/bin/bash
# per-rank workloads of the 1/2/4/8-GPU config-3 runs on one GPU (defaults), then the GPU suite
mkdir -p gpurun_out/ab
b() { timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()})"; }
for M in 32 64 128 256; do echo "M$M default: $(b --mixtures $M)" >> gpurun_out/ab/bench.log; done
echo "cfg1 default: $(b --config 1)" >> gpurun_out/ab/bench.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ab/pytest.log 2>&1; echo rc=$? >> gpurun_out/ab/pytest.log
