#!/bin/bash
# 3xFP16 reconstruction: parity subset, per-kernel timings A/B, short bench lines A/B
mkdir -p gpurun_out/h16
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "recon or cfg0 or cfg3 or edge or gamma or cfg4 or overlap or sharding" > gpurun_out/h16/pytest.log 2>&1; echo rc=$? >> gpurun_out/h16/pytest.log
for v in f16 tf32; do
  export NFHMM_RECON=$v
  timeout 300 python scripts/perf_quick.py --mixtures 64 --iters 10 --check > gpurun_out/h16/quick_$v.log 2>&1
  timeout 300 python scripts/perf_quick.py --config 1 --mixtures 1 --iters 20 --check > gpurun_out/h16/quick1_$v.log 2>&1
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline > gpurun_out/h16/bench3_$v.log 2>&1
  timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline > gpurun_out/h16/bench1_$v.log 2>&1
done
