#!/bin/bash
# quick GPU check: dist + parity tests, then cfg-3 bench lines for the Dirichlet variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -x -q > gpurun_out/q_pytest.log 2>&1; echo rc=$? >> gpurun_out/q_pytest.log
for v in ring pipe; do
  if [ $v = ring ]; then unset NFHMM_DIRICHLET; else export NFHMM_DIRICHLET=$v; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline > gpurun_out/q_bench_$v.log 2>&1
done
