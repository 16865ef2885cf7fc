#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/d5_pytest.log 2>&1; echo rc=$? >> gpurun_out/d5_pytest.log
for c in 3 4 1 2; do for v in ring pipe; do
  if [ $v = ring ]; then unset NFHMM_DIRICHLET; else export NFHMM_DIRICHLET=pipe; fi
  echo "== cfg$c $v" >> gpurun_out/d5_bench.log
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['kernels']['dirichlet']['ms_per_step'],3), round(d['rooflines']['dirichlet']['frac'],3))" >> gpurun_out/d5_bench.log 2>&1
done; done
