#!/bin/bash
# Dirichlet ring kernel A/B: parity subset, then per-config Dirichlet ms per step and roofline fraction
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/rg_pytest.log 2>&1; echo rc=$? >> gpurun_out/rg_pytest.log
for c in 3 4 1 2; do
  echo "== cfg$c" >> gpurun_out/rg_bench.log
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['kernels']['dirichlet']['ms_per_step'],3), round(d['rooflines']['dirichlet']['frac'],3))" >> gpurun_out/rg_bench.log 2>&1
done
