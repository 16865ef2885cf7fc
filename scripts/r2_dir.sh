#!/bin/bash
# Dirichlet ring tile-shape sweep at config 3 (+ parity of the default)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg0 or cfg3 or edge or gamma" > gpurun_out/d_pytest.log 2>&1; echo rc=$? >> gpurun_out/d_pytest.log
for v in default 8,320 4,320 8,160 16,320 6,480 4,160 12,480 2,160; do
  if [ $v = default ]; then unset NFHMM_DIR_RING; else export NFHMM_DIR_RING=$v; fi
  echo "== $v" >> gpurun_out/d_bench.log
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), d['kernels']['dirichlet']['ms_per_step']/50, d['rooflines']['dirichlet']['frac'])" >> gpurun_out/d_bench.log
done
export NFHMM_DIRICHLET=pipe; unset NFHMM_DIR_RING; echo "== pipe" >> gpurun_out/d_bench.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), d['kernels']['dirichlet']['ms_per_step']/50, d['rooflines']['dirichlet']['frac'])" >> gpurun_out/d_bench.log
