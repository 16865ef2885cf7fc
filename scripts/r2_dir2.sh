#!/bin/bash
mkdir -p gpurun_out
for v in 6,128 6,160 8,128 8,160 6,96; do
  export NFHMM_DIR_RING=$v
  echo "== $v" >> gpurun_out/d2_bench.log
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), d['kernels']['dirichlet']['ms_per_step']/50, d['rooflines']['dirichlet']['frac'])" >> gpurun_out/d2_bench.log 2>&1
done
export NFHMM_DIR_RING=6,160
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg0 or cfg3 or edge or gamma or cfg1" > gpurun_out/d2_pytest.log 2>&1; echo rc=$? >> gpurun_out/d2_pytest.log
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:dirichlet_ring" -s 1 -c 1 \
  -o gpurun_out/ncu_ring2 -f python bench.py --steps 1 --warmup 1 --iters 3 --no-e2e --no-bound-off --no-cpu-baseline > gpurun_out/ncu_ring2.log 2>&1
