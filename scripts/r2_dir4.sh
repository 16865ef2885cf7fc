#!/bin/bash
mkdir -p gpurun_out
for lib in libnfhmm_r64.so libnfhmm.so libnfhmm_r128.so; do
 for v in 6,128 8,128 8,160 4,128 6,192; do
  export NFHMM_DIR_RING=$v NFHMM_DIR_WARP=0 NFHMM_LIB=$PWD/paper_1206_6468_b200/lib/$lib
  echo "== $lib $v" >> gpurun_out/d4_bench.log
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), d['kernels']['dirichlet']['ms_per_step']/50, d['rooflines']['dirichlet']['frac'])" >> gpurun_out/d4_bench.log 2>&1
 done
done
