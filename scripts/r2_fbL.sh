#!/bin/bash
mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/L_bench.log; timeout 300 env "$@" python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],2) for k,v in d['kernels'].items() if k in ('recon','backproj','fb','dirichlet','elbo')})" >> gpurun_out/L_bench.log 2>&1; }
for CFG in 1 2; do for L in 24 32 48 64 96 128; do run NFHMM_FB_CHUNK=$L; done; done
