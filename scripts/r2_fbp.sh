#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/p_pytest.log 2>&1; echo rc=$? >> gpurun_out/p_pytest.log
run() { echo "== $*" >> gpurun_out/p_bench.log; timeout 300 env "$@" python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],2) for k,v in d['kernels'].items() if k in ('recon','backproj','fb','dirichlet','elbo')})" >> gpurun_out/p_bench.log 2>&1; }
for CFG in 1 2; do
  run NFHMM_FB_CHUNK=16
  run NFHMM_FB_CHUNK=8
  run NFHMM_FB_CHUNK=32
done

timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launch_fbp.csv python bench.py --config 1 --steps 1 --warmup 1 --iters 3 --no-cpu-baseline --no-e2e --no-bound-off > /dev/null 2>&1
