#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/f_pytest.log 2>&1; echo rc=$? >> gpurun_out/f_pytest.log
for v in "1 0" "1 20" "1 24" "1 32" "1 40" "0 32"; do
  set -- $v
  export NFHMM_FB_MULTI=$1 NFHMM_OVERLAP=$2
  echo "== multi=$1 overlap=$2" >> gpurun_out/f_bench.log
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],1), 'fb', round(d['kernels']['fb']['ms_per_step'],2), 'recon', round(d['kernels']['recon']['ms_per_step'],2))" >> gpurun_out/f_bench.log 2>&1
done
NFHMM_OVERLAP=0 ./scripts/ncu_one.sh fb_multi ncu_fbm
