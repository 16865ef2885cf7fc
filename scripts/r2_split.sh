#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/s_pytest.log 2>&1; echo rc=$? >> gpurun_out/s_pytest.log
for c in 1 2 0; do for v in 1 0; do
  export NFHMM_SPLITK=$v
  echo "== cfg$c split=$v" >> gpurun_out/s_bench.log
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()}, {k:round(v['frac'],3) for k,v in d['rooflines'].items()})" >> gpurun_out/s_bench.log 2>&1
done; done
