#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -x -q -k "dist or cfg1 or sharding or resume" > gpurun_out/q2_pytest.log 2>&1; echo rc=$? >> gpurun_out/q2_pytest.log
for CFG in 1 2; do
  echo "== cfg$CFG" >> gpurun_out/q2_bench.log
  timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), round(d['value_bound_off']/1e6,3), {k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()})" >> gpurun_out/q2_bench.log 2>&1
done
