timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$?; tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --mixtures 64 --iters 4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print({n:round(v['ms_per_step']/v['launches_per_step'],3) for n,v in k.items()})"
