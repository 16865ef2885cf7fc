#!/bin/bash
# HEAD check: full GPU suite + default bench line
mkdir -p gpurun_out/h
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/h/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/h/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/h/bench_cfg3.log 2>&1
for c in 1 2; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/h/bench_cfg$c.log 2>&1; done
