#!/bin/bash
# e2e pipeline check: default bench lines (cfg 3, 1, 4) and the bench contract test
mkdir -p gpurun_out/ab
for c in 3 1 0; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/ab/bench_cfg$c.log 2>&1; echo rc=$? >> gpurun_out/ab/bench_cfg$c.log; done
timeout 600 python -m pytest tests/test_gpu_bench_contract.py -q > gpurun_out/ab/pytest.log 2>&1; echo rc=$? >> gpurun_out/ab/pytest.log
