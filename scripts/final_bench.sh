#!/bin/bash
# final bench lines of the last commit (default options, as the driver runs them, per config)
mkdir -p gpurun_out/fb
timeout 900 python bench.py > gpurun_out/fb/bench_cfg3.log 2>&1
for c in 0 1 2; do timeout 600 python bench.py --config $c > gpurun_out/fb/bench_cfg$c.log 2>&1; done
timeout 1200 python bench.py --config 4 > gpurun_out/fb/bench_cfg4.log 2>&1
for M in 32 64 128; do timeout 600 python bench.py --mixtures $M --no-cpu-baseline > gpurun_out/fb/bench_cfg3_M$M.log 2>&1; done
