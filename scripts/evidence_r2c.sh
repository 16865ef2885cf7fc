#!/bin/bash
# Round-2 evidence on the final build (fourth session): bench lines of every config, the reference arm,
# the launch list of the default bench command and ncu --set full of the config-3 hot kernels.
set -x
D=gpurun_out/ev4
mkdir -p $D
nvidia-smi -q -d CLOCK,POWER > $D/smi.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $D/bench_cfg3.log 2>&1
for c in 0 1 2 4; do timeout 900 python bench.py --config $c > $D/bench_cfg$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $D/bench_reference.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $D/launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-bound-off > $D/ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:tc_gemm_kernel|dirichlet_ring|fb_multi" -s 6 -c 4 -o $D/ncu_full_cfg3 -f python bench.py --steps 1 --warmup 1 --iters 4 --no-cpu-baseline --no-e2e --no-bound-off > $D/ncu_full.log 2>&1
echo done > $D/DONE
