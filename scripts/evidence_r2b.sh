#!/bin/bash
# Round-2 evidence (final, third session): the full GPU test suite, the bench lines (all configs, reference arm, training),
# the launch list of the default bench command, and ncu --set full captures of the hot kernels.
set -x
mkdir -p gpurun_out/ev3
rm -f gpurun_out/parity_records.jsonl
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/ev3/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/ev3/pytest_gpu.log
cp gpurun_out/parity_records.jsonl gpurun_out/ev3/parity_records.jsonl
nvidia-smi -q -d CLOCK,POWER > gpurun_out/ev3/smi.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/ev3/bench_cfg3.log 2>&1
for c in 0 1 2 4; do timeout 900 python bench.py --config $c > gpurun_out/ev3/bench_cfg$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev3/bench_reference.log 2>&1
timeout 600 python bench.py --workload train > gpurun_out/ev3/bench_train.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/ev3/launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-bound-off > gpurun_out/ev3/ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:tc_gemm_kernel|dirichlet_ring|fb_multi" -s 6 -c 4 -o gpurun_out/ev3/ncu_full_cfg3 -f python bench.py --steps 1 --warmup 1 --iters 4 --no-cpu-baseline --no-e2e --no-bound-off > gpurun_out/ev3/ncu_full.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev3/smoke.log 2>&1
