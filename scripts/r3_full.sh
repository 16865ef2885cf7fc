#!/bin/bash
mkdir -p gpurun_out/full
rm -f gpurun_out/parity_records.jsonl
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/full/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/full/pytest_gpu.log
cp gpurun_out/parity_records.jsonl gpurun_out/full/parity_records.jsonl
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/full/bench_cfg3.log 2>&1
