#!/bin/bash
# final check of the committed build: GPU suite + smoke + default bench line
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final/smoke.log
timeout 900 python bench.py > gpurun_out/final/bench.log 2>&1; echo "rc=$?" >> gpurun_out/final/bench.log
