#!/bin/bash
# ncu --set full of one kernel (regex $1) launched by a short bench run; report -> gpurun_out/$2.ncu-rep
# usage: scripts/ncu_one.sh <kernel-regex> <name> [extra bench args...]
K=$1; NAME=$2; shift 2
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" -s 2 -c 1 \
  -o gpurun_out/$NAME -f python bench.py --steps 1 --warmup 1 --iters 3 --no-e2e --no-bound-off --no-cpu-baseline "$@" \
  > gpurun_out/$NAME.log 2>&1
echo "ncu rc=$?" >> gpurun_out/$NAME.log
