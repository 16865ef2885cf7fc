# Round-end style GPU run: tests, smoke, benches (configs 3 / 1 / 2 / 0 / 4), reference arm, profiles.
# Usage: bash scripts/gpu_round.sh TAG
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
nproc
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo pytest_exit=$?; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke_exit=$?; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_cfg3_$TAG.log 2>&1; echo bench3_exit=$?
for c in 1 2 0; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg${c}_$TAG.log 2>&1; echo bench${c}_exit=$?; done
timeout 1200 python bench.py --config 4 --steps 2 --no-cpu-baseline --no-bound-off > gpurun_out/bench_cfg4_$TAG.log 2>&1; echo bench4_exit=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo ref_exit=$?
timeout 600 python bench.py --workload train > gpurun_out/bench_train_$TAG.log 2>&1; echo train_exit=$?
CMD="python bench.py --no-cpu-baseline --no-e2e --no-bound-off"
timeout 900 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu1=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm_kernel|dirichlet|fb_kernel" -s 12 -c 4 -o gpurun_out/prof_full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu2=$?
