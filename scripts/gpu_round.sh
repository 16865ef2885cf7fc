set -x
nproc
CMD="python bench.py"
timeout 900 $CMD > gpurun_out/bench_full.log 2>&1; echo bench_exit=$?; tail -c 3000 gpurun_out/bench_full.log
timeout 900 $CMD > gpurun_out/plain.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1_exit=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm_kernel" -s 8 -c 2 -o gpurun_out/prof_full_r1 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2_exit=$?; tail -3 gpurun_out/ncu_full.log
