set -x
CMD="python bench.py --mixtures 16 --iters 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm_kernel|dirichlet_kernel" -s 6 -c 3 -o gpurun_out/prof_tc1 $CMD > gpurun_out/ncu.log 2>&1; echo ncu_exit=$?; tail -3 gpurun_out/ncu.log
