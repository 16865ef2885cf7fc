set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$?; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 2 --warmup 1 --iters 10 --mixtures 64 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1; echo bench_exit=$?; tail -c 2500 gpurun_out/bench_small.log
CMD="python bench.py --mixtures 16 --iters 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"recon_kernel|backproj_kernel|dirichlet_kernel|fb_kernel" -s 8 -c 4 -o gpurun_out/prof_r1a $CMD > gpurun_out/ncu.log 2>&1; echo ncu_exit=$?; tail -5 gpurun_out/ncu.log
