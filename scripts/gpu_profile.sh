# Profiling evidence for profiles/: plain bench, launch list of the same command, one --set full capture
# per hot kernel (tcgen05 GEMM recon + backproj, Dirichlet, FB).  Usage: bash scripts/gpu_profile.sh TAG
set -x
TAG=${1:-r1}
CMD="python bench.py --no-cpu-baseline --no-e2e"
mkdir -p gpurun_out
timeout 900 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu1=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm_kernel|dirichlet_kernel|fb_kernel" -s 12 -c 4 -o gpurun_out/prof_full_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu2=$?; tail -3 gpurun_out/ncu_full_$TAG.log
