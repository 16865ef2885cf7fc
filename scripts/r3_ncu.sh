#!/bin/bash
# branch-free ratio epilogue + packed converter: bench, decomposition, ncu of the two GEMMs, parity subset
mkdir -p gpurun_out/nc
b() { timeout 300 python bench.py "$@" --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()})"; }
echo "cfg3: $(b)" >> gpurun_out/nc/bench.log
echo "cfg1: $(b --config 1)" >> gpurun_out/nc/bench.log
for d in 0 2 4 8 128 12; do echo "dbg $d: $(NFHMM_TC_DEBUG=$d timeout 120 python scripts/perf_quick.py --mixtures 64 --kernels recon,backproj 2>&1 | tr '\n' ' ')" >> gpurun_out/nc/dbg.log; done
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:tc_gemm_kernel" -s 4 -c 2 -o gpurun_out/nc/ncu_gemm -f python scripts/perf_quick.py --mixtures 64 --iters 2 > gpurun_out/nc/ncu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/nc/pytest.log 2>&1; echo rc=$? >> gpurun_out/nc/pytest.log
