#!/bin/bash
# 3xFP16 back-projection + epilogue L2 prefetch: parity, benches, decomposition
mkdir -p gpurun_out/hb
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/hb/pytest.log 2>&1; echo rc=$? >> gpurun_out/hb/pytest.log
b() { timeout 300 python bench.py "$@" --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()})"; }
echo "cfg3 default: $(b)" >> gpurun_out/hb/bench.log
echo "cfg3 backproj tf32: $(NFHMM_BACKPROJ=tf32 b)" >> gpurun_out/hb/bench.log
for o in 12 16 24; do echo "cfg3 overlap $o: $(NFHMM_OVERLAP=$o b)" >> gpurun_out/hb/bench.log; done
echo "cfg1 default: $(b --config 1)" >> gpurun_out/hb/bench.log
echo "cfg2 default: $(b --config 2)" >> gpurun_out/hb/bench.log
echo "cfg0 default: $(b --config 0)" >> gpurun_out/hb/bench.log
echo "cfg4 default: $(b --config 4 --steps 2 --warmup 1)" >> gpurun_out/hb/bench.log
for d in 0 2 4 8 64 128; do echo "dbg $d: $(NFHMM_TC_DEBUG=$d timeout 120 python scripts/perf_quick.py --mixtures 64 --kernels recon,backproj 2>&1 | tr '\n' ' ')" >> gpurun_out/hb/dbg.log; done
timeout 300 python scripts/perf_quick.py --mixtures 64 --iters 10 --check > gpurun_out/hb/quick.log 2>&1
