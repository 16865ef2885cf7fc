#!/bin/bash
# deferred back-projection beside the forward-backward: parity, overlap sweeps, recon decomposition
mkdir -p gpurun_out/df
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/df/pytest.log 2>&1; echo rc=$? >> gpurun_out/df/pytest.log
b() { timeout 300 python bench.py "$@" --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"; }
for o in 12 16 24 32; do echo "cfg3 overlap $o: $(NFHMM_OVERLAP=$o b)" >> gpurun_out/df/bench.log; done
echo "cfg3 overlap 24 nodefer: $(NFHMM_OVERLAP=24 NFHMM_DEFER=0 b)" >> gpurun_out/df/bench.log
for o in 0 16 32 48 64; do echo "cfg1 overlap $o: $(NFHMM_OVERLAP=$o b --config 1)" >> gpurun_out/df/bench.log; done
echo "cfg1 overlap 32 nodefer: $(NFHMM_OVERLAP=32 NFHMM_DEFER=0 b --config 1)" >> gpurun_out/df/bench.log
for o in 0 32 48; do echo "cfg2 overlap $o: $(NFHMM_OVERLAP=$o b --config 2)" >> gpurun_out/df/bench.log; done
for d in 0 1 2 4 8 32 64 128 12 44; do echo "dbg $d: $(NFHMM_TC_DEBUG=$d timeout 120 python scripts/perf_quick.py --mixtures 64 --kernels recon,backproj 2>&1 | tr '\n' ' ')" >> gpurun_out/df/dbg.log; done
