#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multi or overlap or cfg3 or sharding" > gpurun_out/m_pytest.log 2>&1; echo rc=$? >> gpurun_out/m_pytest.log
run() { echo "== $*" >> gpurun_out/m_bench.log; timeout 300 env "$@" python bench.py --steps 5 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],1), {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items() if k in ('recon','backproj','fb','dirichlet')})" >> gpurun_out/m_bench.log 2>&1; }
for o in 0 4 8 12 16; do run NFHMM_FB_MULTI=2 NFHMM_OVERLAP=$o; done
run NFHMM_FB_MULTI=1 NFHMM_OVERLAP=24
