#!/bin/bash
# A/B: warp-per-frame Wiener kernel (new lib) vs the previous build (lib/libnfhmm_base.so), config 3 and 1
mkdir -p gpurun_out/abw
timeout 600 python -m pytest tests -m gpu -q -k "separ or edge or cfg1 or cfg0 or guard or device_io or resume" > gpurun_out/abw/pytest.log 2>&1; echo rc=$? >> gpurun_out/abw/pytest.log
b() { timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-bound-off --no-cpu-baseline "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"; }
for rep in 1 2; do
echo "cfg3 new: $(b)" >> gpurun_out/abw/bench.log
echo "cfg3 base: $(NFHMM_LIB=$PWD/paper_1206_6468_b200/lib/libnfhmm_base.so b)" >> gpurun_out/abw/bench.log
done
echo "cfg1 new: $(b --config 1)" >> gpurun_out/abw/bench.log
echo "cfg1 base: $(NFHMM_LIB=$PWD/paper_1206_6468_b200/lib/libnfhmm_base.so b --config 1)" >> gpurun_out/abw/bench.log
