#!/bin/bash
mkdir -p gpurun_out/dp
q() { timeout 120 python scripts/perf_quick.py --mixtures 64 --kernels recon,backproj 2>&1 | tr '\n' ' '; }
for st in 2 3 4; do echo "stages $st: $(NFHMM_TC_STAGES=$st q)" >> gpurun_out/dp/dbg.log; done
for pf in 0 4 8 32 64; do echo "prefetch $pf: $(NFHMM_TC_PREFETCH=$pf q)" >> gpurun_out/dp/dbg.log; done
for d in 237 233 205 109 45; do echo "dbg $d: $(NFHMM_TC_DEBUG=$d q)" >> gpurun_out/dp/dbg.log; done
for st in 2 3; do echo "dbg 237 stages $st: $(NFHMM_TC_DEBUG=237 NFHMM_TC_STAGES=$st q)" >> gpurun_out/dp/dbg.log; done
echo "tf32: $(NFHMM_RECON=tf32 q)" >> gpurun_out/dp/dbg.log
echo "tf32 dbg 237: $(NFHMM_RECON=tf32 NFHMM_TC_DEBUG=237 q)" >> gpurun_out/dp/dbg.log
