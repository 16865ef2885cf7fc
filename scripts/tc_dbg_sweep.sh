# GEMM bottleneck experiments (NFHMM_TC_DEBUG bits: 1 no A loads, 2 no MMAs, 4 no epilogue I/O,
# 8 no A TMEM stores, 32 no B loads); numbers are not valid results, only relative times.
for d in 0 1 2 4 8 32 33 36 34 38 39 45; do
  echo "== dbg=$d"; NFHMM_TC_DEBUG=$d timeout 120 python scripts/perf_quick.py --mixtures 64 --iters 1 --kernels recon,backproj 2>&1 | grep -E "alone|Error"
done
