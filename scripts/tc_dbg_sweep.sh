# GEMM bottleneck experiments (NFHMM_TC_DEBUG bits: 1 no A loads, 2 no MMAs, 4 no epilogue I/O,
# 8 no A TMEM stores, 32 no B loads; NFHMM_TC_CHUNK k-blocks per TMEM slot); relative times only.
for c in ${CHUNKS:-4 16}; do for d in ${DBGS:-0 45 4 8 1 36 47}; do
  echo "== chunk=$c dbg=$d $(NFHMM_TC_CHUNK=$c NFHMM_TC_DEBUG=$d timeout 120 python scripts/perf_quick.py --mixtures 64 --iters 1 --kernels recon,backproj 2>&1 | grep -E "alone|Error" | tr '\n' ' ')"
done; done
