# accuracy / speed of the TMEM accumulation chunk (NFHMM_TC_CHUNK k-blocks of 16 per slot)
for c in 4 8 16; do
  echo "== chunk=$c"
  NFHMM_TC_CHUNK=$c timeout 200 python scripts/perf_quick.py --mixtures 64 --iters 5 --check 2>&1 | grep -E "recon|backproj|after|total"
  NFHMM_TC_CHUNK=$c timeout 200 python scripts/perf_quick.py --config 4 --mixtures 1 --T 256 --iters 1 --check 2>&1 | grep -E "recon|backproj|after"
done
