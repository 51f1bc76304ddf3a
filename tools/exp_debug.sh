# NFFTK_DEBUG experiment: 0 = normal, 1 = skip spread flush, 2 = skip spread node loop,
# 4 = node loop without the FMAs
for dbg in ${DBGS:-0 1 2 4}; do
  for c in ${CONFIGS:-C3 C5}; do
    NFFTK_DEBUG=$dbg timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/exp_${c}_$dbg.log 2>&1
  done
done
