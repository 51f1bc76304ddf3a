# A/B an environment knob on the in-tree library: ENVS="NFFTK_NO_DENSE_FLUSH=1" CONFIGS="C3 C4 C5"
i=0
for e in "" ${ENVS}; do
  for c in ${CONFIGS:-C3 C5}; do
    env $e timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abe_${i}_$c.log 2>&1
  done
  i=$((i+1))
done
