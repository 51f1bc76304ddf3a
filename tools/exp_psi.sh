for c in C3 C5 C4; do
  for p in direct tensor; do
    timeout 300 python bench.py --config $c --psi $p --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_$p.log 2>&1
  done
done
