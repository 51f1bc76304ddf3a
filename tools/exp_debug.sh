for dbg in 0 1 2 3; do
  NFFTK_DEBUG=$dbg timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/exp_c5_$dbg.log 2>&1
  NFFTK_DEBUG=$dbg timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/exp_c3_$dbg.log 2>&1
done
