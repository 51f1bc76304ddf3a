# A/B quick: pipe tests on each variant, then C3 / C5 / C3-c64 bench lines.
#   VARIANTS="a b" bash tools/ab_quick.sh   (variants from tools/build_variant.sh)
for v in ${VARIANTS}; do
  lib=paper_1810_09891_b200/variants/libnfftk_$v.so
  NFFTK_LIB=$lib timeout 400 python -m pytest tests/test_gpu_pipe.py -x -q > gpurun_out/t_$v.log 2>&1; echo rc=$? >> gpurun_out/t_$v.log
  for c in ${CONFIGS:-C3 C5}; do
    NFFTK_LIB=$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${v}_$c.log 2>&1
  done
  [ -n "$NO_C64" ] || NFFTK_LIB=$lib timeout 300 python bench.py --config C3 --precision single --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${v}_C3_c64.log 2>&1
done
