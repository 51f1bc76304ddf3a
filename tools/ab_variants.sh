# A/B the built variants against the in-tree library: VARIANTS="a b" CONFIGS="C3 C5"
for v in base ${VARIANTS}; do
  lib=""; [ "$v" = base ] || lib=paper_1810_09891_b200/variants/libnfftk_$v.so
  for c in ${CONFIGS:-C3 C5}; do
    NFFTK_LIB=$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${v}_$c.log 2>&1
  done
done
