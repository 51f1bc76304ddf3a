# A/B of d=2 variants on C4 (c128 and c64): VARIANTS="a b" bash tools/ab_c4.sh
for v in base ${VARIANTS}; do
  lib=""; [ "$v" = base ] || lib=paper_1810_09891_b200/variants/libnfftk_$v.so
  NFFTK_LIB=$lib timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c4_${v}.log 2>&1
  NFFTK_LIB=$lib timeout 300 python bench.py --config C4 --precision single --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c4_${v}_c64.log 2>&1
done
