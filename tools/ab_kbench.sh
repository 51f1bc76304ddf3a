# A/B of built variants with tools/kbench.py (timing + golden parity):
#   VARIANTS="a b" CONFIGS="C5 C3" bash tools/ab_kbench.sh
for c in ${CONFIGS:-C5}; do
  for v in base ${VARIANTS}; do
    lib=""; [ "$v" = base ] || lib=paper_1810_09891_b200/variants/libnfftk_$v.so
    NFFTK_LIB=$lib timeout 300 python tools/kbench.py $c ${KB_ARGS} 2>&1 | tail -1 | sed "s/^/$v /"
  done
done
