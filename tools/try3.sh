timeout 900 python -m pytest tests/test_gpu_residue.py -x -q 2>&1 | tail -3
for c in ${CONFIGS:-C5q}; do
for v in ${VARIANTS:-0 1 2 3 4 5}; do NFFTK_RES_VARIANT=$v timeout 600 python tools/kbench.py $c --reps 5 2>&1 | tail -1 | cut -c1-260| sed "s/^/v$v /"; done
NFFTK_NO_RES=1 timeout 600 python tools/kbench.py $c --reps 5 2>&1 | tail -1 | cut -c1-260| sed "s/^/rows /"
done
