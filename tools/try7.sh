timeout 1500 python -m pytest tests/test_gpu_residue.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -4
for c in ${CONFIGS:-C5q C5}; do
timeout 600 python tools/kbench.py $c --reps 5 2>&1 | tail -1 | cut -c1-330 | sed "s/^/irun /"
NFFTK_NO_IRUN=1 timeout 600 python tools/kbench.py $c --reps 5 2>&1 | tail -1 | cut -c1-330| sed "s/^/pipe /"
done
