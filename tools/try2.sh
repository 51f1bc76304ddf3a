timeout 900 python -m pytest tests/test_gpu_residue.py tests/test_gpu_pipe.py -x -q 2>&1 | tail -3
for c in C5 C3; do
NFFTK_NO_RES=1 timeout 600 python tools/kbench.py $c --reps 5 2>&1 | tail -1 | sed "s/^/rows-blocked /"
NFFTK_NO_RES=1 NFFTK_NO_BLOCK_ORDER=1 timeout 600 python tools/kbench.py $c --reps 5 2>&1 | tail -1 | sed "s/^/rows-plain /"
done
NFFTK_RES_TEAMS=3 timeout 600 python tools/kbench.py C5 --reps 5 2>&1 | tail -1 | sed "s/^/res3 /"
