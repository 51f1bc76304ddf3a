timeout 900 python -m pytest tests/test_gpu_residue.py -x -q 2>&1 | tail -3
for t in 3 4; do NFFTK_RES_TEAMS=$t timeout 600 python tools/kbench.py C5q --reps 5 2>&1 | tail -1 | cut -c1-200| sed "s/^/res$t /"; done
