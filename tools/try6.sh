timeout 1500 python -m pytest tests/test_gpu_residue.py tests/test_gpu_pipe.py -x -q 2>&1 | tail -4
for c in C3 C5; do
timeout 600 python tools/kbench.py $c --reps 5 2>&1 | tail -1 | cut -c1-330 | sed "s/^/res /"
NFFTK_NO_RES=1 timeout 600 python tools/kbench.py $c --reps 5 2>&1 | tail -1 | cut -c1-330| sed "s/^/rows /"
timeout 600 python tools/kbench.py $c --reps 5 --single 2>&1 | tail -1 | cut -c1-330 | sed "s/^/res-c64 /"
NFFTK_NO_RES=1 timeout 600 python tools/kbench.py $c --reps 5 --single 2>&1 | tail -1 | cut -c1-330| sed "s/^/rows-c64 /"
done
NFFTK_RES_VARIANT=1 timeout 600 python tools/kbench.py C3 --reps 5 2>&1 | tail -1 | cut -c1-330 | sed "s/^/res-v1 /"
