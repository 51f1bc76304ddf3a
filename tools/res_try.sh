# residue kernels: parity tests, then timing for both team layouts and the row kernels
timeout 900 python -m pytest tests/test_gpu_residue.py -x -q > gpurun_out/res_pytest.log 2>&1
tail -5 gpurun_out/res_pytest.log
for c in ${CONFIGS:-C5q C5}; do
for t in 4 3; do NFFTK_RES_TEAMS=$t timeout 600 python tools/kbench.py $c --reps 5 2>&1 | tail -1 | sed "s/^/teams$t /"; done | tee -a gpurun_out/res_kbench.log
NFFTK_NO_RES=1 timeout 600 python tools/kbench.py $c --reps 5 2>&1 | tail -1 | sed "s/^/rows /" | tee -a gpurun_out/res_kbench.log
done
