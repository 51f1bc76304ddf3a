timeout 900 python -m pytest tests/test_gpu_residue.py tests/test_gpu_pipe.py -x -q 2>&1 | tail -2
for c in C5 C3 C4; do timeout 600 python tools/kbench.py $c --reps 5 2>&1 | tail -1 | cut -c1-420; done
python tools/profile_config.py C5 1 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_(interp_pipe|spread_res)" -c 2 python tools/profile_config.py C5 1 2>&1 | grep -E "k_|dram__|gpu__time"
