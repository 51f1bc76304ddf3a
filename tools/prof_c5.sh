set -x
python tools/profile_config.py C5 1 > gpurun_out/prof_plain_C5.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_(interp_pipe|spread_pipe)" -c 2 \
    -o gpurun_out/full_C5 python tools/profile_config.py C5 1 > gpurun_out/ncu_full_C5.log 2>&1
python tools/ncu_summary.py gpurun_out/full_C5.ncu-rep > gpurun_out/ncu_full_C5.txt 2>&1
python tools/ncu_hot.py gpurun_out/full_C5.ncu-rep k_spread_pipe 70 > gpurun_out/hot_spread_C5.txt 2>&1
python tools/ncu_hot.py gpurun_out/full_C5.ncu-rep k_interp_pipe 70 > gpurun_out/hot_interp_C5.txt 2>&1
ls -la gpurun_out/
