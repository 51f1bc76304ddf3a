# ncu capture of the residue-geometry kernels on one workload
C=${1:-C5q}
python tools/kbench.py $C --reps 5 2>&1 | tail -1 | cut -c1-250
ncu --set full --clock-control none --import-source on -k regex:"k_(interp_pipe|interp_run|spread_res)" -c 2 \
    -o gpurun_out/res_$C python tools/profile_config.py $C 1 > gpurun_out/ncu_res_$C.log 2>&1
python tools/ncu_summary.py gpurun_out/res_$C.ncu-rep > gpurun_out/ncu_res_$C.txt 2>&1
python tools/ncu_hot.py gpurun_out/res_$C.ncu-rep k_interp 70 > gpurun_out/hot_interp_res_$C.txt 2>&1
python tools/ncu_mix.py gpurun_out/res_$C.ncu-rep k_interp $C > gpurun_out/mix_interp_res_$C.txt 2>&1
