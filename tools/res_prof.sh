# ncu capture of the residue kernels on the quarter-size C5 workload
C=${1:-C5q}
python tools/kbench.py $C --reps 5 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:"k_(interp|spread)_res" -c 2 \
    -o gpurun_out/res_$C python tools/profile_config.py $C 1 > gpurun_out/ncu_res_$C.log 2>&1
python tools/ncu_summary.py gpurun_out/res_$C.ncu-rep > gpurun_out/ncu_res_$C.txt 2>&1
python tools/ncu_hot.py gpurun_out/res_$C.ncu-rep k_spread_res 90 > gpurun_out/hot_spread_res_$C.txt 2>&1
python tools/ncu_hot.py gpurun_out/res_$C.ncu-rep k_interp_res 90 > gpurun_out/hot_interp_res_$C.txt 2>&1
