# Round profile: bench (no ncu) then the ncu launch list of the same command,
# then one ncu --set full capture of the dominant kernels.
set -x
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.log 2>&1 || exit 1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
python tools/profile_config.py C3 1 > gpurun_out/prof_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_(interp|spread_rr)" -c 2 \
    -o gpurun_out/full_C3 python tools/profile_config.py C3 1 > gpurun_out/ncu_full.log 2>&1
