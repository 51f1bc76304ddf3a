# Round profile: bench (no ncu) then the ncu launch list of the same command,
# then one ncu --set full capture of the gridding kernels per config (the C3
# report is kept; the others are summarised on the box to stay small).
set -x
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.log 2>&1 || exit 1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
for c in ${PROFILE_CONFIGS:-C3}; do
  python tools/profile_config.py $c 1 > gpurun_out/prof_plain_$c.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:"k_(interp|spread)" -c 2 \
      -o gpurun_out/full_$c python tools/profile_config.py $c 1 > gpurun_out/ncu_full_$c.log 2>&1
  python tools/ncu_summary.py gpurun_out/full_$c.ncu-rep > gpurun_out/ncu_full_$c.txt 2>&1
  python tools/ncu_traffic.py gpurun_out/full_$c.ncu-rep $c gpurun_out/ncu_traffic.json >> gpurun_out/ncu_full_$c.txt 2>&1
  [ "$c" = C3 ] || rm -f gpurun_out/full_$c.ncu-rep
done
