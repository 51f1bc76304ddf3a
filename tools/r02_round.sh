# Round-2 refresh on the GPU box: GPU tests, the default (C5) bench line, the
# ncu launch list of the same command, one ncu --set full capture of the C5
# gridding kernels, then the per-config lines.  Everything lands in gpurun_out/.
set -x
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
python tools/ncu_launch_summary.py gpurun_out/launches_C5.csv > gpurun_out/launches_C5_summary.txt 2>&1
for c in ${PROFILE_CONFIGS:-C5}; do
  python tools/profile_config.py $c 1 > gpurun_out/prof_plain_$c.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:"k_(interp|spread|fft_pass)" -c 8 \
      -o gpurun_out/full_$c python tools/profile_config.py $c 1 > gpurun_out/ncu_full_$c.log 2>&1
  python tools/ncu_summary.py gpurun_out/full_$c.ncu-rep > gpurun_out/ncu_full_$c.txt 2>&1
  python tools/ncu_traffic.py gpurun_out/full_$c.ncu-rep $c gpurun_out/ncu_traffic.json >> gpurun_out/ncu_full_$c.txt 2>&1
  python tools/ncu_hot.py gpurun_out/full_$c.ncu-rep k_spread 60 > gpurun_out/hot_spread_$c.txt 2>&1
  python tools/ncu_mix.py gpurun_out/full_$c.ncu-rep k_spread $c > gpurun_out/mix_spread_$c.txt 2>&1
  python tools/ncu_mix.py gpurun_out/full_$c.ncu-rep k_interp $c > gpurun_out/mix_interp_$c.txt 2>&1
  python tools/ncu_hot.py gpurun_out/full_$c.ncu-rep k_interp 60 > gpurun_out/hot_interp_$c.txt 2>&1
  [ -n "$KEEP_REP" ] || rm -f gpurun_out/full_$c.ncu-rep   # gpurun_out/ only travels back under 64 MiB
done
for c in ${BENCH_CONFIGS:-C1 C2 C3 C4}; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.log 2>&1; done
for c in ${BENCH_C64:-C3 C4 C5}; do timeout 600 python bench.py --config $c --precision single --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_c64.log 2>&1; done
ls -la gpurun_out/
