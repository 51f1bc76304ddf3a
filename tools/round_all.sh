# Full round refresh: GPU tests, per-config bench lines (c128, and c64 where
# the config names it), then the profile pass.
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
for c in C1 C2 C4 C5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.log 2>&1; done
for c in C3 C4 C5; do timeout 600 python bench.py --config $c --precision single --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_c64.log 2>&1; done
PROFILE_CONFIGS="${PROFILE_CONFIGS:-C3 C4 C5}" bash tools/round_profile.sh
