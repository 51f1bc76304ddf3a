# quick A/B: GPU pipe tests + phase times (CONFIGS, default C3 C5)
timeout 300 python -m pytest tests/test_gpu_pipe.py -x -q > gpurun_out/pipe_tests.log 2>&1; echo rc=$? >> gpurun_out/pipe_tests.log
for c in ${CONFIGS:-C3 C5}; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/q_$c.log 2>&1; done
