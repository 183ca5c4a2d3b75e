timeout 900 python -m pytest tests/test_gpu_query.py tests/test_sharded.py -m gpu -q -x > gpurun_out/pytest_a.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
SUCO_SELECT_VARIANT=8,1,0 timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_a_old.json 2> gpurun_out/bench_a_old.err
SUCO_SELECT_VARIANT=16,0,0 timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_a_16.json 2> gpurun_out/bench_a_16.err
echo done
