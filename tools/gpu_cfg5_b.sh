# half-width dense select: tests, then cfg5 at 10M and 100M
timeout 900 python -m pytest tests/test_gpu_query.py tests/test_gpu_build.py -q -x -k "half or sampled" > gpurun_out/c5b_pytest.log 2>&1
timeout 900 python bench.py --config cfg5 --n 10000000 --queries 2000 --steps 2 --warmup 1 --cpu-seconds 5 > gpurun_out/c5b_10m.json 2> gpurun_out/c5b_10m.err
timeout 1800 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/c5b_full.json 2> gpurun_out/c5b_full.err
echo done
