timeout 900 python -m pytest tests/test_sharded.py -m gpu -q > gpurun_out/pytest_w.log 2>&1
timeout 600 python bench.py --sharded --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_w_sharded1.json 2> gpurun_out/bench_w_sharded1.err
echo done
