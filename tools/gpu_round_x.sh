timeout 900 python -m pytest tests/test_sharded.py -m gpu -q > gpurun_out/pytest_x.log 2>&1
timeout 600 python bench.py --sharded --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_x_sharded1.json 2> gpurun_out/bench_x_sharded1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_x_sharded.csv python bench.py --sharded --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_x.log 2>&1
echo done
