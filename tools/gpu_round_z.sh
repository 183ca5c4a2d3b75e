timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_z.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_z.json 2> gpurun_out/bench_z.err
timeout 600 python bench.py --sharded --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_z_sharded.json 2> gpurun_out/bench_z_sharded.err
echo done
