timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_d.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
timeout 600 python bench.py --sharded --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_d_sh.json 2> gpurun_out/bench_d_sh.err
echo done
