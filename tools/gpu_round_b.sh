timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_b.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
timeout 600 python bench.py --sharded --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_b_sh.json 2> gpurun_out/bench_b_sh.err
echo done
